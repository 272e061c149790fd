timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_project_d64 -s 2 -c 1 -o gpurun_out/ncu_k1_d64 python tools/profile_build.py 5 0.3 > gpurun_out/ncu_k1.log 2>&1
tail -2 gpurun_out/ncu_k1.log
