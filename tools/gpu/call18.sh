MRPT_PIN=fp16 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scan_topk_filter_h -c 1 -o gpurun_out/ncu_scan_fp16_c5 python tools/profile_query.py --config 5 --nq 4000 --reps 1 > gpurun_out/ncu_scan.log 2>&1
tail -2 gpurun_out/ncu_scan.log
