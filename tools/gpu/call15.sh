timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_build_c5.csv python tools/profile_build.py 5 1.0 > gpurun_out/launches_build_c5.log 2>&1
tail -1 gpurun_out/launches_build_c5.log
