timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py --steps 5 --warmup 3 > gpurun_out/c5_r02_c.json 2> gpurun_out/c5_r02_c.err; tail -2 gpurun_out/c5_r02_c.err
MRPT_PIN=fp16 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python tools/profile_query.py --config 5 --reps 1 > gpurun_out/launches_c5.log 2>&1
tail -2 gpurun_out/launches_c5.log
