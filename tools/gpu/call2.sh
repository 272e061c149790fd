# GPU tests, then the default bench (config 5) and the reference arm
df -h /dev/shm | tail -1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
( time python bench.py --steps 5 --warmup 3 ) > gpurun_out/c5_r02_b.json 2> gpurun_out/c5_r02_b.err
tail -5 gpurun_out/c5_r02_b.err
( time python bench.py --impl reference --steps 5 --warmup 2 ) > gpurun_out/ref5_r02_b.json 2> gpurun_out/ref5_r02_b.err
tail -5 gpurun_out/ref5_r02_b.err
