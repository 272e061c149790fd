set -x
nproc; free -g; df -h /tmp | tail -1; nvidia-smi --query-gpu=name,memory.total --format=csv
python -c "import numpy; print(numpy.__version__)"
( time python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline ) > gpurun_out/c5_r02_a.json 2> gpurun_out/c5_r02_a.err
tail -3 gpurun_out/c5_r02_a.err
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
