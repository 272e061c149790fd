./tools/micro/atom_bench2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "stream" 2>&1 | tail -5
