timeout 900 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_bindings.py -x -q 2>&1 | tail -15
