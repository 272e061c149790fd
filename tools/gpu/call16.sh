timeout 1500 python -m pytest tests/test_gpu_configs.py -x -q -s 2>&1 | grep -E "fallbacks|passed|failed|Error|assert" | head -20
