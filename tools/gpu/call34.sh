timeout 900 python -m pytest tests/test_gpu_scan_variants.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -2
python tools/profile_query.py --config 5 --reps 2 --time 2>&1 | grep TIME
MRPT_PIN=fp16 python tools/profile_query.py --config 4 --reps 2 --time 2>&1 | grep TIME
