timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q 2>&1 | tail -2
for o in 0 1; do MRPT_QUERY_ORDER=$o python tools/profile_query.py --config 5 --reps 2 --time 2>&1 | grep TIME; done
for o in 0 1; do MRPT_QUERY_ORDER=$o python tools/profile_query.py --config 3 --votes 2 --reps 2 --time 2>&1 | grep TIME; done
