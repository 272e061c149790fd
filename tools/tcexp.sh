timeout 300 python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep -E "TIME|rror" | sed "s/^/base /"
MRPT_ROUTE_ILV=1 timeout 300 python tools/profile_query.py --config 2 --reps 2 --time 2>&1 | grep -E "TIME|rror" | sed "s/^/ilv /"
MRPT_ROUTE_ILV=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
