timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "stream" 2>&1 | tail -15
python tools/vote_ab.py --config 5 --nq 20000 2>&1 | tail -3
python tools/vote_ab.py --config 4 --nq 1000 2>&1 | tail -3
python tools/vote_ab.py --config 3 --nq 10000 --votes 2 2>&1 | tail -3
