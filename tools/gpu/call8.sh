timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "stream" 2>&1 | tail -2
for u in 1 2 4; do echo "P=$u"; MRPT_VSTREAM_P=$u python tools/vote_ab.py --config 5 --nq 20000 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['same_counts'], d['stream']['ms_per_100k'], d['dir']['ms_per_100k'])"; done
