timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "stream" 2>&1 | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_vote_stream -c 1 -o gpurun_out/ncu_vote_stream_c5 python tools/vote_ab.py --config 5 --nq 2000 --reps 1 > gpurun_out/ncu_vs.log 2>&1
tail -3 gpurun_out/ncu_vs.log
