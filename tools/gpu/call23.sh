MRPT_VOTE_DBG=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_vote_stream -c 1 -o gpurun_out/ncu_vs_dbg3 python tools/vote_ab.py --config 5 --nq 2000 --reps 1 > gpurun_out/ncu_vs3.log 2>&1
tail -1 gpurun_out/ncu_vs3.log
