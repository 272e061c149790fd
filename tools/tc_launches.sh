# per-kernel device times of the tc route on config 2 (ncu launch list), CG from $1
export MRPT_SCAN_ROWS=u8tc_bits MRPT_TC_CG=$1
python tools/profile_query.py --config 2 --reps 2 > gpurun_out/pq_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tc_launches_cg$1.csv python tools/profile_query.py --config 2 --reps 2 > /dev/null 2>&1
