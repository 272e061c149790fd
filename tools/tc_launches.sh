# per-kernel device times of the pinned tc route on config 2 (ncu launch list) + one full capture
export MRPT_PIN=u8tc_bits
python tools/profile_query.py --config 2 --reps 2 > gpurun_out/pq_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/tc_launches.csv python tools/profile_query.py --config 2 --reps 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tc_filter -s 1 -c 1 -o gpurun_out/tc_full4 python tools/profile_query.py --config 2 --reps 2 > /dev/null 2>&1
