# Round evidence for profiles/: bench (plain), launch list + DRAM traffic of the
# pinned headline route, one --set full capture of the fused filter.
set -x
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
export MRPT_PIN=u8tc_bits
python tools/profile_query.py --config 2 --votes 1 --reps 2 > gpurun_out/pq_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/traffic_c2v1.csv python tools/profile_query.py --config 2 --votes 1 --reps 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tc_filter -s 1 -c 1 -o gpurun_out/tc_filter_full \
    python tools/profile_query.py --config 2 --votes 1 --reps 2 > /dev/null 2>&1
