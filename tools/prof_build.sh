set -x
python tools/profile_build.py 3 > gpurun_out/build_c3.log 2>&1 || exit 1
cat gpurun_out/build_c3.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:mrpt --csv --log-file gpurun_out/build_c3_launches.csv python tools/profile_build.py 3 > gpurun_out/build_c3_ncu1.log 2>&1
for k in k_project_smem k_big_keys k_big_hist k_big_scatter k_seg_small k_fnv_perm; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/build_c3_$k -f python tools/profile_build.py 3 > gpurun_out/build_c3_ncu_$k.log 2>&1
done
ls -la gpurun_out/
