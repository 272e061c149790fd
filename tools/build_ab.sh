# build-kernel A/B: launch-list totals per kernel and wall build time under env settings
for e in "$@"; do
  f="gpurun_out/bab_$(echo "$e" | tr ' =' '_-')"
  env $e python tools/profile_build.py 3; env $e python tools/profile_build.py 3
  env $e ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:^k_ --csv --log-file $f.csv python tools/profile_build.py 3 > /dev/null 2>&1
  echo "== $e"; python tools/build_launch_summary.py $f.csv | head -12
done
