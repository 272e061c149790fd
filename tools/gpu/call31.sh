python bench.py --steps 10 --warmup 3 > gpurun_out/c5_r02_d.json 2> gpurun_out/c5_r02_d.err; tail -2 gpurun_out/c5_r02_d.err
for c in 2 3 4; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c${c}_r02_d.json 2> gpurun_out/c${c}_r02_d.err; tail -1 gpurun_out/c${c}_r02_d.err; done
