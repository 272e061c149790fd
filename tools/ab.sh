# usage: ab.sh config scale tag env...
cfg=$1; sc=$2; tag=$3; shift 3
for e in "$@"; do
  env $e timeout 500 python bench.py --config $cfg --scale $sc --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${tag}_$e.json 2>gpurun_out/ab_${tag}_$e.err
  python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], round(d['value']), {k: round(v,2) for k,v in d['stage_ms_per_step'].items()}, round(d['roofline']['frac'],3))" gpurun_out/ab_${tag}_$e.json "$tag $e" || tail -3 gpurun_out/ab_${tag}_$e.err
done
