# A/B of bench.py under env settings: ab.sh config scale tag "ENV=1 ENV2=2" ...
cfg=$1; sc=$2; tag=$3; shift 3
for e in "$@"; do
  f="gpurun_out/ab_${tag}_$(echo "$e" | tr ' =' '_-')"
  env $e timeout 500 python bench.py --config $cfg --scale $sc --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline > "$f.json" 2> "$f.err"
  python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], round(d['value']), {k: round(v,2) for k,v in d['stage_ms_per_step'].items()}, round(d['roofline']['frac'],3), 'e2e', d['e2e'])" "$f.json" "$tag $e" || tail -n 3 "$f.err"
done
