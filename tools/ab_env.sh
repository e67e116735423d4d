# A/B one library under environment settings: tools/ab_env.sh "MSV_X=0" "MSV_X=1" ...
for rep in 1 2; do
  for v in "$@"; do
    echo -n "$v: "
    env $v python bench.py --no-cpu-baseline --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), round(d['ms_per_step'],2), d['stage_ms'], d.get('parity',{}).get('placement_hash_equal'))"
  done
done
