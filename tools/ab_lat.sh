# A/B libraries on the bench grid (throughput) and on the latency-bound configs (stage times)
for v in "$@"; do
  echo -n "$v bench: "
  MSV_LIB=_ab/$v.so python bench.py --no-cpu-baseline --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), round(d['ms_per_step'],2), d['stage_ms']['sim_ms'])"
  MSV_LIB=_ab/$v.so python tools/stage_configs.py 2>&1 | sed "s/^/$v /"
done
