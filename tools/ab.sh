# A/B the library builds in _ab/ on the bench grid: tools/ab.sh name1 name2 ...
for rep in 1 2; do
  for v in "$@"; do
    echo -n "$v: "
    MSV_LIB=_ab/$v.so python bench.py --no-cpu-baseline --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), round(d['ms_per_step'],2), d['stage_ms'])"
  done
done
