for v in "MSV_TRACE_GROUP_FIRST=2" "MSV_TRACE_GROUP_FIRST=16" "MSV_TRACE_GROUP_FIRST=2 MSV_CHUNK_SPLIT=1,1,1,1" "MSV_TRACE_GROUP_FIRST=16 MSV_CHUNK_SPLIT=1,1,1,1" "MSV_TRACE_GROUP_FIRST=16 MSV_CHUNK_SPLIT=1,1" "MSV_TRACE_GROUP_FIRST=2 MSV_CHUNK_SPLIT=3,1,1,1" "MSV_TRACE_GROUP_FIRST=16 MSV_CHUNK_SPLIT=1,1,1,1,1,1,1,1"; do
  echo -n "$v: "
  env $v python bench.py --no-cpu-baseline --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), round(d['ms_per_step'],2))"
done
