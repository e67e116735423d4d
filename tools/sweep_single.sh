# single (non-pipelined) launch time on the bench grid for chunk layouts
for v in "MSV_CHUNK_SPLIT=2,1,1,1" "MSV_CHUNK_SPLIT=1,2,1,1" "MSV_CHUNK_SPLIT=1,1,1,1" "MSV_CHUNK_SPLIT=1,3,2,1" "MSV_CHUNK_SPLIT=2,1,1,1 MSV_TRACE_GROUP_FIRST=1" "MSV_CHUNK_SPLIT=1,2,1,1 MSV_TRACE_GROUP_FIRST=1" "MSV_CHUNK_SPLIT=1,4,2,2 MSV_TRACE_GROUP_FIRST=1"; do
  echo -n "$v: "
  env MSV_PIPELINE=0 $v python bench.py --no-cpu-baseline --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), round(d['ms_per_step'],2), round(d['e2e']['value']/1e9,3))"
done
