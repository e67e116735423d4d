run() { python bench.py --no-cpu-baseline --steps 5 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), round(d['ms_per_step'],2))"; }
for sp in ${SPLITS:-"2,1,1,1" "1,1,1,2" "1,1,1,1" "1,2,1,1" "1,1,2" "1,3"}; do echo -n "split=$sp "; MSV_CHUNK_SPLIT=$sp run; done
