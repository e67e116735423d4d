P=gpurun_out/r02/sort
mkdir -p $P
for rep in 1 2; do for m in "" 1 2; do MSV_BENCH_SORT=$m timeout 900 python bench.py --no-cpu-baseline > $P/b.log 2>&1; echo -n "sort=$m: "; tail -1 $P/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), round(d['e2e']['value']/1e9,3), round(d['ms_per_step'],2))"; done; done
