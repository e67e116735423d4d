for v in base lazyest; do
  echo "== $v"; MSV_LIB=_ab/$v.so timeout 600 python tools/diag_classes.py 16384 1e5 mobilenet 2>&1 | head -5 | cut -c1-60
  MSV_LIB=_ab/$v.so MSV_MAX_CHUNKS=1 timeout 600 ncu --metrics smsp__inst_executed.sum -k regex:sim_warp_kernel -c 1 --csv python tools/prof_k2.py mobilenet k1 4096 2>/dev/null | grep inst_executed | cut -c1-200
done
for rep in 1 2; do for v in base lazyest; do MSV_LIB=_ab/$v.so timeout 900 python bench.py --no-cpu-baseline > gpurun_out/b.log 2>&1; echo -n "$v: "; tail -1 gpurun_out/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), round(d['e2e']['value']/1e9,3), round(d['ms_per_step'],2))"; done; done
