set -x
mkdir -p gpurun_out/r02/ab
for o in default slow; do
  MSV_CLASS_ORDER=$o timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02/ab/bench_c5_order_$o.log 2>&1
  MSV_CLASS_ORDER=$o timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02/ab/bench_c5_order_${o}2.log 2>&1
done
for f in gpurun_out/r02/ab/bench_c5_order_*.log; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/1e9,3), round(d['e2e']['value']/1e9,3), d['stage_ms'])"; done
