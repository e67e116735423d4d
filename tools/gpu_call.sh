set -x
mkdir -p gpurun_out/r02/ab
T=v2n
for i in 1 2; do timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02/ab/bench_c5_${T}_$i.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02/gpu_tests_$T.log 2>&1
tail -n 3 gpurun_out/r02/gpu_tests_$T.log
for f in gpurun_out/r02/ab/bench_c5_${T}*.log; do echo $f; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); print(round(d['value']/1e9,3), round(d['e2e']['value']/1e9,3), d['stage_ms'], d['roofline']['issue'], d['roofline']['traffic'])"; done
