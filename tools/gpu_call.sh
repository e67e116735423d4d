set -x
mkdir -p gpurun_out/r02/ab
for v in base s1b6 s1b8q8; do
  MSV_LIB=_ab/libmsv_$v.so timeout 600 python tools/diag_classes.py 16384 1e5 bert_base > gpurun_out/r02/ab/classes_$v.log 2>&1
  for i in 1 2; do MSV_LIB=_ab/libmsv_$v.so timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02/ab/bench_c5_${v}_$i.log 2>&1; done
done
MSV_LIB=_ab/libmsv_s1b8q8.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fuzz or overload or c5_slice or grid" > gpurun_out/r02/ab/tests_s1b8q8.log 2>&1
tail -2 gpurun_out/r02/ab/tests_s1b8q8.log
for v in base s1b6 s1b8q8; do cat gpurun_out/r02/ab/classes_$v.log | cut -c1-50; for i in 1 2; do python -c "
import json
d=json.loads(open('gpurun_out/r02/ab/bench_c5_${v}_$i.log').read().strip().splitlines()[-1]); print('$v', round(d['value']/1e9,3), round(d['e2e']['value']/1e9,3))"; done; done
