set -x
T=v2m
P=gpurun_out/r02/prof
mkdir -p gpurun_out/r02/ab $P
for i in 1 2; do timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02/ab/bench_c5_${T}_$i.log 2>&1; done
MSV_SEG_WIDTH=8 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02/ab/bench_c5_${T}_w8.log 2>&1
MSV_SEG_WIDTH=16 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02/ab/bench_c5_${T}_w16.log 2>&1
N=$(python -c "import json; d=json.loads(open('$P/bench_1500.log').read().strip().splitlines()[-1]); print(d['gpu_launches']//d['steps'])")
KR='regex:sim_warp_kernel|sim_kernel|trace_gen_kernel|trace_group_kernel|tail_kernel'
MSV_CLASS_STREAMS=0 timeout 1800 ncu --set full --clock-control none --import-source on -k "$KR" --launch-skip $((3 * N)) --launch-count $N \
    -o $P/step_serial python bench.py --no-cpu-baseline --steps 1 --warmup 3 --scenarios 1500 > $P/ncu_step_serial.log 2>&1
for f in gpurun_out/r02/ab/bench_c5_${T}*.log; do echo $f; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); print(round(d['value']/1e9,3), round(d['e2e']['value']/1e9,3), d['clocks'])"; done
