# Round-1 profile capture on one B200 (run under gpurun); summarise here with
#   python tools/summarize_profiles.py r01 gpurun_out/r01/step.ncu-rep --opcodes gpurun_out/r01/k2.ncu-rep \
#       --launches gpurun_out/r01/launches.csv --bench gpurun_out/r01/bench.log --reference gpurun_out/r01/bench_ref.log
set -x
mkdir -p gpurun_out/r01
python bench.py > gpurun_out/r01/bench.log 2>&1 || exit 1
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r01/bench_ref.log 2>&1
# the launch list of the same command (bench numbers never come from a profiled run)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01/launches.csv \
    python bench.py --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/r01/ncu_launch.log 2>&1
# every kernel of one step (after the three warm-up steps)
N=$(python -c "import json; d=json.loads(open('gpurun_out/r01/bench.log').read().strip().splitlines()[-1]); print(d['gpu_launches']//d['steps'])")
KR='regex:sim_warp_kernel|sim_kernel|trace_gen_kernel|trace_group_kernel|tail_kernel'
ncu --set full --clock-control none --import-source on -k "$KR" --launch-skip $((3 * N)) --launch-count $N \
    -o gpurun_out/r01/step python bench.py --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/r01/ncu_step.log 2>&1
# one K2 launch for the SASS opcode histogram (source page)
ncu --set full --clock-control none --import-source on -k regex:sim_warp_kernel --launch-skip 12 --launch-count 1 \
    -o gpurun_out/r01/k2 python bench.py --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/r01/ncu_k2.log 2>&1
tail -n 2 gpurun_out/r01/ncu_step.log gpurun_out/r01/ncu_k2.log
