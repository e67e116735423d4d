# Round-2 capture on one B200 (run under gpurun); summarise here with tools/summarize_profiles.py
# (see profiles/r02/README.md for the exact command).
set -x
P=gpurun_out/r02/prof
mkdir -p $P
python bench.py > $P/bench.log 2>&1 || exit 1
python bench.py --impl reference > $P/bench_ref.log 2>&1
# the launch list of the same command (bench numbers never come from a profiled run)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches.csv \
    python bench.py --no-cpu-baseline --steps 2 --warmup 3 > $P/ncu_launch.log 2>&1
# every kernel of one step of a one-wave C5 grid (300 scenarios x 1e6 queries: every plan and load)
python bench.py --no-cpu-baseline --steps 1 --warmup 3 --scenarios 300 > $P/bench_300.log 2>&1
N=$(python -c "import json; d=json.loads(open('$P/bench_300.log').read().strip().splitlines()[-1]); print(d['gpu_launches']//d['steps'])")
KR='regex:sim_warp_kernel|sim_kernel|trace_gen_kernel|trace_group_kernel|tail_kernel'
MSV_CLASS_STREAMS=0 ncu --set full --clock-control none --import-source on -k "$KR" --launch-skip $((3 * N)) --launch-count $N \
    -o $P/step python bench.py --no-cpu-baseline --steps 1 --warmup 3 --scenarios 300 > $P/ncu_step.log 2>&1
# one K2 launch of the C2-shape grid (one slot per lane) and of a P = 56 grid (two slots), source-level
# (MSV_MAX_CHUNKS=1: one K2 launch simulates every query the script prints)
MSV_MAX_CHUNKS=1 ncu --set full --clock-control none --import-source on -k regex:sim_warp_kernel --launch-count 1 \
    -o $P/k2_c2 python tools/prof_k2.py c2 > $P/ncu_k2_c2.log 2>&1
MSV_MAX_CHUNKS=1 ncu --set full --clock-control none --import-source on -k regex:sim_warp_kernel --launch-count 1 \
    -o $P/k2_p56 python tools/prof_k2.py mobilenet k1 4096 > $P/ncu_k2_p56.log 2>&1
tail -n 2 $P/ncu_step.log $P/ncu_k2_c2.log $P/ncu_k2_p56.log
