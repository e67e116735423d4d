set -x
mkdir -p gpurun_out/r01
python bench.py > gpurun_out/r01/bench.log 2>&1 || exit 1
python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/r01/bench_ref.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01/launches.csv python bench.py --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/r01/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sim_warp_kernel|trace_gen|tail_kernel" -c 3 -o gpurun_out/r01/full python bench.py --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/r01/ncu_full.log 2>&1
tail -2 gpurun_out/r01/ncu_full.log
