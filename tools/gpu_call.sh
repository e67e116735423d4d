set -x
mkdir -p gpurun_out/r02/ab
T=v2g
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02/gpu_tests_$T.log 2>&1
tail -n 3 gpurun_out/r02/gpu_tests_$T.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02/bench_c5_$T.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --workload c2 > gpurun_out/r02/bench_c2_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_warp_kernel --launch-count 1 -o gpurun_out/r02/ab/k2_c2_$T python tools/prof_k2.py c2 > gpurun_out/r02/ab/ncu_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_warp_kernel --launch-count 1 -o gpurun_out/r02/ab/k2_s2_$T python tools/prof_k2.py mobilenet k1 4096 > gpurun_out/r02/ab/ncu_s2_$T.log 2>&1
for f in gpurun_out/r02/bench_*_$T*.log; do echo $f; tail -c 800 $f | head -c 300; echo; done
