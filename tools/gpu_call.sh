set -x
mkdir -p gpurun_out/r02/ab
T=v2j
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02/gpu_tests_$T.log 2>&1
tail -n 3 gpurun_out/r02/gpu_tests_$T.log
timeout 600 python tools/diag_classes.py > gpurun_out/r02/ab/classes_$T.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02/bench_c5_$T.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02/bench_c5_${T}b.log 2>&1
timeout 900 python tools/diag_latency.py > gpurun_out/r02/ab/latency_$T.log 2>&1
timeout 1800 python tools/run_configs.py gpurun_out/r02/configs_$T.json > gpurun_out/r02/configs_$T.log 2>&1
cat gpurun_out/r02/ab/classes_$T.log gpurun_out/r02/ab/latency_$T.log
for f in gpurun_out/r02/bench_*_$T*.log; do echo $f; tail -c 800 $f | head -c 300; echo; done
