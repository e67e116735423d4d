set -x
mkdir -p gpurun_out/r02/final
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02/final/gpu_tests.log 2>&1; tail -3 gpurun_out/r02/final/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02/final/smoke.log 2>&1; tail -2 gpurun_out/r02/final/smoke.log
timeout 900 python bench.py > gpurun_out/r02/final/bench.log 2>&1; tail -1 gpurun_out/r02/final/bench.log | cut -c1-400
timeout 900 python bench.py --impl reference > gpurun_out/r02/final/bench_ref.log 2>&1; tail -1 gpurun_out/r02/final/bench_ref.log | cut -c1-300
timeout 1800 python tools/run_configs.py gpurun_out/r02/final/configs.json > gpurun_out/r02/final/configs.log 2>&1; tail -8 gpurun_out/r02/final/configs.log
