set -x
T=v2l
mkdir -p gpurun_out/r02
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02/gpu_tests_$T.log 2>&1
tail -n 3 gpurun_out/r02/gpu_tests_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke_$T.log 2>&1
timeout 2400 bash tools/profile_r02.sh
tail -c 600 gpurun_out/r02/prof/bench.log
