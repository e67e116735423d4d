P=gpurun_out/r02/noise4
mkdir -p $P
timeout 900 python -m pytest tests -m gpu -x -q -k "noise" > $P/t.log 2>&1; tail -3 $P/t.log
timeout 1800 python -m pytest tests -m gpu -x -q > $P/gpu_tests.log 2>&1; tail -2 $P/gpu_tests.log
