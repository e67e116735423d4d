P=gpurun_out/r02/stream
mkdir -p $P
timeout 1800 python -m pytest tests -m gpu -x -q > $P/gpu_tests.log 2>&1; tail -2 $P/gpu_tests.log
timeout 1800 python tools/run_configs.py $P/configs.json > $P/configs.log 2>&1; tail -6 $P/configs.log | cut -c1-330
