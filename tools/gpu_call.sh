P=gpurun_out/r02/final3
mkdir -p $P
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "constant_latencies" > $P/t_const.log 2>&1; tail -2 $P/t_const.log
timeout 1800 python -m pytest tests -m gpu -x -q > $P/gpu_tests.log 2>&1; tail -2 $P/gpu_tests.log
