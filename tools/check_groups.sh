python -m pytest tests/test_gpu_parity.py -x -q -k "shared_random or chunking" > gpurun_out/t.log 2>&1; echo rc=$? >> gpurun_out/t.log
python bench.py > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 600 python tools/run_c5.py > gpurun_out/c5.log 2>&1
