timeout 900 python -m pytest tests -m gpu -x -q -k "noise" 2>&1 | tail -1
timeout 900 python tools/noise_bench.py 1e5 > gpurun_out/nb.log 2>&1; tail -5 gpurun_out/nb.log | cut -c150-330
