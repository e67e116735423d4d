timeout 900 python -m pytest tests -m gpu -x -q -k "noise" 2>&1 | tail -1
for i in 1 2; do timeout 600 python tools/_nb1.py; done
timeout 900 python tools/noise_bench.py 1e5 2>&1 | tail -5 | cut -c150-330
timeout 900 python tools/noise_grid_bench.py 2>&1 | tail -3
