P=gpurun_out/r02/noise
mkdir -p $P
timeout 900 python -m pytest tests -m gpu -x -q -k "noise" > $P/t.log 2>&1; tail -2 $P/t.log
MSV_HOST_TIMING=1 timeout 900 python tools/noise_grid_bench.py > $P/nb.log 2>&1; grep -E "msv|device:|reference|parity" $P/nb.log | tail -5
timeout 900 python tools/noise_grid_bench.py > $P/nb2.log 2>&1; tail -3 $P/nb2.log
