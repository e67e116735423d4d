mkdir -p gpurun_out/r02/extra
timeout 1500 python tools/diag_lbt.py > gpurun_out/r02/extra/lbt.log 2>&1; cat gpurun_out/r02/extra/lbt.log | cut -c1-300
timeout 900 python tools/noise_bench.py 1e5 > gpurun_out/r02/extra/noise_bench.log 2>&1; tail -5 gpurun_out/r02/extra/noise_bench.log | cut -c1-100
