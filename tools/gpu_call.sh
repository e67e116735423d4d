MSV_HOST_TIMING=1 timeout 1200 python tools/run_configs.py gpurun_out/cfg_t.json > gpurun_out/cfg_t.log 2>&1
grep -n "n=6870\|run_grid n=6870" gpurun_out/cfg_t.log | head -12
grep '"C4"' gpurun_out/cfg_t.log | cut -c1-250
