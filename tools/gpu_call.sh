MSV_HOST_TIMING=1 timeout 600 python tools/diag_host.py 2>&1 | tail -12
