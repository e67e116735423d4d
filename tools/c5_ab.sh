python tools/run_c5.py 10000 1e6 2>&1 | head -1
MSV_CHUNK_SPLIT=1,1 python tools/run_c5.py 10000 1e6 2>&1 | head -1
MSV_MAX_CHUNKS=1 python tools/run_c5.py 10000 1e6 2>&1 | head -1
