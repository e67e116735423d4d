P=gpurun_out/r02/prof2
mkdir -p $P
timeout 900 python bench.py > $P/bench.log 2>&1; tail -1 $P/bench.log | cut -c1-200
MSV_CLASS_STREAMS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_kernel --launch-skip 3 --launch-count 1 \
    -o $P/k3 python bench.py --no-cpu-baseline --steps 1 --warmup 3 --scenarios 300 > $P/ncu_k3.log 2>&1; tail -1 $P/ncu_k3.log
timeout 900 python tools/diag_latency.py > $P/latency.log 2>&1; cat $P/latency.log
