mkdir -p gpurun_out/r02/prof gpurun_out/r02/prof2
bash tools/profile_r02.sh > gpurun_out/r02/prof_run.log 2>&1
tail -3 gpurun_out/r02/prof_run.log
grep -h "^queries" gpurun_out/r02/prof/ncu_k2_*.log
P2=gpurun_out/r02/prof2
MSV_CLASS_STREAMS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tail_kernel --launch-skip 3 --launch-count 1 \
    -o $P2/k3 python bench.py --no-cpu-baseline --steps 1 --warmup 3 --scenarios 300 > $P2/ncu_k3.log 2>&1; tail -1 $P2/ncu_k3.log
