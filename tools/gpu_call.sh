mkdir -p gpurun_out/r02/var
for i in 1 2 3 4; do MSV_HOST_TIMING=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02/var/bench_$i.log 2>&1; grep "wave(s)" gpurun_out/r02/var/bench_$i.log | sort | uniq -c | head -5; tail -1 gpurun_out/r02/var/bench_$i.log | cut -c1-200; done
