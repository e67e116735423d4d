mkdir -p gpurun_out/r02/prof
bash tools/profile_r02.sh > gpurun_out/r02/prof_run.log 2>&1
tail -5 gpurun_out/r02/prof_run.log
grep -h "^queries" gpurun_out/r02/prof/ncu_k2_*.log
