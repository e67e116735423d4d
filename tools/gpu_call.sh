set -x
mkdir -p gpurun_out/r02/ab
MSV_LIB=_ab/libmsv_r01.so timeout 600 python tools/diag_classes.py > gpurun_out/r02/ab/classes_r01.log 2>&1
timeout 600 python tools/diag_classes.py > gpurun_out/r02/ab/classes_v2a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_warp_kernel --launch-count 1 -o gpurun_out/r02/ab/k2_c2_v2a python tools/prof_k2.py c2 > gpurun_out/r02/ab/ncu_v2a.log 2>&1
MSV_LIB=_ab/libmsv_r01.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:sim_warp_kernel --launch-count 1 -o gpurun_out/r02/ab/k2_c2_r01 python tools/prof_k2.py c2 > gpurun_out/r02/ab/ncu_r01.log 2>&1
cat gpurun_out/r02/ab/classes_*.log
