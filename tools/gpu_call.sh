P=gpurun_out/r02/final7
mkdir -p $P
timeout 1800 python -m pytest tests -m gpu -x -q > $P/gpu_tests.log 2>&1; tail -2 $P/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $P/smoke.log 2>&1; tail -1 $P/smoke.log
