P=gpurun_out/r02/final8
mkdir -p $P
timeout 1800 python -m pytest tests -m gpu -x -q > $P/gpu_tests.log 2>&1; tail -1 $P/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $P/smoke.log 2>&1; tail -1 $P/smoke.log
timeout 900 python bench.py > $P/bench.log 2>&1; tail -1 $P/bench.log | cut -c1-120
