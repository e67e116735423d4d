timeout 900 python -m pytest tests -m gpu -x -q -k "noise" 2>&1 | tail -1
for v in base redux base redux; do echo "== $v"; MSV_LIB=_ab/$v.so timeout 600 python tools/_nb1.py; done
MSV_LIB=_ab/redux.so timeout 900 python tools/noise_grid_bench.py 2>&1 | tail -3
