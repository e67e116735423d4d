"""Host-side cost breakdown of one-shot grids (debug helper)."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import ctypes as C
from paper_2202_13481_b200 import Engine
from paper_2202_13481_b200 import workloads as W
from paper_2202_13481_b200 import _native as N
eng = Engine(0)
specs = W.c2(seeds=1024, queries=1e5)
eng.run_grid(specs)
for it in range(3):
    t0 = time.perf_counter(); sc = eng.scenarios(specs); t1 = time.perf_counter()
    n = len(specs); ps = np.array([0.95, 0.99]); res = (N.Result * n)()
    rc = eng._lib.msv_run_grid(eng._h, sc, n, ps.ctypes.data_as(C.POINTER(C.c_double)), 2, res, None); t2 = time.perf_counter()
    from paper_2202_13481_b200.engine import results_to_numpy
    r = results_to_numpy(res, n, 2); t3 = time.perf_counter()
    print(f"marshal {1e3*(t1-t0):.1f} ms  msv_run_grid {1e3*(t2-t1):.1f} ms  unpack {1e3*(t3-t2):.1f} ms", flush=True)
g = eng.grid(specs)
for it in range(3):
    t0 = time.perf_counter(); g.launch(); eng.synchronize(); t1 = time.perf_counter()
    print(f"device-resident launch {1e3*(t1-t0):.1f} ms", g.timing(), flush=True)
