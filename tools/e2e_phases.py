"""Host-side phases of one msv_run_grid call on the bench grid (MSV_HOST_TIMING=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MSV_HOST_TIMING"] = "1"
from paper_2202_13481_b200 import Engine
from paper_2202_13481_b200 import workloads as W
eng = Engine(0)
specs = W.c2(seeds=1024, queries=1e5)
prepared = eng.prepare(specs)
for i in range(4):
    t0 = time.perf_counter()
    eng.run_grid(prepared, (0.95, 0.99))
    print(f"run_grid {i}: {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr, flush=True)
