"""Host-side cost breakdown of one-shot grids (debug helper; MSV_HOST_TIMING=1 for phases)."""
import sys, time
sys.path.insert(0, "/root/repo")
from paper_2202_13481_b200 import Engine
from paper_2202_13481_b200 import workloads as W
eng = Engine(0)
specs = W.c2(seeds=1024, queries=1e5)
prep = eng.prepare(specs)
for it in range(6):
    t0 = time.perf_counter(); eng.run_grid(prep); t1 = time.perf_counter()
    print(f"run_grid(prepared) {1e3*(t1-t0):.1f} ms", flush=True)
g = eng.grid(specs)
for it in range(3):
    t0 = time.perf_counter(); g.launch(); eng.synchronize(); t1 = time.perf_counter()
    print(f"device-resident launch {1e3*(t1-t0):.1f} ms", g.timing(), flush=True)
