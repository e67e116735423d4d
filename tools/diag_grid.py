"""Staged timing of one large grid (debug helper): create, trace, sim, tail."""
import sys, time, faulthandler
sys.path.insert(0, "/root/repo")
faulthandler.dump_traceback_later(100, exit=True)
from paper_2202_13481_b200 import Engine
from paper_2202_13481_b200 import workloads as W
seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 512
eng = Engine(0)
specs = W.c2(seeds=seeds, queries=1e5)
t = time.time(); g = eng.grid(specs); print("create", time.time() - t, flush=True)
for it in range(2):
    t = time.time(); g.launch(); eng.synchronize(); print("launch", it, time.time() - t, g.timing(), flush=True)
t = time.time(); r = g.results(); print("results", time.time() - t, r["status"].max(), flush=True)
t = time.time(); r2 = eng.run_grid(specs); print("run_grid", time.time() - t, flush=True)
t = time.time(); r2 = eng.run_grid(specs); print("run_grid2", time.time() - t, flush=True)
