"""Repeated one-shot grids (debug helper)."""
import sys, time, faulthandler
sys.path.insert(0, "/root/repo")
faulthandler.dump_traceback_later(60, exit=True)
import numpy as np
from paper_2202_13481_b200 import Engine
from paper_2202_13481_b200 import workloads as W
seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 64
eng = Engine(0)
specs = W.c2(seeds=seeds, queries=1e5)
ref = None
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 6):
    t = time.time(); r = eng.run_grid(specs)
    nan = int(np.isnan(r["tail"]).sum())
    same = ref is None or (np.array_equal(r["placement_hash"], ref["placement_hash"]) and np.array_equal(r["tail"], ref["tail"], equal_nan=True))
    ref = ref or r
    print("run_grid", it, round(time.time() - t, 3), "nan_tails", nan, "same", same, flush=True)
