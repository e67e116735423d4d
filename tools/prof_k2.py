"""Launch one C2-shape (or C5 class) grid once, for an ncu capture of K2 (run with
MSV_MAX_CHUNKS=1: one K2 launch simulating every query of the grid):
    python tools/prof_k2.py [c2|MODEL PLAN] [n_scenarios]"""
import sys
sys.path.insert(0, "/root/repo")
from paper_2202_13481_b200 import Engine, homogeneous_plan
from paper_2202_13481_b200 import workloads as W
eng = Engine(0)
if sys.argv[1] == "c2":
    specs = W.c2(seeds=int(sys.argv[2]) if len(sys.argv) > 2 else 1024, queries=1e5)
else:
    m = W.model(sys.argv[1])
    pn = sys.argv[2]
    p = W.paris(m, int(pn[5:])) if pn.startswith("paris") else homogeneous_plan(int(pn[1:]), 56, 8, 7)
    specs = [W._spec(m, p, 0.8 * W.capacity_qps(m, p), 1e5, 1 + s) for s in range(int(sys.argv[3]) if len(sys.argv) > 3 else 4096)]
g = eng.grid(specs)
g.set_usage(False)
g.set_overlap(False)
g.launch()
eng.synchronize()
print("queries", g.queries(), g.timing())
