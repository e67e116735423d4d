"""One class grid (debug helper): python tools/diag_one.py MODEL PLAN [n_scen]  (PLAN: k1..k7, paris1, paris8)."""
import sys
sys.path.insert(0, "/root/repo")
from paper_2202_13481_b200 import Engine, homogeneous_plan
from paper_2202_13481_b200 import workloads as W
name, pn = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
sched = sys.argv[4] if len(sys.argv) > 4 else "elsa"
m = W.model(name)
p = W.paris(m, int(pn[5:])) if pn.startswith("paris") else homogeneous_plan(int(pn[1:]), 56, 8, 7)
rate = 0.8 * W.capacity_qps(m, p)
eng = Engine(0)
g = eng.grid([W._spec(m, p, rate, 1e5, 1 + s, sched) for s in range(n)])
g.set_overlap(False)
g.set_usage(False)
g.launch()
tm = g.timing()
print(f"{name} {pn} {sched} P={p.total_instances()} sim {g.queries() / tm['sim_ms'] * 1e-6:.2f} G q/s", flush=True)
g.close()
