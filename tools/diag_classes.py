"""Per-kernel-class throughput on C5-style plans (debug helper)."""
import sys, time
sys.path.insert(0, "/root/repo")
from paper_2202_13481_b200 import Engine, homogeneous_plan
from paper_2202_13481_b200 import workloads as W
eng = Engine(0)
for name in ("mobilenet", "bert_base"):
    m = W.model(name)
    plans = {"paris8": W.paris(m, 8), "k1": homogeneous_plan(1, 56, 8, 7), "k2": homogeneous_plan(2, 56, 8, 7),
             "k3": homogeneous_plan(3, 56, 8, 7), "k7": homogeneous_plan(7, 56, 8, 7), "paris1": W.paris(m, 1)}
    for pn, p in plans.items():
        rate = 0.8 * W.capacity_qps(m, p)
        specs = [W._spec(m, p, rate, 1e5, 1 + s) for s in range(4096)]
        g = eng.grid(specs); g.launch(); g.set_overlap(False); g.launch(); tm = g.timing()
        q = g.queries()
        print(f"{name:9s} {pn:7s} P={p.total_instances():2d}  sim {q / tm['sim_ms'] * 1e-6:6.2f} G q/s  trace {q / tm['trace_ms'] * 1e-6:6.1f}  tail {q / tm['tail_ms'] * 1e-6:6.1f}", flush=True)
        g.close()
