"""Per-kernel-class simulation throughput on C5's plans at full occupancy (A/B helper):
    python tools/diag_classes.py [n_scenarios] [queries] [models...]"""
import sys
sys.path.insert(0, "/root/repo")
from paper_2202_13481_b200 import Engine, homogeneous_plan
from paper_2202_13481_b200 import workloads as W
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
q = float(sys.argv[2]) if len(sys.argv) > 2 else 1e5
models = sys.argv[3:] or ["mobilenet", "bert_base"]
eng = Engine(0)
for name in models:
    m = W.model(name)
    plans = {"paris8": W.paris(m, 8), "k1": homogeneous_plan(1, 56, 8, 7), "k2": homogeneous_plan(2, 56, 8, 7),
             "k3": homogeneous_plan(3, 56, 8, 7), "k7": homogeneous_plan(7, 56, 8, 7)}
    for pn, p in plans.items():
        specs = [W._spec(m, p, (0.3, 0.5, 0.7, 0.8, 0.9)[s % 5] * W.capacity_qps(m, p), q, 1 + s) for s in range(n)]
        g = eng.grid(specs)
        g.set_usage(False)
        g.set_overlap(False)
        g.launch()
        tm = g.timing()
        qq = g.queries()
        print(f"{name:9s} {pn:7s} P={p.total_instances():2d}  sim {qq / tm['sim_ms'] * 1e-6:6.2f} G q/s  "
              f"trace {qq / tm['trace_ms'] * 1e-6:6.1f}  tail {qq / tm['tail_ms'] * 1e-6:6.1f}", flush=True)
        g.close()
