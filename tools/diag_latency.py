"""Single-scenario latency (debug helper): small grids are bound by one warp's serial chain."""
import sys, time
sys.path.insert(0, "/root/repo")
from paper_2202_13481_b200 import Engine
from paper_2202_13481_b200 import workloads as W
eng = Engine(0)
for name, specs in (("C1 (1 x 1e5)", W.c1(queries=1e5)), ("C3-like (192 x 1e6)", W.c3(seeds=64, queries=1e6)),
                    ("C2 1 seed (10 x 1e5)", W.c2(seeds=1, queries=1e5))):
    g = eng.grid(specs)
    g.set_usage(False)
    g.launch(); eng.synchronize()
    g.set_overlap(False)
    g.launch()
    tm = g.timing()
    q = g.queries()
    print(f"{name}: {q} queries, stages {({k: round(v, 2) for k, v in tm.items()})}, "
          f"{q / tm['total_ms'] * 1e-6:.3f} G q/s, sim ns/arrival/scenario {tm['sim_ms'] * 1e6 / (q / len(specs)):.1f}",
          flush=True)
    g.close()
