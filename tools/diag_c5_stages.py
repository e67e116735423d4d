"""C5 stage breakdown (debug helper): per-class scenario counts and stage times."""
import sys, collections
sys.path.insert(0, "/root/repo")
from paper_2202_13481_b200 import Engine
from paper_2202_13481_b200 import workloads as W
eng = Engine(0)
specs = W.c5(n_scenarios=int(sys.argv[1]) if len(sys.argv) > 1 else 10000, queries=1e6)
print(collections.Counter(s.plan.total_instances() for s in specs))
g = eng.grid(specs)
g.set_usage(False)
g.set_overlap(False)
g.launch()
print(g.timing(), g.queries(), flush=True)
