"""Stage times (K1 / K2 / K3, device events) of the BASELINE configs' grids on one B200."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_13481_b200 import Engine
from paper_2202_13481_b200 import workloads as W
eng = Engine(0)
for name, specs in (("C1", W.c1()), ("C2-160", W.c2()), ("C3", W.c3()), ("C4", W.c4()[0])):
    g = eng.grid(specs, (0.95, 0.99))
    g.set_usage(False)
    g.set_overlap(False)
    g.launch()
    g.results()
    g.launch()
    print(name, len(specs), g.timing(), flush=True)
    g.close()
