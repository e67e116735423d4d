import sys; sys.path.insert(0, "/root/repo")
from paper_2202_13481_b200 import Engine
from paper_2202_13481_b200 import workloads as W
eng = Engine(0)
specs = W.c2(seeds=1024, queries=1e5)
for tails in ((0.95, 0.99), ()):
    g = eng.grid(specs, tails); g.set_usage(False)
    for _ in range(3): g.launch()
    eng.synchronize()
    eng.event_record(0)
    for _ in range(5): g.launch()
    eng.event_record(1)
    print(tails, eng.event_elapsed_ms(0, 1) / 5, flush=True)
    g.close()
