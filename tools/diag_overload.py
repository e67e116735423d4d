"""Throughput at and beyond saturation: device vs the compiled reference (debug helper)."""
import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2202_13481_b200 import Engine
from paper_2202_13481_b200 import workloads as W
from tests import oracle_py as O
eng = Engine(0)
ref = O.best_oracle()
m = W.model("bert_base"); p = W.paris(m, 8); peak = W.capacity_qps(m, p)
cores = len(os.sched_getaffinity(0))
for load in (0.9, 1.0, 1.2, 1.5, 2.0, 3.0):
    q = 2e4
    specs = [W._spec(m, p, load * peak, q, 1 + s) for s in range(1024)]
    eng.run_grid(specs[:64])
    t0 = time.perf_counter(); r = eng.run_grid(specs); dt = time.perf_counter() - t0
    gq = r["total"].sum() / dt
    sub = specs[:cores]
    t0 = time.perf_counter(); rr = ref.run_grid(sub, threads=cores); ct = time.perf_counter() - t0
    cq = rr["total"].sum() / ct
    same = np.array_equal(r["placement_hash"][:cores], rr["placement_hash"])
    print(f"load {load}: device {gq/1e9:.3f} G q/s ({dt*1e3:.0f} ms)  reference {cq/1e6:.3f} M q/s on {cores} cores  ratio {gq/cq:.0f}x  parity {same}", flush=True)
