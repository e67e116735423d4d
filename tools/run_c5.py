"""C5: 1e4 scenarios x 1e6 queries on one B200 (multi-wave), with a reference spot check."""
import sys, time, os, json
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2202_13481_b200 import Engine
from paper_2202_13481_b200 import workloads as W
from tests import oracle_py as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
q = float(sys.argv[2]) if len(sys.argv) > 2 else 1e6
eng = Engine(0)
specs = W.c5(n_scenarios=n, queries=q)
t0 = time.perf_counter(); g = eng.grid(specs); g.set_usage(False); t1 = time.perf_counter()
g.launch(); tm = g.timing(); t2 = time.perf_counter()
r = g.results()
tot = int(r["total"].sum())
print(json.dumps({"scenarios": n, "queries": tot, "create_s": round(t1 - t0, 3), "launch_s": round(t2 - t1, 3),
                  "device_ms": tm["total_ms"], "G_qps": tot / (tm["total_ms"] / 1e3) / 1e9,
                  "status_max": int(r["status"].max())}), flush=True)
cores = len(os.sched_getaffinity(0))
idx = list(range(0, n, max(1, n // cores)))[:cores]
t0 = time.perf_counter(); rr = O.best_oracle().run_grid([specs[i] for i in idx], threads=cores); ct = time.perf_counter() - t0
print(json.dumps({"reference_spot_check": len(idx), "reference_qps": float(rr["total"].sum() / ct),
                  "hash_equal": bool(np.array_equal(r["placement_hash"][idx], rr["placement_hash"])),
                  "tails_equal": bool(np.array_equal(r["tail"][idx], rr["tail"], equal_nan=True))}), flush=True)
