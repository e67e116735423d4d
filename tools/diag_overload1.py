"""One overloaded scenario (LBT-probe-like): device single-warp time vs the reference on one core."""
import sys, time
sys.path.insert(0, "/root/repo")
from paper_2202_13481_b200 import Engine
from paper_2202_13481_b200 import workloads as W
from tests import oracle_py as O
eng = Engine(0)
ref = O.best_oracle()
m = W.model("resnet50"); p = W.paris(m, 1); peak = W.capacity_qps(m, p)
for load, q in ((1.5, 2e4), (2.0, 2e4), (2.0, 1e5)):
    specs = [W._spec(m, p, load * peak, q, 1)]
    eng.run_grid(specs)
    t0 = time.perf_counter(); r = eng.run_grid(specs); dt = time.perf_counter() - t0
    t0 = time.perf_counter(); rr = ref.run_grid(specs, threads=1); ct = time.perf_counter() - t0
    print(f"P={p.total_instances()} load {load} q {q:.0f}: device {dt*1e3:.1f} ms, reference 1 core {ct*1e3:.1f} ms, "
          f"parity {bool((r['placement_hash'] == rr['placement_hash']).all())}", flush=True)
