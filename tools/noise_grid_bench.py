"""Noisy sweep at grid scale: N scenarios with execution noise through
msv_run_grid_noise vs the compiled reference's sample_trace -> run(noise) ->
tail_latency on every host core (ctypes calls release the GIL: one Python thread per
core), with a bit-exactness check on a sample of scenarios.

    python tools/noise_grid_bench.py [n_scenarios] [queries] [sample]"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_13481_b200 import Engine, GridSpec  # noqa: E402
from paper_2202_13481_b200 import workloads as W  # noqa: E402
from tests import oracle_py as O  # noqa: E402
from tests.test_gpu_parity import _digest_sum  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
queries = float(sys.argv[2]) if len(sys.argv) > 2 else 1e5
sample = int(sys.argv[3]) if len(sys.argv) > 3 else 64
rng = np.random.default_rng(1)
specs, sig, seeds = [], [], []
models = [(nm, W.model(nm)) for nm in ("mobilenet", "resnet50", "bert_base")]
for i in range(n):
    nm, m = models[i % 3]
    plan = W.paris(m, 8 if nm != "mobilenet" else 4)  # P <= 64 (K5)
    load = (0.5, 0.7, 0.9)[(i // 3) % 3]
    rate = load * W.capacity_qps(m, plan)
    specs.append(GridSpec(plan, m.table, m.dist, m.sla, rate, queries / rate * 1000.0, 1 + i, "elsa"))
    sig.append((0.1, 0.3)[i % 2])
    seeds.append(1000 + i)
eng = Engine(0)
eng.run_grid_noise(specs[:8], sig[:8], seeds[:8])  # warm-up (module load, buffers)
t0 = time.perf_counter()
got = eng.run_grid_noise(specs, sig, seeds, (0.95, 0.99))
dt = time.perf_counter() - t0
q = int(got["total"].sum())
print(f"device: {n} noisy scenarios, {q} queries in {dt:.3f} s end to end = {q / dt / 1e6:.1f} M q/s", flush=True)

ref = O.best_oracle()
cores = len(os.sched_getaffinity(0))
idx = list(range(0, n, max(1, n // sample)))[:sample]


def one(k):
    s = specs[k]
    arr, bat = ref.sample_trace(s.dist, s.rate_qps, s.duration_ms, s.seed)
    r = ref.run_noise(s.plan, s.scheduler, arr, bat, s.duration_ms, s.table, s.sla, s.warmup_fraction, None, sig[k],
                      seeds[k])
    lat = r["finish_ms"] - arr
    meas = lat[arr >= r["warmup_ms"]]
    return k, len(arr), r, meas


t0 = time.perf_counter()
with ThreadPoolExecutor(cores) as ex:
    out = list(ex.map(one, idx))
rdt = time.perf_counter() - t0
rq = sum(o[1] for o in out)
print(f"reference: {len(idx)} of the scenarios, {rq} queries in {rdt:.2f} s on {cores} threads = "
      f"{rq / rdt / 1e6:.2f} M q/s -> device/reference {q / dt / (rq / rdt):.1f}x", flush=True)
bad = 0
for k, nq, r, meas in out:
    ok = (got["total"][k] == nq and got["violations"][k] == r["violations"] and got["measured"][k] == r["measured"]
          and int(got["placement_hash"][k]) == _digest_sum(r["partition"], r["start_ms"], r["finish_ms"])
          and got["horizon_ms"][k] == r["horizon_ms"]
          and (len(meas) == 0 or got["tail"][k, 1] == ref.tail_latency(meas, 0.99)))
    bad += not ok
print(f"parity on {len(out)} scenarios: {'all equal' if bad == 0 else f'{bad} differ'}")
