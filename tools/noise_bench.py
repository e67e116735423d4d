"""K5 (run() with execution noise, engine.hpp:140-145) on one B200 vs the reference's run()
with EngineOptions::noise_sigma on one host core (oracle/_ref), same trace and noise seed.

Times one API call each way (device: Engine.run(noise_sigma, noise_seed) with per-query records
back on the host; reference: oraref_run_noise), after one warm-up call, and checks that the
records are byte-identical. Usage: python tools/noise_bench.py [max_queries]
"""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
from paper_2202_13481_b200 import Engine  # noqa: E402
from paper_2202_13481_b200 import workloads as W  # noqa: E402
from tests import oracle_py as O  # noqa: E402

eng = Engine(0)
ref = O.best_oracle()
assert ref.kind == "reference", "needs oracle/_ref (the C port has no noise path)"
qmax = float(sys.argv[1]) if len(sys.argv) > 1 else 1e6
rows = []
for m, gpus, sched, load, sigma in (("bert_base", 8, "elsa", 0.5, 0.1), ("bert_base", 8, "elsa", 0.9, 0.3),
                                    ("resnet50", 8, "elsa", 0.9, 0.3), ("mobilenet", 8, "fifs", 0.9, 0.3),
                                    ("bert_base", 8, "elsa", 1.3, 0.3)):  # overloaded: queues grow
    mod = W.model(m)
    plan = W.paris(mod, gpus)
    rate = load * W.capacity_qps(mod, plan)
    for q in (1e5, 1e6):
        if q > qmax:
            continue
        duration = q / rate * 1000.0
        arr, bat = ref.sample_trace(mod.dist, rate, duration, 11)
        args = (plan, sched, arr, bat, duration, mod.table, mod.sla, 0.1, None)
        eng.run(*args, tail_p=(0.99,), noise_sigma=sigma, noise_seed=5)  # warm-up
        t0 = time.perf_counter()
        got = eng.run(*args, tail_p=(0.99,), noise_sigma=sigma, noise_seed=5)
        dt = time.perf_counter() - t0
        t0 = time.perf_counter()
        want = ref.run_noise(*args, sigma, 5)
        ct = time.perf_counter() - t0
        ok = all(np.array_equal(np.asarray(got[k]), np.asarray(want[k]))
                 for k in ("partition", "kind", "start_ms", "finish_ms", "busy_ms", "queries"))
        n = len(arr)
        import ctypes as C
        mult = np.zeros(n)
        t0 = time.perf_counter()
        eng._lib.msv_noise_multipliers(5, float(sigma), n, mult.ctypes.data_as(C.POINTER(C.c_double)))
        mt = time.perf_counter() - t0
        row = dict(model=m, gpus=gpus, partitions=plan.total_instances(), sched=sched, load=load,
                   sigma=sigma, queries=n, device_ms=round(dt * 1e3, 2), host_multiplier_draw_ms=round(mt * 1e3, 2), reference_1core_ms=round(ct * 1e3, 2),
                   device_qps=round(n / dt), reference_qps=round(n / ct), speedup=round(ct / dt, 1),
                   records_identical=ok)
        rows.append(row)
        print(row, flush=True)
assert all(r["records_identical"] for r in rows)
