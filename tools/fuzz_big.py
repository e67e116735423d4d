"""One-off larger randomised differential run (debug helper): device vs compiled reference."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2202_13481_b200 import (BatchDistribution, Engine, GridSpec, PartitionPlan, ProfileTable, SlaConfig,
                                   SyntheticProfileParams, derive_sla_target, lognormal_batch_pdf, synth_profile)
from paper_2202_13481_b200 import workloads as W
from tests import oracle_py as O
from tests.test_gpu_fuzz import _random_table, _same
eng = Engine(0)
ref = O.Oracle("reference")
bad = 0
for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    rng = np.random.default_rng(1000 + seed)
    specs = []
    for i in range(600):
        table = _random_table(rng, i)
        b = table.b_max
        dist = lognormal_batch_pdf(float(rng.uniform(0.0, 2.5)), float(rng.uniform(0.2, 2.0)), b)
        gpus = int(rng.integers(1, 17))
        ks = [int(k) for k in table.sizes]
        per = []
        for _ in range(gpus):
            left, g = 7, []
            while True:
                fit = [k for k in ks if k <= left]
                if not fit:
                    break
                k = int(rng.choice(fit)); g.append(k); left -= k
            per.append(sorted(g, reverse=True))
        plan = PartitionPlan(gpus, 7, per)
        m = W.Model("f", table, dist, SlaConfig(1.0))
        cap = W.capacity_qps(m, plan)
        load = float(rng.choice([0.01, 0.2, 0.5, 0.8, 0.99, 1.02, 1.3, 2.0, 5.0]))
        sla = SlaConfig(derive_sla_target(table, b, float(rng.uniform(0.3, 4.0))),
                        *((1.0, 1.0) if rng.random() < 0.5 else (float(rng.uniform(0.2, 2.0)), float(rng.uniform(0.0, 2.0)))))
        q = float(rng.choice([50, 1000, 8000, 20000]))
        rate = load * cap
        specs.append(GridSpec(plan, table, dist, sla, rate, q / rate * 1000.0, int(rng.integers(1, 1 << 62)),
                              "elsa" if rng.random() < 0.75 else "fifs", float(rng.choice([0.0, 0.05, 0.1, 0.9]))))
    got, want = eng.run_grid(specs, (0.01, 0.5, 0.95, 0.999)), ref.run_grid(specs, (0.01, 0.5, 0.95, 0.999))
    for k in ("total", "violations", "measured", "measured_violations", "horizon_ms", "placement_hash", "tail", "status"):
        if not _same(got[k], want[k]):
            a, b2 = np.asarray(got[k]), np.asarray(want[k])
            idx = np.nonzero(~np.all((a == b2) | (np.isnan(a) & np.isnan(b2)) if a.dtype.kind == 'f' else (a == b2), axis=tuple(range(1, a.ndim))))[0] if a.ndim > 1 else np.nonzero(a != b2)[0]
            print("MISMATCH seed", seed, k, idx[:10], flush=True)
            bad += 1
    print("seed", seed, "ok" if bad == 0 else "BAD", "P range", min(s.plan.total_instances() for s in specs),
          max(s.plan.total_instances() for s in specs), "queries", int(got["total"].sum()), flush=True)
print("bad", bad)
