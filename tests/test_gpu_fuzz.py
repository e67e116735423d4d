"""Randomised differential tests: the device engine vs the compiled reference on random
inputs (fixed seeds): random profiles (synthetic and hand-made), batch distributions,
partition plans (1..64 partitions, any mix of sizes), SLA / alpha / beta, loads from
idle to deep overload, warm-up fractions, both schedulers, and — through run() on host
traces — simultaneous arrivals, segment routing and the wait-consistency check. Every
output is compared bit for bit (per-query records, counts, horizons, tails, hashes)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2202_13481_b200 import (BatchDistribution, Engine, GridSpec, PartitionPlan, ProfileTable, SlaConfig,
                                   SyntheticProfileParams, derive_sla_target, lognormal_batch_pdf, synth_profile)
from paper_2202_13481_b200 import workloads as W
from tests import oracle_py as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    return Engine(0)


@pytest.fixture(scope="module")
def ref():
    if not O.REF_LIB.exists():
        pytest.skip("oracle/_ref not built")
    return O.Oracle("reference")


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype.kind == "f":
        return a.shape == b.shape and np.array_equal(a.view(np.uint64), np.asarray(b, np.float64).view(np.uint64))
    return np.array_equal(a, b)


def _random_table(rng, i):
    sizes = sorted(rng.choice([1, 2, 3, 4, 7], size=int(rng.integers(2, 6)), replace=False).tolist())
    b_max = int(rng.choice([4, 8, 16, 32]))
    if rng.random() < 0.6:
        p = SyntheticProfileParams(float(rng.uniform(0.3, 12.0)), float(rng.uniform(0.2, 6.0)),
                                   float(rng.uniform(0.05, 0.5)), float(rng.uniform(0.6, 1.0)))
        return synth_profile(p, sizes, b_max)
    n = len(sizes)
    row = np.cumsum(rng.uniform(0.05, 4.0, size=b_max))
    lat = np.stack([row * f for f in np.cumprod(rng.uniform(0.3, 1.0, size=n))])
    util = np.sort(rng.uniform(0.0, 1.0, size=(n, b_max)), axis=1)
    return ProfileTable(np.array(sizes, np.int32), b_max, lat, util, f"fuzz{i}")


def _random_plan(rng, sizes):
    gpus = int(rng.integers(1, 9))
    per = []
    for _ in range(gpus):
        left, g = 7, []
        while True:
            fit = [k for k in sizes if k <= left]
            if not fit or (g and rng.random() < 0.15):
                break
            k = int(rng.choice(fit))
            g.append(k)
            left -= k
        per.append(sorted(g, reverse=True))
    if sum(len(g) for g in per) == 0:
        per[0] = [int(sizes[0])]
    return PartitionPlan(gpus, 7, per)


def _fuzz_specs(seed, n):
    rng = np.random.default_rng(seed)
    specs = []
    for i in range(n):
        table = _random_table(rng, i)
        b = table.b_max
        dist = lognormal_batch_pdf(float(rng.uniform(0.0, 2.0)), float(rng.uniform(0.3, 1.5)), b) \
            if rng.random() < 0.7 else BatchDistribution(rng.uniform(0.0, 1.0, size=b) + 1e-3)
        plan = _random_plan(rng, [int(k) for k in table.sizes])
        m = W.Model("fuzz", table, dist, SlaConfig(1.0))
        cap = W.capacity_qps(m, plan)
        load = float(rng.choice([0.05, 0.3, 0.7, 0.95, 1.1, 1.6, 3.0]))
        sla_ms = derive_sla_target(table, b, float(rng.uniform(0.6, 3.0)))
        alpha, beta = (1.0, 1.0) if rng.random() < 0.6 else (float(rng.uniform(0.5, 1.5)), float(rng.uniform(0.5, 1.5)))
        queries = float(rng.choice([200, 1500, 4000]))
        rate = load * cap
        specs.append(GridSpec(plan, table, dist, SlaConfig(sla_ms, alpha, beta), rate, queries / rate * 1000.0,
                              int(rng.integers(1, 1 << 40)), "elsa" if rng.random() < 0.7 else "fifs",
                              float(rng.choice([0.0, 0.1, 0.5]))))
    return specs


def test_fuzz_grids(eng, ref):
    specs = _fuzz_specs(20260, 400)
    got, want = eng.run_grid(specs, (0.5, 0.95, 0.99)), ref.run_grid(specs, (0.5, 0.95, 0.99))
    for k in ("total", "violations", "measured", "measured_violations", "horizon_ms", "placement_hash", "tail",
              "status"):
        assert _same(got[k], want[k]), k


def test_fuzz_device_grid_many_profiles(eng, ref):
    """A device-resident grid whose profiles exceed one shared table (1,024 cells) is held as
    several sub-grids: launches, results, usage, queries and timing still cover the whole grid
    in the caller's order."""
    specs = _fuzz_specs(4242, 120)
    assert sum(s.table.latency.size for s in {id(s.table): s for s in specs}.values()) > 1024
    want = ref.run_grid(specs, (0.5, 0.99))
    use = eng.run_grid(specs, (0.5, 0.99), usage=True)["usage"]  # the split msv_run_grid path
    g = eng.grid(specs, (0.5, 0.99))
    for _ in range(2):
        g.launch()
        got = g.results(usage=True)
        for k in ("total", "violations", "measured", "measured_violations", "horizon_ms", "placement_hash", "tail",
                  "status"):
            assert _same(got[k], want[k]), k
        for k in use:
            assert _same(got["usage"][k], use[k]), k
    assert g.queries() == int(want["total"].sum())
    assert g.timing()["total_ms"] > 0
    g.set_usage(False)
    g.launch()
    assert _same(g.results()["tail"], want["tail"])
    g.close()


KEYS = ("partition", "kind", "start_ms", "finish_ms", "busy_ms", "weighted_busy_ms", "queries", "total",
        "violations", "measured", "measured_violations", "horizon_ms", "max_wait_estimate_diff")


def test_fuzz_runs_with_routing_and_checks(eng, ref):
    rng = np.random.default_rng(777)
    items, wants = [], []
    for i in range(120):
        table = _random_table(rng, 1000 + i)
        plan = _random_plan(rng, [int(k) for k in table.sizes])
        n = int(rng.integers(0, 600))
        gaps = rng.exponential(float(rng.uniform(0.2, 8.0)), size=n)
        gaps[rng.random(n) < 0.2] = 0.0  # simultaneous arrivals
        arrival = np.cumsum(gaps)
        batch = rng.integers(1, table.b_max + 1, size=n).astype(np.int32)
        duration = float(arrival[-1] * rng.uniform(0.5, 1.2)) if n else 100.0
        sla = SlaConfig(derive_sla_target(table, table.b_max, float(rng.uniform(0.5, 3.0))),
                        *((1.0, 1.0) if rng.random() < 0.5 else (float(rng.uniform(0.5, 1.5)), float(rng.uniform(0.5, 1.5)))))
        routing = None
        if rng.random() < 0.5:  # contiguous batch segments per size (paris.hpp:23-30 style)
            ks = [int(k) for k in table.sizes]
            cuts = sorted(rng.choice(np.arange(1, table.b_max), size=len(ks) - 1, replace=False).tolist()) \
                if table.b_max > len(ks) else list(range(1, len(ks)))
            lo, routing = 1, []
            for j, k in enumerate(ks):
                hi = cuts[j] if j < len(cuts) else table.b_max
                routing.append((k, lo, hi))
                lo = hi + 1
        check = bool(rng.random() < 0.5)
        sched = "elsa" if rng.random() < 0.6 else "fifs"
        warm = float(rng.choice([0.0, 0.1, 0.4]))
        got = eng.run(plan, sched, arrival, batch, duration, table, sla, warm, routing, check)
        want = ref.run(plan, sched, arrival, batch, duration, table, sla, warm, routing, check)
        for k in KEYS:
            assert _same(got[k], want[k]), (i, k)
        items.append((plan, sched, arrival, batch, duration, table, sla, warm, routing, check))
        wants.append(want)
    # all cases in one call: more profiles than one device table holds -> split grids
    for i, (got, want) in enumerate(zip(eng.run_many(items), wants)):
        for k in KEYS:
            assert _same(got[k], want[k]), ("batched", i, k)


def _fuzz_shared_stream_specs(seed, n):
    """Random grids whose scenarios share seeds and distributions (so chunked waves
    generate several traces per random stream), at random rates, lengths and plans."""
    rng = np.random.default_rng(seed)
    tables = [_random_table(rng, 5000 + i) for i in range(4)]
    dists = [lognormal_batch_pdf(float(rng.uniform(0.0, 2.0)), float(rng.uniform(0.3, 1.5)), t.b_max) for t in tables]
    specs = []
    for i in range(n):
        j = int(rng.integers(0, len(tables)))
        table, dist = tables[j], dists[j]
        plan = _random_plan(rng, [int(k) for k in table.sizes])
        m = W.Model("fuzz", table, dist, SlaConfig(1.0))
        rate = float(rng.choice([0.1, 0.5, 0.9, 1.2, 2.5])) * W.capacity_qps(m, plan)
        queries = float(rng.choice([50, 400, 1500, 3000]))
        sla_ms = derive_sla_target(table, table.b_max, float(rng.uniform(0.6, 3.0)))
        specs.append(GridSpec(plan, table, dist, SlaConfig(sla_ms), rate, queries / rate * 1000.0,
                              int(rng.integers(1, 12)), "elsa" if rng.random() < 0.7 else "fifs",
                              float(rng.choice([0.0, 0.1]))))
    return specs


def _fuzz_shared_results():
    r = Engine(0).run_grid(_fuzz_shared_stream_specs(99, 500), (0.5, 0.95, 0.99))
    return np.concatenate([r["placement_hash"].view(np.float64), r["tail"].ravel(), r["total"].astype(np.float64),
                           r["violations"].astype(np.float64)])


def test_fuzz_shared_streams_chunked(ref):
    """Random shared-stream grids through forced chunks (grouped trace generation) and the
    default layout: bit-identical to the reference."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    specs = _fuzz_shared_stream_specs(99, 500)
    w = ref.run_grid(specs, (0.5, 0.95, 0.99))
    want = np.concatenate([w["placement_hash"].view(np.float64), w["tail"].ravel(), w["total"].astype(np.float64),
                           w["violations"].astype(np.float64)])
    code = ("import sys, numpy as np; sys.path.insert(0, %r); from tests.test_gpu_fuzz import _fuzz_shared_results; "
            "np.save(sys.argv[1], _fuzz_shared_results())" % str(root))
    for extra in ({"MSV_CHUNK_SPLIT": "2,1,1,1"}, {"MSV_CHUNK_SPLIT": "1,1,1", "MSV_TRACE_GROUP_FIRST": "16"}, {}):
        out = Path(f"/tmp/msv_fz_{os.getpid()}.npy")
        r = subprocess.run([sys.executable, "-c", code, str(out)], capture_output=True, text=True,
                           env=dict(os.environ, **extra), timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        assert np.array_equal(np.load(out).view(np.uint64), want.view(np.uint64)), extra
