"""K4 (batched paris_plan on the device) vs the reference's paris_plan (paris.hpp:329-345):
identical knees, bit-identical ratios / counts, identical packed plans, and the same
exception class for every failing job (test_paris.cpp:264-324 covers the pipeline the
reference pins; here thousands of random profiles/distributions/fleets stress it)."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2202_13481_b200 import (BatchDistribution, Engine, ParisJob, ProfileTable, SyntheticProfileParams,
                                   lognormal_batch_pdf, paris_plan, synth_profile)
from paper_2202_13481_b200 import _native as N
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


def _ref_outcome(ref, j: ParisJob):
    try:
        return ref.paris_plan(j.table, j.dist, j.total_gpcs, j.num_gpus, j.gpcs_per_gpu, j.knee_threshold), None
    except Exception as e:  # noqa: BLE001 - the class is what we compare
        return None, e


def _compare(eng, ref, jobs):
    got = eng.paris_batch(jobs)
    n_ok = 0
    for j, g in zip(jobs, got):
        want, err = _ref_outcome(ref, j)
        if err is not None:
            assert g.error is not None, (j, err)
            code = {v: k for k, v in N._ERRORS.items()}[type(g.error)]
            assert (code, f"[{code}] {g.error}") == (err.code, str(err)), (j, g.error, err)
            continue
        assert g.error is None, (j, g.error)
        ks = [int(k) for k in j.table.sizes]
        assert [g.knees[k] for k in ks] == [int(x) for x in want["knees"]]
        assert np.array_equal(np.array(g.ratios).view(np.uint64), want["ratios"].view(np.uint64))
        assert np.array_equal(np.array(g.counts).view(np.uint64), want["counts"].view(np.uint64))
        assert g.plan.gpus == want["gpus"]
        n_ok += 1
    return n_ok


def test_paris_batch_presets_match_host_and_reference(eng, ref):
    from paper_2202_13481_b200 import workloads as W
    jobs = []
    for name in ("mobilenet", "resnet50", "bert_base"):
        m = W.model(name)
        for gpus in (1, 2, 4, 8):
            for thr in (0.5, 0.8, 0.95, 1.0):
                jobs.append(ParisJob(m.table, m.dist, 7 * gpus, gpus, 7, thr))
    assert _compare(eng, ref, jobs) == len(jobs)
    # the host C++ header path gives the same plan
    for j, g in zip(jobs, eng.paris_batch(jobs)):
        assert paris_plan(j.table, j.dist, j.total_gpcs, j.num_gpus, j.gpcs_per_gpu, j.knee_threshold).gpus == \
            g.plan.gpus


def test_paris_batch_random_synthetic(eng, ref):
    rng = np.random.default_rng(7)
    all_sizes = [1, 2, 3, 4, 7]
    jobs = []
    for _ in range(1500):
        sizes = sorted(rng.choice(all_sizes, size=int(rng.integers(1, 6)), replace=False).tolist())
        b_max = int(rng.choice([4, 8, 16, 32, 40, 64]))
        params = SyntheticProfileParams(float(rng.uniform(0.2, 20.0)), float(rng.uniform(0.1, 10.0)),
                                        float(rng.uniform(0.02, 0.6)), float(rng.uniform(0.5, 1.0)))
        table = synth_profile(params, sizes, b_max)
        dist = lognormal_batch_pdf(float(rng.uniform(0.0, 2.5)), float(rng.uniform(0.2, 1.5)), b_max)
        gpus = int(rng.integers(1, 9))
        gpcs = int(rng.choice([7, 7, 7, 4, 8]))
        total = int(rng.integers(1, gpus * gpcs + 1)) if rng.random() < 0.3 else gpus * gpcs
        thr = float(rng.choice([0.8, 0.5, 0.9, 1.0, float(rng.uniform(0.05, 1.0))]))
        jobs.append(ParisJob(table, dist, total, gpus, gpcs, thr))
    assert _compare(eng, ref, jobs) >= 1000


def test_paris_batch_random_tables_and_errors(eng, ref):
    """Hand-made tables: knees not ordered by size (knee-order violations), zero-mass
    segments, sizes above gpcs_per_gpu (InfeasibleError), bad thresholds / totals /
    fleets, and a distribution whose support differs from the table's."""
    rng = np.random.default_rng(11)
    jobs = []
    for i in range(1200):
        n = int(rng.integers(1, 6))
        sizes = np.array(sorted(rng.choice(np.arange(1, 9), size=n, replace=False)), np.int32)
        b_max = int(rng.choice([3, 8, 16, 33]))
        row = np.cumsum(rng.uniform(0.1, 5.0, size=b_max))  # rises in batch, falls in size
        lat = np.stack([row * f for f in np.cumprod(rng.uniform(0.4, 1.0, size=n))])
        util = np.sort(rng.uniform(0.0, 1.0, size=(n, b_max)), axis=1)  # rows rise in batch
        table = ProfileTable(sizes, b_max, lat, util, f"t{i}")
        w = rng.uniform(0.0, 1.0, size=b_max)
        w[rng.random(b_max) < 0.3] = 0.0
        if w.sum() == 0.0:
            w[0] = 1.0
        if rng.random() < 0.05:
            w = np.append(w, 0.5)  # support mismatch -> ValidationError
        dist = BatchDistribution(w)
        gpus = int(rng.integers(0, 5)) if rng.random() < 0.1 else int(rng.integers(1, 5))
        gpcs = int(rng.choice([0, 3, 7, 8])) if rng.random() < 0.2 else 7
        total = int(rng.integers(-1, 3)) if rng.random() < 0.05 else max(1, gpus * max(gpcs, 1))
        thr = float(rng.choice([0.0, 1.2, -0.5])) if rng.random() < 0.05 else float(rng.uniform(0.05, 1.0))
        jobs.append(ParisJob(table, dist, total, gpus, gpcs, thr))
    n_ok = _compare(eng, ref, jobs)
    assert 200 < n_ok < len(jobs)


def test_paris_batch_error_messages(eng):
    from paper_2202_13481_b200 import workloads as W
    m = W.model("bert_base")
    t = synth_profile(SyntheticProfileParams(), [1, 2, 7], 8)
    d = lognormal_batch_pdf(1.0, 1.0, 8)
    cases = [
        (ParisJob(t, d, 7, 1, 7, 0.0), N.ParamError, "knee: threshold must be in (0,1]"),
        (ParisJob(t, lognormal_batch_pdf(1.0, 1.0, 9), 7, 1, 7, 0.8), N.ValidationError,
         "paris_plan: distribution support must match profile b_max"),
        (ParisJob(t, d, 0, 1, 7, 0.8), N.ParamError, "instance_counts: total_gpcs must be >= 1"),
        (ParisJob(t, d, 7, 0, 7, 0.8), N.ParamError, "pack_plan: num_gpus must be >= 1"),
        (ParisJob(m.table, m.dist, 14, 2, 3, 0.8), N.InfeasibleError,
         "pack_plan: instance of size 4 exceeds gpcs_per_gpu=3"),
    ]
    got = eng.paris_batch([c[0] for c in cases])
    for (job, cls, msg), g in zip(cases, got):
        assert isinstance(g.error, cls) and str(g.error) == msg, (g.error, msg)
