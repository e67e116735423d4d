"""Search drivers on the device vs the reference's own drivers (metrics.hpp:81-209):
identical rates (bit for bit), identical infeasibility flags and simulation counts,
and the GPU(max) winner; plus the exhaustive PARIS search on a 1-GPU fleet set."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2202_13481_b200 import (BatchDistribution, Engine, PartitionPlan, ProfileTable, SlaConfig,
                                   SyntheticProfileParams, derive_sla_target, lognormal_batch_pdf, synth_profile)
from paper_2202_13481_b200 import search as S
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


def flat_k7(latency_at_bmax, b_max):  # test_metrics.cpp:14-20
    lat = np.array([[latency_at_bmax * b / b_max for b in range(1, b_max + 1)]])
    util = np.array([[0.03 * b for b in range(1, b_max + 1)]])
    return ProfileTable(np.array([7], np.int32), b_max, lat, util, "flat7")


@pytest.mark.parametrize("sla", [200.0, 10.0, 40.0, 80.0])
def test_lbt_single_partition_matches_reference(eng, ref, sla):
    t = flat_k7(20.0, 1)
    d = BatchDistribution(np.array([1.0]))
    opt = S.LbtOptions(duration_ms=30000.0, seeds=(1, 2, 3))
    for plan in (PartitionPlan(1, 7, [[7]]), PartitionPlan(2, 7, [[7], [7]])):
        got = S.latency_bounded_throughput(eng, [S.Design(plan, "fifs", t, d, SlaConfig(sla), opt)])[0]
        want = ref.lbt(plan, "fifs", t, SlaConfig(sla), d, opt)
        assert (got.qps, got.infeasible_at_min, got.sims_run) == want


def test_lbt_elsa_paris_matches_reference(eng, ref):
    m = W.model("resnet50")
    p = W.paris(m, 1)
    opt = S.LbtOptions(duration_ms=4000.0, seeds=(1, 2), lambda_min=50.0)
    designs = [S.Design(p, sched, m.table, m.dist, m.sla, opt) for sched in ("elsa", "fifs")]
    got = S.latency_bounded_throughput(eng, designs)
    for d, g in zip(designs, got):
        assert (g.qps, g.infeasible_at_min, g.sims_run) == ref.lbt(d.plan, d.scheduler, m.table, m.sla, m.dist, opt)


def test_best_homogeneous_matches_reference(eng, ref):
    # test_metrics.cpp:193-213 configuration
    table = synth_profile(SyntheticProfileParams(10.0, 5.0, 0.15, 0.95), [1, 2, 3, 4, 7], 16)
    dist = lognormal_batch_pdf(1.0, 0.7, 16)
    sla = SlaConfig(derive_sla_target(table, 16, 1.5))
    opt = S.LbtOptions(duration_ms=8000.0, seeds=(1, 2))
    k, plan, r = S.best_homogeneous(eng, table, dist, sla, 14, 2, 7, opt)
    assert (k, r.qps) == ref.best_homogeneous(table, dist, sla, 14, 2, 7, 8000.0, (1, 2))


def test_paris_search_one_gpu(eng):
    m = W.model("resnet50")
    cands = W.fleet_candidates(1)
    paris = W.paris(m, 1)
    rate = 0.85 * W.capacity_qps(m, paris)
    res = S.paris_search(eng, cands, m.table, m.dist, m.sla, rate, 5000.0, (1, 2, 3), paris=paris)
    assert len(res.mean_p99) == 12 and res.paris_index >= 0
    assert res.mean_p99[res.best_index] == np.min(res.mean_p99)
    # same scoring through the reference oracle
    ref = O.best_oracle()
    from paper_2202_13481_b200.engine import GridSpec
    from paper_2202_13481_b200.distributed import paris_argmin
    specs = [GridSpec(p, m.table, m.dist, m.sla, rate, 5000.0, s, "elsa") for p in cands for s in (1, 2, 3)]
    r = ref.run_grid(specs, (0.95, 0.99))
    best, means = paris_argmin(r["tail"][:, 1], 12, 3)
    assert best == res.best_index and np.array_equal(means, res.mean_p99)
