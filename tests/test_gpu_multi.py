"""Multi-device contexts (msv_create_multi) on the product path: a grid sharded over
several member contexts must equal the single-context run bit for bit (here two or three
members on one B200 — the sharding, upload mirroring, gather and error paths are the
same as on 8 GPUs), plus the world-2 rank-sharded path through Engine (gloo, two ranks
sharing the device), gathered results equal to the compiled reference."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2202_13481_b200 import Engine, LookupError_, ParamError
from paper_2202_13481_b200 import workloads as W
from tests import oracle_py as O

pytestmark = pytest.mark.gpu


def _grid():
    return W.c2(seeds=6, queries=8e3) + W.c3(seeds=4, queries=6e3) + W.c1(queries=5e3)


def _assert_same(a, b):
    for k in ("total", "violations", "measured", "measured_violations", "status"):
        assert np.array_equal(a[k], b[k]), k
    assert np.array_equal(a["placement_hash"], b["placement_hash"])
    assert np.array_equal(a["tail"], b["tail"], equal_nan=True)
    assert np.array_equal(a["horizon_ms"], b["horizon_ms"])


@pytest.mark.parametrize("members", [[0, 0], [0, 0, 0]])
def test_multi_context_run_grid_equals_single(members):
    specs = _grid()
    one = Engine(0).run_grid(specs, (0.95, 0.99), usage=True)
    multi = Engine(members)
    assert multi.devices == members
    got = multi.run_grid(specs, (0.95, 0.99), usage=True)
    _assert_same(got, one)
    for k in ("busy_ms", "weighted_busy_ms", "queries"):
        assert np.array_equal(got["usage"][k], one["usage"][k]), k


def test_multi_context_matches_reference():
    specs = _grid()
    got = Engine([0, 0]).run_grid(specs, (0.95, 0.99))
    _assert_same(got, O.best_oracle().run_grid(specs, (0.95, 0.99)))


def test_multi_context_device_grid_and_replay():
    specs = _grid()
    single = Engine(0)
    multi = Engine([0, 0, 0])
    g1, g2 = single.grid(specs), multi.grid(specs)
    g1.launch()
    g2.launch()
    _assert_same(g2.results(), g1.results())
    assert g2.queries() == g1.queries()
    t = g2.timing()
    assert t["total_ms"] > 0
    # replay with per-query records across members (records land at the caller's offsets)
    items = []
    for s in specs[:9]:
        arr, bat = O.best_oracle().sample_trace(s.dist, s.rate_qps, s.duration_ms, s.seed)
        items.append((s, arr, bat))
    r1 = single.run_many([(s.plan, s.scheduler, a, b, s.duration_ms, s.table, s.sla, 0.1, None, False)
                         for s, a, b in items])
    r2 = multi.run_many([(s.plan, s.scheduler, a, b, s.duration_ms, s.table, s.sla, 0.1, None, False)
                        for s, a, b in items])
    for x, y in zip(r1, r2):
        for k in ("partition", "start_ms", "finish_ms", "kind"):
            assert np.array_equal(x[k], y[k]), k


def test_multi_context_errors_propagate():
    specs = _grid()
    bad = list(specs)
    bad[-1] = W.GridSpec(bad[-1].plan, bad[-1].table, bad[-1].dist, W.SlaConfig(0.0), bad[-1].rate_qps,
                         bad[-1].duration_ms, bad[-1].seed)
    with pytest.raises(ParamError):
        Engine([0, 0]).run_grid(bad, (0.95,))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch.distributed as td
    from paper_2202_13481_b200.distributed import run_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    td.init_process_group("gloo", rank=rank, world_size=world)
    specs = W.c5(n_scenarios=150, queries=1e4)
    eng = Engine(0)
    res = run_sharded(specs, lambda sub: eng.run_grid(sub, (0.95, 0.99)), rank, world)
    q.put((rank, res["placement_hash"].tolist(), res["tail"].tolist(), res["total"].tolist()))
    td.barrier()
    td.destroy_process_group()


def test_world2_ranks_share_one_b200_through_engine():
    """world 2 (gloo), two ranks on one B200 through Engine: the gathered
    grid equals the compiled reference on every scenario."""
    specs = W.c5(n_scenarios=150, queries=1e4)
    ref = O.best_oracle().run_grid(specs, (0.95, 0.99))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for _, hashes, tails, totals in got:
        assert hashes == ref["placement_hash"].tolist()
        assert np.array_equal(np.array(tails), ref["tail"], equal_nan=True)
        assert totals == ref["total"].tolist()
