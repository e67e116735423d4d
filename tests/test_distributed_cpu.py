"""Multi-process host logic of the multi-GPU path on CPU: world_size 2 over gloo.
Each rank runs its shard (here through the CPU oracle port, standing in for the
device), all-gathers, and must end with the full grid identical to a single-process
run plus the same PARIS argmin on both ranks."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def O_REF_EXISTS() -> bool:
    from tests import oracle_py as O
    return O.REF_LIB.exists()


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _specs():
    from paper_2202_13481_b200 import workloads as W
    m = W.model("bert_base")
    cands = W.fleet_candidates(1)[:6]  # six 1-GPU fleets
    rate = 0.6 * W.capacity_qps(m, W.paris(m, 1))
    return [W._spec(m, p, rate, 1500, 1 + s) for p in cands for s in range(3)], len(cands)


def _worker(rank, world, port, out_q):
    import torch.distributed as td
    from paper_2202_13481_b200.distributed import paris_argmin, run_sharded
    from tests import oracle_py as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    td.init_process_group("gloo", rank=rank, world_size=world)
    specs, n_c = _specs()
    port_oracle = O.Oracle("port")
    res = run_sharded(specs, lambda sub: port_oracle.run_grid(sub, (0.95, 0.99), threads=1), rank, world)
    best, means = paris_argmin(res["tail"][:, 1], n_c, 3)
    out_q.put((rank, res["placement_hash"].tolist(), res["tail"].tolist(), best))
    td.barrier()
    td.destroy_process_group()


def test_sharded_gather_matches_single_process():
    from paper_2202_13481_b200.distributed import paris_argmin
    from tests import oracle_py as O
    specs, n_c = _specs()
    ref = O.Oracle("port").run_grid(specs, (0.95, 0.99), threads=1)
    ref_best, _ = paris_argmin(ref["tail"][:, 1], n_c, 3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, hashes, tails, best in got:
        assert hashes == ref["placement_hash"].tolist()
        assert np.array_equal(np.array(tails), ref["tail"])
        assert best == ref_best


def test_shard_bounds_cover_in_order():
    from paper_2202_13481_b200.distributed import shard_bounds
    specs, _ = _specs()
    for world in (1, 2, 3, 8):
        b = shard_bounds(specs, world)
        assert b[0][0] == 0 and b[-1][1] == len(specs)
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))


def test_paris_argmin_ties_and_empty_seeds():
    from paper_2202_13481_b200.distributed import paris_argmin
    p99 = np.array([3.0, 3.0, 2.0, np.nan, 2.0, 2.0, 1.5, 2.5, 2.0])
    best, means = paris_argmin(p99, 3, 3)
    assert means[1] == 2.0 and means[2] == 2.0 and best == 1


def _lbt_designs():
    from paper_2202_13481_b200 import workloads as W
    from paper_2202_13481_b200.search import Design, LbtOptions
    m = W.model("resnet50")
    opt = LbtOptions(duration_ms=1500.0, seeds=(1, 2), rel_tol=0.05)
    out = []
    for p in W.fleet_candidates(1)[:5]:
        for sched in ("elsa", "fifs"):
            out.append(Design(p, sched, m.table, m.dist, m.sla, opt))
    return out


def _lbt_worker(rank, world, port, out_q):
    import torch.distributed as td
    from paper_2202_13481_b200.distributed import lbt_sharded
    from tests import oracle_py as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    td.init_process_group("gloo", rank=rank, world_size=world)
    ref = O.Oracle("reference")
    designs = _lbt_designs()
    res = lbt_sharded(designs, lambda ds: [ref.lbt(d.plan, d.scheduler, d.table, d.sla, d.dist, d.opt) for d in ds],
                      rank, world)
    out_q.put((rank, res))
    td.barrier()
    td.destroy_process_group()


@pytest.mark.skipif(not O_REF_EXISTS(), reason="oracle/_ref not built")
def test_lbt_sharded_matches_single_process():
    """Rank-local LBT searches (3 ranks, 10 designs: uneven shards) + one all-gather give every
    rank the single-process results in design order."""
    from tests import oracle_py as O
    ref = O.Oracle("reference")
    want = [ref.lbt(d.plan, d.scheduler, d.table, d.sla, d.dist, d.opt) for d in _lbt_designs()]
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_lbt_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert got[r] == [(float(a), bool(b), int(c)) for a, b, c in want], r


def _err_worker(rank, world, port, out_q):
    import torch.distributed as td
    from paper_2202_13481_b200 import _native as N
    from paper_2202_13481_b200.distributed import lbt_sharded, run_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    td.init_process_group("gloo", rank=rank, world_size=world)
    specs = list(range(6))  # stand-ins: only the shard split and the failure matter

    class _S:
        def __init__(self, i):
            self.rate_qps, self.duration_ms = 1.0, 1000.0
            self.plan = type("P", (), {"total_instances": lambda self: 1})()

    specs = [_S(i) for i in specs]

    def local(sub):
        if rank == 1:
            raise N.LookupError_("profile: batch 40 outside grid 1..32")
        return {"total": np.ones(len(sub)), "violations": np.zeros(len(sub)), "measured": np.ones(len(sub)),
                "measured_violations": np.zeros(len(sub)), "tail": np.ones((len(sub), 2)),
                "horizon_ms": np.ones(len(sub)), "placement_hash": np.zeros(len(sub), np.uint64),
                "status": np.zeros(len(sub))}
    got = []
    for fn in (lambda: run_sharded(specs, local, rank, world),
               lambda: lbt_sharded(list(range(4)), lambda ds: (_ for _ in ()).throw(N.ParamError("sla <= 0"))
                                   if rank == 0 else [(1.0, False, 3)] * len(ds), rank, world)):
        try:
            fn()
            got.append("ok")
        except N.Error as e:
            got.append(type(e).__name__)
    out_q.put((rank, got))
    td.barrier()
    td.destroy_process_group()


def test_sharded_failure_raises_on_every_rank():
    """a rank whose local work raises must not leave the others in the collective;
    every rank raises the same errors.hpp type."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_err_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0] == got[1] == ["LookupError_", "ParamError"]


def test_grouped_argmin_seed_order_and_ties():
    from paper_2202_13481_b200.distributed import grouped_argmin
    p99 = np.array([3.0, 1.0, 2.0, np.nan, 2.0, 5.0, 1.0, 1.0])
    group = ["a", "a", "a", "a", "b", "b", "b", "b"]
    cand = [0, 1, 0, 1, 7, 8, 8, 7]
    out = grouped_argmin(p99, group, cand)
    assert out["a"][0] == 1 and out["a"][1] == {0: 2.5, 1: 1.0}
    assert out["b"][0] == 7 and out["b"][1] == {7: 1.5, 8: 3.0}
    tie = grouped_argmin(np.array([1.0, 1.0]), ["g", "g"], [5, 4])
    assert tie["g"][0] == 5  # the candidate seen first wins ties
