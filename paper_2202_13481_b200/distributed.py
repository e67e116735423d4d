"""Multi-GPU scenario sharding: one process per GPU (torch.distributed), each rank
simulates a cost-balanced contiguous shard of the scenario list on its own device
(no data-path collective), then one all-gather of fixed-size per-scenario results
(NCCL over NVLink on GPUs; gloo in the CPU tests) gives every rank the whole grid,
from which each rank takes the same deterministic PARIS argmin.
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np

from .workloads import shard

# Per-scenario record exchanged between ranks (float64 lanes; integers < 2^53).
FIELDS = ("total", "violations", "measured", "measured_violations", "p95", "p99", "horizon_ms", "hash_hi",
          "hash_lo", "status")


def pack(res: dict) -> np.ndarray:
    """Engine.run_grid result dict -> (n, len(FIELDS)) float64 rows."""
    n = len(res["total"])
    out = np.zeros((n, len(FIELDS)))
    out[:, 0] = res["total"]
    out[:, 1] = res["violations"]
    out[:, 2] = res["measured"]
    out[:, 3] = res["measured_violations"]
    tail = np.asarray(res["tail"])
    out[:, 4] = tail[:, 0] if tail.shape[1] > 0 else np.nan
    out[:, 5] = tail[:, 1] if tail.shape[1] > 1 else np.nan
    out[:, 6] = res["horizon_ms"]
    h = np.asarray(res["placement_hash"], dtype=np.uint64)
    out[:, 7] = (h >> np.uint64(32)).astype(np.float64)
    out[:, 8] = (h & np.uint64(0xFFFFFFFF)).astype(np.float64)
    out[:, 9] = res["status"]
    return out


def unpack(rows: np.ndarray) -> dict:
    h = (rows[:, 7].astype(np.uint64) << np.uint64(32)) | rows[:, 8].astype(np.uint64)
    return {"total": rows[:, 0].astype(np.int64), "violations": rows[:, 1].astype(np.int64),
            "measured": rows[:, 2].astype(np.int64), "measured_violations": rows[:, 3].astype(np.int64),
            "tail": rows[:, 4:6].copy(), "horizon_ms": rows[:, 6].copy(), "placement_hash": h,
            "status": rows[:, 9].astype(np.int32)}


def shard_bounds(specs: Sequence, world: int) -> list[tuple[int, int]]:
    """[lo, hi) of every rank's shard (the same cut `workloads.shard` makes)."""
    bounds, lo = [], 0
    for r in range(world):
        n = len(shard(list(specs), r, world))
        bounds.append((lo, lo + n))
        lo += n
    return bounds


def _error_code(exc: BaseException) -> int:
    """errors.hpp type of a local failure as the C-ABI status code (MSV_PARAM..MSV_CUDA),
    99 for anything else."""
    from . import _native as N
    for code, cls in N._ERRORS.items():
        if type(exc) is cls:
            return int(code)
    return 99


def _raise_remote(codes: np.ndarray, rank: int, local_exc: BaseException | None, what: str) -> None:
    """After the gather: every rank raises when any rank's local work failed (the failing
    rank re-raises its own exception; the others raise the same errors.hpp type)."""
    bad = [r for r, c in enumerate(codes) if c != 0]
    if not bad:
        return
    if local_exc is not None:
        raise local_exc
    from . import _native as N
    cls = N._ERRORS.get(int(codes[bad[0]]), N.Error)
    raise cls(f"{what}: rank {bad[0]} failed (status {int(codes[bad[0]])})")


def run_sharded(specs: Sequence, run_local: Callable[[list], dict], rank: int, world: int, device=None) -> dict:
    """Run this rank's shard with `run_local` (e.g. Engine.run_grid) and all-gather every
    rank's rows in global scenario order. A failure of one rank's local work (e.g. a
    LookupError from run_grid) still takes part in the gather — row 0 of every rank's
    buffer carries its status — and is raised on every rank, as the single-process
    reference would raise it, instead of leaving the other ranks in the collective."""
    import torch
    import torch.distributed as td
    bounds = shard_bounds(specs, world)
    lo, hi = bounds[rank]
    exc, local = None, np.zeros((0, len(FIELDS)))
    try:
        if hi > lo:
            local = pack(run_local(list(specs[lo:hi])))
    except Exception as e:  # noqa: BLE001 - re-raised after the gather
        if world == 1:
            raise
        exc = e
    if world == 1:
        return unpack(local)
    width = max(h - l for l, h in bounds)
    buf = np.full((width + 1, len(FIELDS)), np.nan)
    buf[0, 0] = _error_code(exc) if exc is not None else 0
    if exc is None:
        buf[1: 1 + hi - lo] = local
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    td.all_gather(parts, t)
    parts = [p.cpu().numpy() for p in parts]
    _raise_remote(np.array([p[0, 0] for p in parts]), rank, exc, "run_sharded")
    rows = np.concatenate([p[1: 1 + h - l] for p, (l, h) in zip(parts, bounds)])
    return unpack(rows)


def grouped_argmin(p99: np.ndarray, group: Sequence, candidate: Sequence) -> dict:
    """PARIS argmin per group (e.g. per (model, load) of the C5 grid): the mean p99 of every
    candidate over its scenarios in list order (seed order; NaN tails skipped, summed like
    mean_tail_at_rate, metrics.hpp:61-74), then the candidate with the least mean; ties go
    to the candidate seen first. Returns {group: (best candidate, {candidate: mean})}."""
    sums: dict = {}
    order: dict = {}
    for v, g, c in zip(np.asarray(p99, float), group, candidate):
        d = sums.setdefault(g, {})
        order.setdefault(g, [])
        if c not in d:
            d[c] = [0.0, 0]
            order[g].append(c)
        if v == v:
            d[c][0] += float(v)
            d[c][1] += 1
    out = {}
    for g, d in sums.items():
        means = {c: (s / n if n else np.inf) for c, (s, n) in d.items()}
        best = order[g][0]
        for c in order[g][1:]:
            if means[c] < means[best]:
                best = c
        out[g] = (best, means)
    return out


def paris_argmin(p99: np.ndarray, n_candidates: int, seeds_per_candidate: int) -> tuple[int, np.ndarray]:
    """Mean p99 per candidate (seed-major rows in candidate order, NaN-free seeds only,
    summed in seed order like mean_tail_at_rate, metrics.hpp:61-74) and the argmin;
    ties break toward the lowest candidate index."""
    p = np.asarray(p99, float).reshape(n_candidates, seeds_per_candidate)
    means = np.empty(n_candidates)
    for c in range(n_candidates):
        s, used = 0.0, 0
        for v in p[c]:
            if v == v:
                s += float(v)
                used += 1
        means[c] = s / used if used else np.inf
    best = 0
    for c in range(1, n_candidates):
        if means[c] < means[best]:
            best = c
    return best, means


def design_bounds(n: int, world: int) -> list[tuple[int, int]]:
    """[lo, hi) contiguous design shards, sizes differing by at most one."""
    base, extra = divmod(n, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def lbt_sharded(designs: Sequence, search_local: Callable[[list], list], rank: int, world: int,
                device=None) -> list[tuple[float, bool, int]]:
    """latency_bounded_throughput (metrics.hpp:81-120) of many designs over `world` ranks
    (SURVEY §8e): each design's whole search — every seed of every probed rate — stays on
    one rank, so the lockstep rounds need no collective; one all-gather of (qps,
    infeasible_at_min, sims_run) at the end gives every rank every design's result, in
    design order. `search_local(designs) -> [(qps, infeasible, sims), ...]` is e.g.
    `search.latency_bounded_throughput(eng, ds)` mapped to tuples."""
    bounds = design_bounds(len(designs), world)
    lo, hi = bounds[rank]
    exc, local = None, []
    try:
        local = [tuple(r) for r in search_local(list(designs[lo:hi]))] if hi > lo else []
    except Exception as e:  # noqa: BLE001 - re-raised on every rank after the gather
        if world == 1:
            raise
        exc = e
    if world == 1:
        return [(float(q), bool(i), int(n)) for q, i, n in local]
    import torch
    import torch.distributed as td
    width = max(1, max(h - l for l, h in bounds))
    buf = np.full((width + 1, 3), np.nan)
    buf[0, 0] = _error_code(exc) if exc is not None else 0
    for j, (q, inf, n) in enumerate(local):
        buf[1 + j] = (q, 1.0 if inf else 0.0, n)
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    td.all_gather(parts, t)
    parts = [p.cpu().numpy() for p in parts]
    _raise_remote(np.array([p[0, 0] for p in parts]), rank, exc, "lbt_sharded")
    rows = np.concatenate([p[1: 1 + h - l] for p, (l, h) in zip(parts, bounds)])
    return [(float(r[0]), bool(r[1]), int(r[2])) for r in rows]
