"""Search drivers over device grids:

    latency_bounded_throughput   metrics.hpp:81-120, every design advanced in lockstep;
                                 each round is one device grid over (design x seed)
    best_homogeneous             metrics.hpp:183-209 (GPU(max) under FIFS)
    paris_search                 exhaustive 8-GPU fleet search scored by ELSA p99 (C4),
                                 with the PARIS closed-form plan's rank

The per-design rate sequence is the reference's exactly (same doubling/bisection,
same comparisons), so the returned rates are bit-identical to the reference's.
"""
from __future__ import annotations

import copy
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _native as N
from .engine import (BatchDistribution, Engine, GridSpec, PartitionPlan, ProfileTable, SlaConfig,
                     homogeneous_plan)


@dataclass
class LbtOptions:
    """LbtOptions (metrics.hpp:39-47), same defaults."""
    duration_ms: float = 20000.0
    seeds: Sequence[int] = (1, 2, 3)
    rel_tol: float = 0.01
    tail_p: float = 0.95
    lambda_min: float = 1.0
    warmup_fraction: float = 0.1
    max_doublings: int = 24


@dataclass
class LbtResult:
    qps: float = 0.0
    infeasible_at_min: bool = False
    sims_run: int = 0


@dataclass
class Design:
    plan: PartitionPlan
    scheduler: str
    table: ProfileTable
    dist: BatchDistribution
    sla: SlaConfig
    opt: LbtOptions = field(default_factory=LbtOptions)


class _Search:
    """One design's bracket + bisection as a resumable state machine."""
    MIN, DOUBLE, BISECT, DONE = range(4)

    def __init__(self, d: Design):
        if not d.sla.sla_target_ms > 0.0:
            raise N.ParamError("latency_bounded_throughput: sla must be > 0")
        if len(d.opt.seeds) == 0:
            raise N.ParamError("latency_bounded_throughput: need at least one seed")
        self.d = d
        self.phase = self.MIN
        self.rate = d.opt.lambda_min
        self.lo = self.hi = self.mid = 0.0
        self.doublings = 0
        self.res = LbtResult()

    def _next_double(self):
        if self.doublings < self.d.opt.max_doublings:
            self.hi *= 2.0
            self.rate = self.hi
            self.phase = self.DOUBLE
        else:
            self.res.qps = self.lo
            self.phase = self.DONE

    def _next_bisect(self):
        if (self.hi - self.lo) / self.lo > self.d.opt.rel_tol:
            self.mid = 0.5 * (self.lo + self.hi)
            self.rate = self.mid
            self.phase = self.BISECT
        else:
            self.res.qps = self.lo
            self.phase = self.DONE

    def feed(self, tail: float):
        self.res.sims_run += len(self.d.opt.seeds)
        sla = self.d.sla.sla_target_ms
        if self.phase == self.MIN:
            if tail > sla:
                self.res.infeasible_at_min = True
                self.phase = self.DONE
                return
            self.lo = self.hi = self.d.opt.lambda_min
            self.doublings = 0
            self._next_double()
        elif self.phase == self.DOUBLE:
            if tail > sla:
                self._next_bisect()
                return
            self.lo = self.hi
            self.doublings += 1
            self._next_double()
        elif self.phase == self.BISECT:
            if tail <= sla:
                self.lo = self.mid
            else:
                self.hi = self.mid
            self._next_bisect()


def _mean_tail(tails: np.ndarray, measured: np.ndarray) -> float:
    """mean_tail_at_rate (metrics.hpp:61-74): sum in seed order over seeds with samples."""
    s, used = 0.0, 0
    for t, m in zip(tails, measured):
        if m == 0:
            continue
        s += float(t)
        used += 1
    return 0.0 if used == 0 else s / used


def _clone(s: _Search) -> _Search:
    c = copy.copy(s)
    c.res = copy.copy(s.res)
    return c


def _probe_tree(s: _Search, depth: int) -> list[tuple[int, float]]:
    """Rates the search may probe in its next `depth` steps: node k's children are 2k+1
    (probe met the SLA) and 2k+2 (violated it); (node, rate) for every live node."""
    out, level = [], [(0, s)]
    for _ in range(depth):
        nxt = []
        for k, st in level:
            if st.phase == _Search.DONE:
                continue
            out.append((k, st.rate))
            for child, tail in ((2 * k + 1, -np.inf), (2 * k + 2, np.inf)):
                c = _clone(st)
                c.feed(tail)
                nxt.append((child, c))
        level = nxt
    return out


def latency_bounded_throughput(eng: Engine, designs: Sequence[Design], lookahead: int = 3) -> list[LbtResult]:
    """Every design's bracket/bisection advanced in lockstep. Each round simulates the
    rates of the next `lookahead` steps of every design's outcome tree (2^L - 1 probes per
    design, all independent scenarios of one device grid) and then walks the tree with
    the measured tails: the same probe sequence, comparisons and rates as the reference
    (metrics.hpp:81-120), in L times fewer rounds. sims_run counts the probes taken."""
    searches = [_Search(d) for d in designs]
    depth = max(1, int(lookahead))
    while True:
        active = [s for s in searches if s.phase != _Search.DONE]
        if not active:
            return [s.res for s in searches]
        by_p: dict[float, list[_Search]] = {}
        for s in active:
            by_p.setdefault(s.d.opt.tail_p, []).append(s)
        for p, group in by_p.items():
            specs, where = [], []
            for s in group:
                o = s.d.opt
                nodes = {}
                for k, rate in _probe_tree(s, depth):
                    nodes[k] = (len(specs), rate)
                    specs += [GridSpec(s.d.plan, s.d.table, s.d.dist, s.d.sla, rate, o.duration_ms, seed,
                                       s.d.scheduler, o.warmup_fraction) for seed in o.seeds]
                where.append(nodes)
            r = eng.run_grid(specs, (p,))
            for s, nodes in zip(group, where):
                k, n_seeds = 0, len(s.d.opt.seeds)
                while k in nodes and s.phase != _Search.DONE:
                    pos, rate = nodes[k]
                    assert rate == s.rate  # the tree followed the search's own rule
                    tail = _mean_tail(r["tail"][pos:pos + n_seeds, 0], r["measured"][pos:pos + n_seeds])
                    sla = s.d.sla.sla_target_ms  # the branch feed() takes
                    bad = not (tail <= sla) if s.phase == _Search.BISECT else tail > sla
                    s.feed(tail)
                    k = 2 * k + (2 if bad else 1)


def best_homogeneous(eng: Engine, table: ProfileTable, dist: BatchDistribution, sla: SlaConfig, total_gpcs: int,
                     num_gpus: int, gpcs_per_gpu: int, opt: LbtOptions | None = None) -> tuple[int, PartitionPlan,
                                                                                             LbtResult]:
    """GPU(max): LBT under FIFS for every homogeneous size; first strictly larger wins."""
    opt = opt or LbtOptions()
    ks, plans = [], []
    for k in [int(x) for x in table.sizes]:
        if k > gpcs_per_gpu or k > total_gpcs:
            continue
        ks.append(k)
        plans.append(homogeneous_plan(k, total_gpcs, num_gpus, gpcs_per_gpu))
    if not ks:
        raise N.InfeasibleError("best_homogeneous: no size fits the server")
    idx = [i for i, p in enumerate(plans) if p.total_instances() > 0]
    res = latency_bounded_throughput(eng, [Design(plans[i], "fifs", table, dist, sla, opt) for i in idx])
    by = dict(zip(idx, res))
    best_k, best_plan, best = 0, None, LbtResult()
    for i, k in enumerate(ks):
        r = by.get(i, LbtResult())
        if best_k == 0 or r.qps > best.qps:
            best_k, best_plan, best = k, plans[i], r
    return best_k, best_plan, best


@dataclass
class SearchResult:
    best_index: int
    best_plan: PartitionPlan
    mean_p99: np.ndarray          # per candidate
    paris_index: int              # index of the PARIS closed-form fleet among the candidates (-1: absent)
    paris_rank: int               # 0 = best
    queries: int


def paris_search(eng: Engine, candidates: Sequence[PartitionPlan], table: ProfileTable, dist: BatchDistribution,
                 sla: SlaConfig, rate_qps: float, duration_ms: float, seeds: Sequence[int],
                 paris: PartitionPlan | None = None, scheduler: str = "elsa", rank: int = 0, world: int = 1,
                 device=None) -> SearchResult:
    """Score every candidate fleet by mean ELSA p99 over `seeds` (one device grid per rank;
    ranks split the candidates and all-gather, then take the same argmin)."""
    from .distributed import paris_argmin, run_sharded
    specs = [GridSpec(p, table, dist, sla, rate_qps, duration_ms, s, scheduler) for p in candidates for s in seeds]
    res = run_sharded(specs, lambda sub: eng.run_grid(sub, (0.95, 0.99)), rank, world, device)
    best, means = paris_argmin(res["tail"][:, 1], len(candidates), len(seeds))
    pidx, prank = -1, -1
    if paris is not None:
        key = sorted(paris.instance_counts())
        for i, c in enumerate(candidates):
            if sorted(c.instance_counts()) == key:
                pidx = i
                break
        if pidx >= 0:
            prank = int(np.sum(means < means[pidx]))
    return SearchResult(best, candidates[best], means, pidx, prank, int(res["total"].sum()))
