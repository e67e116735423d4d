"""Model presets and the five BASELINE.json configurations as scenario grids.

The reference ships no measured ResNet-50 / BERT-base / MobileNet profiles; only
`SyntheticProfileParams` (profile.hpp:43-48) and prose presets. The
presets below are this build's recorded choice ("Inputs the reference
does not define"): knees ascend with partition size, and the 1-GPU PARIS plan of
the ResNet-50 preset serves 1,000 q/s at ~88% of its nominal capacity (C1).

Nominal capacity ("peak QPS") of a plan = sum over partitions of
1000 / E_b[latency(k_p, b)] under the batch distribution.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

from .engine import (BatchDistribution, GridSpec, PartitionPlan, ProfileTable, SlaConfig, SyntheticProfileParams,
                     derive_sla_target, homogeneous_plan, lognormal_batch_pdf, paris_plan, synth_profile)

SIZES = (1, 2, 3, 4, 7)
B_MAX = 32
PRESETS = {
    # name: (work_per_sample ms*GPC, fixed_overhead ms, parallelism_per_sample, util_cap)
    "mobilenet": SyntheticProfileParams(0.4, 0.5, 0.15, 0.95),
    "resnet50": SyntheticProfileParams(0.8, 0.8, 0.25, 0.95),
    "bert_base": SyntheticProfileParams(4.0, 2.0, 0.40, 0.95),
}
SLA_MULTIPLIER = 1.5  # SPEC.md:429-431 default N


@dataclass
class Model:
    name: str
    table: ProfileTable
    dist: BatchDistribution
    sla: SlaConfig


_MODELS: dict[str, Model] = {}


def model(name: str) -> Model:
    if name not in _MODELS:
        t = synth_profile(PRESETS[name], SIZES, B_MAX, name)
        d = lognormal_batch_pdf(1.0, 1.0, B_MAX)  # SPEC.md:167 defaults
        _MODELS[name] = Model(name, t, d, SlaConfig(derive_sla_target(t, B_MAX, SLA_MULTIPLIER), 1.0, 1.0))
    return _MODELS[name]


def capacity_qps(m: Model, plan: PartitionPlan) -> float:
    pmf = np.asarray(m.dist.weights, float)
    pmf = pmf / pmf.sum()
    row = {int(k): i for i, k in enumerate(m.table.sizes)}
    return float(sum(1000.0 / float((pmf * m.table.latency[row[k]]).sum()) for k in plan.flatten()))


def paris(m: Model, gpus: int) -> PartitionPlan:
    return paris_plan(m.table, m.dist, 7 * gpus, gpus, 7)


def _spec(m: Model, plan: PartitionPlan, rate: float, queries: float, seed: int, sched: str = "elsa") -> GridSpec:
    return GridSpec(plan, m.table, m.dist, m.sla, rate, queries / rate * 1000.0, seed, sched)


# ---- C1: ResNet-50, 1-GPU PARIS, Poisson 1k QPS, 1e5 queries, ELSA vs FIFS ----
def c1(queries: float = 1e5, seed: int = 1) -> list[GridSpec]:
    m = model("resnet50")
    p = paris(m, 1)
    return [_spec(m, p, 1000.0, queries, seed, s) for s in ("elsa", "fifs")]


# ---- C2: BERT-base, 8-GPU PARIS, ELSA, load 10%..100% of nominal peak ----
C2_LOADS = tuple(round(0.1 * i, 1) for i in range(1, 11))


def c2(seeds: int = 16, queries: float = 1e5, seed0: int = 1, loads=C2_LOADS) -> list[GridSpec]:
    m = model("bert_base")
    p = paris(m, 8)
    peak = capacity_qps(m, p)
    return [_spec(m, p, load * peak, queries, seed0 + s) for load in loads for s in range(seeds)]


# ---- C3: MobileNet / ResNet-50 / BERT as independent per-model scenarios ----
def c3(seeds: int = 64, queries: float = 1e6, load: float = 0.8, seed0: int = 1) -> list[GridSpec]:
    out = []
    for name in ("mobilenet", "resnet50", "bert_base"):
        m = model(name)
        p = paris(m, 8)
        rate = load * capacity_qps(m, p)
        out += [_spec(m, p, rate, queries, seed0 + s) for s in range(seeds)]
    return out


# ---- C4: exhaustive 8-GPU MIG fleets scored by ELSA p99 ----
def gpu_configs(gpcs: int = 7, sizes=SIZES, full: bool = True) -> list[tuple[int, ...]]:
    """Per-GPU multisets of partition sizes, each sorted descending (as random_plan
    does, paris.hpp:314); `full` keeps those using all gpcs."""
    out = set()

    def rec(rem: int, start: int, cur: list[int]):
        if (rem == 0) or (not full and cur):
            out.add(tuple(sorted(cur, reverse=True)))
        for i in range(start, len(sizes)):
            if sizes[i] <= rem:
                rec(rem - sizes[i], i, cur + [sizes[i]])

    rec(gpcs, 0, [])
    return sorted(out, reverse=True)


def fleet_candidates(gpus: int = 8) -> list[PartitionPlan]:
    """Distinct aggregate fleets (instance counts per size) of `gpus` full GPUs. Each
    is represented by its first GPU-lexicographic placement (GPU configs in
    descending lexicographic order); that placement fixes partition ids."""
    cfgs = gpu_configs()
    seen: dict[tuple, PartitionPlan] = {}
    for combo in itertools.combinations_with_replacement(range(len(cfgs)), gpus):
        plan_gpus = [list(cfgs[i]) for i in combo]
        counts = tuple(sorted(PartitionPlan(gpus, 7, plan_gpus).instance_counts()))
        if counts not in seen:
            seen[counts] = PartitionPlan(gpus, 7, plan_gpus)
    return list(seen.values())


def c4(gpus: int = 8, seeds: int = 2, queries: float = 2e4, model_name: str = "bert_base", load: float = 0.7,
       max_candidates: int | None = None) -> tuple[list[GridSpec], list[PartitionPlan]]:
    m = model(model_name)
    rate = load * capacity_qps(m, paris(m, gpus))
    cands = fleet_candidates(gpus)
    if max_candidates:
        cands = cands[:max_candidates]
    specs = [_spec(m, p, rate, queries, 1 + s) for p in cands for s in range(seeds)]
    return specs, cands


# ---- C5: large Monte-Carlo grid: plans x rates x seeds ----
C5_LOADS = (0.3, 0.5, 0.7, 0.8, 0.9)
C5_PLANS = ("paris", "homog1", "homog2", "homog3", "homog7")


def c5_cells() -> list[tuple[str, Model, str, PartitionPlan, float]]:
    """The 75 (model, plan, load) cells of C5 in grid order: per model its 8-GPU PARIS plan
    and the homogeneous 1g/2g/3g/7g fleets of 56 GPCs, each at five loads."""
    plans = []
    for name in ("mobilenet", "resnet50", "bert_base"):
        m = model(name)
        plans.append((name, m, "paris", paris(m, 8)))
        for k in (1, 2, 3, 7):
            plans.append((name, m, f"homog{k}", homogeneous_plan(k, 56, 8, 7)))
    return [(name, m, tag, p, load) for (name, m, tag, p) in plans for load in C5_LOADS]


def c5(n_scenarios: int = 10_000, queries: float = 1e6, seed0: int = 1) -> list[GridSpec]:
    """Scenario i = cell i mod 75 with seed seed0 + i // 75 (cells interleaved, so any
    prefix or contiguous shard covers every plan and load)."""
    cells = c5_cells()
    out = []
    for i in range(n_scenarios):
        _, m, _, p, load = cells[i % len(cells)]
        out.append(_spec(m, p, load * capacity_qps(m, p), queries, seed0 + i // len(cells)))
    return out


def c5_labels(n_scenarios: int = 10_000) -> tuple[list[tuple[str, float]], list[str]]:
    """Per scenario of c5(): its PARIS decision group (model, load) and candidate plan tag,
    for `distributed.grouped_argmin` (which plan serves each model and load best by p99)."""
    cells = c5_cells()
    group = [(cells[i % len(cells)][0], cells[i % len(cells)][4]) for i in range(n_scenarios)]
    cand = [cells[i % len(cells)][2] for i in range(n_scenarios)]
    return group, cand


def shard(specs: list, rank: int, world: int) -> list:
    """Contiguous, cost-balanced shard of a scenario list (cost ~ expected queries x
    (partitions + 1)); every rank gets whole scenarios, no data-path exchange."""
    cost = np.array([s.rate_qps * s.duration_ms * (s.plan.total_instances() + 1) for s in specs], float)
    if len(specs) == 0:
        return []
    cum = np.cumsum(cost)
    total = cum[-1]
    lo = np.searchsorted(cum, total * rank / world, side="right") if rank else 0
    hi = np.searchsorted(cum, total * (rank + 1) / world, side="right") if rank + 1 < world else len(specs)
    return specs[lo:hi]
