"""TEST INFRASTRUCTURE ONLY: the BASELINE scenario grids built from the compiled
reference alone (oracle/_ref/libmsv_ref.so), for bench.py's reference arm.

The reference arm must not map the product library, so nothing here imports
`paper_2202_13481_b200`: profiles come from the reference's own `synth_profile`
(profile.hpp:183-215, `oraref_synth_profile`), batch distributions from its
`lognormal_batch_pdf` (workload.hpp:81-93, `oraref_lognormal_pdf`), plans from its
`paris_plan` / `homogeneous_plan` (paris.hpp:275-345). The recipe (presets, loads,
cell order, seeds) restates `paper_2202_13481_b200/workloads.py`;
`tests/test_cpu.py::test_ref_workloads_match_product_workloads` pins the two grids
to be identical field for field, bit for bit.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import oracle_py as O

SIZES = (1, 2, 3, 4, 7)
B_MAX = 32
# (work_per_sample, fixed_overhead, parallelism_per_sample, util_cap): DESIGN.md §7
PRESETS = {
    "mobilenet": (0.4, 0.5, 0.15, 0.95),
    "resnet50": (0.8, 0.8, 0.25, 0.95),
    "bert_base": (4.0, 2.0, 0.40, 0.95),
}
SLA_MULTIPLIER = 1.5
C5_LOADS = (0.3, 0.5, 0.7, 0.8, 0.9)
C2_LOADS = tuple(round(0.1 * i, 1) for i in range(1, 11))


@dataclass
class Table:
    sizes: np.ndarray
    b_max: int
    latency: np.ndarray
    utilization: np.ndarray


@dataclass
class Dist:
    weights: np.ndarray


@dataclass
class Plan:
    num_gpus: int
    gpcs_per_gpu: int
    gpus: list

    def flatten(self):
        return [k for g in self.gpus for k in g]

    def total_instances(self):
        return sum(len(g) for g in self.gpus)

    def key(self):
        return (self.num_gpus, self.gpcs_per_gpu, tuple(tuple(g) for g in self.gpus))


@dataclass
class Sla:
    sla_target_ms: float
    alpha: float = 1.0
    beta: float = 1.0


@dataclass
class Spec:
    plan: Plan
    table: Table
    dist: Dist
    sla: Sla
    rate_qps: float
    duration_ms: float
    seed: int
    scheduler: str = "elsa"
    warmup_fraction: float = 0.1


def _ora() -> O.Oracle:
    ora = O.best_oracle()
    if ora.kind != "reference":
        raise FileNotFoundError("oracle/_ref/libmsv_ref.so (build it with oracle/build_oracle.py)")
    return ora


def _check(ora, rc, what):
    if rc:
        raise ora.err(rc)


def synth_profile(params, sizes=SIZES, b_max=B_MAX) -> Table:
    ora = _ora()
    s = np.asarray(sizes, np.int32)
    out = np.zeros(len(s), np.int32)
    lat = np.zeros(len(s) * b_max)
    util = np.zeros_like(lat)
    n = C.c_int()
    f = ora.L.oraref_synth_profile
    f.argtypes = [C.c_double] * 4 + [O._i32p, C.c_int, C.c_int, O._i32p, C.POINTER(C.c_int), O._f64p, O._f64p]
    _check(ora, f(*params, O._p(s, C.c_int32), len(s), b_max, O._p(out, C.c_int32), C.byref(n),
                  O._p(lat, C.c_double), O._p(util, C.c_double)), "synth_profile")
    k = n.value
    return Table(out[:k].copy(), b_max, lat[:k * b_max].reshape(k, b_max).copy(),
                 util[:k * b_max].reshape(k, b_max).copy())


def lognormal_batch_pdf(mu=1.0, sigma=1.0, b_max=B_MAX) -> Dist:
    ora = _ora()
    pmf, cdf = np.zeros(b_max), np.zeros(b_max)
    f = ora.L.oraref_lognormal_pdf
    f.argtypes = [C.c_double, C.c_double, C.c_int, O._f64p, O._f64p]
    _check(ora, f(mu, sigma, b_max, O._p(pmf, C.c_double), O._p(cdf, C.c_double)), "lognormal_batch_pdf")
    return Dist(pmf)


def paris_plan(table: Table, dist: Dist, gpus: int) -> Plan:
    r = _ora().paris_plan(table, dist, 7 * gpus, gpus, 7)
    return Plan(gpus, 7, r["gpus"])


def homogeneous_plan(k: int, total_gpcs: int, num_gpus: int, gpcs_per_gpu: int) -> Plan:
    ora = _ora()
    n_per = np.zeros(num_gpus, np.int32)
    flat = np.zeros(num_gpus * gpcs_per_gpu, np.int32)
    f = ora.L.oraref_homogeneous_plan
    f.argtypes = [C.c_int] * 4 + [O._i32p, O._i32p]
    _check(ora, f(k, total_gpcs, num_gpus, gpcs_per_gpu, O._p(n_per, C.c_int32), O._p(flat, C.c_int32)),
           "homogeneous_plan")
    out, off = [], 0
    for g in range(num_gpus):
        out.append([int(x) for x in flat[off:off + n_per[g]]])
        off += int(n_per[g])
    return Plan(num_gpus, gpcs_per_gpu, out)


_MODELS: dict = {}


def model(name: str):
    if name not in _MODELS:
        t = synth_profile(PRESETS[name])
        d = lognormal_batch_pdf()
        row = int(np.searchsorted(t.sizes, int(t.sizes[-1])))
        sla = SLA_MULTIPLIER * float(t.latency[row, B_MAX - 1])  # derive_sla_target, metrics.hpp:34-37
        _MODELS[name] = (t, d, Sla(sla, 1.0, 1.0))
    return _MODELS[name]


def capacity_qps(table: Table, dist: Dist, plan: Plan) -> float:
    pmf = np.asarray(dist.weights, float)
    pmf = pmf / pmf.sum()
    row = {int(k): i for i, k in enumerate(table.sizes)}
    return float(sum(1000.0 / float((pmf * table.latency[row[k]]).sum()) for k in plan.flatten()))


def _spec(m, plan, rate, queries, seed, sched="elsa") -> Spec:
    t, d, sla = m
    return Spec(plan, t, d, sla, rate, queries / rate * 1000.0, seed, sched)


def c5_cells():
    plans = []
    for name in ("mobilenet", "resnet50", "bert_base"):
        m = model(name)
        plans.append((name, m, paris_plan(m[0], m[1], 8)))
        for k in (1, 2, 3, 7):
            plans.append((name, m, homogeneous_plan(k, 56, 8, 7)))
    return [(name, m, p, load) for (name, m, p) in plans for load in C5_LOADS]


def c5(n_scenarios: int = 10_000, queries: float = 1e6, seed0: int = 1) -> list[Spec]:
    cells = c5_cells()
    out = []
    for i in range(n_scenarios):
        _, m, p, load = cells[i % len(cells)]
        rate = load * capacity_qps(m[0], m[1], p)
        out.append(_spec(m, p, rate, queries, seed0 + i // len(cells)))
    return out


def c2(seeds: int = 16, queries: float = 1e5, seed0: int = 1, loads=C2_LOADS) -> list[Spec]:
    m = model("bert_base")
    p = paris_plan(m[0], m[1], 8)
    peak = capacity_qps(m[0], m[1], p)
    return [_spec(m, p, load * peak, queries, seed0 + s) for load in loads for s in range(seeds)]
