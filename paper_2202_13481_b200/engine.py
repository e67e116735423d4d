"""Python face of the engine: the reference's data types (ProfileTable,
BatchDistribution, PartitionPlan, SlaConfig) as light holders, and `Engine`, one
device context (include/msv.h) with the hot-path calls:

    Engine.run_grid      sample_trace -> run -> tail_latency per scenario (device)
    Engine.run           run() on host traces, per-query records   (engine.hpp:115)
    Engine.sample_trace  sample_trace on the device                (workload.hpp:97)
    Engine.tail_latency  nearest-rank tail on the device           (metrics.hpp:22)
    Engine.dispatch      elsa_dispatch / fifs_dispatch / t_wait    (sched.hpp:77-174)
    Engine.grid          device-resident grid for timing loops

Host-side constructors (synth_profile, lognormal_batch_pdf, paris_plan) call the C++
host headers through libmsv.so, so Python and C++ users get the same bits.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import _native as N
from ._native import check


def _arr(a, dtype):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


# ---------------------------------------------------------------------------
# reference data types
# ---------------------------------------------------------------------------
@dataclass
class SyntheticProfileParams:
    """profile.hpp:43-48 (defaults identical)."""
    work_per_sample: float = 10.0
    fixed_overhead: float = 5.0
    parallelism_per_sample: float = 0.15
    util_cap: float = 0.95


@dataclass
class ProfileTable:
    """Dense [size_idx][batch-1] latency / utilisation grid (profile.hpp:52-132)."""
    sizes: np.ndarray
    b_max: int
    latency: np.ndarray      # (n_sizes, b_max) float64
    utilization: np.ndarray  # (n_sizes, b_max) float64
    model: str = "synthetic"

    def _cell(self, k: int, batch: int) -> tuple[int, int]:
        idx = int(np.searchsorted(self.sizes, k))
        if idx >= len(self.sizes) or int(self.sizes[idx]) != k:
            raise N.LookupError_(f"profile: unknown partition size k={k}")
        if batch < 1 or batch > self.b_max:
            raise N.LookupError_(f"profile: batch {batch} outside grid 1..{self.b_max}")
        return idx, batch - 1

    def latency_ms(self, k: int, batch: int) -> float:
        return float(self.latency[self._cell(k, batch)])

    def util(self, k: int, batch: int) -> float:
        return float(self.utilization[self._cell(k, batch)])

    def max_size(self) -> int:
        return int(self.sizes[-1])


def synth_profile(params: SyntheticProfileParams, sizes: Sequence[int], b_max: int, model: str = "synthetic"
                  ) -> ProfileTable:
    """synth_profile (profile.hpp:183-215), computed by the C++ host header."""
    s = _arr(sizes, np.int32)
    out_sizes = np.zeros(max(len(s), 1), np.int32)
    lat = np.zeros(max(len(s), 1) * max(b_max, 1), np.float64)
    util = np.zeros_like(lat)
    n = C.c_int32(0)
    check(N.lib().msv_synth_profile(params.work_per_sample, params.fixed_overhead, params.parallelism_per_sample,
                                    params.util_cap, len(s), _ptr(s, C.c_int32), b_max, C.byref(n),
                                    _ptr(out_sizes, C.c_int32), _ptr(lat, C.c_double), _ptr(util, C.c_double)),
          "synth_profile")
    k = n.value
    return ProfileTable(out_sizes[:k].copy(), b_max, lat[:k * b_max].reshape(k, b_max).copy(),
                        util[:k * b_max].reshape(k, b_max).copy(), model)


@dataclass
class BatchDistribution:
    """BatchDistribution(weights) (workload.hpp:22-53); `weights` are kept raw so the
    device rebuilds pmf/cdf with the reference's exact arithmetic."""
    weights: np.ndarray

    @property
    def b_max(self) -> int:
        return len(self.weights)

    def tables(self) -> tuple[np.ndarray, np.ndarray]:
        w = [float(x) for x in self.weights]
        total = 0.0
        for x in w:
            total += x
        pmf = np.array([x / total for x in w])
        cdf = np.empty_like(pmf)
        acc = 0.0
        for i, p in enumerate(pmf):
            acc = p if i == 0 else acc + p
            cdf[i] = acc
        cdf[-1] = 1.0
        return pmf, cdf


def lognormal_batch_pdf(mu: float, sigma: float, b_max: int) -> BatchDistribution:
    """lognormal_batch_pdf (workload.hpp:81-93); returned as its exact normalised pmf."""
    pmf = np.zeros(max(b_max, 1))
    cdf = np.zeros_like(pmf)
    check(N.lib().msv_lognormal_pdf(mu, sigma, b_max, _ptr(pmf, C.c_double), _ptr(cdf, C.c_double)),
          "lognormal_batch_pdf")
    return BatchDistribution(pmf)


@dataclass
class PartitionPlan:
    """PartitionPlan (paris.hpp:133-156): sizes per GPU; ids = GPU-major order."""
    num_gpus: int
    gpcs_per_gpu: int
    gpus: list[list[int]]

    def flatten(self) -> list[int]:
        return [k for g in self.gpus for k in g]

    def total_instances(self) -> int:
        return sum(len(g) for g in self.gpus)

    def instance_counts(self) -> list[tuple[int, int]]:
        c: dict[int, int] = {}
        for k in self.flatten():
            c[k] = c.get(k, 0) + 1
        return sorted(c.items())

    def used_gpcs(self) -> int:
        return sum(self.flatten())

    def key(self) -> tuple:
        return (self.num_gpus, self.gpcs_per_gpu, tuple(tuple(g) for g in self.gpus))


def paris_plan(table: ProfileTable, dist: BatchDistribution, total_gpcs: int, num_gpus: int, gpcs_per_gpu: int,
               knee_threshold: float = 0.8) -> PartitionPlan:
    """paris_plan (paris.hpp:329-345) through the C++ host header."""
    n_per = np.zeros(num_gpus, np.int32)
    flat = np.zeros(num_gpus * gpcs_per_gpu, np.int32)
    sizes = _arr(table.sizes, np.int32)
    lat = _arr(table.latency, np.float64)
    util = _arr(table.utilization, np.float64)
    w = _arr(dist.weights, np.float64)
    if len(w) != table.b_max:
        raise N.ValidationError("paris_plan: distribution support must match profile b_max")
    check(N.lib().msv_paris_plan(len(sizes), _ptr(sizes, C.c_int32), table.b_max, _ptr(lat, C.c_double),
                                 _ptr(util, C.c_double), _ptr(w, C.c_double), total_gpcs, num_gpus, gpcs_per_gpu,
                                 knee_threshold, _ptr(n_per, C.c_int32), _ptr(flat, C.c_int32)), "paris_plan")
    gpus, off = [], 0
    for g in range(num_gpus):
        gpus.append([int(x) for x in flat[off:off + n_per[g]]])
        off += int(n_per[g])
    return PartitionPlan(num_gpus, gpcs_per_gpu, gpus)


def homogeneous_plan(k: int, total_gpcs: int, num_gpus: int, gpcs_per_gpu: int) -> PartitionPlan:
    """homogeneous_plan (paris.hpp:275-290)."""
    if k < 1:
        raise N.ParamError("homogeneous_plan: k must be >= 1")
    if num_gpus < 1:
        raise N.ParamError("homogeneous_plan: num_gpus must be >= 1")
    if k > gpcs_per_gpu:
        raise N.InfeasibleError("homogeneous_plan: k exceeds gpcs_per_gpu")
    n = min(num_gpus * (gpcs_per_gpu // k), total_gpcs // k)
    gpus: list[list[int]] = [[] for _ in range(num_gpus)]
    for i in range(n):
        gpus[i % num_gpus].append(k)
    return PartitionPlan(num_gpus, gpcs_per_gpu, gpus)


@dataclass
class ParisJob:
    """One paris_plan call (paris.hpp:329-345) for Engine.paris_batch."""
    table: ProfileTable
    dist: BatchDistribution
    total_gpcs: int
    num_gpus: int
    gpcs_per_gpu: int
    knee_threshold: float = 0.8


@dataclass
class ParisOutcome:
    """ParisResult (paris.hpp:318-324) of one job, or the exception paris_plan throws."""
    knees: dict = field(default_factory=dict)            # k -> knee batch
    segments: list = field(default_factory=list)         # (k, first, last)
    ratios: list = field(default_factory=list)           # RatioEntry::ratio, ascending k
    segment_mass: list = field(default_factory=list)
    counts: list = field(default_factory=list)           # InstanceCounts::counts (real)
    weighted_sum: float = 0.0
    normalizer: float = 0.0
    plan: PartitionPlan | None = None
    error: Exception | None = None


def _paris_error(o, job: ParisJob) -> Exception:
    """The reference's exception (type and message) for a failed device job."""
    st, thr = o.status, job.knee_threshold
    if st == N.MSV_VALIDATION:
        if len(job.dist.weights) != job.table.b_max:
            return N.ValidationError("paris_plan: distribution support must match profile b_max")
        if o.err_b:
            return N.ValidationError(f"instance_ratios: nonpositive throughput at (k={o.err_k}, b={o.err_b})")
        if o.weighted_sum == 0.0 and any(o.ratio[i] < 0.0 for i in range(o.n_sizes)):
            return N.ValidationError("instance_counts: negative ratio")
        return N.ValidationError("segment_batches: knees must be nondecreasing in k")
    if st == N.MSV_PARAM:
        if len(job.table.sizes) > N.MSV_PARIS_MAX_SIZES:
            return N.ParamError(f"paris batch: at most {N.MSV_PARIS_MAX_SIZES} partition sizes per profile")
        if not (thr > 0.0) or thr > 1.0:
            return N.ParamError("knee: threshold must be in (0,1]")
        if job.total_gpcs < 1:
            return N.ParamError("instance_counts: total_gpcs must be >= 1")
        if not (o.weighted_sum > 0.0):
            return N.ParamError("instance_counts: all ratios are zero")
        if job.num_gpus < 1:
            return N.ParamError("pack_plan: num_gpus must be >= 1")
        if job.gpcs_per_gpu < 1:
            return N.ParamError("pack_plan: gpcs_per_gpu must be >= 1")
        return N.ParamError("pack_plan: partition size must be positive")
    if st == N.MSV_INFEASIBLE:
        return N.InfeasibleError(f"pack_plan: instance of size {o.err_k} exceeds gpcs_per_gpu={job.gpcs_per_gpu}")
    return N._ERRORS.get(st, N.Error)(f"paris_plan: status {st}")


@dataclass
class SlaConfig:
    sla_target_ms: float
    alpha: float = 1.0
    beta: float = 1.0


def derive_sla_target(table: ProfileTable, b_max: int, multiplier: float) -> float:
    """derive_sla_target (metrics.hpp:34-37)."""
    if not multiplier > 0.0:
        raise N.ParamError("derive_sla_target: multiplier must be > 0")
    return multiplier * table.latency_ms(table.max_size(), b_max)


@dataclass
class GridSpec:
    """One scenario of a grid (msv_scenario) in Python terms."""
    plan: PartitionPlan
    table: ProfileTable
    dist: BatchDistribution
    sla: SlaConfig
    rate_qps: float
    duration_ms: float
    seed: int
    scheduler: str = "elsa"
    warmup_fraction: float = 0.1
    routing: list[tuple[int, int, int]] | None = None  # (k, first, last) segments
    check_wait: bool = False


# Placeholder distribution of replay scenarios (the trace is the caller's).
_REPLAY_DIST = BatchDistribution(np.ones(1))


# ---------------------------------------------------------------------------
# device context
# ---------------------------------------------------------------------------
@dataclass
class PreparedGrid:
    """A grid's msv_scenario array (include/msv.h), marshalled once for repeated calls."""
    array: object
    n: int
    n_partitions: int


class Engine:
    """One msv_ctx: a CUDA device, its memory and stream — or, given a list of devices,
    a multi-device context (msv_create_multi): grids are cut into cost-balanced
    contiguous shards, one per device, run concurrently and gathered in scenario order."""

    def __init__(self, device: int | Sequence[int] = 0, log1p_variant: int | None = None):
        self._lib = N.lib()
        h = C.c_void_p()
        if isinstance(device, (list, tuple)):
            ids = _arr(list(device), np.int32)
            check(self._lib.msv_create_multi(_ptr(ids, C.c_int32), len(ids), C.byref(h)), "msv_create_multi")
            self.devices = [int(x) for x in ids]
            device = self.devices[0]
        else:
            check(self._lib.msv_create(device, C.byref(h)), "msv_create")
            self.devices = [device]
        self._h = h
        self.device = device
        if log1p_variant is not None:
            check(self._lib.msv_set_log1p_variant(self._h, log1p_variant), "msv_set_log1p_variant")
        self._profiles: dict[int, int] = {}
        self._dists: dict[int, int] = {}
        self._plans: dict[tuple, int] = {}
        self._plan_objs: dict[int, tuple] = {}  # id(plan) -> (plan, handle, contents)
        self._routings: dict[tuple, int] = {}
        self._keep: list = []

    def close(self) -> None:
        if self._h:
            self._lib.msv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def log1p_variant(self) -> int:
        v = C.c_int(-1)
        check(self._lib.msv_get_log1p_variant(self._h, C.byref(v)))
        return v.value

    def kernel_launches(self) -> int:
        return int(self._lib.msv_kernel_launches(self._h))

    # ---- uploads (cached by object identity / value) ----
    def profile(self, t: ProfileTable) -> int:
        key = id(t)
        if key not in self._profiles:
            sizes = _arr(t.sizes, np.int32)
            lat = _arr(t.latency, np.float64)
            util = _arr(t.utilization, np.float64)
            h = C.c_int32(-1)
            check(self._lib.msv_upload_profile(self._h, len(sizes), _ptr(sizes, C.c_int32), t.b_max,
                                               _ptr(lat, C.c_double), _ptr(util, C.c_double), C.byref(h)),
                  "msv_upload_profile")
            self._profiles[key] = h.value
            self._keep.append(t)
        return self._profiles[key]

    def dist(self, d: BatchDistribution) -> int:
        key = id(d)
        if key not in self._dists:
            w = _arr(d.weights, np.float64)
            h = C.c_int32(-1)
            check(self._lib.msv_upload_dist(self._h, len(w), _ptr(w, C.c_double), C.byref(h)), "msv_upload_dist")
            self._dists[key] = h.value
            self._keep.append(d)
        return self._dists[key]

    def plan(self, p: PartitionPlan) -> int:
        hit = self._plan_objs.get(id(p))  # the same, unchanged object again: skip the key
        if hit is not None and hit[0] is p and hit[2] == p.gpus and hit[3] == (p.num_gpus, p.gpcs_per_gpu):
            return hit[1]
        key = p.key()
        if key not in self._plans:
            n_per = _arr([len(g) for g in p.gpus] or [0], np.int32)
            flat = _arr(p.flatten() or [0], np.int32)
            h = C.c_int32(-1)
            check(self._lib.msv_upload_plan(self._h, p.num_gpus, p.gpcs_per_gpu, _ptr(n_per, C.c_int32),
                                            _ptr(flat, C.c_int32), C.byref(h)), "msv_upload_plan")
            self._plans[key] = h.value
        # (holds p, so its id stays unique; a snapshot of its contents catches later edits)
        self._plan_objs[id(p)] = (p, self._plans[key], [list(g) for g in p.gpus], (p.num_gpus, p.gpcs_per_gpu))
        return self._plans[key]

    def routing(self, segs: Sequence[tuple[int, int, int]]) -> int:
        key = tuple(tuple(s) for s in segs)
        if key not in self._routings:
            k = _arr([s[0] for s in segs] or [0], np.int32)
            f = _arr([s[1] for s in segs] or [0], np.int32)
            la = _arr([s[2] for s in segs] or [0], np.int32)
            h = C.c_int32(-1)
            check(self._lib.msv_upload_routing(self._h, len(segs), _ptr(k, C.c_int32), _ptr(f, C.c_int32),
                                               _ptr(la, C.c_int32), C.byref(h)), "msv_upload_routing")
            self._routings[key] = h.value
        return self._routings[key]

    def scenarios(self, specs: Iterable[GridSpec]) -> C.Array:
        """Marshal specs into an msv_scenario array (column-wise through numpy)."""
        specs = list(specs)
        n = len(specs)
        arr = (N.Scenario * max(n, 1))()
        if n == 0:
            return arr
        a = np.ctypeslib.as_array(arr)
        plan_h: dict[int, int] = {}  # per plan object; uploads are cached by value in self.plan

        def ph(p):
            h = plan_h.get(id(p))
            if h is None:
                h = plan_h[id(p)] = self.plan(p)
            return h

        a["profile"] = [self.profile(s.table) for s in specs]
        a["dist"] = [self.dist(s.dist) for s in specs]
        a["plan"] = [ph(s.plan) for s in specs]
        a["scheduler"] = [N.MSV_ELSA if s.scheduler == "elsa" else N.MSV_FIFS for s in specs]
        a["routing"] = [self.routing(s.routing) if s.routing is not None else -1 for s in specs]
        a["flags"] = [N.MSV_FLAG_CHECK_WAIT if s.check_wait else 0 for s in specs]
        a["sla_ms"] = [s.sla.sla_target_ms for s in specs]
        a["alpha"] = [s.sla.alpha for s in specs]
        a["beta"] = [s.sla.beta for s in specs]
        a["rate_qps"] = [s.rate_qps for s in specs]
        a["duration_ms"] = [s.duration_ms for s in specs]
        a["warmup_fraction"] = [s.warmup_fraction for s in specs]
        a["seed"] = np.array([s.seed for s in specs], dtype=np.uint64)
        return arr

    # ---- hot path ----
    def run_grid(self, specs, tail_p: Sequence[float] = (0.95, 0.99), usage: bool = False) -> dict:
        """One msv_run_grid call. `specs` is a list of GridSpec, or the msv_scenario array
        Engine.scenarios() built from one (the C-ABI input, marshalled once)."""
        if isinstance(specs, PreparedGrid):
            sc, n, n_use = specs.array, specs.n, specs.n_partitions
            ps = _arr(list(tail_p) or [0.5], np.float64)
            res = (N.Result * max(n, 1))()
            use = (N.Usage * max(n_use, 1))() if usage else None
            check(self._lib.msv_run_grid(self._h, sc, n, _ptr(ps, C.c_double), len(tail_p), res, use), "run_grid")
            return results_to_numpy(res, n, len(tail_p), use, n_use)
        sc = self.scenarios(specs)
        n = len(specs)
        ps = _arr(list(tail_p) or [0.5], np.float64)
        res = (N.Result * max(n, 1))()
        n_use = sum(s.plan.total_instances() for s in specs)
        use = (N.Usage * max(n_use, 1))() if usage else None
        check(self._lib.msv_run_grid(self._h, sc, n, _ptr(ps, C.c_double), len(tail_p), res, use), "run_grid")
        return results_to_numpy(res, n, len(tail_p), use, n_use)

    def run_grid_noise(self, specs, noise_sigma, noise_seed, tail_p: Sequence[float] = (0.95, 0.99),
                       usage: bool = False) -> dict:
        """One msv_run_grid_noise call: every scenario with execution noise
        (EngineOptions::noise_sigma / noise_seed, engine.hpp:140-145) — sample_trace ->
        run -> tail_latency, batched on the device (K1, K5 one warp per scenario, K3).
        `noise_sigma` / `noise_seed`: one value, or one per scenario."""
        n = len(specs)
        sig = np.broadcast_to(np.asarray(noise_sigma, np.float64), (n,)).copy()
        seed = np.broadcast_to(np.asarray(noise_seed, np.uint64), (n,)).copy()
        sc = self.scenarios(specs)
        ps = _arr(list(tail_p) or [0.5], np.float64)
        res = (N.Result * max(n, 1))()
        n_use = sum(s.plan.total_instances() for s in specs)
        use = (N.Usage * max(n_use, 1))() if usage else None
        check(self._lib.msv_run_grid_noise(self._h, sc, n, _ptr(sig, C.c_double), seed.ctypes.data_as(
            C.POINTER(C.c_uint64)), _ptr(ps, C.c_double), len(tail_p), res, use), "run_grid_noise")
        return results_to_numpy(res, n, len(tail_p), use, n_use)

    def run(self, plan: PartitionPlan, scheduler: str, arrival, batch, duration_ms: float, table: ProfileTable,
            sla: SlaConfig, warmup_fraction: float = 0.1, routing=None, check_wait: bool = False,
            tail_p: Sequence[float] = (), noise_sigma: float = 0.0, noise_seed: int = 1) -> dict:
        """run() (engine.hpp:115-253) on one host trace, with per-query records;
        noise_sigma > 0: execution noise (engine.hpp:140-145) on K5 (msv_run_noise)."""
        if noise_sigma > 0.0:
            return self._run_noise(plan, scheduler, arrival, batch, duration_ms, table, sla, warmup_fraction, routing,
                                   tail_p, noise_sigma, noise_seed)
        return self.run_many([(plan, scheduler, arrival, batch, duration_ms, table, sla, warmup_fraction, routing,
                               check_wait)], tail_p)[0]

    def _run_noise(self, plan, scheduler, arrival, batch, duration_ms, table, sla, warmup_fraction, routing, tail_p,
                   noise_sigma, noise_seed) -> dict:
        arrival, batch = _arr(arrival, np.float64), _arr(batch, np.int32)
        n = len(arrival)
        # the reference's heap serves arrivals by (time, trace index): a stable sort
        order = np.argsort(arrival, kind="stable")
        arr_s, bat_s = np.ascontiguousarray(arrival[order]), np.ascontiguousarray(batch[order])
        spec = GridSpec(plan, table, _REPLAY_DIST, sla, 1.0, duration_ms, 0, scheduler, warmup_fraction, routing, False)
        sc = self.scenarios([spec])
        mult = np.zeros(max(n, 1))
        check(self._lib.msv_noise_multipliers(int(noise_seed), float(noise_sigma), n, _ptr(mult, C.c_double)),
              "noise_multipliers")
        P = plan.total_instances()
        res = (N.Result * 1)()
        use = (N.Usage * max(P, 1))()
        rec = (N.Record * max(n, 1))()
        a = arr_s if n else np.zeros(1)
        b = bat_s if n else np.zeros(1, np.int32)
        check(self._lib.msv_run_noise(self._h, sc, n, _ptr(a, C.c_double), _ptr(b, C.c_int32),
                                      _ptr(mult, C.c_double), res, use, rec), "run")
        agg = results_to_numpy(res, 1, 0, use, P)
        r = {k: v[0] for k, v in agg.items() if k not in ("usage", "tail")}
        rr = np.ctypeslib.as_array(rec)[:n] if n else np.zeros(0, rec._type_)
        inv = np.empty(n, np.int64)
        inv[order] = np.arange(n)
        r["partition"] = np.array(rr["partition"], np.int32)[inv]
        r["start_ms"] = np.array(rr["start_ms"])[inv]
        r["finish_ms"] = np.array(rr["finish_ms"])[inv]
        r["kind"] = np.array(rr["kind"], np.int32)[inv]
        r["busy_ms"] = agg["usage"]["busy_ms"]
        r["weighted_busy_ms"] = agg["usage"]["weighted_busy_ms"]
        r["queries"] = agg["usage"]["queries"]
        if tail_p:
            lat = r["finish_ms"] - arrival
            meas = lat[arrival >= r["warmup_ms"]]
            r["tail"] = (np.array(self.tail_latency(meas, list(tail_p)), dtype=np.float64) if len(meas)
                         else np.full(len(tail_p), np.nan))
        return r

    def run_many(self, items, tail_p: Sequence[float] = ()) -> list[dict]:
        """run() on many host traces in one device grid. Traces need not be sorted: like the
        reference's event heap, which serves arrivals by (time, trace index)
        (engine.hpp:101-107), an unsorted trace is stable-sorted for the device and its
        per-query records are mapped back to trace order."""
        specs, arrs, bats, perms = [], [], [], []
        for plan, scheduler, arrival, batch, duration_ms, table, sla, warm, routing, cw in items:
            specs.append(GridSpec(plan, table, _REPLAY_DIST, sla, 1.0, duration_ms, 0, scheduler, warm, routing,
                                  cw))
            a, b = _arr(arrival, np.float64), _arr(batch, np.int32)
            perm = None
            if len(a) > 1 and np.any(a[1:] < a[:-1]):
                perm = np.argsort(a, kind="stable")
                a, b = np.ascontiguousarray(a[perm]), np.ascontiguousarray(b[perm])
            arrs.append(a)
            bats.append(b)
            perms.append(perm)
        sc = self.scenarios(specs)
        n = len(specs)
        offs = np.zeros(n + 1, np.int64)
        for i, a in enumerate(arrs):
            offs[i + 1] = offs[i] + len(a)
        arrival = np.concatenate(arrs) if offs[-1] else np.zeros(1)
        batch = np.concatenate(bats).astype(np.int32) if offs[-1] else np.zeros(1, np.int32)
        ps = _arr(list(tail_p) or [0.5], np.float64)
        res = (N.Result * max(n, 1))()
        n_use = sum(s.plan.total_instances() for s in specs)
        use = (N.Usage * max(n_use, 1))()
        rec = (N.Record * max(int(offs[-1]), 1))()
        check(self._lib.msv_run_replay(self._h, sc, n, _ptr(offs, C.c_int64), _ptr(arrival, C.c_double),
                                       _ptr(batch, C.c_int32), _ptr(ps, C.c_double), len(tail_p), res, use, rec),
              "run")
        agg = results_to_numpy(res, n, len(tail_p), use, n_use)
        recs = np.ctypeslib.as_array(rec)[: int(offs[-1])] if offs[-1] else np.zeros(0, rec._type_)
        out, uo = [], 0
        for i, s in enumerate(specs):
            P = s.plan.total_instances()
            r = {k: (v[i] if isinstance(v, np.ndarray) and k != "usage" else v) for k, v in agg.items() if k != "usage"}
            rr = recs[offs[i]:offs[i + 1]]
            inv = slice(None)
            if perms[i] is not None:
                inv = np.empty(len(perms[i]), np.int64)
                inv[perms[i]] = np.arange(len(perms[i]))
            r["partition"] = np.array(rr["partition"], np.int32)[inv]
            r["start_ms"] = np.array(rr["start_ms"])[inv]
            r["finish_ms"] = np.array(rr["finish_ms"])[inv]
            r["kind"] = np.array(rr["kind"], np.int32)[inv]
            r["busy_ms"] = agg["usage"]["busy_ms"][uo:uo + P]
            r["weighted_busy_ms"] = agg["usage"]["weighted_busy_ms"][uo:uo + P]
            r["queries"] = agg["usage"]["queries"][uo:uo + P]
            uo += P
            out.append(r)
        return out

    def sample_trace(self, dist: BatchDistribution, rate_qps: float, duration_ms: float, seed: int
                     ) -> tuple[np.ndarray, np.ndarray]:
        h = self.dist(dist)
        mean = rate_qps * duration_ms / 1000.0 if rate_qps > 0 else 0.0
        cap = int(np.ceil(mean + 10 * np.sqrt(max(mean, 0.0)) + 160))
        while True:
            arr = np.zeros(max(cap, 1))
            bat = np.zeros(max(cap, 1), np.int32)
            n = C.c_int64(0)
            rc = self._lib.msv_sample_trace(self._h, h, rate_qps, duration_ms, seed, cap, _ptr(arr, C.c_double),
                                            _ptr(bat, C.c_int32), C.byref(n))
            if rc == N.MSV_PARAM and n.value > cap:
                cap *= 4
                continue
            check(rc, "sample_trace")
            return arr[: n.value].copy(), bat[: n.value].copy()

    def tail_latency(self, samples, p: float | Sequence[float] = 0.95):
        s = _arr(samples, np.float64)
        ps = _arr([p] if np.isscalar(p) else list(p), np.float64)
        out = np.zeros(len(ps))
        check(self._lib.msv_tail_latency(self._h, _ptr(s, C.c_double), len(s), _ptr(ps, C.c_double), len(ps),
                                         _ptr(out, C.c_double)), "tail_latency")
        return float(out[0]) if np.isscalar(p) else out

    def dispatch(self, table: ProfileTable | None, scheduler: str, trials: Sequence[dict], want_t_wait: bool = False):
        """Batched elsa_dispatch / fifs_dispatch. Each trial: dict(parts=[(id, k, busy, cur_est, cur_start,
        [queued batches])...], batch, now, sla, alpha, beta)."""
        part_off, ids, ks, busy, est, start, q_off, qb = [0], [], [], [], [], [], [0], []
        qbatch, now, sla, al, be = [], [], [], [], []
        for t in trials:
            for (pid, k, b, e, s, queue) in t["parts"]:
                ids.append(pid)
                ks.append(k)
                busy.append(1 if b else 0)
                est.append(e)
                start.append(s)
                qb.extend(queue)
                q_off.append(len(qb))
            part_off.append(len(ids))
            qbatch.append(t["batch"])
            now.append(t.get("now", 0.0))
            sla.append(t.get("sla", 1.0))
            al.append(t.get("alpha", 1.0))
            be.append(t.get("beta", 1.0))
        a = {k: _arr(v or [0], dt) for k, v, dt in [
            ("part_off", part_off, np.int64), ("id", ids, np.int32), ("k", ks, np.int32), ("busy", busy, np.uint8),
            ("est", est, np.float64), ("start", start, np.float64), ("q_off", q_off, np.int64),
            ("qb", qb, np.int32), ("qbatch", qbatch, np.int32), ("now", now, np.float64), ("sla", sla, np.float64),
            ("al", al, np.float64), ("be", be, np.float64)]}
        n = len(trials)
        chosen = np.zeros(max(n, 1), np.int32)
        kind = np.zeros(max(n, 1), np.int32)
        tw = np.zeros(max(len(ids), 1))
        prof = self.profile(table) if table is not None else -1
        check(self._lib.msv_dispatch_batch(
            self._h, prof, N.MSV_ELSA if scheduler == "elsa" else N.MSV_FIFS, n, _ptr(a["part_off"], C.c_int64),
            _ptr(a["id"], C.c_int32), _ptr(a["k"], C.c_int32), _ptr(a["busy"], C.c_uint8),
            _ptr(a["est"], C.c_double), _ptr(a["start"], C.c_double), _ptr(a["q_off"], C.c_int64),
            _ptr(a["qb"], C.c_int32), _ptr(a["qbatch"], C.c_int32), _ptr(a["now"], C.c_double),
            _ptr(a["sla"], C.c_double), _ptr(a["al"], C.c_double), _ptr(a["be"], C.c_double),
            _ptr(chosen, C.c_int32), _ptr(kind, C.c_int32), _ptr(tw, C.c_double) if want_t_wait else None),
            "dispatch")
        if want_t_wait:
            return chosen[:n], kind[:n], tw[: len(ids)]
        return chosen[:n], kind[:n]

    def prepare(self, specs: Sequence[GridSpec]) -> PreparedGrid:
        return PreparedGrid(self.scenarios(specs), len(specs), sum(s.plan.total_instances() for s in specs))

    def paris_batch(self, jobs: Sequence[ParisJob]) -> list[ParisOutcome]:
        """Batched paris_plan on the device (K4, msv_paris_batch): one warp per job."""
        n = len(jobs)
        if n == 0:
            return []
        ja = (N.ParisJob * n)()
        n_gpu = n_inst = 0
        for i, j in enumerate(jobs):
            ja[i].profile = self.profile(j.table)
            ja[i].dist = self.dist(j.dist)
            ja[i].total_gpcs = j.total_gpcs
            ja[i].num_gpus = j.num_gpus
            ja[i].gpcs_per_gpu = j.gpcs_per_gpu
            ja[i].knee_threshold = j.knee_threshold
            if j.num_gpus >= 1 and j.gpcs_per_gpu >= 1:
                n_gpu += j.num_gpus
                n_inst += j.num_gpus * j.gpcs_per_gpu
        out = (N.ParisOut * n)()
        per = np.zeros(max(n_gpu, 1), np.int32)
        flat = np.zeros(max(n_inst, 1), np.int32)
        check(self._lib.msv_paris_batch(self._h, ja, n, out, _ptr(per, C.c_int32), _ptr(flat, C.c_int32)),
              "paris_batch")
        res, go, io = [], 0, 0
        for i, j in enumerate(jobs):
            o = out[i]
            r = ParisOutcome()
            if o.status:
                r.error = _paris_error(o, j)
            else:
                ns = o.n_sizes
                r.knees = {int(o.k[s]): int(o.knee[s]) for s in range(ns)}
                r.segments = [(int(o.k[s]), int(o.seg_first[s]), int(o.seg_last[s])) for s in range(ns)]
                r.ratios = [o.ratio[s] for s in range(ns)]
                r.segment_mass = [o.segment_mass[s] for s in range(ns)]
                r.counts = [o.count[s] for s in range(ns)]
                r.weighted_sum, r.normalizer = o.weighted_sum, o.normalizer
                gpus, off = [], io
                for g in range(j.num_gpus):
                    c = int(per[go + g])
                    gpus.append([int(x) for x in flat[off:off + c]])
                    off += c
                r.plan = PartitionPlan(j.num_gpus, j.gpcs_per_gpu, gpus)
            if j.num_gpus >= 1 and j.gpcs_per_gpu >= 1:
                go += j.num_gpus
                io += j.num_gpus * j.gpcs_per_gpu
            res.append(r)
        return res

    def grid(self, specs: Sequence[GridSpec], tail_p: Sequence[float] = (0.95, 0.99)) -> "DeviceGrid":
        return DeviceGrid(self, specs, tail_p)

    def synchronize(self) -> None:
        check(self._lib.msv_synchronize(self._h))

    def event_record(self, slot: int) -> None:
        check(self._lib.msv_event_record(self._h, slot), "msv_event_record")

    def event_elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_float()
        check(self._lib.msv_event_elapsed(self._h, a, b, C.byref(ms)), "msv_event_elapsed")
        return float(ms.value)

    def transfer_bytes(self) -> tuple[int, int]:
        h, d = C.c_int64(), C.c_int64()
        check(self._lib.msv_transfer_bytes(self._h, C.byref(h), C.byref(d)))
        return int(h.value), int(d.value)


class DeviceGrid:
    """msv_grid: scenarios, traces and outputs resident on the device; launch() runs
    trace generation + simulation + tail selection with no host traffic."""

    def __init__(self, eng: Engine, specs: Sequence[GridSpec], tail_p: Sequence[float]):
        self.eng = eng
        self.specs = list(specs)
        self.tail_p = list(tail_p)
        sc = eng.scenarios(self.specs)
        ps = _arr(self.tail_p or [0.5], np.float64)
        g = C.c_void_p()
        check(eng._lib.msv_grid_create(eng._h, sc, len(self.specs), _ptr(ps, C.c_double), len(self.tail_p),
                                       C.byref(g)), "msv_grid_create")
        self._g = g
        self.n_usage = sum(s.plan.total_instances() for s in self.specs)

    def launch(self) -> None:
        check(self.eng._lib.msv_grid_launch(self._g), "msv_grid_launch")

    def timing(self) -> dict:
        t = [C.c_float() for _ in range(4)]
        check(self.eng._lib.msv_grid_timing(self._g, *[C.byref(x) for x in t]), "msv_grid_timing")
        return dict(zip(("total_ms", "trace_ms", "sim_ms", "tail_ms"), (x.value for x in t)))

    def queries(self) -> int:
        return int(self.eng._lib.msv_grid_queries(self._g))

    def set_overlap(self, on: bool) -> None:
        check(self.eng._lib.msv_grid_set_overlap(self._g, 1 if on else 0), "msv_grid_set_overlap")

    def set_usage(self, on: bool) -> None:
        check(self.eng._lib.msv_grid_set_usage(self._g, 1 if on else 0), "msv_grid_set_usage")

    def results(self, usage: bool = False) -> dict:
        n = len(self.specs)
        res = (N.Result * max(n, 1))()
        use = (N.Usage * max(self.n_usage, 1))() if usage else None
        check(self.eng._lib.msv_grid_results(self._g, res, use), "msv_grid_results")
        return results_to_numpy(res, n, len(self.tail_p), use, self.n_usage)

    def close(self) -> None:
        if self._g:
            self.eng._lib.msv_grid_destroy(self._g)
            self._g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def results_to_numpy(res, n: int, n_tails: int, use=None, n_use: int = 0) -> dict:
    a = np.ctypeslib.as_array(res)[:n] if n else np.zeros(0, np.dtype(N.Result))
    out = {
        "total": np.array(a["total"]), "violations": np.array(a["violations"]), "measured": np.array(a["measured"]),
        "measured_violations": np.array(a["measured_violations"]),
        "tail": np.array(a["tail"])[:, :n_tails] if n else np.zeros((0, n_tails)),
        "horizon_ms": np.array(a["horizon_ms"]), "warmup_ms": np.array(a["warmup_ms"]),
        "max_wait_estimate_diff": np.array(a["max_wait_estimate_diff"]),
        "placement_hash": np.array(a["placement_hash"], dtype=np.uint64), "status": np.array(a["status"]),
    }
    if use is not None:
        u = np.ctypeslib.as_array(use)[:n_use]
        out["usage"] = {"busy_ms": np.array(u["busy_ms"]), "weighted_busy_ms": np.array(u["weighted_busy_ms"]),
                        "queries": np.array(u["queries"])}
    return out
