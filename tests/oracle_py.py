"""TEST INFRASTRUCTURE ONLY: ctypes binding of the CPU checkers (oracle/oracle_abi.h).

    Oracle("reference")  oracle/_ref/libmsv_ref.so — the reference headers compiled
                         unmodified (oracle/build_oracle.py)
    Oracle("port")       oracle/libmsv_oracle.so — plain-C restatement

Used by tests/, __graft_entry__.smoke() and bench.py's CPU baseline only.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
REF_LIB = ROOT / "oracle" / "_ref" / "libmsv_ref.so"
PORT_LIB = ROOT / "oracle" / "libmsv_oracle.so"

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_u8p = C.POINTER(C.c_uint8)


class OraProfile(C.Structure):
    _fields_ = [("n_sizes", C.c_int), ("sizes", _i32p), ("b_max", C.c_int), ("lat", _f64p), ("util", _f64p)]


class OraPlan(C.Structure):
    _fields_ = [("num_gpus", C.c_int), ("gpcs_per_gpu", C.c_int), ("n_per_gpu", _i32p), ("sizes_flat", _i32p)]


class OraDist(C.Structure):
    _fields_ = [("b_max", C.c_int), ("weights", _f64p)]


class OraScenario(C.Structure):
    _fields_ = [("profile", C.c_int32), ("dist", C.c_int32), ("plan", C.c_int32), ("scheduler", C.c_int32),
                ("sla_ms", C.c_double), ("alpha", C.c_double), ("beta", C.c_double), ("rate_qps", C.c_double),
                ("duration_ms", C.c_double), ("warmup_fraction", C.c_double), ("seed", C.c_uint64)]


class OraResult(C.Structure):
    _fields_ = [("total", C.c_int64), ("violations", C.c_int64), ("measured", C.c_int64),
                ("measured_violations", C.c_int64), ("tail", C.c_double * 4), ("horizon_ms", C.c_double),
                ("placement_hash", C.c_uint64), ("status", C.c_int32), ("pad", C.c_int32)]


class OraRecords(C.Structure):
    _fields_ = [("partition", _i32p), ("start_ms", _f64p), ("finish_ms", _f64p), ("kind", _i32p)]


class OraReport(C.Structure):
    _fields_ = [("total", C.c_int64), ("violations", C.c_int64), ("measured", C.c_int64),
                ("measured_violations", C.c_int64), ("horizon_ms", C.c_double), ("warmup_ms", C.c_double),
                ("max_wait_estimate_diff", C.c_double), ("busy_ms", _f64p), ("weighted_busy_ms", _f64p),
                ("queries", _i64p)]


def _a(x, dt):
    return np.ascontiguousarray(np.asarray(x, dtype=dt))


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Oracle:
    def __init__(self, kind: str):
        path = REF_LIB if kind == "reference" else PORT_LIB
        if not path.exists():
            raise FileNotFoundError(path)
        self.L = C.CDLL(str(path))
        self.kind = kind
        L = self.L
        L.ora_last_error.restype = C.c_char_p
        L.ora_kind.restype = C.c_char_p
        L.ora_sample_trace.restype = C.c_int64
        L.ora_sample_trace.argtypes = [C.POINTER(OraDist), C.c_double, C.c_double, C.c_uint64, C.c_int64, _f64p, _i32p]
        L.ora_dist_tables.argtypes = [C.POINTER(OraDist), _f64p, _f64p]
        L.ora_run.argtypes = [C.POINTER(OraPlan), C.c_int, _f64p, _i32p, C.c_int64, C.c_double, C.POINTER(OraProfile),
                              C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, _i32p, _i32p, _i32p,
                              C.POINTER(OraRecords), C.POINTER(OraReport)]
        L.ora_tail_latency.argtypes = [_f64p, C.c_int64, C.c_double, _f64p]
        L.ora_run_grid.argtypes = [C.POINTER(OraProfile), C.POINTER(OraDist), C.POINTER(OraPlan),
                                   C.POINTER(OraScenario), C.c_int64, _f64p, C.c_int, C.c_int, C.POINTER(OraResult)]
        self._keep: list = []

    def err(self, code: int):
        return OracleError(code, (self.L.ora_last_error() or b"").decode())

    # -- struct builders --
    def profile(self, t) -> OraProfile:
        s, lat, util = _a(t.sizes, np.int32), _a(t.latency, np.float64), _a(t.utilization, np.float64)
        self._keep += [s, lat, util]
        return OraProfile(len(s), _p(s, C.c_int32), t.b_max, _p(lat, C.c_double), _p(util, C.c_double))

    def plan(self, p) -> OraPlan:
        n = _a([len(g) for g in p.gpus] or [0], np.int32)
        f = _a(p.flatten() or [0], np.int32)
        self._keep += [n, f]
        return OraPlan(p.num_gpus, p.gpcs_per_gpu, _p(n, C.c_int32), _p(f, C.c_int32))

    def dist(self, d) -> OraDist:
        w = _a(d.weights, np.float64)
        self._keep.append(w)
        return OraDist(len(w), _p(w, C.c_double))

    # -- checker entry points --
    def dist_tables(self, d):
        pmf, cdf = np.zeros(d.b_max), np.zeros(d.b_max)
        rc = self.L.ora_dist_tables(C.byref(self.dist(d)), _p(pmf, C.c_double), _p(cdf, C.c_double))
        if rc:
            raise self.err(rc)
        return pmf, cdf

    def sample_trace(self, d, rate, duration, seed):
        mean = rate * duration / 1000.0
        cap = int(mean + 12 * np.sqrt(max(mean, 0)) + 256)
        while True:
            arr, bat = np.zeros(cap), np.zeros(cap, np.int32)
            n = self.L.ora_sample_trace(C.byref(self.dist(d)), rate, duration, seed, cap, _p(arr, C.c_double),
                                        _p(bat, C.c_int32))
            if n < 0:
                raise self.err(-n)
            if n <= cap:
                return arr[:n].copy(), bat[:n].copy()
            cap = n

    def run(self, plan, scheduler, arrival, batch, duration, table, sla, warmup=0.1, routing=None, check_wait=False):
        arrival, batch = _a(arrival, np.float64), _a(batch, np.int32)
        n = len(arrival)
        P = plan.total_instances()
        m = max(n, 1)
        part, start, fin, kind = np.zeros(m, np.int32), np.zeros(m), np.zeros(m), np.zeros(m, np.int32)
        busy, wbusy, nq = np.zeros(max(P, 1)), np.zeros(max(P, 1)), np.zeros(max(P, 1), np.int64)
        rec = OraRecords(_p(part, C.c_int32), _p(start, C.c_double), _p(fin, C.c_double), _p(kind, C.c_int32))
        rep = OraReport(0, 0, 0, 0, 0.0, 0.0, 0.0, _p(busy, C.c_double), _p(wbusy, C.c_double), _p(nq, C.c_int64))
        if routing is None:
            nr, rk, rf, rl = -1, None, None, None
        else:
            rk = _a([s[0] for s in routing] or [0], np.int32)
            rf = _a([s[1] for s in routing] or [0], np.int32)
            rl = _a([s[2] for s in routing] or [0], np.int32)
            nr = len(routing)
            rk, rf, rl = _p(rk, C.c_int32), _p(rf, C.c_int32), _p(rl, C.c_int32)
        rc = self.L.ora_run(C.byref(self.plan(plan)), 1 if scheduler == "elsa" else 0,
                            _p(arrival if n else np.zeros(1), C.c_double), _p(batch if n else np.zeros(1, np.int32),
                                                                            C.c_int32),
                            n, duration, C.byref(self.profile(table)), sla.sla_target_ms, sla.alpha, sla.beta, warmup,
                            1 if check_wait else 0, nr, rk, rf, rl, C.byref(rec), C.byref(rep))
        if rc:
            raise self.err(rc)
        return {"partition": part[:n], "start_ms": start[:n], "finish_ms": fin[:n], "kind": kind[:n],
                "total": rep.total, "violations": rep.violations, "measured": rep.measured,
                "measured_violations": rep.measured_violations, "horizon_ms": rep.horizon_ms,
                "warmup_ms": rep.warmup_ms, "max_wait_estimate_diff": rep.max_wait_estimate_diff,
                "busy_ms": busy[:P], "weighted_busy_ms": wbusy[:P], "queries": nq[:P]}

    def run_noise(self, plan, scheduler, arrival, batch, duration, table, sla, warmup, routing, sigma, seed):
        """The reference's run() with execution noise (oracle/_ref only: oraref_run_noise)."""
        arrival, batch = _a(arrival, np.float64), _a(batch, np.int32)
        n, P = len(arrival), plan.total_instances()
        m = max(n, 1)
        part, start, fin, kind = np.zeros(m, np.int32), np.zeros(m), np.zeros(m), np.zeros(m, np.int32)
        busy, wbusy, nq = np.zeros(max(P, 1)), np.zeros(max(P, 1)), np.zeros(max(P, 1), np.int64)
        rec = OraRecords(_p(part, C.c_int32), _p(start, C.c_double), _p(fin, C.c_double), _p(kind, C.c_int32))
        rep = OraReport(0, 0, 0, 0, 0.0, 0.0, 0.0, _p(busy, C.c_double), _p(wbusy, C.c_double), _p(nq, C.c_int64))
        if routing is None:
            nr, rk, rf, rl = -1, None, None, None
        else:
            nr = len(routing)
            rk, rf, rl = (_a([s[i] for s in routing], np.int32) for i in range(3))
            self._keep += [rk, rf, rl]
            rk, rf, rl = _p(rk, C.c_int32), _p(rf, C.c_int32), _p(rl, C.c_int32)
        fn = self.L.oraref_run_noise
        fn.argtypes = None
        rc = fn(C.byref(self.plan(plan)), C.c_int(1 if scheduler == "elsa" else 0),
                _p(arrival if n else np.zeros(1), C.c_double), _p(batch if n else np.zeros(1, np.int32), C.c_int32),
                C.c_int64(n), C.c_double(duration), C.byref(self.profile(table)), C.c_double(sla.sla_target_ms),
                C.c_double(sla.alpha), C.c_double(sla.beta), C.c_double(warmup), C.c_int(nr), rk, rf, rl,
                C.c_double(sigma), C.c_uint64(seed), C.byref(rec), C.byref(rep))
        if rc:
            raise self.err(rc)
        return {"partition": part[:n], "start_ms": start[:n], "finish_ms": fin[:n], "kind": kind[:n],
                "total": rep.total, "violations": rep.violations, "measured": rep.measured,
                "measured_violations": rep.measured_violations, "horizon_ms": rep.horizon_ms,
                "warmup_ms": rep.warmup_ms, "busy_ms": busy[:P], "weighted_busy_ms": wbusy[:P], "queries": nq[:P]}

    def tail_latency(self, samples, p):
        s = _a(samples, np.float64)
        out = C.c_double()
        rc = self.L.ora_tail_latency(_p(s if len(s) else np.zeros(1), C.c_double), len(s), p, C.byref(out))
        if rc:
            raise self.err(rc)
        return out.value

    def run_grid(self, specs, tail_p=(0.95, 0.99), threads: int | None = None):
        profs, dists, plans = {}, {}, {}
        P, D, L = [], [], []
        sc = (OraScenario * max(len(specs), 1))()
        for i, s in enumerate(specs):
            if id(s.table) not in profs:
                profs[id(s.table)] = len(P)
                P.append(self.profile(s.table))
            if id(s.dist) not in dists:
                dists[id(s.dist)] = len(D)
                D.append(self.dist(s.dist))
            k = s.plan.key()
            if k not in plans:
                plans[k] = len(L)
                L.append(self.plan(s.plan))
            sc[i] = OraScenario(profs[id(s.table)], dists[id(s.dist)], plans[k], 1 if s.scheduler == "elsa" else 0,
                                s.sla.sla_target_ms, s.sla.alpha, s.sla.beta, s.rate_qps, s.duration_ms,
                                s.warmup_fraction, s.seed)
        Pa = (OraProfile * max(len(P), 1))(*P)
        Da = (OraDist * max(len(D), 1))(*D)
        La = (OraPlan * max(len(L), 1))(*L)
        ps = _a(list(tail_p) or [0.5], np.float64)
        out = (OraResult * max(len(specs), 1))()
        threads = threads or int(os.environ.get("MSV_ORACLE_THREADS", os.cpu_count() or 1))
        rc = self.L.ora_run_grid(Pa, Da, La, sc, len(specs), _p(ps, C.c_double), len(tail_p), threads, out)
        if rc:
            raise self.err(rc)
        a = np.ctypeslib.as_array(out)[: len(specs)]
        return {"total": np.array(a["total"]), "violations": np.array(a["violations"]),
                "measured": np.array(a["measured"]), "measured_violations": np.array(a["measured_violations"]),
                "tail": np.array(a["tail"])[:, : len(tail_p)], "horizon_ms": np.array(a["horizon_ms"]),
                "placement_hash": np.array(a["placement_hash"], dtype=np.uint64), "status": np.array(a["status"])}

    # -- reference-only extras (oracle/_ref) --
    def paris_plan(self, table, dist, total, num_gpus, gpcs, thr=0.8):
        L = self.L
        n_sizes = len(table.sizes)
        knees, ratios, counts = np.zeros(n_sizes, np.int32), np.zeros(n_sizes), np.zeros(n_sizes)
        n_per, flat = np.zeros(num_gpus, np.int32), np.zeros(num_gpus * gpcs, np.int32)
        rc = L.oraref_paris_plan(C.byref(self.profile(table)), C.byref(self.dist(dist)), total, num_gpus, gpcs,
                                 C.c_double(thr), _p(knees, C.c_int32), _p(ratios, C.c_double), _p(counts, C.c_double),
                                 _p(n_per, C.c_int32), _p(flat, C.c_int32))
        if rc:
            raise self.err(rc)
        gpus, off = [], 0
        for g in range(num_gpus):
            gpus.append([int(x) for x in flat[off:off + n_per[g]]])
            off += int(n_per[g])
        return {"knees": knees, "ratios": ratios, "counts": counts, "gpus": gpus}


    def lbt(self, plan, scheduler, table, sla, dist, opt):
        """latency_bounded_throughput (metrics.hpp:81-120) of the compiled reference."""
        seeds = _a(list(opt.seeds), np.uint64)
        qps, inf, sims = C.c_double(), C.c_int(), C.c_int()
        rc = self.L.oraref_lbt(C.byref(self.plan(plan)), 1 if scheduler == "elsa" else 0, C.byref(self.profile(table)),
                               C.c_double(sla.sla_target_ms), C.c_double(sla.alpha), C.c_double(sla.beta),
                               C.byref(self.dist(dist)), C.c_double(opt.duration_ms), _p(seeds, C.c_uint64),
                               len(seeds), C.c_double(opt.rel_tol), C.c_double(opt.tail_p),
                               C.c_double(opt.lambda_min), C.c_double(opt.warmup_fraction), opt.max_doublings,
                               C.byref(qps), C.byref(inf), C.byref(sims))
        if rc:
            raise self.err(rc)
        return qps.value, bool(inf.value), sims.value

    def best_homogeneous(self, table, dist, sla, total_gpcs, num_gpus, gpcs_per_gpu, duration_ms, seeds):
        s = _a(list(seeds), np.uint64)
        k, qps = C.c_int(), C.c_double()
        rc = self.L.oraref_best_homogeneous(C.byref(self.profile(table)), C.byref(self.dist(dist)),
                                            C.c_double(sla.sla_target_ms), C.c_double(sla.alpha),
                                            C.c_double(sla.beta), total_gpcs, num_gpus, gpcs_per_gpu,
                                            C.c_double(duration_ms), _p(s, C.c_uint64), len(s), C.byref(k),
                                            C.byref(qps))
        if rc:
            raise self.err(rc)
        return k.value, qps.value


_BEST = None


def best_oracle() -> Oracle:
    """The compiled reference when present, else the C port."""
    global _BEST
    if _BEST is None:
        _BEST = Oracle("reference") if REF_LIB.exists() else Oracle("port")
    return _BEST
