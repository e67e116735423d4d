"""TEST INFRASTRUCTURE ONLY. Generates and checks tests/golden/*.npz.

The fixtures are produced by the reference itself — /root/reference/proj/include
compiled unmodified into oracle/_ref/libmsv_ref.so (oracle/build_oracle.py) — on the
build container (glibc 2.39, whichever log1p build its CPU selects; the variant is
recorded). They pin every hot-path output: traces (sample_trace), per-query
placements and timings (run), per-scenario aggregates and tails (the grid), tail
selection, and the host planning helpers (synth_profile, lognormal_batch_pdf,
paris_plan). Regenerate with:

    python -m tests.golden.gen_golden            # needs oracle/_ref built
"""
from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

PROFILE_CASES = [("mobilenet", (0.4, 0.5, 0.15, 0.95)), ("resnet50", (0.8, 0.8, 0.25, 0.95)),
                 ("bert_base", (4.0, 2.0, 0.40, 0.95)), ("ref_default", (10.0, 5.0, 0.15, 0.95)),
                 ("ref_light", (10.0, 5.0, 0.4, 0.95))]
LOGNORMAL_CASES = [(1.0, 1.0, 32), (1.0, 1.0, 8), (0.5, 0.8, 4), (2.5, 1.7, 32), (1.0, 0.7, 16), (0.0, 0.3, 1)]
PARIS_CASES = [("resnet50", 1), ("bert_base", 8), ("mobilenet", 8), ("resnet50", 8), ("bert_base", 2)]
TRACE_CASES = [(1000.0, 2000.0, 1), (150.0, 20000.0, 17), (250.0, 10000.0, 11), (50.0, 10000.0, 99),
               (100.0, 0.0, 7), (1e5, 200.0, 12345), (1000.0, 100000.0, 1)]  # last: digest only


def _digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _tables():
    from paper_2202_13481_b200 import BatchDistribution, ProfileTable
    sl = ProfileTable(np.array([1, 7], np.int32), 4, np.array([[40.0, 80.0, 110.0, 150.0], [20.0, 25.0, 32.0, 40.0]]),
                      np.array([[0.6, 0.8, 0.9, 0.95], [0.1, 0.2, 0.3, 0.4]]), "scenario")
    return sl, BatchDistribution(np.array([0.3, 0.3, 0.2, 0.2]))


def run_cases():
    """(name, table, dist, plan, sched, rate, duration, seed, sla, routing, check_wait)"""
    from paper_2202_13481_b200 import (PartitionPlan, SlaConfig, SyntheticProfileParams, lognormal_batch_pdf,
                                       synth_profile)
    toy = synth_profile(SyntheticProfileParams(10.0, 5.0, 0.4, 0.95), [1, 2, 3, 7], 8)
    d8 = lognormal_batch_pdf(1.0, 1.0, 8)
    plan3 = PartitionPlan(3, 7, [[3, 2, 1, 1], [7], [2, 1, 1]])
    sl, d4 = _tables()
    cases = []
    for sched in ("fifs", "elsa"):
        cases.append(("toy", toy, d8, plan3, sched, 250.0, 10000.0, 11, SlaConfig(100.0), None, True))
        cases.append(("overload", toy, d8, plan3, sched, 900.0, 3000.0, 5, SlaConfig(60.0, 1.3, 0.7), None, False))
        cases.append(("routing", toy, d8, plan3, sched, 200.0, 5000.0, 3, SlaConfig(100.0),
                      [(1, 1, 2), (2, 3, 4), (3, 5, 6), (7, 7, 8)], False))
        cases.append(("small_large", sl, d4, PartitionPlan(2, 7, [[7], [1, 1, 1, 1, 1, 1, 1]]), sched, 60.0, 5000.0,
                      9, SlaConfig(100.0), None, False))
    return cases


def grid_specs():
    from paper_2202_13481_b200 import workloads as W
    specs = W.c1(queries=2e4) + W.c2(seeds=2, queries=4e3) + W.c3(seeds=1, queries=4e3)
    m = W.model("bert_base")
    p = W.paris(m, 8)
    specs += [W._spec(m, p, 1.5 * W.capacity_qps(m, p), 2000, 3)]
    return specs


TAIL_CASES = [(n, p) for n in (1, 10, 97, 5000) for p in (0.05, 0.5, 0.95, 0.99)]


def tail_samples(n):
    rng = np.random.default_rng(n)
    x = rng.lognormal(3.0, 1.0, n)
    if n > 10:
        x[: n // 4] = x[0]
    return x


def compute(O) -> dict[str, dict]:
    """Every fixture, computed by oracle O (reference or port)."""
    from paper_2202_13481_b200 import lognormal_batch_pdf
    out: dict[str, dict] = {}
    d32 = lognormal_batch_pdf(1.0, 1.0, 32)
    tr = {}
    for i, (rate, dur, seed) in enumerate(TRACE_CASES):
        a, b = O.sample_trace(d32, rate, dur, seed)
        tr[f"n_{i}"] = np.array(len(a))
        tr[f"digest_{i}"] = np.array(_digest(a, b))
        if len(a) <= 40000:
            tr[f"arrival_{i}"], tr[f"batch_{i}"] = a, b
    out["traces"] = tr
    runs = {}
    for i, (name, t, d, plan, sched, rate, dur, seed, sla, routing, cw) in enumerate(run_cases()):
        a, b = O.sample_trace(d, rate, dur, seed)
        r = O.run(plan, sched, a, b, dur, t, sla, 0.1, routing, cw)
        for k in ("partition", "kind", "start_ms", "finish_ms", "busy_ms", "weighted_busy_ms", "queries"):
            runs[f"{k}_{i}"] = np.asarray(r[k])
        for k in ("total", "violations", "measured", "measured_violations", "horizon_ms", "warmup_ms",
                  "max_wait_estimate_diff"):
            runs[f"{k}_{i}"] = np.array(r[k])
    out["runs"] = runs
    g = O.run_grid(grid_specs(), (0.95, 0.99), threads=4)
    out["grid"] = {k: np.asarray(v) for k, v in g.items()}
    out["tails"] = {f"tail_{i}": np.array(O.tail_latency(tail_samples(n), p)) for i, (n, p) in enumerate(TAIL_CASES)}
    return out


def compute_planning(O) -> dict:
    """Planning fixtures (reference oracle only: the port restates the hot path)."""
    import ctypes as C
    from paper_2202_13481_b200 import workloads as W
    L = O.L
    fx = {}
    sizes = np.array([1, 2, 3, 4, 7], np.int32)
    for i, (name, prm) in enumerate(PROFILE_CASES):
        so, n = np.zeros(5, np.int32), C.c_int()
        lat, util = np.zeros(5 * 32), np.zeros(5 * 32)
        rc = L.oraref_synth_profile(*[C.c_double(x) for x in prm], sizes.ctypes.data_as(C.POINTER(C.c_int32)), 5, 32,
                                    so.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(n),
                                    lat.ctypes.data_as(C.POINTER(C.c_double)),
                                    util.ctypes.data_as(C.POINTER(C.c_double)))
        assert rc == 0
        fx[f"lat_{i}"], fx[f"util_{i}"] = lat.reshape(5, 32), util.reshape(5, 32)
    for i, (mu, sigma, b) in enumerate(LOGNORMAL_CASES):
        pmf, cdf = np.zeros(b), np.zeros(b)
        rc = L.oraref_lognormal_pdf(C.c_double(mu), C.c_double(sigma), b, pmf.ctypes.data_as(C.POINTER(C.c_double)),
                                    cdf.ctypes.data_as(C.POINTER(C.c_double)))
        assert rc == 0
        fx[f"pmf_{i}"], fx[f"cdf_{i}"] = pmf, cdf
    for i, (name, gpus) in enumerate(PARIS_CASES):
        m = W.model(name)
        r = O.paris_plan(m.table, m.dist, 7 * gpus, gpus, 7)
        fx[f"paris_flat_{i}"] = np.array([k for g in r["gpus"] for k in g], np.int32)
        fx[f"paris_nper_{i}"] = np.array([len(g) for g in r["gpus"]], np.int32)
        fx[f"paris_counts_{i}"] = r["counts"]
        fx[f"paris_ratios_{i}"] = r["ratios"]
        fx[f"paris_knees_{i}"] = r["knees"]
    return fx


def load(name: str) -> dict:
    with np.load(HERE / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def _eq(a, b) -> bool:
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype.kind == "f" or b.dtype.kind == "f":
        return a.shape == b.shape and np.array_equal(a, b, equal_nan=True)
    return a.shape == b.shape and bool(np.all(a == b))


def check_all(O) -> None:
    got = compute(O)
    for name, fx in got.items():
        want = load(name)
        assert set(want) == set(fx), (name, set(want) ^ set(fx))
        for k in want:
            assert _eq(fx[k], want[k]), f"{name}/{k}: {O.kind} oracle differs from the committed fixture"


def main() -> None:
    from tests import oracle_py as OP
    O = OP.Oracle("reference")
    for name, fx in compute(O).items():
        np.savez_compressed(HERE / f"{name}.npz", **fx)
    np.savez_compressed(HERE / "planning.npz", **compute_planning(O))
    sys.path.insert(0, str(ROOT / "tests"))
    from test_cpu import _log1p_lib
    (HERE / "PROVENANCE.txt").write_text(
        "Generated by tests/golden/gen_golden.py from oracle/_ref/libmsv_ref.so (the reference headers,\n"
        "unmodified, g++ 13.3 -O3 -DNDEBUG), glibc 2.39 libm; host log1p build selected by ifunc: "
        f"{'FMA/AVX2' if _log1p_lib().host_variant() == 1 else 'generic SSE2'}.\n")
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
