"""CPU-only tests: the oracles against each other and the reference's own suite,
the glibc-log1p transcription the device uses, the C-ABI library surface (no
compute without a GPU), and the host-side planning helpers."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
from tests import oracle_py as O  # noqa: E402


def have_ref():
    return O.REF_LIB.exists()


# ---------------------------------------------------------------- the reference's own tests
def test_reference_suite_passes_on_shim():
    exe = ROOT / "oracle" / "_ref" / "ref_unit_tests"
    if not exe.exists():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:]
    assert "42 test cases, 0 failed, 167386 assertions" in r.stdout


# ---------------------------------------------------------------- port vs reference
@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
def test_port_matches_reference_grid():
    from paper_2202_13481_b200 import workloads as W
    specs = W.c1(queries=1e4) + W.c2(seeds=2, queries=4e3) + W.c3(seeds=1, queries=4e3)
    m = W.model("bert_base")
    p = W.paris(m, 8)
    specs += [W._spec(m, p, 1.4 * W.capacity_qps(m, p), 2000, 3)]  # overloaded
    a = O.Oracle("reference").run_grid(specs)
    b = O.Oracle("port").run_grid(specs)
    for k in a:
        assert np.array_equal(a[k], b[k], equal_nan=(a[k].dtype.kind == "f")), k


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
def test_port_matches_reference_records():
    from paper_2202_13481_b200 import PartitionPlan, SlaConfig, lognormal_batch_pdf, synth_profile
    from paper_2202_13481_b200 import SyntheticProfileParams
    ref, port = O.Oracle("reference"), O.Oracle("port")
    t = synth_profile(SyntheticProfileParams(10.0, 5.0, 0.4, 0.95), [1, 2, 3, 7], 8)
    d = lognormal_batch_pdf(1.0, 1.0, 8)
    plan = PartitionPlan(3, 7, [[3, 2, 1, 1], [7], [2, 1, 1]])
    for sched in ("fifs", "elsa"):
        for routing in (None, [(1, 1, 2), (2, 3, 4), (3, 5, 6), (7, 7, 8)]):
            arr, bat = ref.sample_trace(d, 300.0, 8000.0, 4)
            assert np.array_equal(arr, port.sample_trace(d, 300.0, 8000.0, 4)[0])
            a = ref.run(plan, sched, arr, bat, 8000.0, t, SlaConfig(90.0, 1.1, 0.9), 0.1, routing, True)
            b = port.run(plan, sched, arr, bat, 8000.0, t, SlaConfig(90.0, 1.1, 0.9), 0.1, routing, True)
            for k in a:
                assert np.array_equal(np.asarray(a[k]), np.asarray(b[k])), (sched, routing, k)


def test_port_tail_latency_cases():
    port = O.Oracle("port")
    ten = [10, 20, 30, 40, 50, 60, 70, 80, 90, 100]
    assert port.tail_latency(ten, 0.95) == 100.0
    assert port.tail_latency(ten, 0.90) == 90.0
    assert port.tail_latency(ten, 0.05) == 10.0
    assert port.tail_latency([42.0], 0.95) == 42.0
    with pytest.raises(O.OracleError):
        port.tail_latency([], 0.95)


# ---------------------------------------------------------------- golden fixtures
def test_golden_fixtures_against_port():
    """tests/golden/*.npz were produced by the compiled reference (gen_golden.py); the
    C port must reproduce every one bit for bit on this host."""
    from tests.golden import gen_golden as G
    G.check_all(O.Oracle("port"))


@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
def test_golden_fixtures_against_reference():
    from tests.golden import gen_golden as G
    G.check_all(O.Oracle("reference"))


# ---------------------------------------------------------------- device log1p transcription (host side)
def _log1p_lib():
    src = ROOT / "tests" / "log1p_check.c"
    out = ROOT / "tests" / "_log1p_check.so"
    hdr = ROOT / "paper_2202_13481_b200" / "csrc" / "msv_math.h"
    if not out.exists() or out.stat().st_mtime < max(src.stat().st_mtime, hdr.stat().st_mtime):
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", str(out), str(src), "-lm",
                        "-lpthread"], check=True)
    L = C.CDLL(str(out))
    L.check_log1p.restype = C.c_long
    L.check_log1p.argtypes = [C.c_int, C.c_long, C.c_uint64]
    L.variants_differ.restype = C.c_long
    L.variants_differ.argtypes = [C.c_long, C.c_uint64]
    L.host_variant.restype = C.c_int
    L.host_log1p_digest.restype = C.c_int
    L.host_log1p_digest.argtypes = [C.c_uint64, C.c_long, C.c_long, C.POINTER(C.c_uint64), C.c_int]
    L.host_log1p_value.restype = C.c_double
    L.host_log1p_value.argtypes = [C.c_uint64, C.c_long]
    return L


def test_log1p_transcription_matches_host_libm():
    """msv_log1p_neg(variant = the build this host's ifunc picked) == glibc log1p on
    2e6 inputs of the generator's domain (x = -k*2^-53)."""
    L = _log1p_lib()
    v = L.host_variant()
    assert v in (0, 1)
    assert L.check_log1p(v, 2_000_000, 12345) == 0
    assert L.variants_differ(2_000_000, 12345) > 0  # the probe can tell the builds apart


def test_log1p_generic_build_under_tunables():
    """Force glibc's generic (SSE2) build and check the other transcription too."""
    code = ("import sys; sys.path.insert(0, %r); from tests.test_cpu import _log1p_lib; L=_log1p_lib(); "
            "assert L.host_variant()==0, L.host_variant(); assert L.check_log1p(0, 1000000, 7)==0; print('ok')"
            % str(ROOT))
    env = dict(os.environ, GLIBC_TUNABLES="glibc.cpu.hwcaps=-AVX2,-FMA")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    if "assert L.host_variant()==0" in r.stderr:
        pytest.skip("this CPU has no FMA build to switch away from")
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


# ---------------------------------------------------------------- C ABI surface
def test_libmsv_exports_every_declared_symbol():
    from paper_2202_13481_b200 import _native as N
    L = N.lib()
    declared = N.header_symbols()
    assert len(declared) >= 25
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert L.msv_abi_version() == 1


def test_no_silent_cpu_path_without_gpu():
    """On a host without a usable B200 the engine refuses instead of computing on the CPU."""
    import torch
    from paper_2202_13481_b200 import DeviceError, Engine
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(DeviceError):
        Engine(0)


def test_planning_exports_match_reference():
    from paper_2202_13481_b200 import paris_plan, synth_profile, lognormal_batch_pdf, SyntheticProfileParams
    from paper_2202_13481_b200 import workloads as W
    from tests.golden import gen_golden as G
    fx = G.load("planning")
    for i, (name, prm) in enumerate(G.PROFILE_CASES):
        t = synth_profile(SyntheticProfileParams(*prm), [1, 2, 3, 4, 7], 32)
        assert np.array_equal(t.latency, fx[f"lat_{i}"]) and np.array_equal(t.utilization, fx[f"util_{i}"])
    for i, (mu, sigma, b) in enumerate(G.LOGNORMAL_CASES):
        d = lognormal_batch_pdf(mu, sigma, b)
        assert np.array_equal(d.weights, fx[f"pmf_{i}"])
    for i, case in enumerate(G.PARIS_CASES):
        name, gpus = case
        m = W.model(name)
        p = paris_plan(m.table, m.dist, 7 * gpus, gpus, 7)
        assert p.flatten() == list(fx[f"paris_flat_{i}"]), (name, gpus)
        assert [len(g) for g in p.gpus] == list(fx[f"paris_nper_{i}"])


def test_fleet_enumeration_counts():
    from paper_2202_13481_b200 import workloads as W
    assert len(W.gpu_configs()) == 12
    assert [len(W.fleet_candidates(g)) for g in (1, 2, 4)] == [12, 53, 360]


def test_shard_partitions_whole_scenarios():
    from paper_2202_13481_b200 import workloads as W
    specs = W.c2(seeds=7, queries=1e4)
    for world in (1, 2, 4, 8):
        parts = [W.shard(specs, r, world) for r in range(world)]
        flat = [s for p in parts for s in p]
        assert len(flat) == len(specs) and all(a is b for a, b in zip(flat, specs))


# ---------------------------------------------------------------- reference-arm inputs
@pytest.mark.skipif(not have_ref(), reason="oracle/_ref not built")
def test_ref_workloads_match_product_workloads():
    """bench.py's reference arm builds C5 / C2 from oracle/_ref alone (tests/ref_workloads.py);
    the grids must equal the product's (paper_2202_13481_b200/workloads.py) bit for bit."""
    from paper_2202_13481_b200 import workloads as W
    from tests import ref_workloads as R

    for mine, ref in ((W.c5(n_scenarios=300, queries=1e6), R.c5(n_scenarios=300, queries=1e6)),
                      (W.c2(seeds=3, queries=1e5), R.c2(seeds=3, queries=1e5))):
        assert len(mine) == len(ref)
        for a, b in zip(mine, ref):
            assert a.plan.key() == b.plan.key()
            assert np.array_equal(a.table.sizes, b.table.sizes) and a.table.b_max == b.table.b_max
            assert a.table.latency.tobytes() == b.table.latency.tobytes()
            assert a.table.utilization.tobytes() == b.table.utilization.tobytes()
            assert np.asarray(a.dist.weights, float).tobytes() == np.asarray(b.dist.weights, float).tobytes()
            assert (a.sla.sla_target_ms, a.sla.alpha, a.sla.beta) == (b.sla.sla_target_ms, b.sla.alpha, b.sla.beta)
            assert (a.rate_qps, a.duration_ms, a.seed, a.scheduler, a.warmup_fraction) == \
                   (b.rate_qps, b.duration_ms, b.seed, b.scheduler, b.warmup_fraction)


def test_engine_plan_handle_cache_sees_edits():
    """Engine.plan reuses the handle of the same, unchanged plan object without rebuilding its
    by-value key, and re-keys a plan object whose contents were edited after upload (no GPU:
    the upload call is stubbed)."""
    import copy
    from paper_2202_13481_b200 import engine as E
    from paper_2202_13481_b200 import workloads as W

    class Lib:
        def __init__(self):
            self.uploads = 0

        def msv_upload_plan(self, h, num_gpus, gpcs, n_per, flat, out):
            self.uploads += 1
            out._obj.value = self.uploads
            return 0

    eng = E.Engine.__new__(E.Engine)  # no device context
    eng._lib, eng._h = Lib(), None
    eng._plans, eng._plan_objs = {}, {}
    m = W.model("resnet50")
    p = copy.deepcopy(W.paris(m, 8))
    h1 = eng.plan(p)
    assert eng.plan(p) == h1 and eng._lib.uploads == 1  # same object: cached
    q = copy.deepcopy(p)
    assert eng.plan(q) == h1 and eng._lib.uploads == 1  # equal contents: same handle, no upload
    p.gpus[0] = list(reversed(p.gpus[0])) + [1] if p.gpus[0] else [1]  # edited after upload
    h2 = eng.plan(p)
    assert h2 != h1 and eng._lib.uploads == 2
    assert eng.plan(p) == h2 and eng._lib.uploads == 2
