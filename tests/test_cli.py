"""The SPEC's experiment runner: `msv run|plan|sweep`.

One source, paper_2202_13481_b200/cli/msv_cli.cpp, is built twice: against this repo's
drop-in headers + libmsv.so (paper_2202_13481_b200/msv, the product: simulations on the
B200) and against the reference headers (oracle/_ref/msv_cli_ref, the checker: the
reference's CPU engine). CPU tests cover the runner's host logic (config validation, file
layout, determinism, the resolved-config round trip, the host-only `plan` verb on the
product binary); the GPU tests require byte-identical output trees from both builds.
"""
from __future__ import annotations

import json
import os
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
DEV = ROOT / "paper_2202_13481_b200" / "msv"
REF = ROOT / "oracle" / "_ref" / "msv_cli_ref"
EX = ROOT / "examples"

need_ref = pytest.mark.skipif(not REF.exists(), reason="oracle/_ref/msv_cli_ref not built")
need_dev = pytest.mark.skipif(not DEV.exists(), reason="paper_2202_13481_b200/msv not built")


def msv(exe: Path, *args, cwd=None, timeout=900) -> subprocess.CompletedProcess:
    env = dict(os.environ)
    env.pop("MSV_OUTPUT_ROOT", None)
    return subprocess.run([str(exe), *map(str, args)], capture_output=True, text=True, timeout=timeout, cwd=cwd,
                          env=env)


def tree(d: Path) -> dict[str, bytes]:
    return {str(p.relative_to(d)): p.read_bytes() for p in sorted(d.rglob("*")) if p.is_file()}


def write_cfg(tmp: Path, cfg: dict, name="cfg.json") -> Path:
    p = tmp / name
    p.write_text(json.dumps(cfg))
    return p


SMALL = {
    "profile": {"preset": "medium"},
    "workload": {"rate_qps": 600, "duration_ms": 1500, "seeds": [1, 2, 3]},
    "designs": [{"plan": "gpu(7)", "scheduler": "fifs"}, {"plan": "paris", "scheduler": "elsa"}],
}


# ------------------------------------------------------------------ CPU: host logic
@need_ref
def test_run_layout_and_determinism(tmp_path):
    """2 designs x 3 seeds -> 6 reports (+ per-query CSVs) and one summary;
    a re-run is byte-identical (acceptance #7)."""
    cfg = write_cfg(tmp_path, SMALL)
    a, b = tmp_path / "a" / "o", tmp_path / "b" / "o"
    for d in (a, b):
        d.parent.mkdir()
        r = msv(REF, "run", cfg, "--out", "o", cwd=d.parent)
        assert r.returncode == 0, r.stderr
    ta = tree(a)
    assert sorted(k for k in ta if k.endswith(".json") and k.startswith("reports")) == sorted(
        f"reports/{lab}__seed{s}.json" for lab in ("gpu_7__fifs", "paris_elsa") for s in (1, 2, 3))
    assert sum(k.endswith(".csv") and k.startswith("reports") for k in ta) == 6
    assert "summary.csv" in ta and "resolved_config.json" in ta
    rows = ta["summary.csv"].decode().splitlines()
    assert rows[0].startswith("label,scheduler,") and len(rows) == 3
    assert ta == tree(b)
    res = json.loads(ta["resolved_config.json"])
    assert res["sla"]["multiplier"] == 1.5 and res["derived"]["sla_target_ms"] > 0
    assert res["derived"]["designs"][1]["plan"]["gpus"]  # the PARIS plan is echoed for provenance


@need_ref
def test_resolved_config_round_trip(tmp_path):
    """the echoed resolved config re-runs to the same results."""
    cfg = write_cfg(tmp_path, SMALL)
    (tmp_path / "a").mkdir(), (tmp_path / "b").mkdir()
    assert msv(REF, "run", cfg, "--out", "o", cwd=tmp_path / "a").returncode == 0
    r = msv(REF, "run", tmp_path / "a" / "o" / "resolved_config.json", cwd=tmp_path / "b")
    assert r.returncode == 0, r.stderr
    assert tree(tmp_path / "a" / "o") == tree(tmp_path / "b" / "o")


@need_ref
def test_output_root_env_and_set_override(tmp_path):
    cfg = write_cfg(tmp_path, {**SMALL, "output": {"dir": "rel"}})
    env = dict(os.environ, MSV_OUTPUT_ROOT=str(tmp_path / "root"))
    r = subprocess.run([str(REF), "run", str(cfg), "--set", "workload.seeds=[5]", "--set", "output.per_query_csv=false"],
                       capture_output=True, text=True, env=env, cwd=tmp_path, timeout=300)
    assert r.returncode == 0, r.stderr
    t = tree(tmp_path / "root" / "rel")
    assert sorted(k for k in t if k.startswith("reports")) == ["reports/gpu_7__fifs__seed5.json",
                                                               "reports/paris_elsa__seed5.json"]


@need_ref
@pytest.mark.parametrize("patch,field", [
    ({"designs": [{"plan": "paris", "scheduler": "edf"}]}, "designs[0].scheduler"),
    ({"designs": [{"plan": "gpu(x)"}]}, "designs[0].plan"),
    ({"designs": []}, "designs"),
    ({"workload": {"rate_qps": -1}}, "workload.rate_qps"),
    ({"workload": {"rate_qps": 10, "seedz": [1]}}, "workload.seedz"),
    ({"sla": {"tail_p": 1.0}}, "sla.tail_p"),
    ({"profile": {"preset": "huge"}}, "profile.preset"),
    ({"designs": [{"plan": "paris"}, {"plan": "paris", "scheduler": "elsa"}]}, "designs[1].label"),
])
def test_validation_errors_name_the_field(tmp_path, patch, field):
    """validation failures name the offending field; exit code 1."""
    cfg = write_cfg(tmp_path, {**SMALL, **patch})
    r = msv(REF, "run", cfg, "--out", tmp_path / "o")
    assert r.returncode == 1 and f"config: {field}:" in r.stderr, (r.returncode, r.stderr)


@need_ref
def test_library_errors_exit_1(tmp_path):
    """Degenerate inputs raise the library's own errors (empty distribution)."""
    r = msv(REF, "plan", write_cfg(tmp_path, {**SMALL, "workload": {"pmf": []}}))
    assert r.returncode == 1 and "ParamError" in r.stderr, r.stderr
    r = msv(REF, "sweep", write_cfg(tmp_path, {**SMALL, "designs": [{"plan": "paris"}]}))
    assert r.returncode == 1 and "gpu(7)+fifs" in r.stderr  # compare() needs its normalisation baseline
    r = msv(REF, "run", tmp_path / "missing.json")
    assert r.returncode == 1
    assert msv(REF, "frobnicate", tmp_path / "missing.json").returncode == 1


@need_ref
@need_dev
def test_plan_verb_host_only_matches_reference(tmp_path):
    """`plan` prints the PARIS plan without simulating; it is host code in
    both builds, so the product binary runs it without a GPU and prints the same bytes.
    Homogeneous k=3 on 8 GPUs -> 16 instances."""
    cfg = write_cfg(tmp_path, {"profile": {"preset": "heavy"}, "server": {"num_gpus": 8},
                               "designs": [{"plan": "gpu(3)", "scheduler": "fifs"},
                                           {"plan": "paris", "scheduler": "elsa"},
                                           {"plan": "random(3)", "scheduler": "elsa"}]})
    want = msv(REF, "plan", cfg)
    got = msv(DEV, "plan", cfg)
    assert want.returncode == 0 and got.returncode == 0, (want.stderr, got.stderr)
    assert got.stdout == want.stdout
    out = json.loads(got.stdout)
    assert out["designs"][0]["plan"]["instances"] == [{"count": 16, "k": 3}]
    assert sum(c["real_count"] * c["k"] for c in out["paris"]["counts"]) == pytest.approx(56, rel=1e-12)


# ------------------------------------------------------------------ GPU: byte-identical trees
def _both(tmp_path, verb, cfg, *extra):
    a, b = tmp_path / "ref" / "o", tmp_path / "dev" / "o"  # same relative output dir: same resolved config
    a.parent.mkdir(), b.parent.mkdir()
    r1 = msv(REF, verb, cfg, "--out", "o", *extra, cwd=a.parent)
    r2 = msv(DEV, verb, cfg, "--out", "o", *extra, cwd=b.parent)
    assert r1.returncode == 0, r1.stderr
    assert r2.returncode == 0, r2.stderr
    ta, tb = tree(a), tree(b)
    assert sorted(ta) == sorted(tb)
    diff = [k for k in ta if ta[k] != tb[k]]
    assert not diff, diff[:5]
    return ta


@pytest.mark.gpu
@need_ref
@need_dev
@pytest.mark.parametrize("cfg,extra", [
    ("paris_vs_gpu7.json", ()),
    ("bert_8gpu_run.json", ()),
    ("bert_8gpu_run.json", ("--set", "workload.rate_qps=1100", "--set", "engine.warmup_fraction=0")),
])
def test_run_tree_identical_to_reference(tmp_path, cfg, extra):
    t = _both(tmp_path, "run", EX / cfg, *extra)
    assert sum(k.endswith(".csv") for k in t) > 4


@pytest.mark.gpu
@need_ref
@need_dev
@pytest.mark.parametrize("cfg,extra", [
    ("sweep_light_1gpu.json", ()),
    ("sweep_light_1gpu.json", ("--set", "profile={\"preset\": \"medium\"}", "--set", "server.num_gpus=2",
                               "--set", "sla.tail_p=0.99")),
])
def test_sweep_tree_identical_to_reference(tmp_path, cfg, extra):
    t = _both(tmp_path, "sweep", EX / cfg, *extra)
    rows = t["summary.csv"].decode().splitlines()
    assert len(rows) == 5 and rows[1].startswith("gpu(7)+fifs,")
    assert len(t["plot_data.csv"].decode().splitlines()) == 1 + 4 * 6


NOISE_CASES = [
    # (config, overrides): ELSA / FIFS / routing / explicit and random plans on 8 GPUs
    ("bert_8gpu_run.json", ("--set", "engine.noise_sigma=0.3", "--set", "engine.noise_seed=5")),
    # busier, other sigma, no warm-up, wait check requested (skipped under noise, engine.hpp:208)
    ("bert_8gpu_run.json", ("--set", "engine.noise_sigma=0.6", "--set", "workload.rate_qps=1100",
                            "--set", "engine.warmup_fraction=0")),
    # one 7g partition at overload: long queues, completion chains inside one drain
    ("paris_vs_gpu7.json", ("--set", "engine.noise_sigma=0.25", "--set", "workload.duration_ms=1500")),
    # 56 x 1g partitions (both lane slots), FIFS and ELSA
    ("bert_8gpu_run.json", ("--set", "engine.noise_sigma=0.4", "--set", "workload.rate_qps=900",
                            "--set", 'designs=[{"plan": "gpu(1)", "scheduler": "fifs"}, {"plan": "gpu(1)", "scheduler": "elsa"}]')),
]


@pytest.mark.gpu
@need_ref
@need_dev
@pytest.mark.parametrize("cfg,extra", NOISE_CASES)
def test_noise_run_tree_identical_to_reference(tmp_path, cfg, extra):
    """Execution noise (engine.hpp:140-145) on the device (K5): per-query CSVs and reports
    byte-identical to the reference engine's."""
    t = _both(tmp_path, "run", EX / cfg, *extra)
    res = json.loads(t["resolved_config.json"])
    assert res["engine"]["noise_sigma"] > 0
    assert any(json.loads(v)["noise_sigma"] > 0 for k, v in t.items() if k.startswith("reports/") and k.endswith(".json"))


@pytest.mark.gpu
@need_ref
@need_dev
def test_noise_four_slots_and_partition_limit(tmp_path):
    """K5 with four lane slots: a 70-partition plan (10 GPUs of 1g) with execution noise is
    byte-identical to the reference engine, ELSA and FIFS; plans beyond 128 partitions raise
    ParamError (the device engine's limit, with or without noise)."""
    cfg = write_cfg(tmp_path, {**SMALL, "server": {"num_gpus": 10}, "engine": {"noise_sigma": 0.3},
                               "workload": {"rate_qps": 3000, "duration_ms": 800, "seeds": [1, 2]},
                               "designs": [{"plan": "gpu(1)", "scheduler": "elsa"},
                                           {"plan": "gpu(1)", "scheduler": "fifs"}]})
    _both(tmp_path, "run", cfg)
    big = write_cfg(tmp_path, {**SMALL, "server": {"num_gpus": 19}, "engine": {"noise_sigma": 0.1},
                               "designs": [{"plan": "gpu(1)", "scheduler": "elsa"}]}, "big.json")
    r = msv(DEV, "run", big, "--out", tmp_path / "o2")
    assert r.returncode == 1 and "ParamError" in r.stderr and "128" in r.stderr, r.stderr


@pytest.mark.gpu
@need_ref
@need_dev
def test_noise_randomised_against_reference(tmp_path):
    """Random noisy runs (plans of 1-63 partitions on 1-9 GPUs, ELSA/FIFS, routing, alpha/beta,
    sigma 0.05-1, light to overloaded rates): per-query CSVs and reports byte-identical."""
    import random
    rng = random.Random(20261019)
    for case in range(24):
        gpus = rng.randint(1, 9)
        plan = rng.choice(["paris", f"random({rng.randint(0, 99)})", f"gpu({rng.choice([1, 2, 3, 7])})"])
        cfg = {
            "profile": {"preset": rng.choice(["light", "medium", "heavy"])},
            "workload": {"rate_qps": rng.choice([50, 200, 800, 2500]) * gpus, "duration_ms": rng.choice([300, 800]),
                         "seeds": [rng.randint(1, 10**6), rng.randint(1, 10**6)], "sigma": rng.choice([0.5, 1.0, 1.5])},
            "server": {"num_gpus": gpus},
            "sla": {"multiplier": rng.choice([1.0, 1.5, 3.0]), "alpha": rng.choice([1.0, 0.8, 1.3]),
                    "beta": rng.choice([1.0, 0.5, 2.0])},
            "engine": {"noise_sigma": rng.choice([0.05, 0.3, 1.0]), "noise_seed": rng.randint(0, 10**6),
                       "warmup_fraction": rng.choice([0.0, 0.1, 0.5])},
            "designs": [{"plan": plan, "scheduler": "elsa", "segment_routing": rng.random() < 0.3},
                        {"plan": plan, "scheduler": "fifs", "label": "fifs-design"}],
        }
        d = tmp_path / f"c{case}"
        d.mkdir()
        _both(d, "run", write_cfg(d, cfg))
