"""TEST INFRASTRUCTURE ONLY — builds the CPU checkers. Never imported by the product.

Outputs (all git-ignored, all travel to the GPU box with the repo snapshot):
  oracle/libmsv_oracle.so       plain-C restatement (port/msv_oracle.c)
  oracle/_ref/libmsv_ref.so     the reference itself: /root/reference/proj/include,
                                unmodified, behind oracle_abi.h (ref_capi.cpp),
                                built with the reference's Release flags (-O3 -DNDEBUG,
                                no -march; proj/CMakeLists.txt:6-8)
  oracle/_ref/ref_unit_tests    the reference's own Catch2 suite (proj/tests/*.cpp)
                                on the catch_shim, against the reference headers
  oracle/_ref/dropin_unit_tests the same unmodified test sources compiled against THIS
                                repo's include/migserve headers and linked to libmsv.so
                                (every run()/sample_trace()/tail_latency()/dispatch call
                                executes on the GPU) — the drop-in check
  oracle/_ref/msv_cli_ref       paper_2202_13481_b200/cli/msv_cli.cpp (the run/plan/sweep
                                runner) compiled against the reference headers: the
                                checker for the product CLI paper_2202_13481_b200/msv

The _ref targets need /root/reference (present in the build container only); on the
GPU box the prebuilt files are used as they are.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
REF = Path(os.environ.get("MSV_REFERENCE", "/root/reference")) / "proj"
REF_OUT = HERE / "_ref"
PORT_LIB = HERE / "libmsv_oracle.so"


def _json_dir() -> str:
    sys.path.insert(0, str(ROOT))
    try:
        from paper_2202_13481_b200.build import json_include_dir

        return json_include_dir()
    finally:
        sys.path.pop(0)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed: {' '.join(cmd)}\n{r.stdout}{r.stderr}")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.exists() and d.stat().st_mtime > t for d in deps)


def build_port(force: bool = False) -> Path:
    src = HERE / "port" / "msv_oracle.c"
    if force or _stale(PORT_LIB, [src, HERE / "oracle_abi.h"]):
        _run(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", str(PORT_LIB), str(src),
              "-lm", "-lpthread"])
    return PORT_LIB


def reference_available() -> bool:
    return (REF / "include" / "migserve" / "engine.hpp").is_file()


def build_reference(force: bool = False) -> None:
    if not reference_available():
        return  # GPU box: use the prebuilt oracle/_ref files
    REF_OUT.mkdir(exist_ok=True)
    inc = REF / "include"
    ref_headers = sorted(inc.rglob("*.hpp"))
    json_dir = _json_dir()
    flags = ["-std=c++20", "-O3", "-DNDEBUG", "-fPIC", "-pthread", f"-I{inc}", f"-I{json_dir}"]
    lib = REF_OUT / "libmsv_ref.so"
    if force or _stale(lib, [HERE / "ref_capi.cpp", HERE / "oracle_abi.h", *ref_headers]):
        _run(["g++", *flags, "-shared", "-o", str(lib), str(HERE / "ref_capi.cpp")])
    tests = sorted((REF / "tests").glob("test_*.cpp"))
    shim = HERE / "catch_shim"
    unit = REF_OUT / "ref_unit_tests"
    if force or _stale(unit, [*tests, *ref_headers, shim / "catch2" / "catch_amalgamated.hpp"]):
        _run(["g++", *flags, f"-I{shim}", str(shim / "shim_main.cpp"), *map(str, tests), "-o", str(unit)])
    cli_src = ROOT / "paper_2202_13481_b200" / "cli" / "msv_cli.cpp"
    cli_ref = REF_OUT / "msv_cli_ref"  # the SPEC's runner on the reference's CPU engine (the CLI checker)
    if force or _stale(cli_ref, [cli_src, *ref_headers]):
        _run(["g++", *flags, str(cli_src), "-o", str(cli_ref)])
    io_ref = REF_OUT / "io_check_ref"  # oracle/io_check.cpp on the reference's CPU engine
    if force or _stale(io_ref, [HERE / "io_check.cpp", *ref_headers]):
        _run(["g++", *flags, str(HERE / "io_check.cpp"), "-o", str(io_ref)])


def build_dropin(force: bool = False) -> None:
    """Reference test sources against this repo's headers + libmsv.so."""
    if not reference_available():
        return
    libmsv = ROOT / "paper_2202_13481_b200" / "libmsv.so"
    if not libmsv.exists():
        return
    REF_OUT.mkdir(exist_ok=True)
    tests = sorted((REF / "tests").glob("test_*.cpp"))
    shim = HERE / "catch_shim"
    ours = sorted((ROOT / "include").rglob("*.h*"))
    out = REF_OUT / "dropin_unit_tests"
    if force or _stale(out, [*tests, *ours, libmsv, shim / "catch2" / "catch_amalgamated.hpp"]):
        _run(["g++", "-std=c++20", "-O2", "-DNDEBUG", "-pthread", f"-I{ROOT / 'include'}", f"-I{_json_dir()}",
              f"-I{shim}", f"-I{REF / 'tests'}", str(shim / "shim_main.cpp"), *map(str, tests), "-o", str(out),
              f"-L{libmsv.parent}", "-lmsv", f"-Wl,-rpath,{libmsv.parent}", "-Wl,-rpath,$ORIGIN/../../paper_2202_13481_b200"])
    io_dev = REF_OUT / "io_check_dev"  # the same program on the device engine (drop-in headers)
    if force or _stale(io_dev, [HERE / "io_check.cpp", *ours, libmsv]):
        _run(["g++", "-std=c++20", "-O2", "-DNDEBUG", "-pthread", f"-I{ROOT / 'include'}", f"-I{_json_dir()}",
              str(HERE / "io_check.cpp"), "-o", str(io_dev), f"-L{libmsv.parent}", "-lmsv",
              f"-Wl,-rpath,{libmsv.parent}", "-Wl,-rpath,$ORIGIN/../../paper_2202_13481_b200"])


def build(force: bool = False) -> None:
    build_port(force)
    build_reference(force)
    build_dropin(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print("oracle built")
