"""Build recipes for the native pieces (no CUDA device needed: nvcc cross-compiles).

    libmsv.so           csrc/*.cu (sm_100a kernels, -fmad=false) + csrc/*.cpp (host
                        runtime) -> paper_2202_13481_b200/libmsv.so, static cudart.
    msv                 cli/msv_cli.cpp (the SPEC's run/plan/sweep runner) over include/migserve,
                        linked to libmsv.so -> paper_2202_13481_b200/msv.
    oracle (test infra) delegated to oracle/build_oracle.py.

Everything is written in-tree so the built files travel to the GPU box with the
repository snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libmsv.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_INC = "/usr/local/cuda/include"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC"] + os.environ.get("MSV_NVCC_EXTRA", "").split() + [
                     "-Xptxas", "-v"]
CXX_FLAGS = ["-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-Wall", "-Wno-unused-function"]


def json_include_dir() -> str:
    """nlohmann/json 3.11.3 header shipped in this image (needed by include/migserve)."""
    cands = [os.environ.get("MSV_JSON_INCLUDE", "")]
    try:
        import cudnn  # noqa: F401  (not required; only used to locate site-packages)
    except Exception:
        pass
    for sp in sys.path:
        cands.append(os.path.join(sp, "include", "cudnn_frontend", "thirdparty", "nlohmann"))
    cands.append("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")
    for c in cands:
        if c and os.path.isfile(os.path.join(c, "json.hpp")):
            return c
    raise FileNotFoundError("nlohmann json.hpp not found (set MSV_JSON_INCLUDE)")


def _run(cmd: list[str], log: list[str] | None = None) -> str:
    r = subprocess.run(cmd, capture_output=True, text=True)
    out = r.stdout + r.stderr
    if log is not None:
        log.append(" ".join(cmd) + "\n" + out)
    if r.returncode != 0:
        raise RuntimeError(f"build step failed ({r.returncode}): {' '.join(cmd)}\n{out}")
    return out


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build_libmsv(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    headers = sorted(CSRC.glob("*.h")) + sorted(CSRC.glob("*.cuh")) + sorted((ROOT / "include").rglob("*.h*"))
    objs: list[Path] = []
    log: list[str] = []
    steps = []  # independent compiles, run concurrently (the kernel files dominate the build)
    for src in sorted(CSRC.glob("*.cu")):
        obj = BUILD / (src.stem + ".o")
        if force or _stale(obj, [src, *headers]):
            steps.append([NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)])
        objs.append(obj)
    for src in sorted(CSRC.glob("*.cpp")):
        obj = BUILD / (src.stem + ".o")
        if force or _stale(obj, [src, *headers]):
            steps.append(["g++", *CXX_FLAGS, f"-I{CUDA_INC}", f"-I{ROOT / 'include'}", f"-I{json_include_dir()}",
                          "-c", str(src), "-o", str(obj)])
        objs.append(obj)
    if steps:
        from concurrent.futures import ThreadPoolExecutor
        logs: list[list[str]] = [[] for _ in steps]
        with ThreadPoolExecutor(max_workers=min(len(steps), os.cpu_count() or 1)) as ex:
            futs = [ex.submit(_run, cmd, lg) for cmd, lg in zip(steps, logs)]
            for f in futs:
                f.result()  # re-raises a failed step
        for lg in logs:
            log.extend(lg)
    if force or _stale(LIB, objs):
        tmp = LIB.with_suffix(".so.tmp")
        _run([NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-cudart", "static",
              "-Xlinker", "--no-undefined", "-lpthread", "-ldl", "-lrt"], log)
        os.replace(tmp, LIB)
    (BUILD / "build.log").write_text("\n".join(log))
    if verbose:
        print("\n".join(log))
    return LIB


CLI = PKG / "msv"


def build_cli(force: bool = False) -> Path:
    """The experiment runner on the device engine: the drop-in headers + libmsv.so."""
    src = PKG / "cli" / "msv_cli.cpp"
    deps = [src, LIB, *sorted((ROOT / "include").rglob("*.h*"))]
    if force or _stale(CLI, deps):
        tmp = CLI.with_name("msv.tmp")
        _run(["g++", "-std=c++20", "-O2", "-Wall", "-pthread", f"-I{ROOT / 'include'}", f"-I{json_include_dir()}",
              str(src), "-o", str(tmp), f"-L{PKG}", "-lmsv", "-Wl,-rpath,$ORIGIN"])
        os.replace(tmp, CLI)
    return CLI


def build_all(force: bool = False) -> None:
    build_libmsv(force=force)
    build_cli(force=force)
    sys.path.insert(0, str(ROOT / "oracle"))
    try:
        import build_oracle  # type: ignore

        build_oracle.build(force=force)
    finally:
        sys.path.pop(0)


if __name__ == "__main__":
    build_libmsv(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
