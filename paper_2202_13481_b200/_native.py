"""ctypes binding of libmsv.so (include/msv.h). Loads the in-tree library built by
paper_2202_13481_b200/build.py; there is no fallback — a missing library or a host
without a B200 raises instead of silently computing on the CPU."""
from __future__ import annotations

import ctypes as C
import os
import re
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["MSV_LIB"]) if os.environ.get("MSV_LIB") else PKG / "libmsv.so"  # MSV_LIB: A/B builds
HEADER = PKG.parent / "include" / "msv.h"

MSV_OK, MSV_PARAM, MSV_FORMAT, MSV_VALIDATION, MSV_LOOKUP, MSV_INFEASIBLE, MSV_CUDA = range(7)
MSV_FIFS, MSV_ELSA = 0, 1
MSV_FLAG_CHECK_WAIT = 1
KIND_NAMES = ("slack-satisfying", "fastest-fallback", "idle-largest", "shortest-queue")


class Error(RuntimeError):
    """migserve::Error (errors.hpp:11)."""


class ParamError(Error):
    """migserve::ParamError (errors.hpp:16)."""


class FormatError(Error):
    """migserve::FormatError (errors.hpp:22)."""


class ValidationError(Error):
    """migserve::ValidationError (errors.hpp:28)."""


class LookupError_(Error):
    """migserve::LookupError (errors.hpp:33)."""


class InfeasibleError(Error):
    """migserve::InfeasibleError (errors.hpp:38)."""


class DeviceError(Error):
    """CUDA / driver failure (MSV_CUDA)."""


_ERRORS = {MSV_PARAM: ParamError, MSV_FORMAT: FormatError, MSV_VALIDATION: ValidationError,
           MSV_LOOKUP: LookupError_, MSV_INFEASIBLE: InfeasibleError, MSV_CUDA: DeviceError}


class Scenario(C.Structure):
    _fields_ = [("profile", C.c_int32), ("dist", C.c_int32), ("plan", C.c_int32), ("scheduler", C.c_int32),
                ("routing", C.c_int32), ("flags", C.c_int32), ("sla_ms", C.c_double), ("alpha", C.c_double),
                ("beta", C.c_double), ("rate_qps", C.c_double), ("duration_ms", C.c_double),
                ("warmup_fraction", C.c_double), ("seed", C.c_uint64)]


class Result(C.Structure):
    _fields_ = [("total", C.c_int64), ("violations", C.c_int64), ("measured", C.c_int64),
                ("measured_violations", C.c_int64), ("tail", C.c_double * 4), ("horizon_ms", C.c_double),
                ("warmup_ms", C.c_double), ("max_wait_estimate_diff", C.c_double), ("duration_ms", C.c_double),
                ("placement_hash", C.c_uint64), ("status", C.c_int32), ("n_partitions", C.c_int32)]


class Usage(C.Structure):
    _fields_ = [("busy_ms", C.c_double), ("weighted_busy_ms", C.c_double), ("queries", C.c_int64)]


class Record(C.Structure):
    _fields_ = [("start_ms", C.c_double), ("finish_ms", C.c_double), ("partition", C.c_int32), ("kind", C.c_int32)]


MSV_PARIS_MAX_SIZES = 8


class ParisJob(C.Structure):
    _fields_ = [("profile", C.c_int32), ("dist", C.c_int32), ("total_gpcs", C.c_int32), ("num_gpus", C.c_int32),
                ("gpcs_per_gpu", C.c_int32), ("pad", C.c_int32), ("knee_threshold", C.c_double)]


class ParisOut(C.Structure):
    _fields_ = [("status", C.c_int32), ("n_sizes", C.c_int32), ("n_instances", C.c_int32), ("err_k", C.c_int32),
                ("err_b", C.c_int32), ("pad", C.c_int32), ("k", C.c_int32 * MSV_PARIS_MAX_SIZES),
                ("knee", C.c_int32 * MSV_PARIS_MAX_SIZES), ("seg_first", C.c_int32 * MSV_PARIS_MAX_SIZES),
                ("seg_last", C.c_int32 * MSV_PARIS_MAX_SIZES), ("ratio", C.c_double * MSV_PARIS_MAX_SIZES),
                ("segment_mass", C.c_double * MSV_PARIS_MAX_SIZES), ("count", C.c_double * MSV_PARIS_MAX_SIZES),
                ("weighted_sum", C.c_double), ("normalizer", C.c_double)]


_P = C.c_void_p
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)

_SIGNATURES = {
    "msv_last_error": (C.c_char_p, []),
    "msv_abi_version": (C.c_int, []),
    "msv_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "msv_create_multi": (C.c_int, [_i32p, C.c_int, C.POINTER(_P)]),
    "msv_context_devices": (C.c_int, [_P, _i32p, C.c_int]),
    "msv_destroy": (C.c_int, [_P]),
    "msv_set_log1p_variant": (C.c_int, [_P, C.c_int]),
    "msv_get_log1p_variant": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "msv_upload_profile": (C.c_int, [_P, C.c_int, _i32p, C.c_int, _f64p, _f64p, _i32p]),
    "msv_upload_dist": (C.c_int, [_P, C.c_int, _f64p, _i32p]),
    "msv_upload_cdf": (C.c_int, [_P, C.c_int, _f64p, _i32p]),
    "msv_upload_plan": (C.c_int, [_P, C.c_int, C.c_int, _i32p, _i32p, _i32p]),
    "msv_upload_routing": (C.c_int, [_P, C.c_int, _i32p, _i32p, _i32p, _i32p]),
    "msv_run_grid": (C.c_int, [_P, C.POINTER(Scenario), C.c_int64, _f64p, C.c_int, C.POINTER(Result),
                               C.POINTER(Usage)]),
    "msv_run_replay": (C.c_int, [_P, C.POINTER(Scenario), C.c_int64, _i64p, _f64p, _i32p, _f64p, C.c_int,
                                 C.POINTER(Result), C.POINTER(Usage), C.POINTER(Record)]),
    "msv_run_noise": (C.c_int, [_P, C.POINTER(Scenario), C.c_int64, _f64p, _i32p, _f64p, C.POINTER(Result),
                                C.POINTER(Usage), C.POINTER(Record)]),
    "msv_noise_multipliers": (C.c_int, [C.c_uint64, C.c_double, C.c_int64, _f64p]),
    "msv_run_grid_noise": (C.c_int, [_P, C.POINTER(Scenario), C.c_int64, _f64p, C.POINTER(C.c_uint64), _f64p, C.c_int,
                                     C.POINTER(Result), C.POINTER(Usage)]),
    "msv_sample_trace": (C.c_int, [_P, C.c_int32, C.c_double, C.c_double, C.c_uint64, C.c_int64, _f64p, _i32p,
                                   _i64p]),
    "msv_tail_latency": (C.c_int, [_P, _f64p, C.c_int64, _f64p, C.c_int, _f64p]),
    "msv_dispatch_batch": (C.c_int, [_P, C.c_int32, C.c_int, C.c_int64, _i64p, _i32p, _i32p, _u8p, _f64p, _f64p,
                                     _i64p, _i32p, _i32p, _f64p, _f64p, _f64p, _f64p, _i32p, _i32p, _f64p]),
    "msv_paris_batch": (C.c_int, [_P, C.POINTER(ParisJob), C.c_int64, C.POINTER(ParisOut), _i32p, _i32p]),
    "msv_grid_create": (C.c_int, [_P, C.POINTER(Scenario), C.c_int64, _f64p, C.c_int, C.POINTER(_P)]),
    "msv_grid_launch": (C.c_int, [_P]),
    "msv_grid_results": (C.c_int, [_P, C.POINTER(Result), C.POINTER(Usage)]),
    "msv_grid_destroy": (C.c_int, [_P]),
    "msv_grid_timing": (C.c_int, [_P, C.POINTER(C.c_float), C.POINTER(C.c_float), C.POINTER(C.c_float),
                                  C.POINTER(C.c_float)]),
    "msv_grid_queries": (C.c_int64, [_P]),
    "msv_grid_set_overlap": (C.c_int, [_P, C.c_int]),
    "msv_grid_set_usage": (C.c_int, [_P, C.c_int]),
    "msv_synchronize": (C.c_int, [_P]),
    "msv_kernel_launches": (C.c_int64, [_P]),
    "msv_event_record": (C.c_int, [_P, C.c_int]),
    "msv_event_elapsed": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(C.c_float)]),
    "msv_transfer_bytes": (C.c_int, [_P, _i64p, _i64p]),
    "msv_paris_plan": (C.c_int, [C.c_int, _i32p, C.c_int, _f64p, _f64p, _f64p, C.c_int, C.c_int, C.c_int,
                                 C.c_double, _i32p, _i32p]),
    "msv_synth_profile": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, _i32p, C.c_int, _i32p,
                                    _i32p, _f64p, _f64p]),
    "msv_lognormal_pdf": (C.c_int, [C.c_double, C.c_double, C.c_int, _f64p, _f64p]),
    "msv_log1p_digest": (C.c_int, [_P, C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.POINTER(C.c_uint64)]),
    "msv_log1p_values": (C.c_int, [_P, C.c_int, C.c_uint64, C.c_int64, C.c_int64, _f64p]),
    "msv_quotient_check": (C.c_int, [_P, C.c_uint64, C.c_int64, _i64p]),
}

_lib = None


def header_symbols() -> list[str]:
    """Every function include/msv.h declares."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+char\s*\*|int64_t|int)\s+(msv_\w+)\s*\(", text, re.M)))


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGNATURES.items():
            if os.environ.get("MSV_LIB") and not hasattr(L, name):
                continue  # an older A/B build lacks newer entry points
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return (lib().msv_last_error() or b"").decode(errors="replace")


def check(rc: int, where: str = "") -> None:
    if rc != MSV_OK:
        msg = last_error()
        raise _ERRORS.get(rc, Error)(f"{where}: {msg}" if where else msg)
