"""B200-native scenario-grid engine for arXiv 2202.13481 (PARIS x ELSA).

The hot path — grids of (partition plan x latency profile x Poisson rate x seed)
inference-server simulations — runs as sm_100a CUDA kernels behind the C ABI in
include/msv.h (libmsv.so, built in-tree). C++ users include include/migserve/*.hpp
(the reference's API); Python users use this package.
"""
from ._native import (DeviceError, Error, FormatError, InfeasibleError, LookupError_, ParamError, ValidationError,
                      KIND_NAMES, lib)
from .engine import (BatchDistribution, DeviceGrid, Engine, GridSpec, ParisJob, ParisOutcome, PartitionPlan,
                     ProfileTable, SlaConfig,
                     SyntheticProfileParams, derive_sla_target, homogeneous_plan, lognormal_batch_pdf, paris_plan,
                     synth_profile)

__all__ = [
    "BatchDistribution", "DeviceError", "DeviceGrid", "Engine", "Error", "FormatError", "GridSpec", "InfeasibleError",
    "KIND_NAMES", "LookupError_", "ParamError", "ParisJob", "ParisOutcome", "PartitionPlan", "ProfileTable", "SlaConfig", "SyntheticProfileParams",
    "ValidationError", "derive_sla_target", "homogeneous_plan", "lib", "lognormal_batch_pdf", "paris_plan",
    "synth_profile",
]
