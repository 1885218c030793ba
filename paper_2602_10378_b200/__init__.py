"""B200-native Flash-SD-KDE engine (drop-in for the reference's fkde estimator path).

Public API mirrors the reference's ``fkde`` C++ API:

* types: SampleSet, Bandwidth, EstimatorConfig, DensityResult, Method,
  EngineKind, KernelKind and the error hierarchy (types.hpp / errors.hpp);
* ``engine``: TilePlan, EngineOptions, score_accumulate, score_flash,
  kde_flash, sdkde_flash, pairwise_sq_dists_block (engine.hpp);
* ``estimate`` (estimator.hpp).

The arithmetic runs in ``libfkde_b200.so`` (sm_100a CUDA, C ABI in
include/fkde_gpu.h).  There is no CPU fallback.
"""
from .types import (Bandwidth, DegenerateDataError, DensityResult, DeviceError,
                    DimensionMismatchError, EngineKind, EstimatorConfig, InvalidArgumentError,
                    IoError, KernelKind, Method, NonFiniteValueError, SampleSet,
                    ScoreUnderflowError, UnsupportedDimensionError, engine_from_string,
                    method_from_string, to_string)
from . import engine
from . import io
from .engine import (Context, EngineOptions, ScoreAccumulator, TilePlan, default_context,
                     kde_flash, pairwise_sq_dists_block, score_accumulate, score_flash,
                     sdkde_flash)
from .estimator import estimate

__all__ = [
    "Bandwidth", "DegenerateDataError", "DensityResult", "DeviceError", "DimensionMismatchError",
    "EngineKind", "EstimatorConfig", "InvalidArgumentError", "IoError", "KernelKind", "Method",
    "NonFiniteValueError", "SampleSet", "ScoreUnderflowError", "UnsupportedDimensionError",
    "engine_from_string", "method_from_string", "to_string", "engine", "Context",
    "EngineOptions", "ScoreAccumulator", "TilePlan", "default_context", "kde_flash",
    "pairwise_sq_dists_block", "score_accumulate", "score_flash", "sdkde_flash", "estimate",
]
