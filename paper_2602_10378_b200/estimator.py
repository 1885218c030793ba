"""Host mirror of ``fkde::estimate`` (estimator.hpp:9-10, estimator.cpp:14-60).

``EngineKind.Flash`` and ``EngineKind.Gpu`` dispatch to the B200 engine.
``EngineKind.Naive`` is the reference's CPU oracle, which stays in the
reference (it is this project's test oracle, not part of the product):
requesting it raises InvalidArgumentError.
"""
from __future__ import annotations

from typing import Optional

import numpy as np

from . import engine
from .types import (DensityResult, EngineKind, EstimatorConfig, InvalidArgumentError,
                    KernelKind, Method, SampleSet)


def _attach_negative_mass(result: DensityResult) -> None:
    # estimator.cpp:14-20
    v = result.values
    result.negative_mass_estimate = float(np.maximum(0.0, -v).sum() / v.size)


def estimate(train, queries, config: EstimatorConfig, *,
             ctx: Optional[engine.Context] = None) -> DensityResult:
    config.validate()
    if config.engine == EngineKind.Naive:
        raise InvalidArgumentError(
            "estimate: EngineKind.Naive is the reference CPU oracle; use Flash/Gpu")
    train, queries = SampleSet.wrap(train), SampleSet.wrap(queries)
    plan = engine.TilePlan.make(queries.n, train.n, config.tile_m, config.tile_n)
    opts = engine.EngineOptions(config.threads, config.fast_accumulation)
    if config.method == Method.Kde:
        return engine.kde_flash(train, queries, config.bandwidth.h, KernelKind.Gaussian, True,
                                plan, opts, ctx=ctx)
    if config.method == Method.Sdkde:
        return engine.sdkde_flash(train, queries, config.bandwidth, plan, opts, ctx=ctx)
    if config.method == Method.LaplaceKde:
        r = engine.kde_flash(train, queries, config.bandwidth.h, KernelKind.LaplaceCorrected,
                             config.fused, plan, opts, ctx=ctx)
        _attach_negative_mass(r)
        return r
    raise InvalidArgumentError("estimate: unknown method")
