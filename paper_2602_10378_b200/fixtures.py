"""Synthetic inputs exactly as the reference generates them (host side).

* ``mixture_16d()``: the reference's configs/mixture-16d-default.json
  (4 equal-weight components, sigma = 1, d = 16), shipped as package data.
* ``sample_mixture`` / ``random_gaussian`` / ``mix64``: bitwise the reference's
  RNG streams (rng.cpp, mixture.cpp:40-67, test_util.hpp:12-20).
* ``runtime_sweep_inputs(n, m)``: the runtime sweep's seed derivation
  (sweep.cpp:67-69, 173-177): train seed mix64(seed ^ mix64(n)), queries
  mix64(train_seed ^ 0x71).
* bandwidth rules (bandwidth.cpp:9-58) and ``BandwidthPolicy`` Auto
  (sweep.cpp:31-61): SD-KDE rate rule for SD-KDE, Silverman otherwise.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

from . import _native as N

HERE = os.path.dirname(os.path.abspath(__file__))
MIXTURE_16D = os.path.join(HERE, "configs", "mixture-16d-default.json")

_dp = ctypes.POINTER(ctypes.c_double)


def _p(a):
    return a.ctypes.data_as(_dp)


def mixture_16d():
    with open(MIXTURE_16D) as f:
        j = json.load(f)
    return (np.asarray(j["weights"], np.float64), np.asarray(j["means"], np.float64),
            np.asarray(j["sigmas"], np.float64))


def mix64(x: int) -> int:
    return int(N.load().fkde_host_mix64(x & 0xFFFFFFFFFFFFFFFF))


def random_gaussian(n: int, d: int, seed: int, scale: float = 1.0) -> np.ndarray:
    out = np.empty((n, d), np.float64)
    N.load().fkde_host_random_gaussian(n, d, seed, scale, _p(out))
    return out


def sample_mixture(weights, means, sigmas, n: int, seed: int) -> np.ndarray:
    w = np.ascontiguousarray(weights, np.float64)
    mu = np.ascontiguousarray(means, np.float64)
    s = np.ascontiguousarray(sigmas, np.float64)
    out = np.empty((n, mu.shape[1]), np.float64)
    rc = N.load().fkde_host_sample_mixture(_p(w), _p(mu), _p(s), w.size, mu.shape[1], n, seed,
                                           _p(out))
    if rc:
        raise ValueError("sample_mixture: invalid mixture")
    return out


def cell_data_seed(seed: int, n: int) -> int:
    return mix64(seed ^ mix64(n))


def runtime_sweep_inputs(n: int, m: int, seed: int = 0):
    w, mu, s = mixture_16d()
    cs = cell_data_seed(seed, n)
    return sample_mixture(w, mu, s, n, cs), sample_mixture(w, mu, s, m, mix64(cs ^ 0x71))


def mean_stddev(x) -> float:
    a = np.ascontiguousarray(x, np.float64)
    return N.load().fkde_host_mean_stddev(_p(a), a.shape[0], a.shape[1])


def silverman_bandwidth(x) -> float:
    a = np.ascontiguousarray(x, np.float64)
    return N.load().fkde_host_silverman_bandwidth(_p(a), a.shape[0], a.shape[1])


def sdkde_bandwidth(x, c: float | None = None) -> float:
    a = np.ascontiguousarray(x, np.float64)
    lib = N.load()
    if c is None:
        c = lib.fkde_host_silverman_prefactor(a.shape[1])
    return lib.fkde_host_sdkde_bandwidth(_p(a), a.shape[0], a.shape[1], c)


def auto_bandwidth(x, method: str) -> float:
    """BandwidthPolicy Auto (sweep.cpp:31-61)."""
    return sdkde_bandwidth(x) if method == "sdkde" else silverman_bandwidth(x)
