"""Host-side mirror of the reference's domain types and errors.

Mirrors /root/reference/proj/core/include/fkde/types.hpp:15-84 and
errors.hpp:10-56 (same names, same validation rules, same exception
hierarchy) so that code and tests written against the reference's
``fkde::`` API read the same here.
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np


# ---- errors.hpp:10-56 ------------------------------------------------------
class InvalidArgumentError(ValueError):
    """Bad values or flag combinations supplied by the caller."""


class DimensionMismatchError(InvalidArgumentError):
    """Two point sets do not live in the same dimension."""


class DegenerateDataError(RuntimeError):
    """Zero spread in every dimension; bandwidth rules are undefined."""


class ScoreUnderflowError(RuntimeError):
    """The score denominator underflowed to zero at a specific point."""

    def __init__(self, index: int, what: str):
        super().__init__(what)
        self._index = int(index)

    def index(self) -> int:
        return self._index


class NonFiniteValueError(RuntimeError):
    def __init__(self, index: int, what: str):
        super().__init__(what)
        self._index = int(index)

    def index(self) -> int:
        return self._index


class IoError(RuntimeError):
    """fkde::IoError (errors.hpp): file missing, malformed or short write
    (raised by paper_2602_10378_b200.io)."""


class DeviceError(RuntimeError):
    """CUDA / NCCL failure inside the engine (no reference counterpart)."""


class UnsupportedDimensionError(InvalidArgumentError):
    """d beyond the tensor-core path's limit (16)."""


# ---- types.hpp:15-41 -----------------------------------------------------------
class SampleSet:
    """Dense n x d row-major point set (fp64)."""

    __slots__ = ("values", "n", "d")

    def __init__(self, data=None, n_rows: Optional[int] = None, n_cols: Optional[int] = None):
        if data is None:
            self.values = np.zeros((0, 0), dtype=np.float64)
            self.n = 0
            self.d = 0
            return
        a = np.asarray(data, dtype=np.float64)
        if n_rows is not None and n_cols is not None:
            if a.size != n_rows * n_cols:
                raise InvalidArgumentError("SampleSet: storage size does not match n*d")
            a = a.reshape(n_rows, n_cols)
        elif a.ndim == 1:
            a = a.reshape(-1, 1)
        self.values = np.ascontiguousarray(a)
        self.n, self.d = self.values.shape
        self.validate()

    @staticmethod
    def zeros(n_rows: int, n_cols: int) -> "SampleSet":
        s = SampleSet()
        s.values = np.zeros((n_rows, n_cols), dtype=np.float64)
        s.n, s.d = n_rows, n_cols
        return s

    @staticmethod
    def wrap(a) -> "SampleSet":
        return a if isinstance(a, SampleSet) else SampleSet(a)

    def row(self, i: int) -> np.ndarray:
        return self.values[i]

    def data(self) -> np.ndarray:
        return self.values

    def empty(self) -> bool:
        return self.n == 0

    def validate(self) -> None:
        # types.cpp:21-33
        if self.n == 0 or self.d == 0:
            raise InvalidArgumentError("SampleSet: n and d must be >= 1")
        if self.values.shape != (self.n, self.d):
            raise InvalidArgumentError("SampleSet: storage size does not match n*d")
        if not np.isfinite(self.values).all():
            raise InvalidArgumentError("SampleSet: non-finite entry")

    def copy(self) -> "SampleSet":
        s = SampleSet()
        s.values = self.values.copy()
        s.n, s.d = self.n, self.d
        return s

    def __repr__(self) -> str:
        return f"SampleSet(n={self.n}, d={self.d})"


# ---- types.hpp:43-50 ----------------------------------------------------------------
class Method(enum.Enum):
    Kde = "kde"
    Sdkde = "sdkde"
    LaplaceKde = "laplace"


class EngineKind(enum.Enum):
    Naive = "naive"   # the reference's CPU oracle -- not part of this product
    Flash = "flash"   # the reference's blocked engine -> served by the GPU engine here
    Gpu = "gpu"       # explicit name for the B200 engine


class KernelKind(enum.Enum):
    Gaussian = 0
    LaplaceCorrected = 1


def to_string(x) -> str:
    return x.value if isinstance(x, (Method, EngineKind)) else str(x)


def method_from_string(s: str) -> Method:
    for m in Method:
        if m.value == s:
            return m
    raise InvalidArgumentError("unknown method: " + s)


def engine_from_string(s: str) -> EngineKind:
    for e in EngineKind:
        if e.value == s:
            return e
    raise InvalidArgumentError("unknown engine: " + s)


# ---- types.hpp:52-63 ----------------------------------------------------------------
@dataclass
class Bandwidth:
    h: float = 1.0
    h_score: float = 1.0

    @staticmethod
    def uniform(h: float) -> "Bandwidth":
        return Bandwidth(h, h)

    @staticmethod
    def half_variance_score(h: float) -> "Bandwidth":
        return Bandwidth(h, h / math.sqrt(2.0))

    def validate(self) -> None:
        # types.cpp:65-72
        if not (self.h > 0.0) or not math.isfinite(self.h):
            raise InvalidArgumentError("Bandwidth: h must be positive and finite")
        if not (self.h_score > 0.0) or not math.isfinite(self.h_score):
            raise InvalidArgumentError("Bandwidth: h_score must be positive and finite")


# ---- types.hpp:65-76 ----------------------------------------------------------------
@dataclass
class EstimatorConfig:
    method: Method = Method.Kde
    bandwidth: Bandwidth = field(default_factory=Bandwidth)
    engine: EngineKind = EngineKind.Flash
    tile_m: int = 64
    tile_n: int = 1024
    fused: bool = True
    threads: int = 0
    fast_accumulation: bool = False

    def validate(self) -> None:
        # types.cpp:74-79
        self.bandwidth.validate()
        if self.tile_m == 0 or self.tile_n == 0:
            raise InvalidArgumentError("EstimatorConfig: tile_m and tile_n must be >= 1")


# ---- types.hpp:80-84 ----------------------------------------------------------------
@dataclass
class DensityResult:
    values: np.ndarray
    negative_mass_estimate: Optional[float] = None
    debiased_samples: Optional[SampleSet] = None
