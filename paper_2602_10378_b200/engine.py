"""Host mirror of ``fkde::engine`` (engine.hpp:15-76) over the B200 C ABI.

Every function keeps the reference's name, argument meaning, validation
order and exception types; the arithmetic runs in libfkde_b200.so
(tcgen05 kernels, see csrc/pairwise_tc.cuh).  ``TilePlan`` and
``EngineOptions`` are validated exactly like the reference
(engine.cpp:248-259) but do not steer the device schedule, which is the
engine's own (128x128 tensor-core tiles, persistent grid, column splits).
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from .types import (Bandwidth, DensityResult, DeviceError, DimensionMismatchError,
                    InvalidArgumentError, KernelKind, SampleSet, ScoreUnderflowError,
                    UnsupportedDimensionError)

_dp = ctypes.POINTER(ctypes.c_double)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


# ---- engine.hpp:15-38 ------------------------------------------------------------
@dataclass
class TilePlan:
    tile_m: int = 64
    tile_n: int = 1024
    n_tiles_m: int = 0
    n_tiles_n: int = 0

    @staticmethod
    def make(n_queries: int, n_train: int, tile_m: int, tile_n: int) -> "TilePlan":
        if tile_m == 0 or tile_n == 0:
            raise InvalidArgumentError("TilePlan: tile sizes must be >= 1")
        return TilePlan(tile_m, tile_n,
                        0 if n_queries == 0 else (n_queries + tile_m - 1) // tile_m,
                        0 if n_train == 0 else (n_train + tile_n - 1) // tile_n)


@dataclass
class ScoreAccumulator:
    phi_sum: np.ndarray
    weighted_sum: SampleSet


@dataclass
class EngineOptions:
    threads: int = 0                 # 0 = one device; k > 0 = k devices (single process)
    fast_accumulation: bool = False  # accepted for API parity; the device path is deterministic


class Context:
    """Owns one libfkde_b200 context (streams, workspaces, NCCL comm)."""

    def __init__(self, devices: Optional[Sequence[int]] = None, *, rank: Optional[int] = None,
                 world: Optional[int] = None, nccl_id: Optional[bytes] = None,
                 device: Optional[int] = None):
        self._lib = N.load()
        h = ctypes.c_void_p()
        if rank is not None:
            rc = self._lib.fkde_gpu_create_rank(int(device or 0), int(rank), int(world or 1),
                                                nccl_id, ctypes.byref(h))
        else:
            devs = list(devices) if devices else [0]
            arr = (ctypes.c_int * len(devs))(*devs)
            rc = self._lib.fkde_gpu_create(arr, len(devs), ctypes.byref(h))
        if rc != N.OK:
            raise DeviceError(f"fkde_gpu_create failed with status {rc}")
        self._h = h
        self.lock = threading.Lock()

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            self._lib.fkde_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, key: int, value: int):
        rc = self._lib.fkde_gpu_set_option(self._h, key, int(value))
        if rc != N.OK:
            raise InvalidArgumentError(f"set_option({key}, {value}) -> {rc}")

    def last_error(self) -> str:
        return (self._lib.fkde_gpu_last_error(self._h) or b"").decode()

    def last_timing(self) -> list:
        buf = (ctypes.c_float * N.T_COUNT)()
        self._lib.fkde_gpu_last_timing(self._h, buf, N.T_COUNT)
        return list(buf)

    def last_kernel_timing(self) -> list:
        """Device ms of the last call's score / check / density kernels (FKDE_KT_*;
        needs OPT_TIMING) -- fkde_gpu_last_kernel_timing."""
        buf = (ctypes.c_float * N.KT_COUNT)()
        self._lib.fkde_gpu_last_kernel_timing(self._h, buf, N.KT_COUNT)
        return list(buf)

    def last_launch_count(self) -> int:
        return int(self._lib.fkde_gpu_last_launch_count(self._h))

    def skip_stats(self) -> dict:
        """Tile skipping of the last call's score pass (and, under "density",
        its density pass) -- fkde_gpu_last_skip_stats."""
        b = (ctypes.c_uint64 * N.SKIP_STATS_COUNT)()
        self._lib.fkde_gpu_last_skip_stats(self._h, b, N.SKIP_STATS_COUNT)
        return {"tiles_checked": int(b[0]), "tiles_skipped": int(b[1]),
                "tiles_total": int(b[2]), "spatial_order": bool(b[3]),
                "direct_rows": int(b[8]),
                "density": {"tiles_skipped": int(b[4]), "tiles_total": int(b[5]),
                            "spatial_order": bool(b[6]), "direct_rows": int(b[7])}}

    def workspace_bytes(self) -> int:
        b = ctypes.c_size_t(0)
        self._lib.fkde_gpu_workspace_bytes(self._h, ctypes.byref(b))
        return int(b.value)

    def stream(self) -> int:
        return int(self._lib.fkde_gpu_stream(self._h) or 0)

    def world(self):
        r, w = ctypes.c_int(), ctypes.c_int()
        self._lib.fkde_gpu_world(self._h, ctypes.byref(r), ctypes.byref(w))
        return r.value, w.value

    def check(self, rc: int, err_index: Optional[int] = None):
        """Map an fkde_status onto the reference's exception types."""
        if rc == N.OK:
            return
        msg = self.last_error()
        if rc == N.INVALID_ARGUMENT or rc == N.NON_FINITE:
            raise InvalidArgumentError(msg)
        if rc == N.DIMENSION_MISMATCH:
            raise DimensionMismatchError(msg)
        if rc == N.SCORE_UNDERFLOW:
            raise ScoreUnderflowError(err_index if err_index is not None else 0, msg)
        if rc == N.UNSUPPORTED_D:
            raise UnsupportedDimensionError(msg)
        raise DeviceError(f"status {rc}: {msg}")


_default_ctx: dict = {}
_default_lock = threading.Lock()


def nccl_unique_id() -> bytes:
    lib = N.load()
    buf = ctypes.create_string_buffer(128)
    rc = lib.fkde_gpu_nccl_unique_id(buf)
    if rc != N.OK:
        raise DeviceError(f"fkde_gpu_nccl_unique_id -> {rc}")
    return buf.raw


def device_count() -> int:
    c = ctypes.c_int(0)
    N.load().fkde_gpu_device_count(ctypes.byref(c))
    return int(c.value)


def default_context(threads: int = 0) -> Context:
    """Process-wide context: threads <= 1 -> device 0; k > 1 -> devices
    0..min(k, visible devices)-1.  The reference accepts any worker count
    (parallel.cpp:12-24); here it is capped by the GPUs present, like the CLI."""
    k = max(1, min(int(threads), device_count()))
    with _default_lock:
        if k not in _default_ctx:
            _default_ctx[k] = Context(list(range(k)))
        return _default_ctx[k]


def _ctx(opts: Optional[EngineOptions], ctx: Optional[Context]) -> Context:
    if ctx is not None:
        return ctx
    return default_context(opts.threads if opts else 0)


def _check_pair(train: SampleSet, queries: SampleSet):
    # engine.cpp:27-34
    train.validate()
    queries.validate()
    if train.d != queries.d:
        raise DimensionMismatchError(f"engine: train.d={train.d} != queries.d={queries.d}")


# ---- engine.hpp:46-49 ----------------------------------------------------------------
def pairwise_sq_dists_block(a, b, *, ctx: Optional[Context] = None) -> SampleSet:
    a, b = SampleSet.wrap(a), SampleSet.wrap(b)
    _check_pair(a, b)
    c = _ctx(None, ctx)
    out = np.empty((a.n, b.n), dtype=np.float64)
    with c.lock:
        rc = c._lib.fkde_gpu_pairwise_sq_dists(c.handle, _ptr(a.values), a.n, _ptr(b.values), b.n,
                                               a.d, _ptr(out))
        c.check(rc)
    s = SampleSet.zeros(a.n, b.n)
    s.values = out
    return s


# ---- engine.hpp:58-59 ----------------------------------------------------------------
def score_accumulate(train, h_score: float, plan: TilePlan = None,
                     opts: EngineOptions = None, *, ctx: Optional[Context] = None
                     ) -> ScoreAccumulator:
    train = SampleSet.wrap(train)
    train.validate()
    Bandwidth(h_score, h_score).validate()
    TilePlan.make(train.n, train.n, (plan or TilePlan()).tile_m, (plan or TilePlan()).tile_n)
    c = _ctx(opts, ctx)
    phi = np.empty(train.n, dtype=np.float64)
    w = np.empty((train.n, train.d), dtype=np.float64)
    with c.lock:
        rc = c._lib.fkde_gpu_score_accumulate(c.handle, _ptr(train.values), train.n, train.d,
                                              float(h_score), _ptr(phi), _ptr(w))
        c.check(rc)
    ws = SampleSet.zeros(train.n, train.d)
    ws.values = w
    return ScoreAccumulator(phi, ws)


# ---- engine.hpp:63-64 ----------------------------------------------------------------
def score_flash(train, h_score: float, plan: TilePlan = None, opts: EngineOptions = None, *,
                ctx: Optional[Context] = None) -> SampleSet:
    train = SampleSet.wrap(train)
    train.validate()
    Bandwidth(h_score, h_score).validate()
    TilePlan.make(train.n, train.n, (plan or TilePlan()).tile_m, (plan or TilePlan()).tile_n)
    c = _ctx(opts, ctx)
    out = np.empty((train.n, train.d), dtype=np.float64)
    idx = ctypes.c_size_t(0)
    with c.lock:
        rc = c._lib.fkde_gpu_score(c.handle, _ptr(train.values), train.n, train.d,
                                   float(h_score), _ptr(out), ctypes.byref(idx))
        c.check(rc, idx.value)
    s = SampleSet.zeros(train.n, train.d)
    s.values = out
    return s


# ---- engine.hpp:70-72 ----------------------------------------------------------------
def kde_flash(train, queries, h: float, kernel: KernelKind = KernelKind.Gaussian,
              fused: bool = True, plan: TilePlan = None, opts: EngineOptions = None, *,
              ctx: Optional[Context] = None) -> DensityResult:
    train, queries = SampleSet.wrap(train), SampleSet.wrap(queries)
    _check_pair(train, queries)
    Bandwidth(h, h).validate()
    p = plan or TilePlan()
    TilePlan.make(queries.n, train.n, p.tile_m, p.tile_n)
    c = _ctx(opts, ctx)
    out = np.empty(queries.n, dtype=np.float64)
    kk = N.KERNEL_GAUSSIAN if kernel == KernelKind.Gaussian else N.KERNEL_LAPLACE_CORRECTED
    with c.lock:
        rc = c._lib.fkde_gpu_kde(c.handle, _ptr(train.values), train.n, _ptr(queries.values),
                                 queries.n, train.d, float(h), kk, 1 if fused else 0, _ptr(out))
        c.check(rc)
    return DensityResult(out)


# ---- engine.hpp:74-76 ----------------------------------------------------------------
def sdkde_flash(train, queries, bw: Bandwidth, plan: TilePlan = None,
                opts: EngineOptions = None, *, ctx: Optional[Context] = None,
                want_debiased: bool = True) -> DensityResult:
    train, queries = SampleSet.wrap(train), SampleSet.wrap(queries)
    _check_pair(train, queries)
    bw.validate()
    p = plan or TilePlan()
    TilePlan.make(queries.n, train.n, p.tile_m, p.tile_n)
    c = _ctx(opts, ctx)
    out = np.empty(queries.n, dtype=np.float64)
    deb = np.empty((train.n, train.d), dtype=np.float64) if want_debiased else None
    idx = ctypes.c_size_t(0)
    with c.lock:
        rc = c._lib.fkde_gpu_sdkde(c.handle, _ptr(train.values), train.n, _ptr(queries.values),
                                   queries.n, train.d, float(bw.h), float(bw.h_score), _ptr(out),
                                   _ptr(deb) if deb is not None else None, ctypes.byref(idx))
        c.check(rc, idx.value)
    res = DensityResult(out)
    if deb is not None:
        ds = SampleSet.zeros(train.n, train.d)
        ds.values = deb
        res.debiased_samples = ds
    return res
