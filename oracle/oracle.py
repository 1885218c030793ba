"""TEST INFRASTRUCTURE ONLY -- numpy/ctypes binding of the CPU oracle.

Two interchangeable back ends with the same function set:

* ``Oracle("port")``  -> ``oracle/liboracle.so``: the plain-C restatement of the
  reference oracle (``fkde_oracle.c``; reference oracle.cpp:36-118).
* ``Oracle("reference")`` -> ``oracle/_ref/libfkde_ref.so``: the reference's own
  ``fkde::oracle`` compiled from /root/reference (``oracle/Makefile ref``).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` leg may import this module.  The product package never
does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfkde_ref.so")

_c_double_p = ctypes.POINTER(ctypes.c_double)
_size_t = ctypes.c_size_t


class OracleError(RuntimeError):
    def __init__(self, status: int, index: int | None = None):
        self.status = status
        self.index = index
        names = {1: "invalid argument", 2: "dimension mismatch", 3: "score underflow"}
        super().__init__(f"oracle status {status} ({names.get(status, 'error')}), index={index}")


def build(ref: bool = False) -> None:
    """Compile the C restatement (and, when /root/reference exists, _ref)."""
    targets = ["all"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_c_double_p)


def _as2d(x) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return a


class Oracle:
    def __init__(self, kind: str = "port"):
        if kind not in ("port", "reference"):
            raise ValueError(kind)
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            if kind == "port":
                build(ref=False)
            else:
                raise FileNotFoundError(f"{path} (build with `make -C oracle ref`)")
        self.kind = kind
        self.path = path
        self.lib = ctypes.CDLL(path)
        p = "fko_" if kind == "port" else "fkr_"
        self._p = p
        L = self.lib
        self._mix64 = getattr(L, p + "mix64")
        self._mix64.restype = ctypes.c_uint64
        self._mix64.argtypes = [ctypes.c_uint64]
        self._rg = getattr(L, p + "random_gaussian")
        self._rg.restype = None
        self._rg.argtypes = [_size_t, _size_t, ctypes.c_uint64, ctypes.c_double, _c_double_p]
        self._u01 = getattr(L, p + "uniform01")
        self._u01.restype = None
        self._u01.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _size_t, _c_double_p]
        self._mix = getattr(L, p + "sample_mixture")
        self._mix.argtypes = [_c_double_p, _c_double_p, _c_double_p, _size_t, _size_t, _size_t,
                              ctypes.c_uint64, _c_double_p]
        for name in ("gaussian_norm_const",):
            f = getattr(L, p + name)
            f.restype = ctypes.c_double
            f.argtypes = [ctypes.c_double, _size_t]
        for name in ("gaussian_kernel", "laplace_corrected_kernel"):
            f = getattr(L, p + name)
            f.restype = ctypes.c_double
            f.argtypes = [ctypes.c_double, ctypes.c_double, _size_t]
        f = getattr(L, p + "mean_stddev")
        f.restype = ctypes.c_double
        f.argtypes = [_c_double_p, _size_t, _size_t]
        f = getattr(L, p + "silverman_prefactor")
        f.restype = ctypes.c_double
        f.argtypes = [_size_t]
        f = getattr(L, p + "silverman_bandwidth")
        f.restype = ctypes.c_double
        f.argtypes = [_c_double_p, _size_t, _size_t]
        f = getattr(L, p + "sdkde_bandwidth")
        f.restype = ctypes.c_double
        f.argtypes = [_c_double_p, _size_t, _size_t, ctypes.c_double]
        for name in ("kde_naive", "laplace_naive"):
            f = getattr(L, p + name)
            f.restype = ctypes.c_int
            f.argtypes = [_c_double_p, _size_t, _c_double_p, _size_t, _size_t, ctypes.c_double,
                          _size_t, _size_t, ctypes.c_int, _c_double_p]
        f = getattr(L, p + "score_naive")
        f.restype = ctypes.c_int
        f.argtypes = [_c_double_p, _size_t, _c_double_p, _size_t, _size_t, ctypes.c_double,
                      _size_t, _size_t, ctypes.c_int, _c_double_p, ctypes.POINTER(_size_t)]

    # -- fixtures ----------------------------------------------------------
    def mix64(self, x: int) -> int:
        return int(self._mix64(ctypes.c_uint64(x & 0xFFFFFFFFFFFFFFFF)))

    def random_gaussian(self, n: int, d: int, seed: int, scale: float = 1.0) -> np.ndarray:
        out = np.empty((n, d), dtype=np.float64)
        self._rg(n, d, seed, scale, _ptr(out))
        return out

    def uniform01(self, seed: int, count: int, stream: int = 0) -> np.ndarray:
        out = np.empty(count, dtype=np.float64)
        self._u01(seed, stream, count, _ptr(out))
        return out

    def sample_mixture(self, weights, means, sigmas, n: int, seed: int) -> np.ndarray:
        w = np.ascontiguousarray(weights, dtype=np.float64)
        mu = _as2d(means)
        s = np.ascontiguousarray(sigmas, dtype=np.float64)
        k, d = mu.shape
        out = np.empty((n, d), dtype=np.float64)
        st = self._mix(_ptr(w), _ptr(mu), _ptr(s), k, d, n, seed, _ptr(out))
        if st:
            raise OracleError(st)
        return out

    # -- scalar kernels ----------------------------------------------------
    def gaussian_norm_const(self, h, d):
        return getattr(self.lib, self._p + "gaussian_norm_const")(h, d)

    def gaussian_kernel(self, r2, h, d):
        return getattr(self.lib, self._p + "gaussian_kernel")(r2, h, d)

    def laplace_corrected_kernel(self, r2, h, d):
        return getattr(self.lib, self._p + "laplace_corrected_kernel")(r2, h, d)

    # -- bandwidth rules ---------------------------------------------------
    def mean_stddev(self, x):
        a = _as2d(x)
        return getattr(self.lib, self._p + "mean_stddev")(_ptr(a), a.shape[0], a.shape[1])

    def silverman_prefactor(self, d):
        return getattr(self.lib, self._p + "silverman_prefactor")(d)

    def silverman_bandwidth(self, x):
        a = _as2d(x)
        return getattr(self.lib, self._p + "silverman_bandwidth")(_ptr(a), a.shape[0], a.shape[1])

    def sdkde_bandwidth(self, x, c):
        a = _as2d(x)
        return getattr(self.lib, self._p + "sdkde_bandwidth")(_ptr(a), a.shape[0], a.shape[1], c)

    # -- naive estimators --------------------------------------------------
    def _rows(self, m, rows):
        if rows is None:
            return 0, m
        return int(rows[0]), int(rows[1])

    def kde_naive(self, train, queries, h, rows=None, threads=1) -> np.ndarray:
        t, q = _as2d(train), _as2d(queries)
        b, e = self._rows(q.shape[0], rows)
        out = np.empty(e - b, dtype=np.float64)
        st = getattr(self.lib, self._p + "kde_naive")(_ptr(t), t.shape[0], _ptr(q), q.shape[0],
                                                      t.shape[1], h, b, e, threads, _ptr(out))
        if st:
            raise OracleError(st)
        return out

    def laplace_naive(self, train, queries, h, rows=None, threads=1) -> np.ndarray:
        t, q = _as2d(train), _as2d(queries)
        b, e = self._rows(q.shape[0], rows)
        out = np.empty(e - b, dtype=np.float64)
        st = getattr(self.lib, self._p + "laplace_naive")(_ptr(t), t.shape[0], _ptr(q),
                                                          q.shape[0], t.shape[1], h, b, e,
                                                          threads, _ptr(out))
        if st:
            raise OracleError(st)
        return out

    def score_naive(self, train, eval_points, h_score, rows=None, threads=1) -> np.ndarray:
        t, q = _as2d(train), _as2d(eval_points)
        b, e = self._rows(q.shape[0], rows)
        out = np.empty((e - b, t.shape[1]), dtype=np.float64)
        idx = _size_t(0)
        st = getattr(self.lib, self._p + "score_naive")(_ptr(t), t.shape[0], _ptr(q), q.shape[0],
                                                        t.shape[1], h_score, b, e, threads,
                                                        _ptr(out), ctypes.byref(idx))
        if st:
            raise OracleError(st, int(idx.value) if st == 3 else None)
        return out

    def sdkde_naive(self, train, queries, h, h_score=None, threads=1):
        """Returns (densities, debiased_samples) -- oracle.cpp:87-101."""
        h_score = h if h_score is None else h_score
        t = _as2d(train)
        scores = self.score_naive(t, t, h_score, threads=threads)
        debiased = t + (0.5 * h * h) * scores
        return self.kde_naive(debiased, queries, h, threads=threads), debiased


_cache: dict[str, Oracle] = {}


def get(kind: str = "port") -> Oracle:
    if kind not in _cache:
        _cache[kind] = Oracle(kind)
    return _cache[kind]


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def default_mixture_16d():
    """The reference's configs/mixture-16d-default.json (data file shipped with the package)."""
    import json
    path = os.path.join(os.path.dirname(HERE), "paper_2602_10378_b200", "configs",
                        "mixture-16d-default.json")
    with open(path) as f:
        j = json.load(f)
    return (np.asarray(j["weights"], dtype=np.float64), np.asarray(j["means"], dtype=np.float64),
            np.asarray(j["sigmas"], dtype=np.float64))
