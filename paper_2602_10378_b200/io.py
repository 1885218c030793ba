"""Sample / value files (include/fkde_io.h over ctypes) -- the Python mirror of
the reference's fkde::io (proj/core/include/fkde/io.hpp:11-38): same names,
same formats, IoError / InvalidArgumentError on the same conditions.

    read_samples(path, pinned=False) -> SampleSet     io.cpp:177-190
    write_samples_bin / write_samples_csv(s, path)    io.cpp:55-74, 106-127
    write_values(values, path, format) / read_values  io.cpp:192-258
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .types import InvalidArgumentError, IoError, SampleSet

_dp = ctypes.POINTER(ctypes.c_double)

__all__ = ["IoError", "read_samples", "write_samples_bin", "write_samples_csv", "write_values",
           "read_values"]


def _check(rc: int) -> None:
    if rc == N.IO_OK:
        return
    msg = N.load().fkde_io_last_error().decode()
    if rc == N.IO_INVALID_ARGUMENT:
        raise InvalidArgumentError(msg)
    raise IoError(msg)


def _arr(values) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(values, dtype=np.float64))


def read_samples(path: str, pinned: bool = False) -> SampleSet:
    """FKDE binary (by magic) or CSV.  pinned=True reads into page-locked host
    memory (needs a CUDA driver; silently ordinary memory without one) -- the
    returned SampleSet owns a copy either way."""
    lib = N.load()
    out = _dp()
    n, d = ctypes.c_size_t(), ctypes.c_size_t()
    pin = ctypes.c_int(1 if pinned else 0)
    _check(lib.fkde_io_read_samples(str(path).encode(), ctypes.byref(out), ctypes.byref(n),
                                    ctypes.byref(d), ctypes.byref(pin)))
    try:
        vals = np.ctypeslib.as_array(out, shape=(n.value * d.value,)).copy()
    finally:
        lib.fkde_io_free(out, pin.value)
    return SampleSet(vals.reshape(n.value, d.value))


def write_samples_bin(s, path: str) -> None:
    v = _arr(s.values if isinstance(s, SampleSet) else s)
    v2 = v.reshape(v.shape[0], -1) if v.ndim > 1 else v.reshape(-1, 1)
    _check(N.load().fkde_io_write_samples_bin(str(path).encode(), v2.ctypes.data_as(_dp),
                                              v2.shape[0], v2.shape[1]))


def write_samples_csv(s, path: str) -> None:
    v = _arr(s.values if isinstance(s, SampleSet) else s)
    v2 = v.reshape(v.shape[0], -1) if v.ndim > 1 else v.reshape(-1, 1)
    _check(N.load().fkde_io_write_samples_csv(str(path).encode(), v2.ctypes.data_as(_dp),
                                              v2.shape[0], v2.shape[1]))


def write_values(values, path: str, fmt: str) -> None:
    v = _arr(values).ravel()
    _check(N.load().fkde_io_write_values(str(path).encode(), v.ctypes.data_as(_dp), v.size,
                                         fmt.encode()))


def read_values(path: str) -> np.ndarray:
    lib = N.load()
    out = _dp()
    m = ctypes.c_size_t()
    _check(lib.fkde_io_read_values(str(path).encode(), ctypes.byref(out), ctypes.byref(m)))
    try:
        return np.ctypeslib.as_array(out, shape=(m.value,)).copy()
    finally:
        lib.fkde_io_free(out, 0)
