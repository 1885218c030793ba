"""ctypes binding of the C ABI (include/fkde_gpu.h) in libfkde_b200.so.

The shared library is built in-tree (``python -m paper_2602_10378_b200.build``
or ``__graft_entry__.build()``).  There is no fallback: if the library is
missing or cannot load, importing the engine raises ImportError.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FKDE_B200_LIB overrides the library path (A/B timing of two in-tree builds)
LIB_PATH = os.environ.get("FKDE_B200_LIB") or os.path.join(HERE, "libfkde_b200.so")

# fkde_status
OK = 0
INVALID_ARGUMENT = 1
DIMENSION_MISMATCH = 2
SCORE_UNDERFLOW = 3
NON_FINITE = 4
CUDA_ERROR = 5
NCCL_ERROR = 6
UNSUPPORTED_D = 7
NO_DEVICE = 8

KERNEL_GAUSSIAN = 0
KERNEL_LAPLACE_CORRECTED = 1
METHOD_KDE, METHOD_SDKDE, METHOD_LAPLACE = 0, 1, 2

OPT_ENGINE, OPT_SPLITS, OPT_TIMING, OPT_MAX_CTAS, OPT_FLUSH_TILES = 1, 2, 3, 4, 5
OPT_SPATIAL = 7
SKIP_STATS_COUNT = 9   # FKDE_SKIP_STATS_COUNT
OPT_PDL = 8
ENGINE_TC = 0

T_PREP, T_SCORE, T_FINALIZE, T_GATHER, T_QUERY, T_REDUCE, T_TOTAL, T_COUNT = range(8)
KT_SCORE, KT_CHECK, KT_DENSITY, KT_COUNT = range(4)   # FKDE_KT_*

EXPORTED_SYMBOLS = (
    "fkde_gpu_device_count", "fkde_gpu_create", "fkde_gpu_nccl_unique_id",
    "fkde_gpu_create_rank", "fkde_gpu_destroy", "fkde_gpu_last_error", "fkde_gpu_set_option",
    "fkde_gpu_world", "fkde_gpu_stream", "fkde_gpu_last_timing", "fkde_gpu_last_kernel_timing",
    "fkde_gpu_last_launch_count",
    "fkde_gpu_score", "fkde_gpu_score_accumulate", "fkde_gpu_kde", "fkde_gpu_sdkde",
    "fkde_gpu_estimate", "fkde_gpu_pairwise_sq_dists", "fkde_gpu_sdkde_device",
    "fkde_gpu_kde_device", "fkde_gpu_score_device", "fkde_gpu_shard_range",
    "fkde_gpu_workspace_bytes", "fkde_gpu_last_skip_stats",
)
HOST_SYMBOLS = (
    "fkde_host_mix64", "fkde_host_random_gaussian", "fkde_host_sample_mixture",
    "fkde_host_mean_stddev", "fkde_host_silverman_prefactor", "fkde_host_silverman_bandwidth",
    "fkde_host_sdkde_bandwidth",
)

IO_SYMBOLS = (
    "fkde_io_read_samples", "fkde_io_free", "fkde_io_alloc", "fkde_io_write_samples_bin",
    "fkde_io_write_samples_csv", "fkde_io_write_values", "fkde_io_read_values",
    "fkde_io_last_error",
)
# fkde_io_status
IO_OK, IO_ERROR, IO_INVALID_ARGUMENT = 0, 1, 2

_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_sz = ctypes.c_size_t
_szp = ctypes.POINTER(ctypes.c_size_t)
_vp = ctypes.c_void_p


def _declare(lib):
    lib.fkde_gpu_device_count.argtypes = [ctypes.POINTER(ctypes.c_int)]
    lib.fkde_gpu_create.argtypes = [ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                    ctypes.POINTER(_vp)]
    lib.fkde_gpu_nccl_unique_id.argtypes = [ctypes.c_char_p]
    lib.fkde_gpu_create_rank.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_char_p, ctypes.POINTER(_vp)]
    lib.fkde_gpu_destroy.argtypes = [_vp]
    lib.fkde_gpu_destroy.restype = None
    lib.fkde_gpu_last_error.argtypes = [_vp]
    lib.fkde_gpu_last_error.restype = ctypes.c_char_p
    lib.fkde_gpu_set_option.argtypes = [_vp, ctypes.c_int, ctypes.c_int64]
    lib.fkde_gpu_world.argtypes = [_vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
    lib.fkde_gpu_stream.argtypes = [_vp]
    lib.fkde_gpu_stream.restype = _vp
    lib.fkde_gpu_last_timing.argtypes = [_vp, ctypes.POINTER(ctypes.c_float), ctypes.c_int]
    lib.fkde_gpu_last_kernel_timing.argtypes = [_vp, ctypes.POINTER(ctypes.c_float), ctypes.c_int]
    lib.fkde_gpu_last_launch_count.argtypes = [_vp]
    lib.fkde_gpu_last_launch_count.restype = ctypes.c_int64
    lib.fkde_gpu_workspace_bytes.argtypes = [_vp, _szp]
    lib.fkde_gpu_last_skip_stats.argtypes = [_vp, ctypes.POINTER(ctypes.c_uint64), ctypes.c_size_t]
    lib.fkde_gpu_score.argtypes = [_vp, _dp, _sz, _sz, ctypes.c_double, _dp, _szp]
    lib.fkde_gpu_score_accumulate.argtypes = [_vp, _dp, _sz, _sz, ctypes.c_double, _dp, _dp]
    lib.fkde_gpu_kde.argtypes = [_vp, _dp, _sz, _dp, _sz, _sz, ctypes.c_double, ctypes.c_int,
                                 ctypes.c_int, _dp]
    lib.fkde_gpu_sdkde.argtypes = [_vp, _dp, _sz, _dp, _sz, _sz, ctypes.c_double, ctypes.c_double,
                                   _dp, _dp, _szp]
    lib.fkde_gpu_estimate.argtypes = [_vp, _dp, _sz, _dp, _sz, _sz, ctypes.c_int, ctypes.c_double,
                                      ctypes.c_double, _sz, _sz, ctypes.c_int, _dp, _dp, _dp, _szp]
    lib.fkde_gpu_pairwise_sq_dists.argtypes = [_vp, _dp, _sz, _dp, _sz, _sz, _dp]
    lib.fkde_gpu_sdkde_device.argtypes = [_vp, _vp, _sz, _vp, _sz, _sz, ctypes.c_double,
                                          ctypes.c_double, _vp]
    lib.fkde_gpu_score_device.argtypes = [_vp, _vp, _sz, _sz, ctypes.c_double, _vp]
    lib.fkde_gpu_kde_device.argtypes = [_vp, _vp, _sz, _vp, _sz, _sz, ctypes.c_double,
                                        ctypes.c_int, ctypes.c_int, _vp]
    lib.fkde_gpu_shard_range.argtypes = [_sz, ctypes.c_int, ctypes.c_int, _sz, _szp, _szp, _szp]
    lib.fkde_host_mix64.argtypes = [ctypes.c_uint64]
    lib.fkde_host_mix64.restype = ctypes.c_uint64
    lib.fkde_host_random_gaussian.argtypes = [_sz, _sz, ctypes.c_uint64, ctypes.c_double, _dp]
    lib.fkde_host_random_gaussian.restype = None
    lib.fkde_host_sample_mixture.argtypes = [_dp, _dp, _dp, _sz, _sz, _sz, ctypes.c_uint64, _dp]
    for f in ("fkde_host_mean_stddev", "fkde_host_silverman_bandwidth"):
        getattr(lib, f).argtypes = [_dp, _sz, _sz]
        getattr(lib, f).restype = ctypes.c_double
    lib.fkde_host_silverman_prefactor.argtypes = [_sz]
    lib.fkde_host_silverman_prefactor.restype = ctypes.c_double
    lib.fkde_host_sdkde_bandwidth.argtypes = [_dp, _sz, _sz, ctypes.c_double]
    lib.fkde_host_sdkde_bandwidth.restype = ctypes.c_double
    ip = ctypes.POINTER(ctypes.c_int)
    lib.fkde_io_read_samples.argtypes = [ctypes.c_char_p, ctypes.POINTER(_dp), _szp, _szp, ip]
    lib.fkde_io_free.argtypes = [_dp, ctypes.c_int]
    lib.fkde_io_free.restype = None
    lib.fkde_io_alloc.argtypes = [_sz, ip]
    lib.fkde_io_alloc.restype = _dp
    lib.fkde_io_write_samples_bin.argtypes = [ctypes.c_char_p, _dp, _sz, _sz]
    lib.fkde_io_write_samples_csv.argtypes = [ctypes.c_char_p, _dp, _sz, _sz]
    lib.fkde_io_write_values.argtypes = [ctypes.c_char_p, _dp, _sz, ctypes.c_char_p]
    lib.fkde_io_read_values.argtypes = [ctypes.c_char_p, ctypes.POINTER(_dp), _szp]
    lib.fkde_io_last_error.argtypes = []
    lib.fkde_io_last_error.restype = ctypes.c_char_p
    return lib


def shard_range(n: int, world: int, rank: int, align: int = 1):
    """(begin, rows, chunk) of rank's slice -- the engine's own partition."""
    lib = load()
    b, r, c = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
    rc = lib.fkde_gpu_shard_range(n, world, rank, align, ctypes.byref(b), ctypes.byref(r),
                                  ctypes.byref(c))
    if rc != OK:
        raise ValueError(f"fkde_gpu_shard_range({n}, {world}, {rank}, {align}) -> {rc}")
    return b.value, r.value, c.value


def load():
    """Load libfkde_b200.so (raises ImportError loudly if absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not found: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')")
        _lib = _declare(ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL))
    return _lib


def loaded_path() -> str:
    return LIB_PATH
