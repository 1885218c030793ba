"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every
entry point include/fkde_gpu.h declares, and the host mirror validates
exactly like the reference (types.cpp:21-33, 65-79; engine.cpp:27-34,
248-259) before touching a device.  No compute calls here."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

import paper_2602_10378_b200 as fk
from paper_2602_10378_b200 import _native as N


def header_symbols(name="fkde_gpu.h"):
    src = open(os.path.join(ROOT, "include", name)).read()
    return sorted(set(re.findall(r"\b(fkde_(?:gpu|host|io)_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = N.load()
    syms = header_symbols()
    assert len(syms) >= 19
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(N.EXPORTED_SYMBOLS) | set(N.HOST_SYMBOLS)


def test_library_exports_every_io_symbol():
    lib = N.load()
    syms = header_symbols("fkde_io.h")
    assert set(syms) == set(N.IO_SYMBOLS)
    for s in syms:
        assert hasattr(lib, s), s


def test_every_header_is_covered():
    # every include/*.h entry point is in one of the checked symbol lists
    listed = set(N.EXPORTED_SYMBOLS) | set(N.HOST_SYMBOLS) | set(N.IO_SYMBOLS)
    for name in os.listdir(os.path.join(ROOT, "include")):
        if name.endswith(".h"):
            assert set(header_symbols(name)) <= listed, name


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_library_has_tcgen05_and_bulk_copy_sass():
    out = subprocess.run(["cuobjdump", "-sass", N.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    sass = out.stdout
    for mnem in ("UTCHMMA", "LDTM", "UBLKCP", "MUFU.EX2"):
        assert mnem in sass, mnem
    assert "HMMA" not in sass.replace("UTCHMMA", "")  # no legacy mma.sync path


def test_shard_range_partition():
    for n in (1, 7, 128, 1000, 1 << 20):
        for world in (1, 2, 3, 8):
            for align in (1, 128):
                covered = 0
                chunks = set()
                for r in range(world):
                    b, rows, chunk = N.shard_range(n, world, r, align)
                    chunks.add(chunk)
                    assert b == min(n, r * chunk) and rows <= chunk
                    assert b == covered or rows == 0
                    covered += rows
                    if align > 1:
                        assert chunk % align == 0
                assert covered == n and len(chunks) == 1


def test_no_device_fails_loudly():
    c = ctypes.c_int(0)
    N.load().fkde_gpu_device_count(ctypes.byref(c))
    if c.value > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(fk.DeviceError):
        fk.Context([0])


# ---- host validation mirrors the reference (no device needed) ---------------------
def test_sampleset_validation():
    with pytest.raises(fk.InvalidArgumentError):
        fk.SampleSet(np.zeros((0, 2)))
    with pytest.raises(fk.InvalidArgumentError):
        fk.SampleSet([1.0, np.nan])
    with pytest.raises(fk.InvalidArgumentError):
        fk.SampleSet([1.0, 2.0, 3.0], 2, 2)
    s = fk.SampleSet([0.0, 0.0, 3.0, 4.0], 2, 2)
    assert s.n == 2 and s.d == 2


def test_tileplan_ceiling_counts():
    p = fk.TilePlan.make(100, 5000, 64, 1024)
    assert (p.n_tiles_m, p.n_tiles_n) == (2, 5)
    with pytest.raises(fk.InvalidArgumentError):
        fk.TilePlan.make(10, 10, 0, 4)


def test_bandwidth_validation():
    with pytest.raises(fk.InvalidArgumentError):
        fk.Bandwidth(-1.0, 1.0).validate()
    with pytest.raises(fk.InvalidArgumentError):
        fk.Bandwidth(1.0, float("inf")).validate()
    b = fk.Bandwidth.half_variance_score(2.0)
    assert b.h == 2.0 and abs(b.h_score - 2.0 / 2 ** 0.5) < 1e-15


def test_engine_validation_before_device():
    tr = np.random.default_rng(0).normal(size=(10, 2))
    q = np.random.default_rng(1).normal(size=(10, 3))
    with pytest.raises(fk.DimensionMismatchError):
        fk.kde_flash(tr, q, 1.0)
    with pytest.raises(fk.InvalidArgumentError):
        fk.score_flash(tr, 0.0)
    with pytest.raises(fk.InvalidArgumentError):
        fk.sdkde_flash(tr, tr, fk.Bandwidth(1.0, -1.0))
    cfg = fk.EstimatorConfig(method=fk.Method.Kde, bandwidth=fk.Bandwidth(-1.0, 1.0))
    with pytest.raises(fk.InvalidArgumentError):
        fk.estimate(tr, tr, cfg)
    cfg = fk.EstimatorConfig(method=fk.Method.Kde, bandwidth=fk.Bandwidth.uniform(0.5), tile_m=0)
    with pytest.raises(fk.InvalidArgumentError):
        fk.estimate(tr, tr, cfg)
    cfg = fk.EstimatorConfig(engine=fk.EngineKind.Naive, bandwidth=fk.Bandwidth.uniform(0.5))
    with pytest.raises(fk.InvalidArgumentError):
        fk.estimate(tr, tr, cfg)


def test_enum_strings():
    assert fk.method_from_string("sdkde") == fk.Method.Sdkde
    assert fk.engine_from_string("flash") == fk.EngineKind.Flash
    with pytest.raises(fk.InvalidArgumentError):
        fk.method_from_string("nope")


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2602_10378_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "liboracle" not in src, f
                assert "fkde_oracle" not in src and "libfkde_ref" not in src, f


def test_host_fixtures_match_reference_rng(port):
    # the product's input generators reproduce the reference's RNG bitwise
    from paper_2602_10378_b200 import fixtures as F
    assert F.mix64(12345) == port.mix64(12345)
    assert np.array_equal(F.random_gaussian(100, 3, 41, 1.5), port.random_gaussian(100, 3, 41, 1.5))
    w, mu, s = F.mixture_16d()
    seed = F.cell_data_seed(0, 4096)
    a = F.sample_mixture(w, mu, s, 500, seed)
    assert np.array_equal(a, port.sample_mixture(w, mu, s, 500, seed))
    assert F.sdkde_bandwidth(a) == port.sdkde_bandwidth(a, port.silverman_prefactor(16))
    assert F.silverman_bandwidth(a) == port.silverman_bandwidth(a)
    tr, q = F.runtime_sweep_inputs(4096, 64)
    from conftest import golden
    c = golden("config1")
    assert np.array_equal(tr[:8], c["train_head"]) and np.array_equal(q[:8], c["query_head"])
