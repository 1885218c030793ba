"""FKDE sample / value files (include/fkde_io.h, csrc/host_io.cpp) against the
reference's own fkde::io (io.cpp, compiled into oracle/_ref): byte-identical
files in both directions plus the reference's test_io.cpp cases
(proj/tests/test_io.cpp:31-102).  CPU only."""
import ctypes
import os
import struct

import numpy as np
import pytest

import paper_2602_10378_b200 as fk
from paper_2602_10378_b200 import io as fio

_dp = ctypes.POINTER(ctypes.c_double)
_sz = ctypes.c_size_t


@pytest.fixture(scope="module")
def reflib(ref):
    L = ref.lib
    for f in ("fkr_write_samples_bin", "fkr_write_samples_csv"):
        getattr(L, f).argtypes = [ctypes.c_char_p, _dp, _sz, _sz]
    L.fkr_write_values.argtypes = [ctypes.c_char_p, _dp, _sz, ctypes.c_char_p]
    L.fkr_read_samples.argtypes = [ctypes.c_char_p, _dp, _sz, ctypes.POINTER(_sz), ctypes.POINTER(_sz)]
    L.fkr_read_values.argtypes = [ctypes.c_char_p, _dp, _sz, ctypes.POINTER(_sz)]
    return L


def _p(a):
    return a.ctypes.data_as(_dp)


def ref_read_samples(L, path):
    n, d = _sz(), _sz()
    assert L.fkr_read_samples(path.encode(), None, 0, ctypes.byref(n), ctypes.byref(d)) == 0
    out = np.empty(n.value * d.value)
    assert L.fkr_read_samples(path.encode(), _p(out), out.size, ctypes.byref(n), ctypes.byref(d)) == 0
    return out.reshape(n.value, d.value)


def ref_read_values(L, path):
    m = _sz()
    assert L.fkr_read_values(path.encode(), None, 0, ctypes.byref(m)) == 0
    out = np.empty(m.value)
    assert L.fkr_read_values(path.encode(), _p(out), out.size, ctypes.byref(m)) == 0
    return out


def awkward(n=37, d=5, seed=3):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(n, d)) * 10.0 ** rng.integers(-30, 30, size=(n, d))
    special = [0.1, -0.0, 5e-324, 1.7976931348623157e308, 1.0 / 3.0]
    for k, v in enumerate(special[:min(n, d)]):
        x[k, k] = v
    return x


def test_binary_round_trip_is_bitwise(tmp_path):
    x = awkward()
    p = str(tmp_path / "s.bin")
    fio.write_samples_bin(fk.SampleSet(x), p)
    y = fio.read_samples(p).values
    assert y.tobytes() == x.tobytes()
    raw = open(p, "rb").read()
    assert raw[:4] == b"FKDE" and struct.unpack("<IQQ", raw[4:24]) == (1, 37, 5)
    assert len(raw) == 24 + x.size * 8


def test_csv_round_trip_is_exact(tmp_path):
    x = awkward()
    p = str(tmp_path / "s.csv")
    fio.write_samples_csv(x, p)
    assert open(p).readline().strip() == ",".join(f"x{k}" for k in range(5))
    assert fio.read_samples(p).values.tobytes() == x.tobytes()


def test_pinned_read_matches(tmp_path):
    x = awkward()
    p = str(tmp_path / "s.bin")
    fio.write_samples_bin(x, p)
    assert fio.read_samples(p, pinned=True).values.tobytes() == x.tobytes()


def test_sniffs_binary_vs_csv(tmp_path):
    x = awkward(8, 3)
    fio.write_samples_bin(x, str(tmp_path / "a"))
    fio.write_samples_csv(x, str(tmp_path / "b"))
    a, b = fio.read_samples(str(tmp_path / "a")), fio.read_samples(str(tmp_path / "b"))
    assert a.values.tobytes() == b.values.tobytes() == x.tobytes()


@pytest.mark.parametrize("fmt", ["csv", "bin", "json"])
def test_value_formats_round_trip(tmp_path, fmt):
    v = awkward(50, 1).ravel()
    p = str(tmp_path / ("v." + fmt))
    fio.write_values(v, p, fmt)
    assert fio.read_values(p).tobytes() == v.tobytes()


def test_files_are_byte_identical_to_the_reference(tmp_path, reflib):
    x = awkward()
    for kind, ours, theirs in (("bin", fio.write_samples_bin, reflib.fkr_write_samples_bin),
                               ("csv", fio.write_samples_csv, reflib.fkr_write_samples_csv)):
        a, b = str(tmp_path / ("ours." + kind)), str(tmp_path / ("ref." + kind))
        ours(x, a)
        assert theirs(b.encode(), _p(x), x.shape[0], x.shape[1]) == 0
        assert open(a, "rb").read() == open(b, "rb").read(), kind
        # and each side reads the other's file bitwise
        assert ref_read_samples(reflib, a).tobytes() == x.tobytes()
        assert fio.read_samples(b).values.tobytes() == x.tobytes()
    v = np.ascontiguousarray(x[:, 0])
    for fmt in ("csv", "bin"):
        a, b = str(tmp_path / ("vo." + fmt)), str(tmp_path / ("vr." + fmt))
        fio.write_values(v, a, fmt)
        assert reflib.fkr_write_values(b.encode(), _p(v), v.size, fmt.encode()) == 0
        assert open(a, "rb").read() == open(b, "rb").read(), fmt
    # json: both sides serialise with nlohmann::json -> byte-identical, including
    # integral values ("0.0", "-0.0", "3.0"), large/small magnitudes and non-finite
    specials = np.array([0.0, -0.0, 3.0, -7.0, 1e22, 1e-7, 123456789012345678.0, 2.5e-310,
                         np.nan, np.inf])
    for tag, vv in (("v", v), ("s", specials)):
        a, b = str(tmp_path / f"vo_{tag}.json"), str(tmp_path / f"vr_{tag}.json")
        fio.write_values(vv, a, "json")
        assert reflib.fkr_write_values(b.encode(), _p(vv), vv.size, b"json") == 0
        assert open(a, "rb").read() == open(b, "rb").read(), tag
    a, b = str(tmp_path / "vo_v.json"), str(tmp_path / "vr_v.json")
    assert ref_read_values(reflib, a).tobytes() == v.tobytes()
    assert fio.read_values(b).tobytes() == v.tobytes()


def test_io_error_is_the_package_io_error():
    # one exception type: `except fk.IoError` catches what fkde.io raises
    import paper_2602_10378_b200 as fk
    assert fio.IoError is fk.IoError


def test_missing_file_is_io_error(tmp_path):
    with pytest.raises(fio.IoError):
        fio.read_samples(str(tmp_path / "nope.bin"))
    with pytest.raises(fio.IoError):
        fio.read_values(str(tmp_path / "nope.csv"))


def test_bad_header_is_io_error(tmp_path):
    p = str(tmp_path / "v.bin")
    open(p, "wb").write(b"FKDE" + struct.pack("<IQQ", 2, 1, 1) + b"\0" * 8)
    with pytest.raises(fio.IoError, match="version"):
        fio.read_samples(p)
    open(p, "wb").write(b"FKDE" + struct.pack("<IQQ", 1, 0, 1))
    with pytest.raises(fio.IoError, match="implausible"):
        fio.read_samples(p)


def test_truncated_payload_is_io_error(tmp_path):
    p = str(tmp_path / "t.bin")
    fio.write_samples_bin(awkward(10, 2), p)
    raw = open(p, "rb").read()
    open(p, "wb").write(raw[:-8])
    with pytest.raises(fio.IoError, match="truncated"):
        fio.read_samples(p)


def test_ragged_and_non_numeric_csv_are_io_errors(tmp_path):
    p = str(tmp_path / "r.csv")
    open(p, "w").write("x0,x1\n1,2\n3\n")
    with pytest.raises(fio.IoError, match="width"):
        fio.read_samples(p)
    open(p, "w").write("x0,x1\n1,abc\n")
    with pytest.raises(fio.IoError, match="number"):
        fio.read_samples(p)
    open(p, "w").write("x0\n")
    with pytest.raises(fio.IoError, match="no data rows"):
        fio.read_samples(p)


def test_invalid_arguments(tmp_path):
    with pytest.raises(fk.InvalidArgumentError):
        fio.write_values(np.ones(3), str(tmp_path / "v"), "xml")
    with pytest.raises(fk.InvalidArgumentError):
        fio.write_values(np.ones(0), str(tmp_path / "v"), "csv")
    with pytest.raises(fk.InvalidArgumentError):
        fio.write_samples_bin(np.array([[1.0, np.nan]]), str(tmp_path / "s"))
    p = str(tmp_path / "nan.csv")
    open(p, "w").write("x0\nnan\n")
    with pytest.raises(fk.InvalidArgumentError):
        fio.read_samples(p)
