"""Builds and runs the C++ facade test (tests/cpp/test_facade.cpp) against
libfkde_b200.so -- the drop-in C++ API a reference caller would use."""
import os
import subprocess

import pytest

from conftest import ROOT

LIBDIR = os.path.join(ROOT, "paper_2602_10378_b200")
SRC = os.path.join(ROOT, "tests", "cpp", "test_facade.cpp")
REF_INC = "/root/reference/proj/core/include"
REF_TYPES_O = os.path.join(ROOT, "oracle", "_ref", "obj", "types.o")
# prebuilt by __graft_entry__.build() where /root/reference exists (it does not on
# the GPU box): the facade compiled against the reference's own fkde:: types
PREBUILT_REF = os.path.join(ROOT, "tests", "cpp", "bin", "test_facade_ref")


def _build(out, extra=()):
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), *extra, SRC,
           "-L", LIBDIR, "-l:libfkde_b200.so", f"-Wl,-rpath,{LIBDIR}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return out


def test_facade_builds_and_validates_on_host(tmp_path):
    exe = _build(str(tmp_path / "test_facade"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.skipif(not (os.path.isdir(REF_INC) and os.path.exists(REF_TYPES_O)),
                    reason="reference headers / oracle/_ref build not present")
def test_facade_compiles_against_reference_types(tmp_path):
    # drop-in proof: the facade accepts the reference's own fkde::SampleSet etc.
    exe = _build(str(tmp_path / "test_facade_ref"),
                 ["-DFKDE_B200_USE_REFERENCE_TYPES", "-I", REF_INC, REF_TYPES_O])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_facade_runs_engine_on_gpu(tmp_path):
    exe = _build(str(tmp_path / "test_facade"))
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_facade_with_reference_types_runs_engine_on_gpu():
    # the reference's own SampleSet / DensityResult / exceptions driving the GPU
    # engine through the facade (binary built by build() against
    # /root/reference/proj/core/include + the reference's types.cpp)
    assert os.path.exists(PREBUILT_REF), "run __graft_entry__.build() where /root/reference exists"
    r = subprocess.run([PREBUILT_REF, "gpu"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
