"""The engine's multi-rank C++ path on one B200: NCCL is replaced (FKDE_NCCL_LIB)
by an in-process emulator (tests/cpp/nccl_emu.cpp) whose ranks share the device,
so the row-sharded score pass, the x^SD allgather layout, the query shards and
the density gather all run for real.  At a fixed column-split count every output
must be bitwise identical to the single-device engine, for the single-process
multi-device context and for one context per rank driven from threads (the
torchrun form bench.py uses)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

EMU_SRC = os.path.join(ROOT, "tests", "cpp", "nccl_emu.cpp")


@pytest.fixture(scope="module")
def emu_lib(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("emu") / "libnccl_emu.so")
    cmd = ["g++", "-std=c++17", "-O2", "-shared", "-fPIC", "-I/usr/local/cuda/include", EMU_SRC,
           "-L/usr/local/cuda/lib64/stubs", "-lcuda", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_emulator_builds(emu_lib):
    assert os.path.exists(emu_lib)


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,world,splits", [(1000, 300, 2, 2), (2049, 129, 3, 3), (4096, 4096, 4, 2)])
def test_multirank_path_is_bitwise_single_device(emu_lib, n, m, world, splits):
    env = dict(os.environ, FKDE_NCCL_LIB=emu_lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "multirank_emu_check.py"),
                        str(n), str(m), str(world), str(splits)],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    print(res)
    assert "per_rank_error" not in res, res
    assert "device_api_error" not in res, res
    assert all(v == 0.0 for v in res["device_api"]), res
    for form in [res["multi_device"]] + res["per_rank"]:
        for k, v in form.items():
            assert v == 0.0, (k, v, res)


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,world,splits", [(5000, 1000, 2, 2), (9000, 777, 3, 3)])
def test_multirank_spatial_order(emu_lib, n, m, world, splits):
    # the spatial order with tile skipping, multi-rank: the score pass's row shards
    # start on tile boundaries of the same sorted order, so scores and debiased
    # samples are bitwise the single-device ones; query shards are not tile
    # aligned, so the density pass's skip decisions (per query tile) differ from
    # the single-device run by at most the 2^-24 relative skip guarantee
    env = dict(os.environ, FKDE_NCCL_LIB=emu_lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "multirank_emu_check.py"),
                        str(n), str(m), str(world), str(splits), "1"],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    print(res)
    assert "per_rank_error" not in res and "device_api_error" not in res, res
    for form in [res["multi_device"]] + res["per_rank"]:
        assert form["score"] == 0.0 and form["debiased"] == 0.0, form
        for k in ("sdkde", "kde", "laplace"):
            assert form[k] <= 1e-6 * res["scale"][k], (k, form, res)
    assert all(v <= 1e-6 * res["scale"]["sdkde"] for v in res["device_api"]), res
