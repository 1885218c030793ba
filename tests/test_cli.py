"""fkde-b200, the command-line drop-in for the reference's `fkde` tool
(proj/tools/src/main.cpp), mirroring proj/tests/test_cli.cpp: same
subcommands, flags, outputs and exit codes (0 ok, 1 comparison failure,
2 usage, 3 I/O, 4 numeric).  File outputs of `gen` are checked byte for byte
against the reference's own sampler + writer, `model` against the
reference's perfmodel (oracle/_ref).  Engine runs are @gpu."""
import ctypes
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden, max_component_rel

from paper_2602_10378_b200 import build as B
from paper_2602_10378_b200 import io as fio

CFG = os.path.join(ROOT, "paper_2602_10378_b200", "configs")
MIX1 = os.path.join(CFG, "mixture-1d-default.json")
MIX16 = os.path.join(CFG, "mixture-16d-default.json")
HW = os.path.join(CFG, "hw")


@pytest.fixture(scope="module")
def cli():
    return B.build_cli()


def run(cli, *args, timeout=600):
    r = subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout, r.stderr


def gen(cli, tmp_path, name, mix, n, seed, fmt="bin"):
    p = str(tmp_path / name)
    rc, _, err = run(cli, "gen", "--config", mix, "--n", n, "--seed", seed, "--out", p, "--format", fmt)
    assert rc == 0, err
    return p


# ---------------------------------------------------------------- CPU
def test_gen_round_trips_and_is_deterministic(cli, tmp_path):
    a = gen(cli, tmp_path, "a.bin", MIX1, 100, 7)
    b = gen(cli, tmp_path, "b.bin", MIX1, 100, 7)
    assert open(a, "rb").read() == open(b, "rb").read()
    assert open(a + ".meta.json").read() == open(b + ".meta.json").read()
    s = fio.read_samples(a)
    assert (s.n, s.d) == (100, 1)
    meta = json.load(open(a + ".meta.json"))
    assert meta["n"] == 100 and meta["d"] == 1 and meta["seed"] == 7 and meta["format"] == "bin"
    assert meta["format_version"] == 1 and meta["mixture_hash"].startswith("0x")


def test_gen_matches_reference_sampler_and_hash(cli, tmp_path, ref):
    mix = json.load(open(MIX16))
    p = gen(cli, tmp_path, "g.bin", MIX16, 333, 11)
    x = ref.sample_mixture(mix["weights"], mix["means"], mix["sigmas"], 333, 11)
    L = ref.lib
    L.fkr_write_samples_bin.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double),
                                        ctypes.c_size_t, ctypes.c_size_t]
    q = str(tmp_path / "ref.bin")
    x = np.ascontiguousarray(x)
    assert L.fkr_write_samples_bin(q.encode(), x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                   333, 16) == 0
    assert open(p, "rb").read() == open(q, "rb").read()
    L.fkr_mixture_hash.argtypes = [ctypes.c_char_p]
    L.fkr_mixture_hash.restype = ctypes.c_uint64
    for cfg in (MIX1, MIX16):
        pp = gen(cli, tmp_path, "h.csv", cfg, 5, 1, "csv")
        assert json.load(open(pp + ".meta.json"))["mixture_hash"] == \
            "0x%016x" % L.fkr_mixture_hash(cfg.encode())


def test_gen_zero_count_is_usage_error(cli, tmp_path):
    rc, _, _ = run(cli, "gen", "--config", MIX1, "--n", 0, "--seed", 0, "--out", tmp_path / "z.bin")
    assert rc == 2
    assert not os.path.exists(tmp_path / "z.bin")


def test_usage_errors(cli, tmp_path):
    assert run(cli)[0] == 2
    assert run(cli, "frobnicate")[0] == 2
    assert run(cli, "gen", "--n", 5)[0] == 2                      # missing --config/--seed/--out
    tr = gen(cli, tmp_path, "tr.bin", MIX1, 50, 1)
    q = gen(cli, tmp_path, "q.bin", MIX1, 10, 2)
    o = str(tmp_path / "o.csv")
    assert run(cli, "estimate", tr, q, "--out", o, "--method", "bogus")[0] == 2
    assert run(cli, "estimate", tr, q, "--out", o, "--h-rule", "fixed")[0] == 2
    assert run(cli, "estimate", tr, q, "--out", o, "--engine", "naive")[0] == 2
    assert run(cli, "estimate", tr, q, "--out", o, "--format", "xml")[0] == 2
    assert run(cli, "bench", "--mode", "runtime", "--config", MIX1, "--n-grid", "64",
               "--out", tmp_path / "b.csv")[0] == 2               # runtime mode requires --seed
    assert not os.path.exists(o)


def test_missing_query_file_is_io_error_with_no_output(cli, tmp_path):
    tr = gen(cli, tmp_path, "tr.bin", MIX1, 50, 1)
    o = str(tmp_path / "out.csv")
    rc, _, err = run(cli, "estimate", tr, tmp_path / "missing.bin", "--out", o)
    assert rc == 3, err
    assert not os.path.exists(o)


def test_dimension_mismatch_is_numeric_error(cli, tmp_path):
    tr = gen(cli, tmp_path, "tr.bin", MIX1, 50, 1)
    q2 = str(tmp_path / "q2.csv")
    fio.write_samples_csv(np.ones((4, 2)), q2)
    rc, _, _ = run(cli, "estimate", tr, q2, "--out", tmp_path / "o.csv")
    assert rc == 4


def test_compare_gates(cli, tmp_path):
    v = np.linspace(1.0, 2.0, 40)
    a, b, c = (str(tmp_path / f) for f in ("a.csv", "b.bin", "c.json"))
    fio.write_values(v, a, "csv")
    fio.write_values(v, b, "bin")
    w = v.copy()
    w[3] *= 1 + 1e-6
    fio.write_values(w, c, "json")
    rc, out, _ = run(cli, "compare", a, b)
    assert rc == 0 and json.loads(out)["pass"] is True and json.loads(out)["count"] == 40
    rc, out, _ = run(cli, "compare", a, c, "--rtol", "1e-8")
    assert rc == 1 and json.loads(out)["pass"] is False
    rc, out, _ = run(cli, "compare", a, c, "--rtol", "1e-5", "--per-component")
    r = json.loads(out)
    assert rc == 0 and abs(r["max_rel_per_component"] - 1e-6 / (1 + 1e-6)) < 1e-12
    fio.write_values(v[:10], b, "bin")
    assert run(cli, "compare", a, b)[0] == 4


def test_model_matches_reference_perfmodel(cli, tmp_path, ref):
    L = ref.lib
    for f, at in (("fkr_flops_nd", [ctypes.c_size_t] * 2), ("fkr_flops_1d", [ctypes.c_size_t]),
                  ("fkr_bytes_nd", [ctypes.c_size_t] * 4), ("fkr_bytes_1d", [ctypes.c_size_t]),
                  ("fkr_bytes_linear", [ctypes.c_size_t] * 2),
                  ("fkr_intensity_asymptotic", [ctypes.c_size_t])):
        getattr(L, f).argtypes = at
        getattr(L, f).restype = ctypes.c_double
    spec = str(tmp_path / "hw.txt")
    open(spec, "w").write("# test\nname = t\npeak_flops = 40e12\nmem_bw = 770e9\nexp_cost = 8\n")
    for d, k, tm, tn in ((16, 1 << 20, 64, 1024), (16, 32768, 32, 128), (1, 4096, 64, 1024),
                         (3, 1000, 7, 13)):
        rc, out, err = run(cli, "model", "--d", d, "--k", k, "--tile-m", tm, "--tile-n", tn, "--hw", spec)
        assert rc == 0, err
        r = json.loads(out)
        fl = L.fkr_flops_1d(k) if d == 1 else L.fkr_flops_nd(d, k)
        by = L.fkr_bytes_1d(k) if d == 1 else L.fkr_bytes_nd(d, k, tm, tn)
        assert r["flops"] == fl and r["bytes"] == by
        assert r["intensity"] == fl / by and r["machine_balance"] == 40e12 / 770e9
        assert r["classification"] == ("compute-bound" if fl / by >= 40e12 / 770e9 else "memory-bound")
        if d > 1:
            assert r["intensity_asymptotic_per_k"] == L.fkr_intensity_asymptotic(d)
            assert r["bytes_linear"] == L.fkr_bytes_linear(d, k)


def test_model_b200_presets(cli):
    # the B200 presets put the exponential, not the GEMM, on the roof: the MUFU
    # bound of the headline SD-KDE (n = 2^20, m = n/8) is ~0.27 s on either preset
    for spec in ("b200-fp32.txt", "b200-tensorcore.txt"):
        rc, out, err = run(cli, "model", "--d", 16, "--k", 1 << 20, "--hw", os.path.join(HW, spec))
        assert rc == 0, err
        r = json.loads(out)
        assert r["exp_count"] == (1 << 40) + (1 << 20) * (1 << 17)
        assert 0.25 < r["exp_bound_s"] < 0.29, r
    # the reference's byte model (tile re-reads, perfmodel.cpp) vs the FP32 roof
    rc, out, _ = run(cli, "model", "--d", 16, "--k", 1 << 20, "--hw", os.path.join(HW, "b200-fp32.txt"))
    assert json.loads(out)["classification"] == "compute-bound"


def test_bad_hw_spec(cli, tmp_path):
    spec = str(tmp_path / "hw.txt")
    open(spec, "w").write("name = x\npeak_flops = 1e12\nmem_bw = 1e9\nbogus = 3\n")
    assert run(cli, "model", "--d", 2, "--k", 10, "--hw", spec)[0] == 4
    assert run(cli, "model", "--d", 2, "--k", 10, "--hw", tmp_path / "none.txt")[0] == 3


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("method", ["kde", "sdkde", "laplace"])
def test_estimate_matches_oracle(cli, tmp_path, port, method):
    tr = gen(cli, tmp_path, "tr.bin", MIX16, 2048, 1)
    q = gen(cli, tmp_path, "q.bin", MIX16, 256, 2)
    o = str(tmp_path / "o.csv")
    rc, out, err = run(cli, "estimate", tr, q, "--method", method, "--h", 1.4, "--out", o)
    assert rc == 0, err
    s = json.loads(out)
    assert s["engine"] == "gpu" and s["n_train"] == 2048 and s["n_test"] == 256 and s["h"] == 1.4
    assert ("negative_mass" in s) == (method == "laplace")
    got = fio.read_values(o)
    X, Y = fio.read_samples(tr).values, fio.read_samples(q).values
    if method == "kde":
        want = port.kde_naive(X, Y, 1.4)
    elif method == "laplace":
        want = port.laplace_naive(X, Y, 1.4)
    else:
        want, _ = port.sdkde_naive(X, Y, 1.4)
    if method == "laplace":
        assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 1e-4
    else:
        assert max_component_rel(got, want) < 1e-4


@pytest.mark.gpu
def test_estimate_summary_and_determinism(cli, tmp_path):
    tr = gen(cli, tmp_path, "tr.bin", MIX16, 1000, 3)
    q = gen(cli, tmp_path, "q.bin", MIX16, 100, 4)
    for fmt in ("csv", "bin", "json"):
        f1, f2 = str(tmp_path / ("1." + fmt)), str(tmp_path / ("2." + fmt))
        for f in (f1, f2):
            rc, out, err = run(cli, "estimate", tr, q, "--method", "laplace", "--out", f, "--format", fmt)
            assert rc == 0, err
        assert open(f1, "rb").read() == open(f2, "rb").read(), fmt
    for k in ("wall_time_s", "negative_mass", "h_score", "tile_m", "tile_n", "fused"):
        assert k in json.loads(out)


@pytest.mark.gpu
def test_laplace_fused_vs_nofuse_agree(cli, tmp_path):
    tr = gen(cli, tmp_path, "tr.bin", MIX1, 4000, 5)
    q = gen(cli, tmp_path, "q.bin", MIX1, 500, 6)
    a, b = str(tmp_path / "a.csv"), str(tmp_path / "b.csv")
    assert run(cli, "estimate", tr, q, "--method", "laplace", "--out", a)[0] == 0
    assert run(cli, "estimate", tr, q, "--method", "laplace", "--no-fuse", "--out", b)[0] == 0
    rc, out, _ = run(cli, "compare", a, b, "--rtol", "1e-5")
    assert rc == 0, out


@pytest.mark.gpu
def test_bench_runtime_mode_emits_tile_columns(cli, tmp_path):
    o = str(tmp_path / "rt.csv")
    rc, out, err = run(cli, "bench", "--mode", "runtime", "--config", MIX1, "--n-grid", "512,1024",
                       "--methods", "kde,sdkde", "--tile-m", "32,64", "--tile-n", "128", "--seed", 0,
                       "--repeats", 2, "--hw", os.path.join(HW, "b200-fp32.txt"), "--out", o)
    assert rc == 0, err
    assert json.loads(out) == {"rows": 8, "failed": 0, "out": o}
    text = open(o).read()
    assert text.startswith("schema_version,method,engine,n_train,n_test,d,tile_m,tile_n,repeats,"
                           "median_seconds,model_flops,utilization,failed,error")
    assert ",32,128," in text and ",64,128," in text
    rows = [l.split(",") for l in text.strip().split("\n")[1:]]
    assert all(float(r[9]) > 0 and r[12] == "0" for r in rows)


@pytest.mark.gpu
def test_bench_error_mode_writes_csv_deterministically(cli, tmp_path):
    args = ["bench", "--mode", "error", "--config", MIX1, "--methods", "kde,sdkde",
            "--n-grid", "200,400", "--seeds", "1,2", "--n-eval", 256]
    for f in ("s1.csv", "s2.csv"):
        rc, _, err = run(cli, *args, "--out", tmp_path / f)
        assert rc == 0, err
    s1 = open(tmp_path / "s1.csv").read()
    assert s1 == open(tmp_path / "s2.csv").read()
    lines = s1.strip().split("\n")
    assert "mise" in lines[0] and len(lines) == 1 + 8
    assert all(l.split(",")[14] == "0" for l in lines[1:])
    mise = [float(l.split(",")[8]) for l in lines[1:]]
    assert all(0 < m < 0.05 for m in mise)
