"""§8(f) row 4 pinned to the reference: the oracle-error sweep of `fkde-b200 bench
--mode error` (sweep.cpp:105-154 + metrics.cpp:47-120 restated in
cli/fkde_cli.cpp) against the reference's own `fkde::bench::error_metrics`,
compiled from /root/reference into oracle/_ref (ref_shim.cpp:fkr_error_metrics),
with the estimator plugged in as a callback.

Per sweep cell (method x n x seed) on the 1-D mixture (Grid1D trapezoid) and the
16-D mixture (importance MC):
  * the reference's metrics evaluated on OUR engine's estimates equal the CLI's
    cells (same estimates, same formulas: the restatement of the metric code);
  * the reference's metrics evaluated on the reference ORACLE's estimates agree
    with the CLI's cells within the engine's stated fp32-class tolerance
    (end-to-end parity of the sweep: estimator + metrics).
"""
import ctypes
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

from paper_2602_10378_b200 import build as B

CFG = os.path.join(ROOT, "paper_2602_10378_b200", "configs")
MIX1 = os.path.join(CFG, "mixture-1d-default.json")
MIX16 = os.path.join(CFG, "mixture-16d-default.json")

CB = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_size_t,
                      ctypes.c_size_t, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p)


def _ref_metrics(ref, cfg, grid, n_eval, seed, estimate):
    f = ref.lib.fkr_error_metrics
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_uint64, CB,
                  ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]

    def cb(pts, n, d, out, user):
        try:
            z = np.ctypeslib.as_array(pts, shape=(n * d,)).reshape(n, d).copy()
            v = np.ascontiguousarray(estimate(z), dtype=np.float64)
            ctypes.memmove(out, v.ctypes.data, n * 8)
            return 0
        except Exception:   # noqa: BLE001 -- reported as a failed call
            return 1

    out = (ctypes.c_double * 6)()
    rc = f(cfg.encode(), 1 if grid else 0, n_eval, seed, CB(cb), None, out)
    assert rc == 0
    return np.array(out[:])


def _cells(cli, cfg, methods, n_grid, seeds, n_eval, tmp_path):
    o = str(tmp_path / "err.csv")
    r = subprocess.run([cli, "bench", "--mode", "error", "--config", cfg, "--methods", methods,
                        "--n-grid", n_grid, "--seeds", seeds, "--n-eval", str(n_eval), "--out", o],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr
    lines = open(o).read().strip().split("\n")
    head = lines[0].split(",")
    return [dict(zip(head, ln.split(","))) for ln in lines[1:]]


def _cell_inputs(ref, cfg, n, seed, method):
    mix = json.load(open(cfg))
    cs = ref.mix64(seed ^ ref.mix64(n))                      # sweep.cpp:67-69
    tr = ref.sample_mixture(mix["weights"], mix["means"], mix["sigmas"], n, cs)
    d = tr.shape[1]
    if method == "sdkde":                                    # BandwidthPolicy Auto, sweep.cpp:31-61
        h = ref.sdkde_bandwidth(tr, ref.silverman_prefactor(d))
    else:
        h = ref.silverman_bandwidth(tr)
    return tr, h


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,grid", [(MIX1, True), (MIX16, False)])
def test_error_sweep_matches_reference_error_metrics(ref, port, tmp_path, cfg, grid):
    import paper_2602_10378_b200 as fk
    cli = B.build_cli()
    n_eval = 512
    rows = _cells(cli, cfg, "kde,sdkde,laplace", "1024,4096", "0,1", n_eval, tmp_path)
    assert len(rows) == 3 * 2 * 2 and all(r["failed"] == "0" for r in rows)
    keys = ["mise", "mise_se", "miae", "miae_se", "negative_mass", "negative_mass_se"]
    ctx = fk.Context([0])
    worst_same, worst_oracle = 0.0, 0.0
    for r in rows:
        method, n, seed = r["method"], int(r["n_train"]), int(r["seed"])
        tr, h = _cell_inputs(ref, cfg, n, seed, method)
        assert float(r["h"]) == h, (method, n, seed)
        ours = np.array([float(r[k]) for k in keys])
        m = {"kde": fk.Method.Kde, "sdkde": fk.Method.Sdkde, "laplace": fk.Method.LaplaceKde}[method]
        conf = fk.EstimatorConfig(m, fk.Bandwidth.uniform(h))

        def gpu_est(z):
            return fk.estimate(tr, z, conf, ctx=ctx).values

        def oracle_est(z):
            if method == "kde":
                return ref.kde_naive(tr, z, h, threads=os.cpu_count())
            if method == "sdkde":
                return ref.sdkde_naive(tr, z, h, threads=os.cpu_count())[0]
            return ref.laplace_naive(tr, z, h, threads=os.cpu_count())

        same = _ref_metrics(ref, cfg, grid, n_eval, seed, gpu_est)
        orac = _ref_metrics(ref, cfg, grid, n_eval, seed, oracle_est)
        # (1) the CLI's metric code == the reference's metric code on the same estimates
        rel_same = np.abs(ours - same) / np.maximum(np.abs(same), 1e-300)
        rel_same[(ours == 0) & (same == 0)] = 0.0
        worst_same = max(worst_same, float(rel_same.max()))
        assert rel_same.max() < 1e-12, (method, n, seed, ours, same)
        # (2) end to end vs the reference estimator: MISE / MIAE (and their standard
        # errors) within the engine's density tolerance; negative mass (Laplace only)
        # relative to the MIAE scale
        den = np.abs(orac[:4])
        rel = np.where(den > 0, np.abs(ours[:4] - orac[:4]) / np.where(den > 0, den, 1.0),
                       np.abs(ours[:4]))   # Grid1D has no standard errors (both 0)
        worst_oracle = max(worst_oracle, float(rel.max()))
        assert rel.max() < 2e-3, (method, n, seed, ours, orac)
        assert abs(ours[4] - orac[4]) <= 1e-4 * max(orac[2], 1e-300), (method, ours, orac)
    ctx.close()
    print(f"error sweep vs reference error_metrics: same-estimate rel {worst_same:.2e}, "
          f"vs oracle estimates rel {worst_oracle:.2e}")
