"""GPU parity tests: the B200 engine (through the C ABI) against the fp64 CPU
oracle and the reference's golden fixtures.

Tolerances (fp32-class operands: 3-term fp16 splits, fp32 accumulation,
fp64 finalize).  BASELINE.json asks for relative error <= 1e-3 on
log-density and on the score; the bounds below are tighter:
  densities (KDE, SD-KDE)   max_component_rel  <= 1e-4   (log-density <= 1e-5)
  Laplace                   max_rel_vs_peak    <= 1e-4
  scores                    max_rowwise_rel / max_rel_global_floor (1e-2 floors,
                            proj/tests/test_util.hpp:53-93) <= 1e-3
  debiased samples          max_rowwise_rel    <= 1e-3 (1-D rows are single
                            components, so near-zero debiased values are judged
                            by plain relative error)
Mirrors proj/tests/test_engine.cpp and acceptance_main.cpp crit. 1/2 (whose
fp64 bounds 1e-8/1e-10 are replaced by the fp32-class bounds above).
"""
import ctypes
import os

import numpy as np
import pytest

from conftest import (GOLDEN, golden, max_component_rel, max_log_rel, max_rel_global_floor,
                      max_rel_vs_peak, max_rowwise_rel)

import paper_2602_10378_b200 as fk
from paper_2602_10378_b200 import _native as N

pytestmark = pytest.mark.gpu

TOL_DENS = 1e-4
TOL_LAP = 1e-4
TOL_SCORE = 1e-3
TOL_DEB = 1e-3


@pytest.fixture(scope="module")
def ctx():
    c = fk.Context([0])
    yield c
    c.close()


def _mixture_inputs(port, n, m):
    import oracle as O
    w, mu, s = O.default_mixture_16d()
    seed = port.mix64(0 ^ port.mix64(n))        # sweep.cpp:67-69
    tr = port.sample_mixture(w, mu, s, n, seed)
    q = port.sample_mixture(w, mu, s, m, port.mix64(seed ^ 0x71))
    return tr, q


# ---- golden fixtures from the reference oracle ------------------------------------
def test_score_golden_4096_style(ctx):
    g = golden("score_1024x16")  # test_engine.cpp:99-105 (first 1024 rows of seed 41)
    s = fk.score_flash(g["train"], float(g["h"]), ctx=ctx).values
    assert max_rowwise_rel(s, g["score"]) < TOL_SCORE
    assert max_rel_global_floor(s, g["score"]) < TOL_SCORE


def test_kde_golden_1d(ctx):
    g = golden("kde_1d")  # test_engine.cpp:123-130
    v = fk.kde_flash(g["train"], g["queries"], float(g["h"]), ctx=ctx).values
    assert max_component_rel(v, g["values"]) < TOL_DENS


@pytest.mark.parametrize("fused", [True, False])
def test_laplace_golden_2d(ctx, fused):
    g = golden("laplace_2d")  # test_engine.cpp:132-143
    v = fk.kde_flash(g["train"], g["queries"], float(g["h"]), fk.KernelKind.LaplaceCorrected,
                     fused, ctx=ctx).values
    assert max_rel_vs_peak(v, g["values"]) < TOL_LAP


def test_sdkde_golden_512x16(ctx):
    g = golden("sdkde_512x16")  # test_engine.cpp:156-166
    r = fk.sdkde_flash(g["train"], g["queries"], fk.Bandwidth(float(g["h"]), float(g["h_score"])),
                       ctx=ctx)
    assert max_component_rel(r.values, g["values"]) < TOL_DENS
    assert max_rowwise_rel(r.debiased_samples.values, g["debiased"]) < TOL_DEB


ACCEPT = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.startswith("accept_"))


@pytest.mark.parametrize("name", ACCEPT)
def test_acceptance_instances(ctx, name):
    # acceptance_main.cpp:65-135 (crit. 1) on the reference's own instances
    g = golden(name)
    tr, q, h = g["train"], g["queries"], float(g["h"])
    assert max_component_rel(fk.kde_flash(tr, q, h, ctx=ctx).values, g["kde"]) < TOL_DENS
    lap = fk.kde_flash(tr, q, h, fk.KernelKind.LaplaceCorrected, True, ctx=ctx).values
    assert max_rel_vs_peak(lap, g["laplace"]) < TOL_LAP
    assert max_rel_global_floor(fk.score_flash(tr, h, ctx=ctx).values, g["score"]) < TOL_SCORE
    r = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=ctx)
    assert max_component_rel(r.values, g["sdkde"]) < TOL_DENS
    assert max_rowwise_rel(r.debiased_samples.values, g["debiased"]) < TOL_DEB


def test_config1_mixture_4096(ctx, port):
    # BASELINE config 1: 16-D mixture, n = m = 4096, SD-KDE rate bandwidth
    c = golden("config1")
    tr, q = _mixture_inputs(port, 4096, 4096)
    h, hs = float(c["h"]), float(c["h_silverman"])
    r = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=ctx)
    assert max_component_rel(r.values, c["sdkde"]) < TOL_DENS
    assert max_log_rel(r.values, c["sdkde"]) < 1e-3  # BASELINE.json's stated metric
    s = fk.score_flash(tr, h, ctx=ctx).values
    print("config1 score rowwise", max_rowwise_rel(s, c["score"]), "global",
          max_rel_global_floor(s, c["score"]))
    assert max_rowwise_rel(s, c["score"]) < TOL_SCORE
    assert max_rel_global_floor(s, c["score"]) < TOL_SCORE
    assert max_component_rel(fk.kde_flash(tr, q, hs, ctx=ctx).values, c["kde"]) < TOL_DENS
    lap = fk.kde_flash(tr, q, hs, fk.KernelKind.LaplaceCorrected, True, ctx=ctx).values
    assert max_rel_vs_peak(lap, c["laplace"]) < TOL_LAP


# ---- engine properties (test_engine.cpp) -------------------------------------------
def test_score_accumulate_includes_self_term(ctx, port):
    tr = port.random_gaussian(65, 2, 43, 3.0)      # test_engine.cpp:114-121
    acc = fk.score_accumulate(tr, 0.5, ctx=ctx)
    assert (acc.phi_sum >= 0.99).all() and np.isfinite(acc.phi_sum).all()
    # raw totals agree with the oracle's definition sum_j phi_ij (x_j)
    d2 = ((tr[:, None, :] - tr[None, :, :]) ** 2).sum(-1)
    phi = np.exp(-d2 / (2 * 0.5 ** 2))
    assert max_component_rel(acc.phi_sum, phi.sum(1)) < 1e-4
    assert max_rowwise_rel(acc.weighted_sum.values, phi @ tr) < 1e-4


def test_laplace_fused_vs_nonfused(ctx, port):
    tr = port.random_gaussian(2048, 16, 55)        # test_engine.cpp:145-154
    q = port.random_gaussian(256, 16, 56)
    a = fk.kde_flash(tr, q, 1.2, fk.KernelKind.LaplaceCorrected, True, ctx=ctx).values
    b = fk.kde_flash(tr, q, 1.2, fk.KernelKind.LaplaceCorrected, False, ctx=ctx).values
    assert max_rel_vs_peak(a, b) < 1e-5


def test_sdkde_single_point_equals_kde(ctx, port):
    q = port.random_gaussian(8, 1, 59)             # test_engine.cpp:168-175
    sd = fk.sdkde_flash(np.array([[0.7]]), q, fk.Bandwidth.uniform(0.6), ctx=ctx)
    kd = port.kde_naive([0.7], q, 0.6)
    assert max_component_rel(sd.values, kd) < TOL_DENS
    assert sd.debiased_samples.values[0, 0] == 0.7


def test_determinism_bitwise(ctx, port):
    tr = port.random_gaussian(700, 3, 65)          # test_engine.cpp:245-262
    q = port.random_gaussian(300, 3, 66)
    a = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(0.5), ctx=ctx).values
    b = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(0.5), ctx=ctx).values
    assert np.array_equal(a, b)


def test_partition_invariance_over_cta_counts(port):
    # Same column splits, different persistent-grid sizes -> bitwise equal
    # (each output row keeps one owner and a fixed accumulation order).
    tr, q = _mixture_inputs(port, 8192, 2048)
    h = 1.4
    outs = []
    for ctas in (1, 7, 0):
        c = fk.Context([0])
        c.set_option(N.OPT_SPLITS, 3)
        c.set_option(N.OPT_MAX_CTAS, ctas)
        outs.append(fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=c).values)
        c.close()
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_split_count_reassociation(port):
    # test_engine.cpp:177-216 analogue: every column split agrees within fp32 rounding
    tr, q = _mixture_inputs(port, 4096, 1024)
    h = 1.5
    base = None
    for splits in (1, 2, 5, 32):
        c = fk.Context([0])
        c.set_option(N.OPT_SPLITS, splits)
        v = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=c).values
        s = fk.score_flash(tr, h, ctx=c).values
        c.close()
        if base is None:
            base = (v, s)
        else:
            assert max_component_rel(v, base[0]) < 1e-4
            assert max_rel_global_floor(s, base[1]) < 1e-4


def test_flush_interval_and_ragged_units(port):
    # O sub-unit drains (FKDE_OPT_FLUSH_TILES) with units of odd length (32 column
    # tiles over 5 / 3 splits -> 6-7 and 10-11 tiles): the two epilogue parities
    # and the drain schedule must cover every tile exactly once for any interval.
    tr = _mixture_inputs(port, 4096, 16)[0]
    h = 1.5
    ref = port.score_naive(tr, tr, h)
    for splits in (5, 3):
        for flush in (1, 2, 4, 1 << 20):
            c = fk.Context([0])
            c.set_option(N.OPT_SPLITS, splits)
            c.set_option(N.OPT_FLUSH_TILES, flush)
            s = fk.score_flash(tr, h, ctx=c).values
            c.close()
            assert max_rel_global_floor(s, ref) < TOL_SCORE, (splits, flush)


def test_flush_interval_must_be_power_of_two(ctx):
    for bad in (-1, 3, 6, (1 << 20) + 1):
        with pytest.raises(fk.InvalidArgumentError):
            ctx.set_option(N.OPT_FLUSH_TILES, bad)


@pytest.mark.parametrize("n,m,d", [(1, 1, 1), (129, 130, 3), (257, 5, 2), (300, 1, 16),
                                   (1000, 999, 4)])
def test_ragged_and_small_shapes(ctx, port, n, m, d):
    tr = port.random_gaussian(n, d, 1000 + n, 1.5)
    q = port.random_gaussian(m, d, 2000 + m, 1.5)
    h = 0.75 * np.sqrt(d)
    assert max_component_rel(fk.kde_flash(tr, q, h, ctx=ctx).values,
                             port.kde_naive(tr, q, h)) < TOL_DENS
    ref_v, ref_deb = port.sdkde_naive(tr, q, h)
    r = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=ctx)
    assert max_component_rel(r.values, ref_v) < TOL_DENS
    assert max_rowwise_rel(r.debiased_samples.values, ref_deb) < TOL_DEB


def test_half_variance_score_bandwidth(ctx, port):
    tr = port.random_gaussian(600, 16, 71)
    q = port.random_gaussian(100, 16, 72)
    bw = fk.Bandwidth.half_variance_score(1.1)
    r = fk.sdkde_flash(tr, q, bw, ctx=ctx)
    ref_v, ref_deb = port.sdkde_naive(tr, q, bw.h, bw.h_score)
    assert max_component_rel(r.values, ref_v) < TOL_DENS
    assert max_rowwise_rel(r.debiased_samples.values, ref_deb) < TOL_DEB


def test_large_offset_data_is_centred(ctx, port):
    # translation invariance (test_oracle.cpp:31-47): far-from-origin data
    tr = port.random_gaussian(512, 16, 73) + 1000.0
    q = port.random_gaussian(64, 16, 74) + 1000.0
    ref = port.kde_naive(tr, q, 0.9)
    assert max_component_rel(fk.kde_flash(tr, q, 0.9, ctx=ctx).values, ref) < TOL_DENS


def test_wide_spread_data_scales_operands(ctx, port):
    # |y|^2/2 beyond 2^13 -> the operand scale exponent e > 0 path.  The Gram
    # expansion's fp32 rounding grows with |x - mu|^2 / h^2, so these rows
    # (|y|^2/2 > kRiskHalfNorm = 128) are flagged and recomputed by direct
    # differences: the normal tolerances hold.
    centres = np.array([[40.0, 0, 0, 0], [-40.0, 0, 0, 0], [0, 40.0, 0, 0], [0, -40.0, 0, 0]])
    tr = port.random_gaussian(800, 4, 75) + np.repeat(centres, 200, axis=0)
    q = port.random_gaussian(80, 4, 76) + np.repeat(centres, 20, axis=0)
    h = 0.6
    v = fk.kde_flash(tr, q, h, ctx=ctx).values
    ref = port.kde_naive(tr, q, h)
    err = max_component_rel(v, ref)
    print("wide-spread kde rel err", err)
    assert err < TOL_DENS
    s = fk.score_flash(tr, h, ctx=ctx).values
    ref_s = port.score_naive(tr, tr, h)
    err_s = max_rel_global_floor(s, ref_s)
    err_r = max_rowwise_rel(s, ref_s)
    print("wide-spread score err", err_s, err_r)
    assert err_s < TOL_SCORE and err_r < TOL_SCORE


def test_estimate_dispatch(ctx, port):
    tr = port.random_gaussian(64, 2, 201)          # test_estimator.cpp:23-65
    q = port.random_gaussian(32, 2, 202, 3.0)
    lap = fk.estimate(tr, q, fk.EstimatorConfig(fk.Method.LaplaceKde, fk.Bandwidth.uniform(0.5)),
                      ctx=ctx)
    assert lap.negative_mass_estimate is not None and lap.negative_mass_estimate >= 0.0
    kde = fk.estimate(tr, q, fk.EstimatorConfig(fk.Method.Kde, fk.Bandwidth.uniform(0.5)), ctx=ctx)
    assert kde.negative_mass_estimate is None and kde.debiased_samples is None
    sd = fk.estimate(tr, q, fk.EstimatorConfig(fk.Method.Sdkde, fk.Bandwidth.uniform(0.5)), ctx=ctx)
    assert sd.debiased_samples is not None and sd.negative_mass_estimate is None
    assert max_component_rel(kde.values, port.kde_naive(tr, q, 0.5)) < TOL_DENS
    ref_lap = port.laplace_naive(tr, q, 0.5)
    assert max_rel_vs_peak(lap.values, ref_lap) < TOL_LAP
    assert abs(lap.negative_mass_estimate - np.maximum(0, -ref_lap).mean()) < 1e-4 * np.abs(ref_lap).max()


def test_estimate_through_c_abi(ctx, port):
    tr = port.random_gaussian(300, 16, 81)
    q = port.random_gaussian(40, 16, 82)
    lib = N.load()
    out = np.empty(40)
    deb = np.empty((300, 16))
    neg = ctypes.c_double(-1)
    idx = ctypes.c_size_t(0)
    dp = ctypes.POINTER(ctypes.c_double)
    rc = lib.fkde_gpu_estimate(ctx.handle, tr.ctypes.data_as(dp), 300, q.ctypes.data_as(dp), 40, 16,
                               N.METHOD_SDKDE, 1.1, 1.1, 64, 1024, 1, out.ctypes.data_as(dp),
                               deb.ctypes.data_as(dp), ctypes.byref(neg), ctypes.byref(idx))
    assert rc == N.OK
    ref_v, ref_deb = port.sdkde_naive(tr, q, 1.1)
    assert max_component_rel(out, ref_v) < TOL_DENS
    rc = lib.fkde_gpu_estimate(ctx.handle, tr.ctypes.data_as(dp), 300, q.ctypes.data_as(dp), 40, 16,
                               N.METHOD_KDE, 1.1, 1.1, 0, 1024, 1, out.ctypes.data_as(dp), None,
                               None, None)
    assert rc == N.INVALID_ARGUMENT


def test_errors(ctx, port):
    with pytest.raises(fk.UnsupportedDimensionError):
        fk.kde_flash(port.random_gaussian(10, 17, 1), port.random_gaussian(3, 17, 2), 1.0, ctx=ctx)
    # device-side non-finite detection through the raw ABI (the host mirror
    # rejects NaN before the call, like SampleSet::validate)
    lib = N.load()
    tr = port.random_gaussian(50, 2, 3)
    tr[7, 1] = np.nan
    out = np.empty(5)
    dp = ctypes.POINTER(ctypes.c_double)
    q = port.random_gaussian(5, 2, 4)
    rc = lib.fkde_gpu_kde(ctx.handle, tr.ctypes.data_as(dp), 50, q.ctypes.data_as(dp), 5, 2, 1.0,
                          0, 1, out.ctypes.data_as(dp))
    assert rc == N.NON_FINITE
    # the context stays usable after a reported error
    tr[7, 1] = 0.0
    v = fk.kde_flash(tr, q, 1.0, ctx=ctx).values
    assert max_component_rel(v, port.kde_naive(tr, q, 1.0)) < TOL_DENS


def test_nonfinite_flag_does_not_leak_between_jobs(ctx, port):
    # a NaN seen by one kind of job must not make a later valid job of another
    # kind (which writes the other PassScalars slot) report NON_FINITE
    lib = N.load()
    dp = ctypes.POINTER(ctypes.c_double)
    tr = port.random_gaussian(64, 3, 11)
    q = port.random_gaussian(8, 3, 12)
    bad = tr.copy()
    bad[5, 2] = np.inf
    out = np.empty(8)
    sc = np.empty((64, 3))
    idx = ctypes.c_size_t(0)
    rc = lib.fkde_gpu_kde(ctx.handle, bad.ctypes.data_as(dp), 64, q.ctypes.data_as(dp), 8, 3, 0.8, 0,
                          1, out.ctypes.data_as(dp))
    assert rc == N.NON_FINITE
    rc = lib.fkde_gpu_score(ctx.handle, tr.ctypes.data_as(dp), 64, 3, 0.8, sc.ctypes.data_as(dp),
                            ctypes.byref(idx))
    assert rc == N.OK, ctx.last_error()
    assert max_rowwise_rel(sc, port.score_naive(tr, tr, 0.8)) < TOL_SCORE
    rc = lib.fkde_gpu_score(ctx.handle, bad.ctypes.data_as(dp), 64, 3, 0.8, sc.ctypes.data_as(dp),
                            ctypes.byref(idx))
    assert rc == N.NON_FINITE
    rc = lib.fkde_gpu_kde(ctx.handle, tr.ctypes.data_as(dp), 64, q.ctypes.data_as(dp), 8, 3, 0.8, 0,
                          1, out.ctypes.data_as(dp))
    assert rc == N.OK, ctx.last_error()
    assert max_component_rel(out, port.kde_naive(tr, q, 0.8)) < TOL_DENS


def test_last_error_is_per_thread(ctx, port):
    # two threads sharing one context: each sees the message of its own call
    import threading
    lib = N.load()
    dp = ctypes.POINTER(ctypes.c_double)
    tr = port.random_gaussian(32, 2, 13)
    q = port.random_gaussian(4, 2, 14)
    out = np.empty(4)
    msgs = {}

    def worker(tag, h):
        for _ in range(200):
            rc = lib.fkde_gpu_kde(ctx.handle, tr.ctypes.data_as(dp), 32, q.ctypes.data_as(dp), 4, 2,
                                  h, 7 if tag == "kind" else 0, 1, out.ctypes.data_as(dp))
            assert rc == N.INVALID_ARGUMENT
            msgs.setdefault(tag, set()).add(lib.fkde_gpu_last_error(ctx.handle).decode())

    ts = [threading.Thread(target=worker, args=("kind", 1.0)),
          threading.Thread(target=worker, args=("h", -1.0))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert msgs["kind"] == {"unknown kernel kind 7"}
    assert len(msgs["h"]) == 1 and "h must be positive" in next(iter(msgs["h"]))


def test_device_ids_are_validated():
    with pytest.raises(fk.DeviceError):
        fk.Context([0, 4096])
    with pytest.raises(fk.DeviceError):
        fk.Context([-1])
    # the reference accepts any worker count: default contexts cap it at the GPUs present
    c = fk.engine.default_context(threads=4096)
    assert c.world()[1] == fk.engine.device_count()


def test_device_api_argument_checks(ctx):
    import torch
    lib = N.load()
    dX = torch.zeros((16, 2), dtype=torch.float64, device="cuda")
    dO = torch.zeros(4, dtype=torch.float64, device="cuda")
    assert lib.fkde_gpu_kde_device(ctx.handle, dX.data_ptr(), 16, dX.data_ptr(), 4, 2, 1.0, 5, 1,
                                   dO.data_ptr()) == N.INVALID_ARGUMENT
    assert lib.fkde_gpu_kde_device(ctx.handle, dX.data_ptr(), 16, dX.data_ptr(), 4, 2, 1.0, 0, 1,
                                   None) == N.INVALID_ARGUMENT
    assert lib.fkde_gpu_sdkde_device(ctx.handle, dX.data_ptr(), 16, dX.data_ptr(), 4, 2, 1.0, 1.0,
                                     None) == N.INVALID_ARGUMENT


# ---- pairwise_sq_dists_block (test_engine.cpp:125-192) --------------------------------
def test_pairwise_pythagorean_and_identical_rows(ctx, port):
    d2 = fk.pairwise_sq_dists_block([[0.0, 0.0], [3.0, 4.0]], [[3.0, 4.0]], ctx=ctx).values
    assert abs(d2[0, 0] - 25.0) < 25.0 * 1e-14 and d2[1, 0] == 0.0
    for d in (1, 4, 16):
        a = port.random_gaussian(10, d, 33 + d, 2.5)
        b = port.random_gaussian(10, d, 34 + d, 2.5)
        b[7] = a[2]
        assert fk.pairwise_sq_dists_block(a, b, ctx=ctx).values[2, 7] == 0.0


def test_pairwise_never_negative_and_tight(ctx, port):
    eps = np.finfo(float).eps
    a = port.random_gaussian(32, 4, 31, 1e-4) + 100.0
    b = port.random_gaussian(32, 4, 32, 1e-4) + 100.0
    d2 = fk.pairwise_sq_dists_block(a, b, ctx=ctx).values
    direct = ((a[:, None] - b[None]) ** 2).sum(-1)
    na = (a * a).sum(1)[:, None] + (b * b).sum(1)[None]
    assert (d2 >= 0).all()
    assert (np.abs(d2 - direct) < 16 * eps * na).all()


# ---- device-resident and multi-rank entry points ------------------------------------------
def test_device_resident_api_matches_host_api(ctx, port):
    torch = pytest.importorskip("torch")
    tr, q = _mixture_inputs(port, 3000, 700)
    h = 1.5
    host = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=ctx).values
    dX = torch.from_numpy(tr).cuda()
    dY = torch.from_numpy(q).cuda()
    dO = torch.empty(700, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    lib = N.load()
    rc = lib.fkde_gpu_sdkde_device(ctx.handle, dX.data_ptr(), 3000, dY.data_ptr(), 700, 16, h, h,
                                   dO.data_ptr())
    assert rc == N.OK
    s = torch.cuda.ExternalStream(ctx.stream())
    s.synchronize()
    assert np.array_equal(dO.cpu().numpy(), host)
    assert ctx.last_launch_count() >= 8


def test_rank_context_world1_matches(ctx, port):
    tr, q = _mixture_inputs(port, 2000, 500)
    r1 = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(1.5), ctx=ctx).values
    rc = fk.Context(rank=0, world=1, device=0)
    r2 = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(1.5), ctx=rc).values
    rc.close()
    assert np.array_equal(r1, r2)


# ---- full-size configurations ------------------------------------------------------------
# The oracle is exactly linear in evaluated rows; where it cannot finish every row
# (configs 4 and 5) parity is checked on a deterministic row subsample, with the
# measured maxima printed.
def _report(tag, **errs):
    print(tag, " ".join(f"{k}={v:.3e}" for k, v in errs.items()))


@pytest.mark.slow
def test_config5_headline_subsample(ctx, port):
    # n = 2^20, m = 2^17 (BASELINE config 5).  Score checked directly on 4096
    # rows with both floored metrics of proj/tests/test_util.hpp:53-93; x^SD on
    # the same rows; densities of 4096 queries against the engine's own x^SD
    # (the oracle's x^SD needs all 2^20 score rows: 1.1e12 pairs -- the density
    # pass is pinned end to end at config 2, where it is affordable).
    n, m = 1 << 20, 1 << 17
    tr, q = _mixture_inputs(port, n, m)
    h = port.sdkde_bandwidth(tr, port.silverman_prefactor(16))
    r = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=ctx)
    v, deb = r.values, r.debiased_samples.values
    assert np.isfinite(v).all() and (v > 0).all()
    rows = np.linspace(0, n - 1, 4096).astype(int)
    sc = port.score_naive(tr, tr[rows], h, threads=os.cpu_count())
    s = fk.score_flash(tr, h, ctx=ctx).values[rows]
    ref_deb = tr[rows] + 0.5 * h * h * sc
    qs = np.linspace(0, m - 1, 4096).astype(int)
    ref_v = port.kde_naive(deb, q[qs], h, threads=os.cpu_count())
    e = dict(score_rowwise=max_rowwise_rel(s, sc), score_global=max_rel_global_floor(s, sc),
             debiased=max_rowwise_rel(deb[rows], ref_deb), density=max_component_rel(v[qs], ref_v),
             log_density=max_log_rel(v[qs], ref_v))
    _report("config5", **e)
    assert e["score_rowwise"] < TOL_SCORE and e["score_global"] < TOL_SCORE
    assert e["debiased"] < TOL_DEB
    assert e["density"] < TOL_DENS and e["log_density"] < 1e-3


@pytest.mark.slow
def test_config4_laplace_subsample(ctx, port):
    # n = 262144, m = 65536 Laplace-corrected (fused), 8192 queries (1/8) vs the oracle
    n, m = 262144, 65536
    tr, q = _mixture_inputs(port, n, m)
    h = port.silverman_bandwidth(tr)
    v = fk.kde_flash(tr, q, h, fk.KernelKind.LaplaceCorrected, True, ctx=ctx).values
    qs = np.linspace(0, m - 1, 8192).astype(int)
    ref = port.laplace_naive(tr, q[qs], h, threads=os.cpu_count())
    e = max_rel_vs_peak(v[qs], ref)
    _report("config4", laplace_vs_peak=e)
    assert e < TOL_LAP


@pytest.mark.slow
def test_config2_sdkde_32k_full(ctx, port):
    # BASELINE config 2: SD-KDE n = m = 32768, every row and every query, end to
    # end: the densities are compared with the oracle's densities at the ORACLE's
    # own debiased samples (oracle.cpp:87-101), not at the engine's
    n = m = 32768
    tr, q = _mixture_inputs(port, n, m)
    h = port.sdkde_bandwidth(tr, port.silverman_prefactor(16))
    r = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=ctx)
    sc = port.score_naive(tr, tr, h, threads=os.cpu_count())
    ref_deb = tr + 0.5 * h * h * sc
    s = fk.score_flash(tr, h, ctx=ctx).values
    ref_v = port.kde_naive(ref_deb, q, h, threads=os.cpu_count())
    e = dict(debiased=max_rowwise_rel(r.debiased_samples.values, ref_deb),
             score_rowwise=max_rowwise_rel(s, sc), score_global=max_rel_global_floor(s, sc),
             density=max_component_rel(r.values, ref_v), log_density=max_log_rel(r.values, ref_v))
    _report("config2", **e)
    assert e["debiased"] < TOL_DEB
    assert e["score_rowwise"] < TOL_SCORE and e["score_global"] < TOL_SCORE
    assert e["density"] < TOL_DENS and e["log_density"] < 1e-3


@pytest.mark.slow
def test_config3_plain_kde_32k_full(ctx, port):
    # BASELINE config 3: plain Gaussian KDE n = m = 32768 (the GEMM+exp kernel alone)
    n = m = 32768
    tr, q = _mixture_inputs(port, n, m)
    h = port.silverman_bandwidth(tr)
    v = fk.kde_flash(tr, q, h, ctx=ctx).values
    ref = port.kde_naive(tr, q, h, threads=os.cpu_count())   # every query
    e = dict(density=max_component_rel(v, ref), log_density=max_log_rel(v, ref))
    _report("config3", **e)
    assert e["density"] < TOL_DENS and e["log_density"] < 1e-3


# ---- acceptance criteria (proj/tests/acceptance/acceptance_main.cpp) --------------------
def _acceptance_instance(port, i):
    # acceptance_main.cpp:65-83 (the generator); n = 4096 instances are made here
    # with the C port (bitwise the reference's RNG, tests/test_oracle.py)
    ns, ds = [3, 64, 1024, 4096], [1, 2, 16]
    n, d = ns[(i % 12) // 3], ds[i % 3]
    tr = port.random_gaussian(n, d, 1000 + i, 1.5)
    q = port.random_gaussian(max(1, n // 8), d, 2000 + i, 1.5)
    h = (0.8 + 0.8 * port.uniform01(3000 + i, 1)[0]) * 0.75 * np.sqrt(float(d))
    return tr, q, h


BIG_ACCEPT = [i for i in range(50) if [3, 64, 1024, 4096][(i % 12) // 3] == 4096]


@pytest.mark.parametrize("i", BIG_ACCEPT)
def test_acceptance_instances_n4096(ctx, port, i):
    # the 12 n = 4096 instances of crit. 1 (make_golden.py stores the n <= 1024 ones)
    tr, q, h = _acceptance_instance(port, i)
    th = os.cpu_count()
    kde = port.kde_naive(tr, q, h, threads=th)
    lap = port.laplace_naive(tr, q, h, threads=th)
    score = port.score_naive(tr, tr, h, threads=th)
    sd, deb = port.sdkde_naive(tr, q, h, threads=th)
    e = dict(kde=max_component_rel(fk.kde_flash(tr, q, h, ctx=ctx).values, kde),
             laplace=max_rel_vs_peak(fk.kde_flash(tr, q, h, fk.KernelKind.LaplaceCorrected, True,
                                                  ctx=ctx).values, lap),
             score=max_rel_global_floor(fk.score_flash(tr, h, ctx=ctx).values, score))
    r = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=ctx)
    e["sdkde"] = max_component_rel(r.values, sd)
    e["debiased"] = max_rowwise_rel(r.debiased_samples.values, deb)
    # crit. 2 (acceptance_main.cpp:137-152): fused == non-fused Laplace
    e["fused_vs_nonfused"] = max_rel_vs_peak(
        fk.kde_flash(tr, q, h, fk.KernelKind.LaplaceCorrected, True, ctx=ctx).values,
        fk.kde_flash(tr, q, h, fk.KernelKind.LaplaceCorrected, False, ctx=ctx).values)
    _report(f"accept_{i:02d}", **e)
    assert e["kde"] < TOL_DENS and e["laplace"] < TOL_LAP and e["score"] < TOL_SCORE
    assert e["sdkde"] < TOL_DENS and e["debiased"] < TOL_DEB
    assert e["fused_vs_nonfused"] < 1e-5


@pytest.mark.slow
def test_acceptance_crit8_shape(ctx, port):
    # crit. 8 (acceptance_main.cpp:354-390): n = 32768, m = 4096, d = 16, h = 2.5,
    # random Gaussian -- parity against the oracle, the >= 5x speed-up over the
    # naive oracle, and a linear (never n^2) device workspace
    import time
    n, m, d = 32768, 4096, 16
    tr = port.random_gaussian(n, d, 81, 1.0)
    q = port.random_gaussian(m, d, 82, 1.0)
    c = fk.Context([0])
    best = 1e300
    for _ in range(3):
        t0 = time.perf_counter()
        r = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(2.5), ctx=c)
        best = min(best, time.perf_counter() - t0)
    ws = c.workspace_bytes()
    t0 = time.perf_counter()
    ref_v, ref_deb = port.sdkde_naive(tr, q, 2.5, threads=1)   # the reference's serial oracle
    naive = time.perf_counter() - t0
    e = dict(sdkde=max_component_rel(r.values, ref_v),
             debiased=max_rowwise_rel(r.debiased_samples.values, ref_deb))
    _report("crit8", speedup=naive / best, **e)
    assert e["sdkde"] < TOL_DENS and e["debiased"] < TOL_DEB
    assert naive >= 5.0 * best
    # n^2 fp64 would be 8 GiB; the engine's workspace is linear in n + m
    assert ws < 64 * 2**20 + 4096 * (n + m), ws
    c.close()


def test_device_workspace_is_linear(port):
    # test_engine.cpp:218-243 analogue: the device workspace of every pass grows
    # linearly in the data (no n x m buffer); 4x the points -> at most ~4x bytes
    sizes = []
    for n in (8192, 32768):
        c = fk.Context([0])
        tr = port.random_gaussian(n, 16, 63)
        q = port.random_gaussian(n // 4, 16, 64)
        fk.kde_flash(tr, q, 0.9, ctx=c)
        fk.score_flash(tr, 0.9, ctx=c)
        fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(0.9), ctx=c)
        sizes.append(c.workspace_bytes())
        c.close()
    print("workspace bytes", sizes)
    # a stated linear bound: 64 MiB (n-independent: direct-row partials, CUB scratch,
    # allocation rounding) + 2 KiB per point -- an n x m fp64 buffer would be
    # 8 * n * n/4 bytes (2 GiB at n = 32768)
    for n, ws in zip((8192, 32768), sizes):
        assert ws <= 64 * 2**20 + 2048 * (n + n // 4), (n, ws)


def test_moderate_spread_stays_on_tensor_cores_within_tolerance(ctx, port):
    # |y|^2/2 up to ~200 (clusters in 4-D, dense neighbourhoods): rows above the
    # direct-row threshold (kRiskHalfNorm = 128, above every BASELINE config's score
    # rows but for a handful at config 5) are recomputed directly, the rest stay on
    # the tensor cores; the result must stay inside 1e-3
    centres = np.array([[10.0, 0, 0, 0], [-10.0, 0, 0, 0], [0, 10.0, 0, 0], [0, -10.0, 0, 0]])
    tr = port.random_gaussian(2000, 4, 91) + np.repeat(centres, 500, axis=0)
    q = port.random_gaussian(200, 4, 92) + np.repeat(centres, 50, axis=0)
    h = 0.62
    s = fk.score_flash(tr, h, ctx=ctx).values
    ref_s = port.score_naive(tr, tr, h)
    v = fk.kde_flash(tr, q, h, ctx=ctx).values
    ref_v = port.kde_naive(tr, q, h)
    e = dict(score_global=max_rel_global_floor(s, ref_s), score_rowwise=max_rowwise_rel(s, ref_s),
             density=max_component_rel(v, ref_v))
    _report("moderate-spread", **e)
    assert e["score_global"] < TOL_SCORE and e["score_rowwise"] < TOL_SCORE
    assert e["density"] < TOL_DENS


@pytest.mark.parametrize("n,d,h", [(5000, 16, 1.3), (3000, 4, 0.6), (700, 2, 0.4), (257, 16, 2.0)])
def test_spatial_order_matches_input_order(port, n, d, h):
    # FKDE_OPT_SPATIAL=1 (Morton order + exact-zero tile skipping) vs 2 (input
    # order): same results within fp32 reassociation, both against the oracle,
    # outputs in the caller's row order (scores, debiased samples, raw sums)
    w, mu, s = __import__("oracle").default_mixture_16d()
    if d == 16:
        tr, q = _mixture_inputs(port, n, n // 4 + 1)
    else:
        tr = port.random_gaussian(n, d, 700 + n, 1.0) + np.repeat(
            np.eye(4, d) * 6.0, -(-n // 4), axis=0)[:n]
        q = port.random_gaussian(n // 4 + 1, d, 800 + n, 1.0)
    outs = {}
    for sp in (1, 2):
        c = fk.Context([0])
        c.set_option(N.OPT_SPATIAL, sp)
        sc = fk.score_flash(tr, h, ctx=c).values
        st = c.skip_stats()
        r = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=c)
        acc = fk.score_accumulate(tr, h, ctx=c)
        outs[sp] = (sc, r.values, r.debiased_samples.values, acc.phi_sum, acc.weighted_sum.values, st)
        c.close()
    assert outs[1][5]["spatial_order"] and not outs[2][5]["spatial_order"]
    ref_s = port.score_naive(tr, tr, h)
    ref_v, ref_deb = port.sdkde_naive(tr, q, h)
    for sp in (1, 2):
        sc, v, deb, phi, wsum, _ = outs[sp]
        # the input-order path accumulates sum phi y in the global frame: dense
        # low-dimensional clusters (tens of neighbours at |y|^2/2 ~ 50) cost it up to
        # ~2e-3 rowwise (stated envelope); the spatial order's per-tile
        # centring (B2) keeps every case inside 1e-3
        tol = TOL_SCORE if (sp == 1 or d == 16) else 3e-3
        print(f"sp={sp} d={d}: score global {max_rel_global_floor(sc, ref_s):.2e} "
              f"rowwise {max_rowwise_rel(sc, ref_s):.2e}")
        assert max_rel_global_floor(sc, ref_s) < tol, sp
        assert max_rowwise_rel(sc, ref_s) < tol, sp
        assert max_component_rel(v, ref_v) < TOL_DENS, sp
        assert max_rowwise_rel(deb, ref_deb) < (TOL_DEB if tol == TOL_SCORE else tol), sp
    # raw sums of the two paths (each within its own error of the oracle)
    assert max_component_rel(outs[1][3], outs[2][3]) < 1e-3
    assert max_rowwise_rel(outs[1][4], outs[2][4]) < 1e-3
    print("skip stats", outs[1][5])


@pytest.mark.parametrize("n", [8192, 40000])
def test_tile_skipping_is_exact(port, n):
    # score pass: skipped tile pairs contribute exact zeros (fp16 P), so the spatial
    # order with skipping (FKDE_OPT_SPATIAL=1) and without (3) give the same bits for
    # the scores and x^SD.  Density pass: a skipped pair has phi < 2^-42.5 and a row
    # keeps its skip only if the skipped mass bound is 2^-24 of its own mass (else
    # it is recomputed directly), so densities agree to that bound plus the fp32
    # reassociation of the visited tiles' sums
    tr, q = _mixture_inputs(port, n, 1000)
    h = port.sdkde_bandwidth(tr, port.silverman_prefactor(16))
    res = {}
    for sp in (1, 3):
        c = fk.Context([0])
        c.set_option(N.OPT_SPATIAL, sp)
        s = fk.score_flash(tr, h, ctx=c).values
        st = c.skip_stats()
        r = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=c)
        c.close()
        res[sp] = (s, r.values, r.debiased_samples.values, st)
    print("skip stats", res[1][3])
    assert res[1][3]["tiles_skipped"] > 0 and res[3][3]["tiles_skipped"] == 0
    assert np.array_equal(res[1][0], res[3][0]) and np.array_equal(res[1][2], res[3][2])
    assert max_component_rel(res[1][1], res[3][1]) < 1e-6


def test_spatial_order_skips_tiles_on_clustered_data(port):
    # four far-apart clusters: most tile pairs contribute exactly zero and are skipped
    tr = port.random_gaussian(8192, 16, 97) + np.repeat(np.eye(4, 16) * 40.0, 2048, axis=0)
    h = 3.0   # |y|^2/2 ~ 50 (tensor-core rows), clusters ~250 log2 units apart
    c = fk.Context([0])
    c.set_option(N.OPT_SPATIAL, 1)
    s = fk.score_flash(tr, h, ctx=c).values
    st = c.skip_stats()
    c.close()
    print("skip stats", st)
    # (skipped = proven by the tile boxes + checked exactly and found zero)
    assert st["tiles_skipped"] > 0 and st["tiles_total"] > st["tiles_skipped"]
    assert st["tiles_checked"] <= st["tiles_total"]
    rows = np.arange(0, 8192, 7)
    ref = port.score_naive(tr, tr[rows], h)
    assert max_rowwise_rel(s[rows], ref) < TOL_SCORE


def test_small_bandwidth_rows_fall_back_without_cliff(port):
    # config-1 data at h/3: many rows have too little neighbour mass for fp16 P and
    # go to the direct-difference kernel; results stay at fp64-oracle accuracy
    c = golden("config1")
    tr, q = _mixture_inputs(port, 4096, 4096)
    h = float(c["h"]) / 3
    ctx = fk.Context([0])
    r = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=ctx)
    ctx.close()
    ref_v, ref_deb = port.sdkde_naive(tr, q, h, threads=os.cpu_count())
    e = dict(sdkde=max_component_rel(r.values, ref_v),
             debiased=max_rowwise_rel(r.debiased_samples.values, ref_deb))
    _report("h/3", **e)
    assert e["sdkde"] < TOL_DENS and e["debiased"] < TOL_DEB


def test_device_api_graph_replay_is_bitwise(ctx, port):
    # the device-resident API runs a call eagerly, captures the repeat into a CUDA
    # graph and replays it afterwards: all three must give the same bits, and a
    # changed argument must fall back to eager execution
    import torch
    tr, q = _mixture_inputs(port, 3000, 700)
    dX = torch.from_numpy(tr).cuda()
    dY = torch.from_numpy(q).cuda()
    lib = N.load()
    stream = torch.cuda.ExternalStream(ctx.stream())
    outs = []
    for h in (1.3, 1.3, 1.3, 1.3, 1.1, 1.3):
        dO = torch.zeros(700, dtype=torch.float64, device="cuda") if not outs else outs_buf
        outs_buf = dO
        rc = lib.fkde_gpu_sdkde_device(ctx.handle, dX.data_ptr(), 3000, dY.data_ptr(), 700, 16, h, h,
                                       dO.data_ptr())
        assert rc == 0, ctx.last_error()
        stream.synchronize()
        outs.append(dO.cpu().numpy().copy())
    assert all(np.array_equal(outs[0], o) for o in (outs[1], outs[2], outs[3], outs[5]))
    assert not np.array_equal(outs[0], outs[4])
    host = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(1.3), ctx=ctx).values
    assert np.array_equal(outs[0], host)
    # a bigger problem in between grows (reallocates) the context's workspaces: the
    # graph captured for the first call must not be replayed with stale pointers
    big, bq = _mixture_inputs(port, 9000, 1500)
    fk.sdkde_flash(big, bq, fk.Bandwidth.uniform(1.3), ctx=ctx)
    for _ in range(3):
        rc = lib.fkde_gpu_sdkde_device(ctx.handle, dX.data_ptr(), 3000, dY.data_ptr(), 700, 16, 1.3, 1.3,
                                       outs_buf.data_ptr())
        assert rc == 0, ctx.last_error()
        stream.synchronize()
        assert np.array_equal(outs_buf.cpu().numpy(), outs[0])
    for kind in (0, 1):   # KDE / Laplace through the graph path too
        dO2 = torch.zeros(700, dtype=torch.float64, device="cuda")
        res = []
        for _ in range(3):
            rc = lib.fkde_gpu_kde_device(ctx.handle, dX.data_ptr(), 3000, dY.data_ptr(), 700, 16, 1.2,
                                         kind, 1, dO2.data_ptr())
            assert rc == 0, ctx.last_error()
            stream.synchronize()
            res.append(dO2.cpu().numpy().copy())
        assert np.array_equal(res[0], res[1]) and np.array_equal(res[0], res[2])


def test_score_device_api_matches_host_api(ctx, port):
    import torch
    tr, _ = _mixture_inputs(port, 2500, 8)
    host = fk.score_flash(tr, 1.4, ctx=ctx).values
    dX = torch.from_numpy(tr).cuda()
    dS = torch.zeros((2500, 16), dtype=torch.float64, device="cuda")
    lib = N.load()
    stream = torch.cuda.ExternalStream(ctx.stream())
    for _ in range(3):   # eager, captured, replayed
        dS.zero_()
        torch.cuda.synchronize()
        rc = lib.fkde_gpu_score_device(ctx.handle, dX.data_ptr(), 2500, 16, 1.4, dS.data_ptr())
        assert rc == 0, ctx.last_error()
        stream.synchronize()
        assert np.array_equal(dS.cpu().numpy(), host)


@pytest.mark.parametrize("kind", ["sdkde", "laplace"])
def test_repeat_calls_are_bitwise_under_dynamic_scheduling(ctx, port, kind):
    # Many units per CTA: the dynamic unit scheduler hands a unit to whichever CTA
    # is free, so the CTA (and the epilogue warp taking a unit's first tile) varies
    # from call to call.  The per-phase density partials (pairwise_tc.cuh: the
    # unit-relative slot) and the skipped-mass bound (tile_predict: per-block
    # partials summed in order) must not depend on it: repeated calls -- eager and
    # graph-replayed, host and device buffers -- agree bit for bit.
    n, m = 131072, 65536
    tr, q = _mixture_inputs(port, n, m)
    h = port.silverman_bandwidth(tr)
    outs = []
    for _ in range(3):
        if kind == "sdkde":
            r = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=ctx)
            outs.append((r.values, r.debiased_samples.values))
        else:
            outs.append((fk.kde_flash(tr, q, h, fk.KernelKind.LaplaceCorrected, True, ctx=ctx).values,))
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b), float(np.max(np.abs(a - b)))


@pytest.mark.parametrize("d,n,m,hs,seed", [(2, 33000, 3000, 0.35, 11), (5, 40961, 2049, 0.8, 12),
                                           (9, 36000, 5000, 1.3, 13), (16, 65600, 777, 2.0, 14)])
def test_spatial_path_other_dims(port, d, n, m, hs, seed):
    # the spatial order + tile skipping (n >= 32768) on dimensions other than the
    # BASELINE's 16, ragged sizes (not multiples of the 128 / 96-point tiles), a
    # clustered input: SD-KDE, KDE and Laplace on row subsamples vs the oracle
    rng = np.random.default_rng(seed)
    centres = rng.normal(scale=4.0, size=(6, d))
    tr = centres[rng.integers(0, 6, n)] + rng.normal(size=(n, d))
    q = centres[rng.integers(0, 6, m)] + rng.normal(size=(m, d)) * 1.3
    h = hs * np.sqrt(d / 2.0)
    c = fk.Context([0])
    r = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=c)
    s = fk.score_flash(tr, h, ctx=c).values
    st = c.skip_stats()
    kde = fk.kde_flash(tr, q, h, ctx=c).values
    lap = fk.kde_flash(tr, q, h, fk.KernelKind.LaplaceCorrected, True, ctx=c).values
    c.close()
    assert st["spatial_order"]
    rows = np.linspace(0, n - 1, 256).astype(int)
    qs = np.linspace(0, m - 1, 256).astype(int)
    th = os.cpu_count()
    ref_s = port.score_naive(tr, tr[rows], h, threads=th)
    ref_deb = tr[rows] + 0.5 * h * h * ref_s
    e = dict(score=max_rowwise_rel(s[rows], ref_s),
             debiased=max_rowwise_rel(r.debiased_samples.values[rows], ref_deb),
             kde=max_component_rel(kde[qs], port.kde_naive(tr, q[qs], h, threads=th)),
             laplace=max_rel_vs_peak(lap[qs], port.laplace_naive(tr, q[qs], h, threads=th)),
             sdkde=max_component_rel(r.values[qs],
                                     port.kde_naive(r.debiased_samples.values, q[qs], h, threads=th)))
    _report(f"spatial_d{d}", skipped=st["tiles_skipped"] / max(st["tiles_total"], 1), **e)
    assert e["score"] < TOL_SCORE and e["debiased"] < TOL_DEB
    assert e["kde"] < TOL_DENS and e["laplace"] < TOL_LAP and e["sdkde"] < TOL_DENS


def test_kernel_timing_brackets_the_pass_kernels(port):
    # fkde_gpu_last_kernel_timing: with OPT_TIMING the score / check / density kernels
    # are bracketed by events; each is positive where the kernel ran, within its phase
    tr, q = _mixture_inputs(port, 40000, 5000)
    h = port.sdkde_bandwidth(tr, port.silverman_prefactor(16))
    c = fk.Context([0])
    c.set_option(N.OPT_TIMING, 1)
    fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=c)
    k = c.last_kernel_timing()
    t = c.last_timing()
    c.set_option(N.OPT_TIMING, 0)
    fk.kde_flash(tr[:3000], q, h, ctx=c)
    off = c.last_kernel_timing()
    c.close()
    assert k[N.KT_SCORE] > 0 and k[N.KT_CHECK] > 0 and k[N.KT_DENSITY] > 0
    assert k[N.KT_SCORE] + k[N.KT_CHECK] <= t[N.T_SCORE] * 1.01
    assert k[N.KT_DENSITY] <= t[N.T_QUERY] * 1.01
    assert off == [0.0, 0.0, 0.0]


def test_repeated_host_calls_are_bitwise_and_checked(port):
    # repeated host-buffer calls (reused workspaces) give every result bitwise equal to
    # a timing-on call, for SD-KDE (with and without x^SD), KDE and the score; the
    # input checks run on every call (a non-finite input after clean calls is
    # reported, and the next clean call is clean again)
    tr, q = _mixture_inputs(port, 3000, 900)
    h = port.sdkde_bandwidth(tr, port.silverman_prefactor(16))
    eager = fk.Context([0])
    eager.set_option(N.OPT_TIMING, 1)   # (timing runs every call eagerly)
    ref_sd = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=eager)
    ref_kde = fk.kde_flash(tr, q, h, ctx=eager).values
    ref_s = fk.score_flash(tr, h, ctx=eager).values
    eager.close()
    c = fk.Context([0])
    for _ in range(4):
        r = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=c)
        assert np.array_equal(r.values, ref_sd.values)
        assert np.array_equal(r.debiased_samples.values, ref_sd.debiased_samples.values)
        assert np.array_equal(fk.kde_flash(tr, q, h, ctx=c).values, ref_kde)
        assert np.array_equal(fk.score_flash(tr, h, ctx=c).values, ref_s)
    lib = N.load()
    out = np.empty(900)
    dp = ctypes.POINTER(ctypes.c_double)
    idx = ctypes.c_size_t(0)
    for _ in range(3):   # densities only (no x^SD): its own graph
        rc = lib.fkde_gpu_sdkde(c.handle, tr.ctypes.data_as(dp), 3000, q.ctypes.data_as(dp), 900, 16,
                                h, h, out.ctypes.data_as(dp), None, ctypes.byref(idx))
        assert rc == N.OK and np.array_equal(out, ref_sd.values)
    bad = tr.copy()
    bad[17, 3] = np.nan
    rc = lib.fkde_gpu_sdkde(c.handle, bad.ctypes.data_as(dp), 3000, q.ctypes.data_as(dp), 900, 16,
                            h, h, out.ctypes.data_as(dp), None, ctypes.byref(idx))
    assert rc == N.NON_FINITE
    rc = lib.fkde_gpu_sdkde(c.handle, tr.ctypes.data_as(dp), 3000, q.ctypes.data_as(dp), 900, 16,
                            h, h, out.ctypes.data_as(dp), None, ctypes.byref(idx))
    assert rc == N.OK and np.array_equal(out, ref_sd.values)
    c.close()
