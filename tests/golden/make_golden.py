"""Regenerate tests/golden/*.npz from the REFERENCE's own oracle.

Runs only in the build container (needs oracle/_ref/libfkde_ref.so, compiled
from /root/reference by ``make -C oracle ref``).  The fixtures pin both the
C restatement (tests/test_oracle.py) and the GPU engine (tests/test_gpu_*.py)
to the reference's outputs on the reference's own seeded inputs.

Cases mirror the reference tests:
  score_1024x16      test_engine.cpp:99-105 (seed 41, h=0.9; first 1024 rows)
  kde_1d             test_engine.cpp:123-130 (seeds 51/52, h=0.3)
  laplace_2d         test_engine.cpp:132-143 (seeds 53/54 scale 2, h=0.4)
  sdkde_512x16       test_engine.cpp:156-166 (seeds 57/58, h=0.8)
  accept_<i>         acceptance_main.cpp:65-135 instances (n<=1024)
  config1            BASELINE config 1: 16-D mixture, n=m=4096, sweep seeds
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import oracle as O  # noqa: E402


def cell_data_seed(R, seed, n):
    # sweep.cpp:67-69
    return R.mix64(seed ^ R.mix64(n))


def main():
    R = O.get("reference")
    out = {}

    tr = R.random_gaussian(1024, 16, 41)
    out["score_1024x16"] = dict(train=tr, h=0.9, score=R.score_naive(tr, tr, 0.9, threads=8))

    tr = R.random_gaussian(1024, 1, 51)
    q = R.random_gaussian(128, 1, 52)
    out["kde_1d"] = dict(train=tr, queries=q, h=0.3, values=R.kde_naive(tr, q, 0.3))

    tr = R.random_gaussian(512, 2, 53)
    q = R.random_gaussian(64, 2, 54, 2.0)
    out["laplace_2d"] = dict(train=tr, queries=q, h=0.4, values=R.laplace_naive(tr, q, 0.4))

    tr = R.random_gaussian(512, 16, 57)
    q = R.random_gaussian(64, 16, 58)
    vals = np.empty(64)
    deb = np.empty((512, 16))
    f = R.lib.fkr_sdkde_naive
    f.argtypes = [O._c_double_p, O._size_t, O._c_double_p, O._size_t, O._size_t, O.ctypes.c_double,
                  O.ctypes.c_double, O._c_double_p, O._c_double_p, O.ctypes.c_void_p]
    st = f(tr.ctypes.data_as(O._c_double_p), 512, q.ctypes.data_as(O._c_double_p),
                               64, 16, 0.8, 0.8, vals.ctypes.data_as(O._c_double_p),
                               deb.ctypes.data_as(O._c_double_p), None)
    assert st == 0
    out["sdkde_512x16"] = dict(train=tr, queries=q, h=0.8, h_score=0.8, values=vals, debiased=deb)

    # acceptance_main.cpp:65-83 instance generator, n <= 1024 only
    ns = [3, 64, 1024, 4096]
    ds = [1, 2, 16]
    for i in range(50):
        n = ns[(i % 12) // 3]
        d = ds[i % 3]
        if n > 1024:
            continue
        tr = R.random_gaussian(n, d, 1000 + i, 1.5)
        q = R.random_gaussian(max(1, n // 8), d, 2000 + i, 1.5)
        h = (0.8 + 0.8 * R.uniform01(3000 + i, 1)[0]) * 0.75 * np.sqrt(float(d))
        kde = R.kde_naive(tr, q, h)
        lap = R.laplace_naive(tr, q, h)
        score = R.score_naive(tr, tr, h)
        sd, deb = R.sdkde_naive(tr, q, h)
        out[f"accept_{i:02d}"] = dict(train=tr, queries=q, h=h, kde=kde, laplace=lap,
                                      score=score, sdkde=sd, debiased=deb)

    # BASELINE config 1: 16-D default mixture, runtime-sweep seeds (sweep.cpp:173-177)
    w, mu, s = O.default_mixture_16d()
    n = 4096
    cs = cell_data_seed(R, 0, n)
    tr = R.sample_mixture(w, mu, s, n, cs)
    q = R.sample_mixture(w, mu, s, n, R.mix64(cs ^ 0x71))
    h = R.sdkde_bandwidth(tr, R.silverman_prefactor(16))
    hs = R.silverman_bandwidth(tr)
    score = R.score_naive(tr, tr, h, threads=8)
    deb = tr + (0.5 * h * h) * score
    vals = R.kde_naive(deb, q, h, threads=8)
    kde_vals = R.kde_naive(tr, q, hs, threads=8)
    lap_vals = R.laplace_naive(tr, q, hs, threads=8)
    out["config1"] = dict(seed=np.uint64(cs), h=h, h_silverman=hs, train_head=tr[:8],
                          query_head=q[:8], score=score, sdkde=vals, kde=kde_vals,
                          laplace=lap_vals)

    for name, arrays in out.items():
        np.savez_compressed(os.path.join(HERE, name + ".npz"),
                            **{k: np.asarray(v) for k, v in arrays.items()})
    print(f"wrote {len(out)} fixtures to {HERE}")


if __name__ == "__main__":
    main()
