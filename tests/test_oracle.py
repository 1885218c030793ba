"""CPU tests pinning the oracle restatement (oracle/fkde_oracle.c).

1. The reference's own known-answer tests (proj/tests/test_kernels.cpp:14-55,
   test_oracle.cpp:21-227, test_bandwidth.cpp) against the C port.
2. Bitwise agreement with the committed golden fixtures, which were produced by
   the reference's oracle itself (tests/golden/make_golden.py).
3. Bitwise agreement with oracle/_ref/libfkde_ref.so (the reference compiled
   from /root/reference) on fresh seeded inputs, when present.
"""
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, max_component_rel, max_rowwise_rel

PI = math.pi


# ---- test_kernels.cpp ------------------------------------------------------------
def test_gaussian_kernel_known_values(port):
    assert abs(port.gaussian_kernel(0.0, 1.0, 1) - 0.39894228040143268) < 1e-15
    assert abs(port.gaussian_kernel(0.0, 2.0, 2) - 0.039788735772973836) < 1e-15
    assert abs(port.gaussian_kernel(1.0, 1.0, 1) - 0.24197072451914337) < 1e-15


def test_gaussian_kernel_monotone(port):
    prev = math.inf
    r2 = 0.0
    while r2 <= 20.0:
        v = port.gaussian_kernel(r2, 0.8, 3)
        assert 0.0 < v < prev
        prev = v
        r2 += 0.37


def test_laplace_kernel_known_values(port):
    assert abs(port.laplace_corrected_kernel(0.0, 1.0, 2) - 0.3183098861837907) < 1e-15
    assert port.laplace_corrected_kernel(3.0, 1.0, 1) == 0.0
    assert port.laplace_corrected_kernel(4.0 * 2.25, 1.5, 2) == 0.0
    assert abs(port.laplace_corrected_kernel(4.0, 1.0, 1) + 0.026995483256594026) < 1e-15


def test_laplace_sign_rule(port):
    u = port.uniform01(123, 30000)
    for t in range(10000):
        h = 0.1 + 3.0 * u[3 * t]
        d = 1 + int(u[3 * t + 1] * 24)
        r2 = 10.0 * (2.0 + d) * h * h * u[3 * t + 2]
        v = port.laplace_corrected_kernel(r2, h, d)
        assert (v < 0.0) == (r2 > (2.0 + d) * h * h)


# ---- test_oracle.cpp -----------------------------------------------------------------
def test_kde_naive_hand_values(port):
    assert abs(port.kde_naive([0.0], [0.0], 1.0)[0] - 0.39894228040143268) < 1e-15
    assert abs(port.kde_naive([-1.0, 1.0], [0.0], 1.0)[0] - 0.24197072451914337) < 1e-15


def test_kde_translation_invariance(port):
    tr = port.random_gaussian(48, 2, 11)
    q = port.random_gaussian(16, 2, 12)
    base = port.kde_naive(tr, q, 0.7)
    sh = np.array([5.0, -2.0])
    assert max_component_rel(base, port.kde_naive(tr + sh, q + sh, 0.7)) < 1e-12


def test_score_known_answers(port):
    assert port.score_naive([1.5], [1.5], 0.8)[0, 0] == 0.0
    for h in (0.3, 1.0, 2.5):
        assert port.score_naive([-0.9, 0.9], [0.0], h)[0, 0] == 0.0
    s = port.score_naive([0.0], [0.35, -2.0], 1.0)
    assert abs(s[0, 0] + 0.35) < 1e-12 and abs(s[1, 0] - 2.0) < 1e-12


def test_score_underflow_names_row(port):
    import oracle as O
    with pytest.raises(O.OracleError) as e:
        port.score_naive([0.0], [0.001, 1e6], 1e-2)
    assert e.value.status == 3 and e.value.index == 1


def test_score_matches_fd_log_density(port):
    for d in (1, 2):
        tr = port.random_gaussian(64, d, 77 + d)
        ev = port.random_gaussian(12, d, 99 + d, 0.8)
        h = 0.6
        s = port.score_naive(tr, ev, h)
        step = 1e-5 * h
        fd = np.zeros_like(s)
        for j in range(ev.shape[0]):
            for k in range(d):
                p, m = ev.copy(), ev.copy()
                p[j, k] += step
                m[j, k] -= step
                fd[j, k] = (math.log(port.kde_naive(tr, p, h)[j]) -
                            math.log(port.kde_naive(tr, m, h)[j])) / (2 * step)
        assert max_rowwise_rel(s, fd, 1e-3) < 1e-5


def test_sdkde_known_answers(port):
    vals, deb = port.sdkde_naive([0.4], [-1.0, 0.0, 2.0], 0.9)
    assert deb[0, 0] == 0.4
    assert np.array_equal(vals, port.kde_naive([0.4], [-1.0, 0.0, 2.0], 0.9))
    vals, deb = port.sdkde_naive([-1.0, 1.0], [0.0], 0.5)
    assert abs(deb[0, 0] + deb[1, 0]) < 1e-15
    assert abs(vals[0] - 0.10812685292024610) < 1e-12


def test_sdkde_two_pass_script(port):
    train = [-1.3, -0.2, 0.5, 2.1]
    h, hs, q = 0.45, 0.6, 0.3
    deb = []
    for xi in train:
        num = den = 0.0
        for xj in train:
            diff = xi - xj
            phi = math.exp(-diff * diff / (2 * hs * hs))
            num += -diff * phi
            den += phi
        deb.append(xi + 0.5 * h * h * num / (hs * hs * den))
    exp = sum(math.exp(-(q - x) ** 2 / (2 * h * h)) / (math.sqrt(2 * PI) * h) for x in deb) / 4
    got, _ = port.sdkde_naive(train, [q], h, hs)
    assert abs(got[0] - exp) < 1e-12 * exp


def test_laplace_known_answers(port):
    assert abs(port.laplace_naive([[0.0, 0.0]], [[0.0, 0.0]], 1.0)[0] - 0.3183098861837907) < 1e-15
    v = port.laplace_naive([0.0], [2.0], 1.0)[0]
    assert abs(v + 0.026995483256594026) < 1e-15 and v < 0


def test_nonnegativity(port):
    tr = port.random_gaussian(40, 2, 5)
    q = port.random_gaussian(30, 2, 6, 4.0)
    for h in (0.05, 0.5, 2.0):
        assert (port.kde_naive(tr, q, h) >= 0).all()
        assert (port.sdkde_naive(tr, q, h)[0] >= 0).all()


def test_sharded_rows_bitwise(port):
    tr = port.random_gaussian(300, 3, 7)
    q = port.random_gaussian(97, 3, 8)
    full = port.kde_naive(tr, q, 0.6)
    assert np.array_equal(full, port.kde_naive(tr, q, 0.6, threads=4))
    assert np.array_equal(full[10:50], port.kde_naive(tr, q, 0.6, rows=(10, 50)))
    s = port.score_naive(tr, tr, 0.6)
    assert np.array_equal(s, port.score_naive(tr, tr, 0.6, threads=3))


# ---- test_bandwidth.cpp ----------------------------------------------------------------
def test_bandwidth_known_values(port):
    assert abs(port.silverman_prefactor(1) - (4.0 / 3.0) ** 0.2) < 1e-15
    x = np.array([[1.0], [2.0], [3.0], [4.0], [5.0]])
    sd = math.sqrt(2.5)
    assert abs(port.mean_stddev(x) - sd) < 1e-15
    assert abs(port.silverman_bandwidth(x) - sd * (4 / 3) ** 0.2 * 5 ** -0.2) < 1e-15
    assert abs(port.sdkde_bandwidth(x, 0.5) - 0.5 * sd * 5 ** (-1 / 9)) < 1e-15


# ---- golden fixtures (the reference's own outputs) ----------------------------------------
GOLDEN_CASES = sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz"))


@pytest.mark.parametrize("name", [c for c in GOLDEN_CASES if c.startswith("accept_")])
def test_port_matches_reference_golden_acceptance(port, name):
    g = golden(name)
    tr, q, h = g["train"], g["queries"], float(g["h"])
    assert np.array_equal(port.kde_naive(tr, q, h), g["kde"])
    assert np.array_equal(port.laplace_naive(tr, q, h), g["laplace"])
    assert np.array_equal(port.score_naive(tr, tr, h), g["score"])
    vals, deb = port.sdkde_naive(tr, q, h)
    assert np.array_equal(vals, g["sdkde"]) and np.array_equal(deb, g["debiased"])


def test_port_matches_reference_golden_engine_cases(port):
    g = golden("score_1024x16")
    assert np.array_equal(port.score_naive(g["train"], g["train"], float(g["h"]), threads=8),
                          g["score"])
    g = golden("kde_1d")
    assert np.array_equal(port.kde_naive(g["train"], g["queries"], float(g["h"])), g["values"])
    g = golden("laplace_2d")
    assert np.array_equal(port.laplace_naive(g["train"], g["queries"], float(g["h"])),
                          g["values"])
    g = golden("sdkde_512x16")
    vals, deb = port.sdkde_naive(g["train"], g["queries"], float(g["h"]), float(g["h_score"]))
    assert np.array_equal(vals, g["values"]) and np.array_equal(deb, g["debiased"])


def test_port_regenerates_reference_inputs(port):
    # the fixtures' inputs are exactly what the port's RNG produces
    g = golden("sdkde_512x16")
    assert np.array_equal(port.random_gaussian(512, 16, 57), g["train"])
    assert np.array_equal(port.random_gaussian(64, 16, 58), g["queries"])
    import oracle as O
    w, mu, s = O.default_mixture_16d()
    c = golden("config1")
    seed = int(c["seed"])
    assert seed == port.mix64(0 ^ port.mix64(4096))
    tr = port.sample_mixture(w, mu, s, 4096, seed)
    q = port.sample_mixture(w, mu, s, 4096, port.mix64(seed ^ 0x71))
    assert np.array_equal(tr[:8], c["train_head"]) and np.array_equal(q[:8], c["query_head"])
    assert port.sdkde_bandwidth(tr, port.silverman_prefactor(16)) == float(c["h"])
    assert port.silverman_bandwidth(tr) == float(c["h_silverman"])


def test_port_config1_against_reference_golden(port):
    import oracle as O
    w, mu, s = O.default_mixture_16d()
    c = golden("config1")
    seed = int(c["seed"])
    tr = port.sample_mixture(w, mu, s, 4096, seed)
    q = port.sample_mixture(w, mu, s, 4096, port.mix64(seed ^ 0x71))
    h = float(c["h"])
    rows = (0, 256)  # bounded CPU time; rows are independent
    assert np.array_equal(port.score_naive(tr, tr, h, rows=rows, threads=8), c["score"][:256])
    assert np.array_equal(port.kde_naive(tr, q, float(c["h_silverman"]), rows=rows, threads=8),
                          c["kde"][:256])


# ---- direct comparison with the reference build (only where /root/reference built) --------
def test_port_bitwise_equals_reference_build(port, ref):
    for (n, d, seed) in [(64, 1, 3), (301, 3, 4), (700, 16, 5)]:
        a = port.random_gaussian(n, d, seed, 1.3)
        assert np.array_equal(a, ref.random_gaussian(n, d, seed, 1.3))
        q = port.random_gaussian(n // 3 + 1, d, seed + 100)
        h = 0.7
        assert np.array_equal(port.kde_naive(a, q, h), ref.kde_naive(a, q, h))
        assert np.array_equal(port.laplace_naive(a, q, h), ref.laplace_naive(a, q, h))
        assert np.array_equal(port.score_naive(a, a, h, threads=4), ref.score_naive(a, a, h, threads=4))
        import oracle as O
        w, mu, s = O.default_mixture_16d()
        assert np.array_equal(port.sample_mixture(w, mu, s, 257, seed),
                              ref.sample_mixture(w, mu, s, 257, seed))
