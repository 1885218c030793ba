"""Score error of the tensor-core path vs data spread (|y|^2/2 = |x-mu|^2 log2(e)/(2h^2)).
Clusters in 4-D / 16-D pushed apart by a factor f; prints the worst rows' |y|^2/2, S and
the error split, for several O-drain intervals (FKDE_OPT_FLUSH_TILES)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N  # noqa: E402
from conftest import max_rel_global_floor, max_rowwise_rel  # noqa: E402


def rowwise_per_row(a, b, row_floor=1e-2):
    rs = np.maximum(np.abs(a).max(axis=1), np.abs(b).max(axis=1))[:, None]
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), row_floor * rs)
    return (np.abs(a - b) / den).max(axis=1)


def main():
    P = O.get("port")
    for d, h, n in ((4, 0.62, 2000), (16, 1.2, 4096)):
        for f in (0.0, 2.5, 5.0, 10.0, 14.0):
            k = 4
            centres = np.zeros((k, d))
            for c in range(k):
                centres[c, c % d] = f * (1 if c % 2 == 0 else -1) if d == 4 else 0
            if d == 16:
                rng = np.random.default_rng(5)
                centres = rng.normal(size=(k, d)) * f / 3
            tr = P.random_gaussian(n, d, 91) + np.repeat(centres, n // k, axis=0)
            ref = P.score_naive(tr, tr, h, threads=os.cpu_count())
            mu = tr.mean(0)
            y2 = ((tr - mu) ** 2).sum(1) * 1.4426950408889634 / (2 * h * h)
            for flush in (1, 2, 4):
                c = fk.Context([0])
                c.set_option(N.OPT_FLUSH_TILES, flush)
                s = fk.score_flash(tr, h, ctx=c).values
                acc = fk.score_accumulate(tr, h, ctx=c)
                c.close()
                rr = rowwise_per_row(s, ref)
                w = np.argsort(rr)[-3:]
                print(f"d={d} f={f:5.1f} flush={flush} max|y|^2/2={y2.max():7.1f} "
                      f"global={max_rel_global_floor(s, ref):.2e} rowwise={max_rowwise_rel(s, ref):.2e} "
                      f"worst rows: " + " ".join(
                          f"[y2/2={y2[i]:.0f} S={acc.phi_sum[i]:.3g} |s|max={np.abs(ref[i]).max():.3g} err={rr[i]:.1e}]"
                          for i in w), flush=True)


if __name__ == "__main__":
    main()
