"""Quick on-device diagnostic: run each pass at small sizes and print the
error against the CPU oracle."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def rowwise(a, b, floor=1e-2):
    scale = np.maximum(np.abs(a).max(axis=1, keepdims=True), np.abs(b).max(axis=1, keepdims=True))
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), floor * scale)
    return float(np.max(np.abs(a - b) / den))


def main():
    P = O.get("port")
    for eng in ["tc"]:
        ctx = fk.Context([0])
        for (n, m, d, h) in [(200, 50, 2, 0.5), (1024, 300, 16, 0.9), (4096, 4096, 16, 1.5)]:
            tr = P.random_gaussian(n, d, 41)
            q = P.random_gaussian(m, d, 42)
            t0 = time.time()
            try:
                kd = fk.kde_flash(tr, q, h, ctx=ctx).values
            except Exception as e:  # noqa
                print(eng, "kde FAILED", n, m, d, e, flush=True)
                raise
            t1 = time.time()
            ref = P.kde_naive(tr, q, h, threads=8)
            print(f"{eng} kde n={n} m={m} d={d}: rel={rel(kd, ref):.3e} ({t1-t0:.3f}s)", flush=True)
            la = fk.kde_flash(tr, q, h, fk.KernelKind.LaplaceCorrected, True, ctx=ctx).values
            lref = P.laplace_naive(tr, q, h, threads=8)
            print(f"{eng} laplace: peak-rel={np.max(np.abs(la-lref))/np.max(np.abs(lref)):.3e}",
                  flush=True)
            sc = fk.score_flash(tr, h, ctx=ctx).values
            sref = P.score_naive(tr, tr, h, threads=8)
            print(f"{eng} score: rowwise={rowwise(sc, sref):.3e}", flush=True)
            sd = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=ctx)
            dref, debref = P.sdkde_naive(tr, q, h, threads=8)
            print(f"{eng} sdkde: rel={rel(sd.values, dref):.3e} "
                  f"debiased rowwise={rowwise(sd.debiased_samples.values, debref):.3e}",
                  flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
