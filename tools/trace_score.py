"""clock64 trace of the score kernel's block 0 (FKDE_OPT_TRACE_PTR): where does a tile's time go?"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N, fixtures as F  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    flush = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    X, _ = F.runtime_sweep_inputs(n, 8)
    h = F.sdkde_bandwidth(X)
    ctx = fk.Context([0])
    ctx.set_option(N.OPT_FLUSH_TILES, flush)
    fk.score_flash(X, h, ctx=ctx)
    buf = torch.zeros(11 * 8 * 256, dtype=torch.int64, device="cuda")
    ctx.set_option(6, buf.data_ptr())
    fk.score_flash(X, h, ctx=ctx)
    torch.cuda.synchronize()
    t = buf.view(11, 8, 256).cpu().numpy().astype(np.float64)
    lo, hi = 16, 200
    print(f"n={n} flush={flush}: tiles {lo}..{hi} of block 0 (cycles)")
    per = np.diff(t[2, 0, lo:hi + 1])
    print(f"  epilogue tile period (warp 2): mean {per.mean():.0f}  min {per.min():.0f}  max {per.max():.0f}")
    for w in range(2, 10):
        ldl = t[w, 6, lo:hi] - t[w, 1, lo:hi]
        cmp_ = t[w, 7, lo:hi] - t[w, 6, lo:hi]
        stl = t[w, 2, lo:hi] - t[w, 7, lo:hi]
        print(f"  warp {w}: LDTM latency {ldl.mean():5.0f}  compute {cmp_.mean():5.0f}  STTM wait+arrive {stl.mean():5.0f}")
    for w in range(2, 10):
        s_wait = t[w, 1, lo:hi] - t[w, 0, lo:hi]
        comp = t[w, 2, lo:hi] - t[w, 1, lo:hi]
        d = t[w, 3, lo:hi] - t[w, 2, lo:hi]
        d = d[(t[w, 3, lo:hi] > 0) & (d > 0) & (d < 1e6)]
        print(f"  warp {w}: s_full wait {s_wait.mean():6.0f}  ld+exp+P store {comp.mean():6.0f}  "
              f"drain {d.mean() if d.size else 0:6.0f} ({d.size} drains)")
    bwait = t[1, 1, lo:hi] - t[1, 0, lo:hi]
    pwait = t[10, 3, lo:hi] - t[10, 2, lo:hi]
    g2 = t[10, 5, lo:hi] - t[10, 3, lo:hi]
    g1 = t[1, 4, lo:hi] - t[1, 1, lo:hi]
    print(f"  GEMM1 warp: b_full+s_free wait {bwait.mean():.0f}  GEMM1 issue {g1.mean():.0f}")
    print(f"  GEMM2 warp: p_full wait {pwait.mean():.0f}  GEMM2 issue {g2.mean():.0f}")
    extra(t, lo, hi)




def extra(t, lo=16, hi=200):
    arr = t[2:10, 2, lo:hi]            # P-arrive times of the 8 epilogue warps
    spread = arr.max(0) - arr.min(0)
    print(f"  P-arrive spread across warps per tile: mean {spread.mean():.0f} max {spread.max():.0f}")
    g1 = t[1, 4, lo:hi]                # GEMM1(t) issued
    ready = t[2:10, 1, lo:hi].min(0)   # first warp passing s_full(t)
    print(f"  GEMM1 issue -> first s_full pass: mean {np.mean(ready - g1):.0f}")
    last_arrive = arr.max(0)
    print(f"  GEMM1(t) issue minus last P-arrive(t-3): {np.mean(g1[3:] - last_arrive[:-3]):.0f}")
    print(f"  GEMM1(t) issue minus last P-arrive(t-2): {np.mean(g1[2:] - last_arrive[:-2]):.0f}")


def mma_timeline(t, lo=16, hi=200):
    g1_issue = t[1, 4, lo:hi] - t[1, 1, lo:hi]
    # gemm2 for tile i is called in iteration i+2; slots 2/3 are indexed by that tile
    g2_issue = t[1, 0, lo + 3:hi + 3] - t[1, 3, lo + 1:hi + 1]
    print(f"  MMA: GEMM1 issue {g1_issue.mean():.0f}  GEMM2 issue (+loop) {g2_issue.mean():.0f}  "
          f"b_full wait {np.mean(t[1, 1, lo:hi] - t[1, 0, lo:hi]):.0f}  "
          f"p_full wait {np.mean(t[1, 3, lo:hi] - t[1, 2, lo:hi]):.0f}  "
          f"iteration {np.mean(np.diff(t[1, 0, lo:hi + 1])):.0f}")


if __name__ == "__main__":
    main()
