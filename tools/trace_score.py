"""clock64 trace of the score kernel's block 0 (FKDE_OPT_TRACE_PTR): where does a tile's time go?"""
import os
import sys

import numpy as np

NP = int(os.environ.get('FKDE_EPI_NP', '3'))   # epilogue warps per lane quadrant
G2 = 2 + 4 * NP                                # GEMM2 issuer warp
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
    buf = torch.zeros(16 * 8 * 256, dtype=torch.int64, device="cuda")
    ctx.set_option(6, buf.data_ptr())
    fk.score_flash(X, h, ctx=ctx)
    torch.cuda.synchronize()
    t = buf.view(16, 8, 256).cpu().numpy().astype(np.float64)
    lo, hi = 16, 200
    print(f"n={n} flush={flush}: tiles {lo}..{hi} of block 0 (cycles)")
    for w in range(2, 2 + 4 * NP):
        own = np.arange(lo, hi)
        own = own[t[w, 1, own] > 0]          # tiles this warp processed (its parity)
        per = np.diff(t[w, 1, own])
        s_wait = t[w, 1, own] - t[w, 0, own]
        ldl = t[w, 6, own] - t[w, 1, own]
        comp = t[w, 7, own] - t[w, 1, own]
        stl = t[w, 2, own] - t[w, 7, own]
        d = t[w, 3, own] - t[w, 2, own]
        d = d[(t[w, 3, own] > 0) & (d > 0) & (d < 1e6)]
        gap = t[w, 0, own[1:]] - t[w, 2, own[:-1]]
        dr = (t[w, 3, own[:-1]] > 0)
        gd = gap[dr] - (t[w, 3, own[:-1]] - t[w, 2, own[:-1]])[dr]
        ow = (t[w, 4, own] - t[w, 2, own])[t[w, 3, own] > 0]
        lw = (t[w, 5, own] - t[w, 4, own])[t[w, 3, own] > 0]
        aw = (t[w, 3, own] - t[w, 5, own])[t[w, 3, own] > 0]
        print(f"      drain: o_full wait {ow.mean():5.0f}  ld {lw.mean():5.0f}  accumulate {aw.mean():5.0f}; "
              f"after-drain gap {gd.mean():5.0f}  no-drain gap {gap[~dr].mean():5.0f}")
        print(f"  warp {w}: {own.size} tiles, period {per.mean():6.0f}  s_full wait {s_wait.mean():5.0f}  "
              f"first ld {ldl.mean():4.0f}  ld+exp+st issue {comp.mean():6.0f}  st wait+arrive {stl.mean():4.0f}  "
              f"drain {d.mean() if d.size else 0:5.0f} ({d.size})  other {gap.mean():5.0f}")
    bwait = t[1, 1, lo:hi] - t[1, 0, lo:hi]
    pwait = t[G2, 3, lo:hi] - t[G2, 2, lo:hi]
    g2 = t[G2, 5, lo:hi] - t[G2, 3, lo:hi]
    fwait = t[1, 5, lo:hi] - t[1, 1, lo:hi]
    g1 = t[1, 4, lo:hi] - t[1, 5, lo:hi]
    print(f"  GEMM1 warp: b_full wait {bwait.mean():.0f}  s_free wait {fwait.mean():.0f}  GEMM1 issue {g1.mean():.0f}")
    print(f"  GEMM2 warp: p_full wait {pwait.mean():.0f}  GEMM2 issue {g2.mean():.0f}")
    extra(t, lo, hi)
    ring(t, lo, hi)




def extra(t, lo=16, hi=200):
    arr = t[2:2 + 4 * NP, 2, lo:hi]            # P-arrive times of the epilogue warps (0 = not its tile)
    arr = np.where(arr > 0, arr, np.nan)
    spread = np.nanmax(arr, 0) - np.nanmin(arr, 0)
    print(f"  P-arrive spread across warps per tile: mean {spread.mean():.0f} max {spread.max():.0f}")
    g1 = t[1, 4, lo:hi]                # GEMM1(t) issued
    ready = np.nanmin(np.where(t[2:2 + 4 * NP, 1, lo:hi] > 0, t[2:2 + 4 * NP, 1, lo:hi], np.nan), 0)
    print(f"  GEMM1 issue -> first s_full pass: mean {np.mean(ready - g1):.0f}")
    per = np.diff(t[1, 4, lo:hi + 1])
    print(f"  GEMM1 tile period: mean {per.mean():.0f}")
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


def ring(t, lo=16, hi=200, nbuf=int(os.environ.get("FKDE_SBUF", "4"))):
    """Life of one S/P buffer use: GEMM1 issued -> first epilogue warp starts ->
    last quadrant's P arrives -> GEMM2 passes p_full -> GEMM2 issued -> GEMM1
    of the buffer's next tile issued."""
    E = slice(2, 2 + 4 * NP)
    g1 = t[1, 4, lo:hi]
    st = np.nanmin(np.where(t[E, 1, lo:hi] > 0, t[E, 1, lo:hi], np.nan), 0)
    pl = np.nanmax(np.where(t[E, 2, lo:hi] > 0, t[E, 2, lo:hi], np.nan), 0)
    pf = np.nanmin(np.where(t[E, 2, lo:hi] > 0, t[E, 2, lo:hi], np.nan), 0)
    g2p = t[G2, 3, lo:hi]
    g2d = t[G2, 5, lo:hi]
    g1n = t[1, 4, lo + nbuf:hi + nbuf]
    print(f"  ring ({nbuf} buffers): GEMM1->epi start {np.mean(st - g1):.0f}  epi start->first P "
          f"{np.mean(pf - st):.0f}  first->last P {np.mean(pl - pf):.0f}  last P->GEMM2 pass "
          f"{np.mean(g2p - pl):.0f}  GEMM2 issue {np.mean(g2d - g2p):.0f}  GEMM2 issued->next GEMM1 "
          f"{np.mean(g1n - g2d):.0f}  | cycle {np.mean(g1n - g1):.0f} = {np.mean(g1n - g1) / nbuf:.0f}/tile")


if __name__ == "__main__":
    main()
