"""Per-SM-sub-partition view of the score kernel's clock64 trace (block 0):
how much of the time at least one epilogue warp of a sub-partition is inside
its ld+exp+st phase, the first-chunk tcgen05.ld latency and the drain split.
    FKDE_B200_LIB=ab/lib_trace.so python tools/trace_cover.py [n]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N, fixtures as F  # noqa: E402

NP = int(os.environ.get("FKDE_SCORE_NP", "3"))
E0 = 8          # first epilogue warp (0-3 control, 4-7 O drain warps)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
    X, _ = F.runtime_sweep_inputs(n, 8)
    h = F.sdkde_bandwidth(X)
    ctx = fk.Context([0])
    fk.score_flash(X, h, ctx=ctx)
    buf = torch.zeros(32 * 8 * 256, dtype=torch.int64, device="cuda")
    ctx.set_option(6, buf.data_ptr())
    fk.score_flash(X, h, ctx=ctx)
    torch.cuda.synchronize()
    t = buf.view(32, 8, 256).cpu().numpy().astype(np.float64)
    lo, hi = 16, 200
    t0 = np.nanmin(np.where(t[E0:E0 + 4 * NP, 1, lo:hi] > 0, t[E0:E0 + 4 * NP, 1, lo:hi], np.nan))
    t1 = np.nanmax(np.where(t[E0:E0 + 4 * NP, 7, lo:hi] > 0, t[E0:E0 + 4 * NP, 7, lo:hi], np.nan))
    span = t1 - t0
    ntiles = hi - lo
    print(f"n={n}: window {span:.0f} cycles for ~{ntiles} tiles = {span / ntiles:.0f}/tile")
    for s in range(4):
        warps = [w for w in range(E0, E0 + 4 * NP) if w % 4 == s]
        cov = np.zeros(int(span) + 1, dtype=np.int8)
        for w in warps:
            for k in range(lo, hi):
                a, b = t[w, 1, k], t[w, 7, k]
                if a > 0 and b > 0 and a >= t0 and b <= t1:
                    cov[int(a - t0):int(b - t0)] += 1
        frac = [(cov >= j).mean() for j in (1, 2, 3)]
        comp_s = np.concatenate([(t[w, 7, lo:hi] - t[w, 1, lo:hi])[(t[w, 7, lo:hi] > 0) & (t[w, 1, lo:hi] > 0)]
                                 for w in warps])
        wait_s = np.concatenate([(t[w, 1, lo:hi] - t[w, 0, lo:hi])[(t[w, 1, lo:hi] > 0) & (t[w, 0, lo:hi] > 0)]
                                 for w in warps])
        print(f"  SMSP {s} (warps {warps}): >=1 warp computing {frac[0]*100:.1f}%  >=2 {frac[1]*100:.1f}%  3 {frac[2]*100:.1f}%"
              f" | per tile: s_full wait {wait_s.mean():5.0f}, ld..st {comp_s.mean():5.0f} cycles")
    E = range(E0, E0 + 4 * NP)
    ldl = np.concatenate([(t[w, 6, lo:hi] - t[w, 1, lo:hi])[t[w, 6, lo:hi] > 0] for w in E])
    print(f"  first-chunk ld latency (s_full pass -> ld done): mean {ldl.mean():.0f} median {np.median(ldl):.0f}")
    dw = np.concatenate([(t[w, 5, :] - t[w, 4, :])[(t[w, 4, :] > 0) & (t[w, 5, :] > 0)] for w in range(4, 8)])
    print(f"  drain warps: o_full wait per sub-unit mean {dw.mean():.0f} (includes idle time)")
    comp = np.concatenate([(t[w, 7, lo:hi] - t[w, 6, lo:hi])[t[w, 6, lo:hi] > 0] for w in E])
    print(f"  compute after first ld (3 chunks): mean {comp.mean():.0f}")


if __name__ == "__main__":
    main()
