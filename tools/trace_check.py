"""clock64 trace of the check pass (kModeCheck) of block 0: per-tile GEMM1 issue
timeline and epilogue waits.  Build: python -m paper_2602_10378_b200.build --trace ab/lib_trace.so
    FKDE_B200_LIB=ab/lib_trace.so FKDE_TRACE_CHECK=1 python tools/trace_check.py [n]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N, fixtures as F  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
    X, _ = F.runtime_sweep_inputs(n, 8)
    h = F.sdkde_bandwidth(X)
    ctx = fk.Context([0])
    ctx.set_option(N.OPT_SPATIAL, 1)
    fk.score_flash(X, h, ctx=ctx)
    buf = torch.zeros(32 * 8 * 256, dtype=torch.int64, device="cuda")
    ctx.set_option(6, buf.data_ptr())
    fk.score_flash(X, h, ctx=ctx)
    torch.cuda.synchronize()
    t = buf.view(32, 8, 256).cpu().numpy().astype(np.float64)
    g = t[1]   # GEMM1 warp: 0 before b_full, 1 after b_full, 5 after s_empty, 4 after commit
    ok = (g[0] > 0) & (g[4] > 0)
    idx = np.nonzero(ok)[0]
    base = g[0, idx[0]]
    print("GEMM1 per tile (cycles rel. to first): tile, b_full wait, s_empty wait, issue, period")
    for k in idx[:60]:
        per = g[4, k] - g[4, k - 1] if k > 0 and g[4, k - 1] > 0 else 0
        print(f"  {k:3d} t={g[0, k] - base:9.0f} bfull={g[1, k] - g[0, k]:6.0f} sempty={g[5, k] - g[1, k]:6.0f} "
              f"issue={g[4, k] - g[5, k]:6.0f} period={per:6.0f}")
    print("epilogue warps (2..9): tile, s_full wait, ld, rest")
    for w in range(2, 10):
        e = t[w]
        ks = np.nonzero((e[0] > 0) & (e[7] > 0))[0][:6]
        for k in ks:
            print(f"  w{w} tile {k:3d} t={e[0, k] - base:9.0f} sfull_wait={e[1, k] - e[0, k]:6.0f} "
                  f"ld={e[6, k] - e[1, k]:6.0f} rest={e[7, k] - e[6, k]:6.0f}")
    periods = np.diff(g[4, idx])
    print(f"GEMM1 median period {np.median(periods):.0f} cycles, mean {periods.mean():.0f}")


if __name__ == "__main__":
    main()
