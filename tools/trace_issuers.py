"""clock64 trace of the score kernel's GEMM1 / GEMM2 issuers (block 0).
    FKDE_B200_LIB=ab/lib_trace.so python tools/trace_issuers.py [n]"""
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
    ctx.set_option(N.OPT_SPATIAL, int(os.environ.get("SPATIAL", "1")))
    fk.score_flash(X, h, ctx=ctx)
    buf = torch.zeros(32 * 8 * 256, dtype=torch.int64, device="cuda")
    ctx.set_option(6, buf.data_ptr())
    fk.score_flash(X, h, ctx=ctx)
    torch.cuda.synchronize()
    t = buf.view(32, 8, 256).cpu().numpy().astype(np.float64)
    g1, g2 = t[1], t[2]
    base = g1[0][g1[0] > 0].min()
    print("tile  G1: bfull  sfree  issue | G2: pfull  issue+commit | G1 period")
    for k in range(40, 80):
        print(f"{k:4d} {g1[1, k] - g1[0, k]:7.0f} {g1[5, k] - g1[1, k]:6.0f} {g1[4, k] - g1[5, k]:6.0f} | "
              f"{g2[3, k] - g2[2, k]:7.0f} {g2[5, k] - g2[3, k]:7.0f} | {g1[4, k] - g1[4, k - 1]:6.0f}")


if __name__ == "__main__":
    main()
