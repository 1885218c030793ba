"""Critical-chain view of the score kernel's clock64 trace (block 0, tiles 16..239):
per tile, when S became ready for the epilogue, when P was complete (slowest
quadrant), when GEMM2 passed p_full / o_empty and issued, when the drain passed
o_full, when GEMM1 passed b_full / s_free.  Prints mean waits per role.
    python -m paper_2602_10378_b200.build --trace ab/lib_trace.so
    FKDE_B200_LIB=ab/lib_trace.so python tools/trace_chain.py [n]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N, fixtures as F  # noqa: E402

NP = 3
E0 = 8


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
    X, _ = F.runtime_sweep_inputs(n, 8)
    h = F.sdkde_bandwidth(X)
    lib = N.load()
    ctx = fk.Context([0])
    dX = torch.from_numpy(X).cuda()
    dS = torch.empty((n, 16), dtype=torch.float64, device="cuda")
    rc = lib.fkde_gpu_score_device(ctx.handle, dX.data_ptr(), n, 16, h, dS.data_ptr())
    buf = torch.zeros(32 * 8 * 256, dtype=torch.int64, device="cuda")
    ctx.set_option(6, buf.data_ptr())
    rc = lib.fkde_gpu_score_device(ctx.handle, dX.data_ptr(), n, 16, h, dS.data_ptr())
    assert rc == 0, ctx.last_error()
    torch.cuda.synchronize()
    t = buf.view(32, 8, 256).cpu().numpy().astype(np.float64)
    t[t == 0] = np.nan
    T = range(16, 240)
    epi = {}
    for w in range(E0, E0 + 4 * NP):
        for k in T:
            if not np.isnan(t[w, 1, k]):
                epi.setdefault(k, []).append(w)
    rows = []
    for k in T:
        ws = epi.get(k, [])
        if len(ws) != 4:
            continue
        s_wait = np.mean([t[w, 1, k] - t[w, 0, k] for w in ws])
        s_ready = np.max([t[w, 1, k] for w in ws])
        ld = np.mean([t[w, 6, k] - t[w, 1, k] for w in ws])
        comp = np.mean([t[w, 7, k] - t[w, 1, k] for w in ws])
        pfull = np.max([t[w, 2, k] for w in ws])
        qspread = np.max([t[w, 2, k] for w in ws]) - np.min([t[w, 2, k] for w in ws])
        g1_b = t[1, 1, k] - t[1, 0, k]
        g1_s = t[1, 5, k] - t[1, 1, k]
        g1_iss = t[1, 4, k] - t[1, 5, k]
        g2_p = t[2, 3, k] - t[2, 2, k]
        g2_o = t[2, 5, k] - t[2, 3, k]
        g2_lag = t[2, 3, k] - pfull
        dr_w = np.mean([t[w, 5, k] - t[w, 4, k] for w in range(4, 8)])
        dr_lag = np.max([t[w, 5, k] for w in range(4, 8)]) - t[2, 5, k]
        rows.append((s_wait, ld, comp, qspread, g1_b, g1_s, g1_iss, g2_p, g2_o, g2_lag, dr_w, dr_lag,
                     s_ready - t[1, 4, k]))
    a = np.array(rows)
    names = ["epi s_full wait", "epi first ld", "epi ld..st", "p_full quadrant spread", "G1 b_full wait",
             "G1 s_free wait", "G1 issue", "G2 p_full wait", "G2 o_empty wait + issue", "G2 start - p_full",
             "drain o_full wait", "drain o_full pass - G2 issued", "S ready - G1 issued"]
    print(f"n={n}: {len(rows)} tiles of block 0 (cycles, mean / median)")
    for i, nm in enumerate(names):
        print(f"  {nm:32s} {np.nanmean(a[:, i]):8.0f} {np.nanmedian(a[:, i]):8.0f}")
    # tile interval
    g2 = t[2, 5, 16:240]
    g2 = g2[~np.isnan(g2)]
    print(f"  GEMM2 issue interval: {np.median(np.diff(g2)):.0f} cycles (median)")
    ctx.close()


if __name__ == "__main__":
    main()
