"""Score-phase device time on the BASELINE mixture for one build / env variant
(A/B driver: run once per variant).  Options through argv: spatial=<0..3>
flush=<tiles> n=<points>.  Prints the score-phase time (check + score kernels),
visited tiles and the per-tile cost.
    FKDE_B200_LIB=ab/lib_x.so python tools/score_ab.py label spatial=0 flush=0"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N, fixtures as F  # noqa: E402


def main():
    label = sys.argv[1] if len(sys.argv) > 1 else "default"
    kv = dict(a.split("=") for a in sys.argv[2:])
    n = int(kv.get("n", 1 << 20))
    reps = int(kv.get("reps", 3))
    X, _ = F.runtime_sweep_inputs(n, 8)
    h = F.sdkde_bandwidth(X)
    lib = N.load()
    ctx = fk.Context([0])
    ctx.set_option(N.OPT_SPATIAL, int(kv.get("spatial", 0)))
    ctx.set_option(N.OPT_FLUSH_TILES, int(kv.get("flush", 0)))
    ctx.set_option(N.OPT_TIMING, 1)
    dX = torch.from_numpy(X).cuda()
    dS = torch.empty((n, 16), dtype=torch.float64, device="cuda")
    ts = []
    for _ in range(reps + 1):
        rc = lib.fkde_gpu_score_device(ctx.handle, dX.data_ptr(), n, 16, h, dS.data_ptr())
        assert rc == 0, ctx.last_error()
        ts.append(ctx.last_timing()[N.T_SCORE])
    st = ctx.skip_stats()
    score = float(np.median(ts[1:]))
    vis = st["tiles_total"] - st["tiles_skipped"] if st["spatial_order"] else st["tiles_total"]
    s = dS.cpu().numpy()
    print(f"{label:24s} n={n} score phase {score:8.3f} ms  visited tiles {vis}  "
          f"{score * 1e3 / max(vis, 1) * 148:.4f} us/tile/CTA  checksum {np.abs(s).sum():.10e}", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
