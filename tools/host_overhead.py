"""Wall time of one host-buffer API call vs the device phases it contains
(where does the non-kernel time of a small estimate go?)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N, fixtures as F  # noqa: E402


def main():
    ctx = fk.Context([0])
    ctx.set_option(N.OPT_TIMING, 1)
    for n, m in ((4096, 512), (32768, 4096), (262144, 32768)):
        X, Y = F.runtime_sweep_inputs(n, m)
        tr, q = fk.SampleSet(X), fk.SampleSet(Y)
        h = F.sdkde_bandwidth(X)
        for kind in ("kde", "sdkde"):
            f = (lambda: fk.kde_flash(tr, q, h, ctx=ctx)) if kind == "kde" else \
                (lambda: fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=ctx))
            f()
            ws = []
            for _ in range(5):
                t = time.perf_counter()
                f()
                ws.append(time.perf_counter() - t)
            tm = ctx.last_timing()
            print(f"{kind:5s} n={n:7d} m={m:6d}: wall {np.median(ws) * 1e3:8.3f} ms | device phases "
                  + " ".join(f"{v:.3f}" for v in tm), flush=True)


if __name__ == "__main__":
    main()
