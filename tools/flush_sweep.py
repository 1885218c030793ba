"""Score-pass accuracy / speed vs FKDE_OPT_FLUSH_TILES (tensor-core accumulation length)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from conftest import golden, max_rel_global_floor, max_rowwise_rel  # noqa: E402
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N, fixtures as F  # noqa: E402


def main():
    c = golden("config1")
    tr, q = F.runtime_sweep_inputs(4096, 4096)
    h = float(c["h"])
    big, bq = F.runtime_sweep_inputs(1 << 18, 1 << 14)
    hb = F.sdkde_bandwidth(big)
    for flush in [int(a) for a in (sys.argv[1:] or ["1", "2", "4", "8", "1000000"])]:
        ctx = fk.Context([0])
        try:
            ctx.set_option(N.OPT_FLUSH_TILES, flush)
        except Exception:
            if flush != 1000000:
                ctx.close()
                continue
        s = fk.score_flash(tr, h, ctx=ctx).values
        rw, gl = max_rowwise_rel(s, c["score"]), max_rel_global_floor(s, c["score"])
        ctx.set_option(N.OPT_TIMING, 1)
        fk.sdkde_flash(big, bq, fk.Bandwidth.uniform(hb), ctx=ctx, want_debiased=False)
        ts = []
        for _ in range(7):
            fk.sdkde_flash(big, bq, fk.Bandwidth.uniform(hb), ctx=ctx, want_debiased=False)
            ts.append(ctx.last_timing()[N.T_SCORE])
        print(f"{os.environ.get('FKDE_B200_LIB', 'current')[-24:]} flush={flush:8d}: config1 score "
              f"rowwise={rw:.3e} global={gl:.3e} | n=262144 score pass min {min(ts):.2f} "
              f"median {sorted(ts)[3]:.2f} ms", flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
