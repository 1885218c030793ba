"""Density-pass A/B: device time of the Gaussian KDE pass (n = 2^20 x m = 2^17
and 32k x 32k) for the library in FKDE_B200_LIB."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N, fixtures as F  # noqa: E402


def main():
    ctx = fk.Context([0])
    ctx.set_option(N.OPT_TIMING, 1)
    for n, m in ((1 << 20, 1 << 17), (32768, 32768)):
        X, Y = F.runtime_sweep_inputs(n, m)
        tr, q = fk.SampleSet(X), fk.SampleSet(Y)
        h = F.sdkde_bandwidth(X)
        ref = fk.kde_flash(tr, q, h, ctx=ctx).values
        ts = []
        for _ in range(5):
            fk.kde_flash(tr, q, h, ctx=ctx)
            ts.append(ctx.last_timing()[N.T_QUERY])
        print(f"{os.environ.get('FKDE_B200_LIB', 'current')[-16:]} kde n={n} m={m}: query pass "
              f"median {np.median(ts):.3f} ms  checksum {float(np.sum(ref)):.12e}", flush=True)


if __name__ == "__main__":
    main()
