"""Score-pass time and accuracy with / without the spatial order + tile skipping
(FKDE_OPT_SPATIAL), on the BASELINE mixture.  python tools/spatial_probe.py [n ...]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N  # noqa: E402
from paper_2602_10378_b200 import fixtures as F  # noqa: E402
from conftest import max_rel_global_floor, max_rowwise_rel  # noqa: E402


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [1 << 18, 1 << 20]
    P = O.get("port")
    lib = N.load()
    for n in sizes:
        X, Y = F.runtime_sweep_inputs(n, n // 8)
        h = F.sdkde_bandwidth(X)
        dX = torch.from_numpy(X).cuda()
        dS = torch.empty((n, 16), dtype=torch.float64, device="cuda")
        rows = np.linspace(0, n - 1, 1024).astype(int)
        ref = P.score_naive(X, X[rows], h, threads=os.cpu_count())
        for sp, fl in ((2, 0), (1, 0), (1, 1)):
            c = fk.Context([0])
            c.set_option(N.OPT_SPATIAL, sp)
            c.set_option(N.OPT_FLUSH_TILES, fl)
            c.set_option(N.OPT_TIMING, 1)
            stream = torch.cuda.ExternalStream(c.stream())
            ts = []
            for it in range(4):
                rc = lib.fkde_gpu_score_device(c.handle, dX.data_ptr(), n, 16, h, dS.data_ptr())
                assert rc == 0, c.last_error()
                t = c.last_timing()
                ts.append((t[N.T_PREP], t[N.T_SCORE], t[N.T_FINALIZE], t[N.T_TOTAL]))
            stream.synchronize()
            st = c.skip_stats()
            s = dS.cpu().numpy()[rows]
            prep, score, fin, tot = np.median(np.array(ts[1:]), axis=0)
            print(f"n={n} spatial={'on' if sp == 1 else 'off'} flush={fl} pred={os.environ.get('FKDE_SKIP_PRED', 'default')} prep={prep:.3f} score_kernel={score:.3f} "
                  f"finalize+={fin:.3f} total={tot:.3f} ms  skip={st}  "
                  f"err global={max_rel_global_floor(s, ref):.2e} rowwise={max_rowwise_rel(s, ref):.2e}",
                  flush=True)
            c.close()


if __name__ == "__main__":
    main()
