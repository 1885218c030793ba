"""Score-pass time vs column-split count on the spatial order (load-balance probe).
python tools/splits_probe.py N [splits ...]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N  # noqa: E402
from paper_2602_10378_b200 import fixtures as F  # noqa: E402

n = int(sys.argv[1])
splits = [int(a) for a in sys.argv[2:]] or [0, 1, 12, 24, 48, 64]
X, _ = F.runtime_sweep_inputs(n, 16)
h = F.sdkde_bandwidth(X)
dX = torch.from_numpy(X).cuda()
dS = torch.empty((n, 16), dtype=torch.float64, device="cuda")
lib = N.load()
ref = None
for s in splits:
    c = fk.Context([0])
    c.set_option(N.OPT_SPATIAL, 1)
    c.set_option(N.OPT_SPLITS, s)
    c.set_option(N.OPT_TIMING, 1)
    ts = []
    for _ in range(4):
        assert lib.fkde_gpu_score_device(c.handle, dX.data_ptr(), n, 16, h, dS.data_ptr()) == 0, c.last_error()
        t = c.last_timing()
        ts.append((t[N.T_SCORE], t[N.T_TOTAL]))
    torch.cuda.synchronize()
    out = dS.cpu().numpy()
    if ref is None:
        ref = out
    diff = float(np.max(np.abs(out - ref)) / np.max(np.abs(ref)))
    sc, tot = np.median(np.array(ts[1:]), axis=0)
    print(f"n={n} splits={s} score_phase={sc:.3f} total={tot:.3f} ms maxdiff_vs_first={diff:.2e}", flush=True)
    c.close()
