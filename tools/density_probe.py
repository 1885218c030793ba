"""Density pass with / without the spatial order and tile skipping (FKDE_OPT_SPATIAL
2 = off, 3 = order only, 1 = order + skipping): time, skip statistics and the
largest relative change against the unordered pass.
    python tools/density_probe.py [case ...]   cases: sdkde1m sdkde32k kde262k lap262k"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N  # noqa: E402
from paper_2602_10378_b200 import fixtures as F  # noqa: E402

CASES = {"sdkde1m": ("sdkde", 1 << 20, 1 << 17), "sdkde32k": ("sdkde", 1 << 15, 1 << 15),
         "kde262k": ("kde", 1 << 18, 1 << 16), "lap262k": ("lap", 1 << 18, 1 << 16)}


def run(kind, n, m):
    X, Y = F.runtime_sweep_inputs(n, m)
    h = F.sdkde_bandwidth(X) if kind == "sdkde" else F.silverman_bandwidth(X)
    dX, dY = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    dO = torch.empty(m, dtype=torch.float64, device="cuda")
    lib = N.load()
    base = None
    for sp in (2, 3, 1):
        c = fk.Context([0])
        c.set_option(N.OPT_SPATIAL, sp)
        c.set_option(N.OPT_TIMING, 1)
        ts = []
        for _ in range(3):
            if kind == "sdkde":
                rc = lib.fkde_gpu_sdkde_device(c.handle, dX.data_ptr(), n, dY.data_ptr(), m, 16, h, h, dO.data_ptr())
            else:
                rc = lib.fkde_gpu_kde_device(c.handle, dX.data_ptr(), n, dY.data_ptr(), m, 16, h,
                                             0 if kind == "kde" else 1, 1, dO.data_ptr())
            assert rc == 0, c.last_error()
            t = c.last_timing()
            ts.append((t[N.T_QUERY] + t[N.T_REDUCE], t[N.T_TOTAL]))
        torch.cuda.synchronize()
        out = dO.cpu().numpy().copy()
        st = c.skip_stats()
        c.close()
        if base is None:
            base = out
        rel = np.abs(out - base) / np.maximum(np.abs(base), 1e-300)
        peak = float(np.max(np.abs(out - base)) / np.max(np.abs(base)))
        dens, tot = np.median(np.array(ts[1:]), axis=0)
        print(f"{kind} n={n} m={m} spatial={sp} density_phase={dens:.3f} total={tot:.3f} ms "
              f"max_rel_vs_off={float(rel.max()):.2e} vs_peak={peak:.2e} finite={bool(np.isfinite(out).all())} "
              f"density_stats={st['density']}", flush=True)


for name in sys.argv[1:] or list(CASES):
    run(*CASES[name])
