"""Small-bandwidth cost probe (no fp64 cliff): config-1 data (SD-KDE n = m = 4096,
d = 16) at the config's bandwidth h and at h/3, h/6 -- device time per call through
the device-resident ABI (graph-replayed), the rows sent to the direct-difference
kernel, and that kernel's share of the call (per-kernel CUDA times from
torch.profiler-free event bracketing: the whole call with and without the rows)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N  # noqa: E402
from paper_2602_10378_b200 import fixtures as F  # noqa: E402

n = m = 4096
X, Y = F.runtime_sweep_inputs(n, m, seed=0)
h0 = F.sdkde_bandwidth(X)
dX, dY = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
dO = torch.empty(m, dtype=torch.float64, device="cuda")
lib = N.load()
for div in (1, 3, 6):
    ctx = fk.Context([0])
    stream = torch.cuda.ExternalStream(ctx.stream())
    h = h0 / div

    def call():
        rc = lib.fkde_gpu_sdkde_device(ctx.handle, dX.data_ptr(), n, dY.data_ptr(), m, 16, h, h,
                                       dO.data_ptr())
        assert rc == 0, ctx.last_error()

    for _ in range(5):
        call()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(100):
        call()
    b.record(stream)
    b.synchronize()
    st = ctx.skip_stats()
    print(f"h = h0/{div} = {h:.4f}: {a.elapsed_time(b) / 100 * 1e3:7.1f} us per SD-KDE; direct rows "
          f"score {st['direct_rows']} / {n}, density {st['density']['direct_rows']} / {m}; "
          f"finite {bool(np.isfinite(dO.cpu().numpy()).all())}", flush=True)
    ctx.close()
