"""One SD-KDE at BASELINE config 5 (or n, m given) through the device API, for ncu.
    python tools/prof_sdkde.py [n m reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N  # noqa: E402
from paper_2602_10378_b200 import fixtures as F  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 17
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
X, Y = F.runtime_sweep_inputs(n, m)
h = F.sdkde_bandwidth(X)
dX, dY = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
dO = torch.empty(m, dtype=torch.float64, device="cuda")
c = fk.Context([0])
c.set_option(N.OPT_TIMING, 1)   # eager launches (no graph) for the profiler
lib = N.load()
for _ in range(reps):
    assert lib.fkde_gpu_sdkde_device(c.handle, dX.data_ptr(), n, dY.data_ptr(), m, 16, h, h,
                                     dO.data_ptr()) == 0, c.last_error()
torch.cuda.synchronize()
print("timing", c.last_timing(), "skip", c.skip_stats())
