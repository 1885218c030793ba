"""One score pass (device API) for ncu: python tools/prof_score.py N SPATIAL(0/1/2) [reps]."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N  # noqa: E402
from paper_2602_10378_b200 import fixtures as F  # noqa: E402

n = int(sys.argv[1])
sp = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
X, _ = F.runtime_sweep_inputs(n, 16)
h = F.sdkde_bandwidth(X)
dX = torch.from_numpy(X).cuda()
dS = torch.empty((n, 16), dtype=torch.float64, device="cuda")
c = fk.Context([0])
c.set_option(N.OPT_SPATIAL, sp)
lib = N.load()
for _ in range(reps):
    assert lib.fkde_gpu_score_device(c.handle, dX.data_ptr(), n, 16, h, dS.data_ptr()) == 0
torch.cuda.synchronize()
print(c.skip_stats())
