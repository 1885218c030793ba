"""Interleaved sweep of a runtime engine option on the bench workload (n = 2^20,
m = 2^17): python tools/knob_probe.py OPTION v1 v2 ... [--rounds R]
(OPTION: a name of paper_2602_10378_b200._native, e.g. OPT_SPLITS; value 0 = engine
default).  Prints the score / density phase times per (round, value)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N  # noqa: E402
from paper_2602_10378_b200 import fixtures as F  # noqa: E402

args = sys.argv[1:]
rounds = 3
if "--rounds" in args:
    i = args.index("--rounds")
    rounds = int(args[i + 1])
    del args[i:i + 2]
opt = getattr(N, args[0])
vals = [int(v) for v in args[1:]]
n, m = 1 << 20, 1 << 17
X, Y = F.runtime_sweep_inputs(n, m, seed=0)
h = F.sdkde_bandwidth(X)
dX, dY = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
dO = torch.empty(m, dtype=torch.float64, device="cuda")
lib = N.load()
ctx = fk.Context([0])
ctx.set_option(N.OPT_TIMING, 1)
for r in range(rounds):
    for v in vals:
        ctx.set_option(opt, v)
        for _ in range(2):
            rc = lib.fkde_gpu_sdkde_device(ctx.handle, dX.data_ptr(), n, dY.data_ptr(), m, 16, h, h,
                                           dO.data_ptr())
            assert rc == 0, ctx.last_error()
        t = ctx.last_timing()
        print(f"{args[0]}={v:3d} round {r}: total {t[N.T_TOTAL]:8.3f} ms score {t[N.T_SCORE]:8.3f} "
              f"query {t[N.T_QUERY]:7.3f}", flush=True)
