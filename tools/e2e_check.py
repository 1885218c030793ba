"""Diagnoses bench.py's e2e output check at the headline size: finiteness and
positivity of the densities from the host C ABI (pinned and pageable buffers) and
bitwise agreement of the two with each other and with the device-resident call."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else bench.N_TRAIN
m = int(sys.argv[2]) if len(sys.argv) > 2 else bench.N_QUERY
X, Y, h = bench.make_inputs(n, m)
d = X.shape[1]
ctx = fk.Context([0])
lib = N.load()
dp = ctypes.POINTER(ctypes.c_double)
idx = ctypes.c_size_t(0)


def host(x, y, o, db):
    rc = lib.fkde_gpu_sdkde(ctx.handle, ctypes.cast(x, dp), n, ctypes.cast(y, dp), m, d, h, h,
                            ctypes.cast(o, dp), ctypes.cast(db, dp), ctypes.byref(idx))
    print("rc", rc, ctx.last_error() if rc else "")


pX, pY = torch.from_numpy(X).pin_memory(), torch.from_numpy(Y).pin_memory()
pO, pD = torch.empty(m, dtype=torch.float64).pin_memory(), torch.empty((n, d), dtype=torch.float64).pin_memory()
for rep in range(2):
    host(pX.data_ptr(), pY.data_ptr(), pO.data_ptr(), pD.data_ptr())
    o = pO.numpy().copy()
    print(f"pinned[{rep}]: nonfinite {int((~np.isfinite(o)).sum())} nonpositive {int((o <= 0).sum())}"
          f" min {o[np.isfinite(o)].min():.3e}")
gO, gD = np.empty(m), np.empty((n, d))
host(X.ctypes.data, Y.ctypes.data, gO.ctypes.data, gD.ctypes.data)
print("pageable == pinned:", np.array_equal(gO, o), "max rel diff",
      float(np.nanmax(np.abs(gO - o) / np.maximum(np.abs(o), 1e-300))),
      "deb equal:", np.array_equal(gD, pD.numpy()))
bad = np.where(~np.isfinite(o) | (o <= 0))[0][:10]
print("bad queries:", bad.tolist(), o[bad].tolist())
