"""Device time per call of the BASELINE configs through the device-resident ABI,
back to back (the repeated call is replayed as a CUDA graph): the small configs are
launch-bound, so this is the number the prologue fusion moves.
python tools/latency_probe.py [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N  # noqa: E402
from paper_2602_10378_b200 import fixtures as F  # noqa: E402

MUFU = 148 * 16 * 1.965e9


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    lib = N.load()
    ctx = fk.Context([0])
    if os.environ.get("SPATIAL"):
        ctx.set_option(N.OPT_SPATIAL, int(os.environ["SPATIAL"]))
    stream = torch.cuda.ExternalStream(ctx.stream())
    cases = [("config1 sdkde", "sdkde", 4096, 4096), ("config2 sdkde", "sdkde", 32768, 32768),
             ("paper sdkde 32k/4k", "sdkde", 32768, 4096), ("config3 kde", "kde", 32768, 32768),
             ("config4 laplace", "laplace", 262144, 65536)]
    for name, kind, n, m in cases:
        X, Y = F.runtime_sweep_inputs(n, m)
        h = F.sdkde_bandwidth(X) if kind == "sdkde" else F.silverman_bandwidth(X)
        dX = torch.from_numpy(X).cuda()
        dY = torch.from_numpy(Y).cuda()
        dO = torch.empty(m, dtype=torch.float64, device="cuda")

        def call():
            if kind == "sdkde":
                rc = lib.fkde_gpu_sdkde_device(ctx.handle, dX.data_ptr(), n, dY.data_ptr(), m, 16, h, h,
                                               dO.data_ptr())
            else:
                rc = lib.fkde_gpu_kde_device(ctx.handle, dX.data_ptr(), n, dY.data_ptr(), m, 16, h,
                                             0 if kind == "kde" else 1, 1, dO.data_ptr())
            assert rc == 0, ctx.last_error()

        for _ in range(3):
            call()
        torch.cuda.synchronize()
        stream.synchronize()
        r = reps if n * max(n, m) < (1 << 31) else 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(r):
            call()
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / r
        exps = (n * n + n * m) if kind == "sdkde" else n * m
        print(f"{name:20s} n={n:7d} m={m:6d}: {ms * 1e3:9.1f} us/call  launches={ctx.last_launch_count()}"
              f"  MUFU floor {exps / MUFU * 1e6:7.1f} us  ({exps / MUFU * 1e3 / ms * 100:5.1f}% of it)",
              flush=True)


if __name__ == "__main__":
    main()
