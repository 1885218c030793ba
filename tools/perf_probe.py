"""Device-time probe of every BASELINE config through the device-resident ABI.
Prints per-phase CUDA-event times and the MUFU-roof fraction."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N  # noqa: E402

MUFU_PEAK = 148 * 16 * 1.965e9


def run(ctx, kind, n, m, reps=5, seed=0):
    rng = np.random.default_rng(seed)
    means = rng.normal(scale=3.0, size=(4, 16))
    X = means[rng.integers(0, 4, n)] + rng.normal(size=(n, 16))
    Y = means[rng.integers(0, 4, m)] + rng.normal(size=(m, 16))
    h = 2.324 * (4 / 18) ** (1 / 20) * n ** (-1 / 24)
    dX = torch.from_numpy(X).cuda()
    dY = torch.from_numpy(Y).cuda()
    dO = torch.empty(m, dtype=torch.float64, device="cuda")
    lib = N.load()
    stream = torch.cuda.ExternalStream(ctx.stream())
    ctx.set_option(N.OPT_TIMING, 1)

    def once():
        if kind == "sdkde":
            rc = lib.fkde_gpu_sdkde_device(ctx.handle, dX.data_ptr(), n, dY.data_ptr(), m, 16, h, h,
                                           dO.data_ptr())
        elif kind == "kde":
            rc = lib.fkde_gpu_kde_device(ctx.handle, dX.data_ptr(), n, dY.data_ptr(), m, 16, h, 0, 1,
                                         dO.data_ptr())
        else:
            rc = lib.fkde_gpu_kde_device(ctx.handle, dX.data_ptr(), n, dY.data_ptr(), m, 16, h, 1, 1,
                                         dO.data_ptr())
        assert rc == 0, ctx.last_error()

    torch.cuda.synchronize()
    s0 = torch.cuda.Event(enable_timing=True)
    e0 = torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    once()
    e0.record(stream)
    e0.synchronize()
    times = [s0.elapsed_time(e0)]
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record(stream)
        once()
        e.record(stream)
        e.synchronize()
        times.append(s.elapsed_time(e))
    tm = ctx.last_timing()
    ms = float(np.median(times[1:] if len(times) > 1 else times))
    exps = (n * n + n * m) if kind == "sdkde" else n * m
    print(f"{kind:7s} n={n:8d} m={m:7d}: {ms:9.3f} ms  q/s={m / ms * 1e3:.3e}  "
          f"exp/s={exps / ms * 1e3:.3e} ({exps / ms * 1e3 / MUFU_PEAK * 100:.1f}% of MUFU@1.965GHz) "
          f"phases prep={tm[0]:.3f} score={tm[1]:.3f} fin={tm[2]:.3f} gath={tm[3]:.3f} "
          f"query={tm[4]:.3f} red={tm[5]:.3f}", flush=True)
    st = ctx.skip_stats()
    print(f"        direct rows: score {st['direct_rows']} density {st['density']['direct_rows']}; "
          f"tiles skipped score {st['tiles_skipped']}/{st['tiles_total']} "
          f"density {st['density']['tiles_skipped']}/{st['density']['tiles_total']}", flush=True)
    v = dO.cpu().numpy()
    assert np.isfinite(v).all()


def run_bench(ctx, n, m, reps=1):
    from paper_2602_10378_b200 import fixtures as F
    X, Y = F.runtime_sweep_inputs(n, m, seed=0)
    h = F.sdkde_bandwidth(X)
    dX = torch.from_numpy(X).cuda()
    dY = torch.from_numpy(Y).cuda()
    dO = torch.empty(m, dtype=torch.float64, device="cuda")
    lib = N.load()
    ctx.set_option(N.OPT_TIMING, 1)
    for _ in range(reps + 1):
        rc = lib.fkde_gpu_sdkde_device(ctx.handle, dX.data_ptr(), n, dY.data_ptr(), m, 16, h, h, dO.data_ptr())
        assert rc == 0, ctx.last_error()
    tm = ctx.last_timing()
    st = ctx.skip_stats()
    print(f"bench   n={n:8d} m={m:7d}: {tm[N.T_TOTAL]:9.3f} ms phases prep={tm[0]:.3f} score={tm[1]:.3f} "
          f"fin={tm[2]:.3f} gath={tm[3]:.3f} query={tm[4]:.3f} red={tm[5]:.3f} | direct rows score "
          f"{st['direct_rows']} density {st['density']['direct_rows']}", flush=True)


def main():
    ctx = fk.Context([0])
    which = sys.argv[1:] or ["small", "big"]
    if "sd1m" in which:
        run(ctx, "sdkde", 1 << 20, 1 << 17, reps=0)
    if "bench1m" in which:   # the bench.py workload (reference mixture, SD-KDE rate bandwidth)
        run_bench(ctx, 1 << 20, 1 << 17)
    if "sd256k" in which:
        run(ctx, "sdkde", 1 << 18, 1 << 14, reps=0)
    if "sd32k" in which:
        run(ctx, "sdkde", 32768, 32768, reps=1)
    if "small" in which:
        run(ctx, "sdkde", 4096, 4096)
        run(ctx, "sdkde", 32768, 32768)
        run(ctx, "sdkde", 32768, 4096)
        run(ctx, "kde", 32768, 32768)
    if "big" in which:
        run(ctx, "laplace", 262144, 65536, reps=3)
        run(ctx, "sdkde", 1 << 20, 1 << 17, reps=2)


if __name__ == "__main__":
    main()
