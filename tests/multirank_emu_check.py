"""Subprocess body of tests/test_multirank_emu.py (needs FKDE_NCCL_LIB set to the
in-process NCCL emulator before the engine first loads NCCL).  Runs the engine's
multi-rank C++ path -- single-process multi-device contexts and one context per
rank driven from threads -- on ONE GPU and prints max differences against the
single-device engine at a fixed column-split count (results are expected to be
bitwise identical: every row / query sees the same per-unit reduction order).
Optional 5th argument 1: every context runs on the spatial order with tile
skipping (FKDE_OPT_SPATIAL = 1, the default for n >= 32768), so the sorted-order
row shards, the sorted x^SD gather and the un-permutation run multi-rank too."""
import ctypes
import json
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N  # noqa: E402


def run_all(ctx, X, Y, h):
    tr, q = fk.SampleSet(X), fk.SampleSet(Y)
    r = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=ctx)
    return {
        "score": fk.score_flash(tr, h, ctx=ctx).values,
        "sdkde": r.values,
        "debiased": r.debiased_samples.values,
        "kde": fk.kde_flash(tr, q, h, ctx=ctx).values,
        "laplace": fk.kde_flash(tr, q, h, fk.KernelKind.LaplaceCorrected, True, ctx=ctx).values,
    }


def main():
    n, m, world, splits = (int(a) for a in sys.argv[1:5])
    spatial = int(sys.argv[5]) if len(sys.argv) > 5 else 0

    def setup(c):
        c.set_option(N.OPT_SPLITS, splits)
        if spatial:
            c.set_option(N.OPT_SPATIAL, 1)
    rng = np.random.default_rng(7)
    X = rng.normal(size=(n, 16)) * 1.5 + rng.integers(0, 3, size=(n, 1))
    Y = rng.normal(size=(m, 16)) * 1.5
    h = 1.3
    one = fk.Context([0])
    setup(one)
    ref = run_all(one, X, Y, h)
    one.close()

    out = {}
    multi = fk.Context([0] * world)           # single process, world "devices"
    setup(multi)
    got = run_all(multi, X, Y, h)
    multi.close()
    out["multi_device"] = {k: float(np.max(np.abs(got[k] - ref[k]))) for k in ref}

    # device-resident API per rank (what bench.py drives under torchrun)
    import torch
    dX = torch.from_numpy(X).cuda()
    dY = torch.from_numpy(Y).cuda()
    lib = N.load()
    uid_d = fk.engine.nccl_unique_id()
    dev_res, dev_errs = [None] * world, []

    def rank_dev(r):
        try:
            c = fk.Context(rank=r, world=world, device=0, nccl_id=uid_d)
            setup(c)
            dO = torch.zeros(m, dtype=torch.float64, device="cuda")
            for _ in range(2):
                rc = lib.fkde_gpu_sdkde_device(c.handle, dX.data_ptr(), n, dY.data_ptr(), m, 16, h, h,
                                               dO.data_ptr())
                if rc != 0:
                    raise RuntimeError(c.last_error())
                torch.cuda.ExternalStream(c.stream()).synchronize()
            dev_res[r] = dO.cpu().numpy()
            c.close()
        except Exception as e:  # noqa: BLE001
            dev_errs.append(repr(e))

    th = [threading.Thread(target=rank_dev, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if dev_errs:
        out["device_api_error"] = dev_errs
    else:
        out["device_api"] = [float(np.max(np.abs(dev_res[r] - ref["sdkde"]))) for r in range(world)]

    uid = fk.engine.nccl_unique_id()          # one context per rank, one thread each
    res, errs = [None] * world, []

    def rank_main(r):
        try:
            c = fk.Context(rank=r, world=world, device=0, nccl_id=uid)
            setup(c)
            res[r] = run_all(c, X, Y, h)
            c.close()
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        out["per_rank_error"] = errs
    else:
        out["per_rank"] = [{k: float(np.max(np.abs(res[r][k] - ref[k]))) for k in ref}
                           for r in range(world)]
    out["scale"] = {k: float(np.max(np.abs(ref[k]))) for k in ref}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
