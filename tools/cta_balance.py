"""Load balance of the persistent pairwise kernels across CTAs: per-CTA start /
end (globaltimer) and visited-tile counts of the check, score and density
kernels of one SD-KDE on the BASELINE mixture.
    python -c "from paper_2602_10378_b200 import build as B; B.build(out='ab/lib_cta.so', defines=['FKDE_CTA_TIMES'])"
    FKDE_B200_LIB=ab/lib_cta.so python tools/cta_balance.py [n] [m]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N, fixtures as F  # noqa: E402

NAMES = {3: "check", 0: "score", 1: "density"}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
    m = int(sys.argv[2]) if len(sys.argv) > 2 else n // 8
    X, Y = F.runtime_sweep_inputs(n, m)
    h = F.sdkde_bandwidth(X)
    lib = N.load()
    ctx = fk.Context([0])
    dX = torch.from_numpy(X).cuda()
    dY = torch.from_numpy(Y).cuda()
    dO = torch.empty(m, dtype=torch.float64, device="cuda")
    buf = torch.zeros(4 * 4096, dtype=torch.int64, device="cuda")
    ctx.set_option(N.OPT_TIMING, 1)
    for it in range(2):
        if it == 1:
            ctx.set_option(6, buf.data_ptr())
        rc = lib.fkde_gpu_sdkde_device(ctx.handle, dX.data_ptr(), n, dY.data_ptr(), m, 16, h, h, dO.data_ptr())
        assert rc == 0, ctx.last_error()
        torch.cuda.synchronize()
    t = ctx.last_timing()
    print(f"n={n} m={m}: score phase {t[N.T_SCORE]:.2f} ms, density phase {t[N.T_QUERY]:.2f} ms")
    b = buf.view(4, 4096).cpu().numpy()
    for mode in (3, 0, 1):
        st, en = b[mode, 0:2048:2], b[mode, 1:2048:2]
        ok = (st > 0) & (en > 0)
        if not ok.any():
            continue
        st, en, tiles = st[ok], en[ok], b[mode, 2048:2048 + 1024][ok]
        t0 = st.min()
        dur = (en - st) / 1e3
        print(f"  {NAMES[mode]:8s} ctas={ok.sum():4d} span {(en.max() - t0) / 1e3:8.1f} us | per-CTA busy "
              f"min {dur.min():8.1f} med {np.median(dur):8.1f} max {dur.max():8.1f} us "
              f"(max/mean {dur.max() / dur.mean():.3f}) | start spread {(st.max() - t0) / 1e3:.1f} us | "
              f"tiles min {tiles.min()} med {int(np.median(tiles))} max {tiles.max()} "
              f"(max/mean {tiles.max() / tiles.mean():.3f}) | us/tile {np.sum(dur) / max(tiles.sum(), 1):.4f}")
        if mode == 0:
            zc = b[mode, 3072:3072 + 1024][ok].sum()
            print(f"           all-zero 32x32 sub-blocks: {zc} of {tiles.sum() * 12} "
                  f"({zc / max(tiles.sum() * 12, 1) * 100:.1f}%)")
    ctx.close()


if __name__ == "__main__":
    main()
