import os, sys, numpy as np
ROOT='/root/repo'; sys.path.insert(0, ROOT); sys.path.insert(0, ROOT+'/oracle'); sys.path.insert(0, ROOT+'/tests')
import oracle as O, paper_2602_10378_b200 as fk
from paper_2602_10378_b200 import _native as N
from conftest import max_rowwise_rel, max_rel_global_floor
port=O.get('port')
for i in (9, 21, 33, 45):
    ns, ds = [3, 64, 1024, 4096], [1, 2, 16]
    n, d = ns[(i % 12) // 3], ds[i % 3]
    tr = port.random_gaussian(n, d, 1000 + i, 1.5)
    q = port.random_gaussian(max(1, n // 8), d, 2000 + i, 1.5)
    h = (0.8 + 0.8 * port.uniform01(3000 + i, 1)[0]) * 0.75 * np.sqrt(float(d))
    sd, deb = port.sdkde_naive(tr, q, h, threads=os.cpu_count())
    for fl in (0, 1, 2):
        ctx = fk.Context([0])
        if fl: ctx.set_option(N.OPT_FLUSH_TILES, fl)
        r = fk.sdkde_flash(tr, q, fk.Bandwidth.uniform(h), ctx=ctx)
        e = np.abs(r.debiased_samples.values - deb)
        rel = max_rowwise_rel(r.debiased_samples.values, deb)
        k = int(np.argmax(e[:,0] / np.maximum(np.abs(deb[:,0]), 1e-300)))
        print(i, 'flush', fl, 'deb rel', rel, 'abs max', e.max(), 'worst row x_sd', deb[k,0], 'abs err', e[k,0])
        ctx.close()
