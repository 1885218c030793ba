"""Accuracy of the tensor-core path on spread rows: config-1 data (SD-KDE n = m = 4096,
d = 16) at h0/2 and h0/3 with the spread-row threshold FKDE_RISK_HALF_NORM (|y|^2/2
above which a row is recomputed directly) given on the command line -- score errors
(the reference's floored metrics) and densities vs the fp64 oracle, rows sent to the
direct path.  python tools/risk_probe.py   (run once per threshold: the value is
read at library load)"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import fixtures as F  # noqa: E402
from conftest import max_component_rel, max_rel_global_floor, max_rowwise_rel  # noqa: E402

port = O.get("port")
X, Y = F.runtime_sweep_inputs(4096, 4096, seed=0)
h0 = F.sdkde_bandwidth(X)
for div in (2, 3):
    h = h0 / div
    ctx = fk.Context([0])
    s = fk.score_flash(X, h, ctx=ctx).values
    st = ctx.skip_stats()
    r = fk.sdkde_flash(X, Y, fk.Bandwidth.uniform(h), ctx=ctx)
    ctx.close()
    ref_s = port.score_naive(X, X, h, threads=os.cpu_count())
    ref_v, ref_deb = port.sdkde_naive(X, Y, h, threads=os.cpu_count())
    print(f"risk={os.environ.get('FKDE_RISK_HALF_NORM', 'default')} h0/{div}: score rowwise "
          f"{max_rowwise_rel(s, ref_s):.2e} global {max_rel_global_floor(s, ref_s):.2e} "
          f"x^SD {max_rowwise_rel(r.debiased_samples.values, ref_deb):.2e} density "
          f"{max_component_rel(r.values, ref_v):.2e} direct rows {st['direct_rows']}", flush=True)
