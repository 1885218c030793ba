"""Score pass at n = 2^18 in a loop with nvidia-smi sampling SM clock and board
power: is the kernel power-capped, and by how much does a variant change that?
    FKDE_B200_LIB=ab/lib_x.so python tools/power_probe.py"""
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_10378_b200 as fk  # noqa: E402
from paper_2602_10378_b200 import _native as N, fixtures as F  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
    secs = float(sys.argv[2]) if len(sys.argv) > 2 else 6.0
    X, _ = F.runtime_sweep_inputs(n, 8)
    h = F.sdkde_bandwidth(X)
    ctx = fk.Context([0])
    ctx.set_option(N.OPT_TIMING, 1)
    tr = fk.SampleSet(X)
    for _ in range(3):
        fk.score_flash(tr, h, ctx=ctx)
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "100"], stdout=subprocess.PIPE, text=True)
    ts = []
    t0 = time.time()
    while time.time() - t0 < secs:
        fk.score_flash(tr, h, ctx=ctx)
        ts.append(ctx.last_timing()[N.T_SCORE])
    smi.terminate()
    rows = [l.split(",") for l in smi.communicate()[0].strip().split("\n") if "," in l]
    clk = [float(r[0]) for r in rows[5:]]
    pw = [float(r[1]) for r in rows[5:]]
    print(f"{os.environ.get('FKDE_B200_LIB', 'current')[-20:]} n={n}: score pass median {np.median(ts):.2f} ms; "
          f"SM clock median {np.median(clk):.0f} MHz; power median {np.median(pw):.0f} W", flush=True)


if __name__ == "__main__":
    main()
