"""bench.py's launch and reference-arm plumbing (no GPU needed)."""
import json
import os
import subprocess
import sys

import numpy as np

from conftest import ROOT

BENCH = os.path.join(ROOT, "bench.py")


def _last_json(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


def test_gpus_n_spawns_n_ranks():
    # outside torchrun, --gpus 2 re-executes itself under torch.distributed.run;
    # every rank joins the process group and rank 0 prints n_gpus = 2
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--steps", "1", "--warmup", "3",
                        "--dry-run"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = _last_json(r.stdout)
    assert line["n_gpus"] == 2 and line["max_over_ranks"] == 2.0


def test_reference_arm_inputs_equal_product_inputs():
    # the reference arm builds its inputs from the oracle library only; they are
    # bitwise the product arm's inputs (same config)
    sys.path.insert(0, ROOT)
    import bench
    import oracle as O
    n, m = 4096, 512
    X1, Y1, h1 = bench.make_inputs(n, m)
    X2, Y2, h2 = bench.make_inputs_oracle(n, m, O.get("port"))
    assert np.array_equal(X1, X2) and np.array_equal(Y1, Y2) and h1 == h2
    if O.reference_available():
        X3, Y3, h3 = bench.make_inputs_oracle(n, m, O.get("reference"))
        assert np.array_equal(X1, X3) and np.array_equal(Y1, Y3) and h1 == h3


def test_reference_arm_never_loads_the_product():
    # run the reference arm's setup in a fresh interpreter and list the shared
    # objects it mapped: the product library must not be among them
    code = (
        "import sys, os; sys.path.insert(0, %r); import bench\n"
        "kind, orc = bench.oracle_handle()\n"
        "X, Y, h = bench.make_inputs_oracle(2048, 256, orc)\n"
        "bench.cpu_oracle_sample(orc, kind, X, Y, h, 4, 4)\n"
        "maps = open('/proc/self/maps').read()\n"
        "print('PRODUCT' if 'libfkde_b200' in maps else 'CLEAN')\n"
        "print('PKG' if 'paper_2602_10378_b200' in sys.modules else 'NOPKG')\n" % ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "CLEAN" in r.stdout and "NOPKG" in r.stdout, r.stdout


def test_reference_arm_every_workload_config():
    # --workload K (BASELINE.json config K) through the reference arm, CPU only:
    # the same metric / config keys as the product arm, the reference's own oracle
    # timed (config 1 and 3: score + density, density only; bounded samples)
    sys.path.insert(0, ROOT)
    import bench
    for wl in (1, 3):
        env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
        r = subprocess.run([sys.executable, BENCH, "--impl", "reference", "--workload", str(wl),
                            "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                           timeout=600, env=env)
        assert r.returncode == 0, r.stderr[-2000:]
        line = _last_json(r.stdout)
        job, n, m, name = bench.WORKLOADS[wl]
        assert line["impl"] == "reference" and line["config"]["workload"] == name
        assert line["config"]["n_train"] == n and line["config"]["n_query"] == m
        assert line["metric"] == bench.metric_of(wl) and line["value"] > 0
        assert ("score_naive" in line["cpu_baseline"]["sample"]) == (job == "sdkde")
