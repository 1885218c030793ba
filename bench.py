#!/usr/bin/env python3
"""Benchmark: Flash-SD-KDE headline workload (BASELINE config 5) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full SD-KDE over n = 2^20 training points and m = 2^17 queries
in d = 16 (score pass -> x + h^2/2 s -> density pass), inputs drawn from the
reference's 16-D Gaussian mixture with its runtime-sweep seeds and SD-KDE
rate bandwidth.  N > 1 runs one process per GPU: launched by the driver under
torchrun, or -- when WORLD_SIZE is unset -- bench.py re-executes itself under
``python -m torch.distributed.run --nproc-per-node N``.  Rows are sharded for
the score pass, the debiased samples are allgathered (NCCL), queries are
sharded for the density pass (total work fixed: strong scaling).

value  = queries/s of the whole job, inputs resident in HBM (fp64), timed on
         the engine's stream with CUDA events, max over ranks.
e2e    = same metric through the host C ABI call (fkde_gpu_sdkde) from pinned
         host buffers: H2D of X and Y, D2H of densities and debiased samples
         (e2e_pageable: the same from ordinary pageable numpy buffers, what a
         std::vector caller of the C++ facade gets).
--impl reference: the reference's own CPU oracle (oracle/_ref built from
         /root/reference, or the C port when _ref is absent) on a bounded row
         sample with all host threads, extrapolated linearly in evaluated rows
         (rank 0 only).  This arm never imports the product package: inputs
         and bandwidth come from the reference's own sampler and rules.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_TRAIN = 1 << 20
N_QUERY = 1 << 17
DIM = 16
METRIC = "SD-KDE wall s & queries/sec, n=1M d=16, 131k queries, at 1/2/4/8 B200 vs CPU ref"
PAPER_WALL_S = 2.3  # PAPER.md:30, 592 (RTX A6000), BASELINE.md section 1
MUFU_EX2_PER_CLK_SM = 16
# BASELINE.json configs: --workload K (default 5, the headline the metric names;
# the others give per-config lines under the same timing contract)
WORKLOADS = {
    1: ("sdkde", 4096, 4096, "SD-KDE n=4096 m=4096 d=16 (BASELINE config 1)"),
    2: ("sdkde", 32768, 32768, "SD-KDE n=32768 m=32768 d=16 (BASELINE config 2)"),
    3: ("kde", 32768, 32768, "Gaussian KDE n=32768 m=32768 d=16 (BASELINE config 3)"),
    4: ("laplace", 262144, 65536, "Laplace-corrected fused KDE n=262144 m=65536 d=16 (BASELINE config 4)"),
    5: ("sdkde", N_TRAIN, N_QUERY, "SD-KDE n=1048576 m=131072 d=16 (BASELINE config 5)"),
}


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


# ---- clocks sampler ------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---- inputs -------------------------------------------------------------------------
def make_inputs(n, m, kind="sdkde"):
    from paper_2602_10378_b200 import fixtures as F
    X, Y = F.runtime_sweep_inputs(n, m, seed=0)
    # BandwidthPolicy Auto (sweep.cpp:31-61): SD-KDE rate for SD-KDE, Silverman otherwise
    h = F.sdkde_bandwidth(X) if kind == "sdkde" else F.silverman_bandwidth(X)
    return X, Y, h


def make_inputs_oracle(n, m, orc, kind="sdkde"):
    """The same inputs from the oracle library alone (reference arm: the product
    package is never imported).  Bitwise equal to make_inputs (tests/test_bench.py)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    w, mu, s = O.default_mixture_16d()
    cs = orc.mix64(0 ^ orc.mix64(n))             # sweep.cpp:67-69 cell_data_seed
    X = orc.sample_mixture(w, mu, s, n, cs)
    Y = orc.sample_mixture(w, mu, s, m, orc.mix64(cs ^ 0x71))
    h = (orc.sdkde_bandwidth(X, orc.silverman_prefactor(X.shape[1])) if kind == "sdkde"
         else orc.silverman_bandwidth(X))
    return X, Y, h


def workload_config(n, m, d, h, wl=5):
    """Identical in both arms (the driver compares them)."""
    big = n * d * 8 > (126 << 20)
    return {"workload": WORKLOADS[wl][3], "h": h, "n_train": n, "n_query": m, "d": d,
            "l2": (f"inputs larger than L2 (X fp64 {n * d * 8 >> 20} MiB)" if big else
                   f"L2 flushed before every timed step (256 MiB write; X fp64 "
                   f"{n * d * 8 >> 20} MiB fits the 126 MiB L2)")}


def metric_of(wl):
    if wl == 5:
        return METRIC
    kind, n, m, name = WORKLOADS[wl]
    return f"{name}: wall s & queries/sec on B200 vs CPU ref"


# ---- CPU baseline (the reference oracle, bounded sample) ------------------------------
ROWS_SCORE, ROWS_QUERY = 1024, 512


def oracle_handle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    kind = "reference" if O.reference_available() else "port"
    return kind, O.get(kind)


def cpu_oracle_sample(orc, kind, X, Y, h, rows_score=ROWS_SCORE, rows_query=ROWS_QUERY,
                      job="sdkde"):
    """Times the reference's naive oracle on a row sample; returns (sample wall s,
    extrapolated full-workload s, details).  Cost is exactly linear in evaluated rows."""
    threads = os.cpu_count() or 1
    n, m = X.shape[0], Y.shape[0]
    rows_score = 0 if job != "sdkde" else min(rows_score, n)
    rows_query = min(rows_query * (4 if job != "sdkde" else 1), m)
    rs = np.linspace(0, n - 1, max(rows_score, 1)).astype(np.int64)
    t0 = time.perf_counter()
    if rows_score:
        orc.score_naive(X, X[rs], h, threads=threads)
    t1 = time.perf_counter()
    qs = np.linspace(0, m - 1, rows_query).astype(np.int64)
    if job == "laplace":
        orc.laplace_naive(X, Y[qs], h, threads=threads)
    else:
        orc.kde_naive(X, Y[qs], h, threads=threads)  # same cost as against the debiased set
    t2 = time.perf_counter()
    full = (t1 - t0) * n / max(rows_score, 1) + (t2 - t1) * m / rows_query
    fn = "laplace_naive" if job == "laplace" else "kde_naive"
    sample = ((f"score_naive on {rows_score} of {n} rows + " if rows_score else "") +
              f"{fn} on {rows_query} of {m} queries (x {n} train), {threads} threads, "
              "extrapolated linearly in rows")
    return t2 - t0, full, {"kind": kind, "cores": threads, "sample": sample,
                           "sample_s": t2 - t0, "extrapolated": True,
                           "sample_rows": {"score": rows_score, "query": rows_query}}


REF_FLASH_NOTE = ("the reference's CPU flash engine (engine.cpp, Eigen3) is not buildable in "
                  "this image (Eigen3 absent here and on the GPU box); the timed path is its "
                  "naive oracle (oracle.cpp), the reference's declared ground truth")


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    kind, orc = oracle_handle()
    job, n_tr, n_q, _ = WORKLOADS[args.workload]
    X, Y, h = make_inputs_oracle(n_tr, n_q, orc, job)
    for _ in range(args.warmup):
        cpu_oracle_sample(orc, kind, X, Y, h, 16, 16, job=job)
    samples, fulls = [], []
    info = None
    for _ in range(args.steps):
        smp, full, info = cpu_oracle_sample(orc, kind, X, Y, h, job=job)
        samples.append(smp)
        fulls.append(full)
    wall = float(np.median(fulls))
    qps = n_q / wall
    line = {
        "impl": "reference", "metric": metric_of(args.workload), "value": qps, "unit": "queries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        # ms_per_step is what one timed step actually took (the bounded sample);
        # value is the full workload's rate extrapolated from it
        "ms_per_step": float(np.mean(samples)) * 1e3,
        "extrapolated": True, "full_workload_wall_s": wall,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference 16-D Gaussian mixture, runtime-sweep seeds",
        "config": workload_config(n_tr, n_q, DIM, h, args.workload),
        "parallelism": f"{info['cores']} host threads on rank 0 (CPU only; no GPU used)",
        "reference_path": f"oracle/_ref ({'reference sources compiled' if kind == 'reference' else 'C port'})",
        "reference_flash_engine": REF_FLASH_NOTE,
        "cpu_baseline": dict(info, value=qps, unit="queries/s"),
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- our arm ---------------------------------------------------------------------------
def run_ours(args):
    import torch

    rank, world, local = env_rank()
    if args.dry_run:
        return run_dry(args, rank, world)
    import paper_2602_10378_b200 as fk
    from paper_2602_10378_b200 import _native as N

    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = [fk.engine.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx = fk.Context(rank=rank, world=world, device=local, nccl_id=uid[0])
    else:
        torch.cuda.set_device(local)
        ctx = fk.Context([local])
    lib = N.load()
    dev = torch.device("cuda", local)

    job, n_tr, n_q, _ = WORKLOADS[args.workload]
    X, Y, h = make_inputs(n_tr, n_q, job)
    n, m, d = X.shape[0], Y.shape[0], X.shape[1]
    kern = N.KERNEL_LAPLACE_CORRECTED if job == "laplace" else N.KERNEL_GAUSSIAN
    dX = torch.from_numpy(X).to(dev)
    dY = torch.from_numpy(Y).to(dev)
    dO = torch.empty(m, dtype=torch.float64, device=dev)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=dev)

    def step():
        if job == "sdkde":
            rc = lib.fkde_gpu_sdkde_device(ctx.handle, dX.data_ptr(), n, dY.data_ptr(), m, d, h, h,
                                           dO.data_ptr())
        else:   # configs 3 / 4: density pass only (Laplace: fused, as BASELINE names it)
            rc = lib.fkde_gpu_kde_device(ctx.handle, dX.data_ptr(), n, dY.data_ptr(), m, d, h, kern,
                                         1, dO.data_ptr())
        if rc != 0:
            raise RuntimeError(ctx.last_error())

    def barrier():
        torch.cuda.synchronize(dev)
        stream.synchronize()
        if dist:
            dist.barrier()

    for _ in range(max(3, args.warmup)):
        step()
    barrier()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches = 0
    if n * d * 8 > (126 << 20):   # inputs larger than L2: steps back to back, no host sync
        ev0.record(stream)
        for _ in range(args.steps):
            step()
            launches += ctx.last_launch_count()
        ev1.record(stream)
        barrier()
        dev_ms = ev0.elapsed_time(ev1)
    else:   # L2-resident working set: L2 flushed (256 MiB write) before every timed step
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        with torch.cuda.stream(stream):
            for a, b in evs:
                flush.fill_(1)
                a.record(stream)
                step()
                b.record(stream)
                launches += ctx.last_launch_count()
        barrier()
        dev_ms = sum(a.elapsed_time(b) for a, b in evs)
    clocks = sampler.stop()
    # per-phase CUDA-event times (score / density pass): separate, untimed steps with
    # the engine's phase events on (they make the call run eagerly: single-rank
    # device calls are otherwise replayed from a captured CUDA graph)
    ctx.set_option(N.OPT_TIMING, 1)
    score_ms, query_ms, kern_ms = [], [], []
    for _ in range(2):
        step()
        t = ctx.last_timing()  # syncs on this step's last event
        score_ms.append(t[N.T_SCORE])
        query_ms.append(t[N.T_QUERY])
        kern_ms.append(ctx.last_kernel_timing())   # events bracketing each pass kernel
    ctx.set_option(N.OPT_TIMING, 0)
    kern_avg = [float(np.mean([k[i] for k in kern_ms])) for i in range(N.KT_COUNT)]
    skip = ctx.skip_stats()   # tile skipping of the last score pass (this rank)

    # e2e through the host C ABI: H2D of this step's inputs and D2H of its results
    # inside the timed region, from pinned (headline) and from pageable buffers
    import ctypes
    dp = ctypes.POINTER(ctypes.c_double)
    idx = ctypes.c_size_t(0)
    pX = torch.from_numpy(X).pin_memory()
    pY = torch.from_numpy(Y).pin_memory()
    pO = torch.empty(m, dtype=torch.float64).pin_memory()
    pD = torch.empty((n, d), dtype=torch.float64).pin_memory()
    gX, gY = np.ascontiguousarray(X), np.ascontiguousarray(Y)
    gO, gD = np.empty(m), np.empty((n, d))

    def host_step(bufs):
        x, y, o, db = bufs
        if job == "sdkde":
            rc = lib.fkde_gpu_sdkde(ctx.handle, ctypes.cast(x, dp), n, ctypes.cast(y, dp), m, d, h,
                                    h, ctypes.cast(o, dp), ctypes.cast(db, dp), ctypes.byref(idx))
        else:
            rc = lib.fkde_gpu_kde(ctx.handle, ctypes.cast(x, dp), n, ctypes.cast(y, dp), m, d, h,
                                  kern, 1, ctypes.cast(o, dp))
        if rc != 0:
            raise RuntimeError(ctx.last_error())

    small = dev_ms / args.steps < 10.0

    def e2e_time(bufs):
        # warm-up calls as for the device value (a repeated small host call is replayed
        # from a CUDA graph from its third call on: the capture is part of warm-up)
        for _ in range(3 if small else 1):
            host_step(bufs)
        barrier()
        steps = max(3, min(args.steps, 50)) if small else max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(steps):
            host_step(bufs)
        barrier()
        return (time.perf_counter() - t0) / steps

    pinned = (pX.data_ptr(), pY.data_ptr(), pO.data_ptr(), pD.data_ptr())
    pageable = (gX.ctypes.data, gY.ctypes.data, gO.ctypes.data, gD.ctypes.data)
    e2e_s = e2e_time(pinned)
    # densities: finite; Gaussian ones also positive (the Laplace-corrected kernel
    # takes negative values by construction)
    out_ok = bool(np.isfinite(pO.numpy()).all() and (job == "laplace" or (pO.numpy() > 0).all()))
    e2e_pg_s = e2e_time(pageable)
    out_ok = out_ok and bool(np.array_equal(gO, pO.numpy()))

    # max over ranks
    vals = torch.tensor([dev_ms, e2e_s, e2e_pg_s, float(np.mean(score_ms)), float(np.mean(query_ms))]
                        + kern_avg, dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
        lsum = torch.tensor([launches], dtype=torch.float64, device=dev)
        dist.all_reduce(lsum)
        launches = int(lsum.item())
    dev_ms, e2e_s, e2e_pg_s, score_avg, query_avg = [float(v) for v in vals.tolist()[:5]]
    k_score, k_check, k_density = [float(v) for v in vals.tolist()[5:8]]

    if rank == 0:
        ms_step = dev_ms / args.steps
        wall = ms_step / 1e3
        qps = m / wall
        peaks, src = measured_peaks()
        sm_mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
        max_mhz = peaks.get("sm_max_mhz", 1965.0)
        # dominant kernel.  SD-KDE: the score pass (check + score kernels, the
        # T_SCORE phase); KDE / Laplace: the density pass (T_QUERY).  Algorithmic
        # work = every (row, column) pair of this rank's rows; executed work = the
        # pairs of the tiles the pass did not prove / check to be exact zeros
        # (128 x 96 per score tile, 128 x 128 per density tile).
        # the dominant kernel's own launch, timed by CUDA events bracketing it on the
        # engine's stream (fkde_gpu_last_kernel_timing); the whole phase beside it
        sd = job == "sdkde"
        if sd:
            rows_rank, st, tile_pairs = -(-n // world), skip, 128 * 96
            phase_ms = k_score if k_score > 0 else score_avg
            kname = "pairwise_tc_kernel<Score> (score pass)"
        else:
            rows_rank, st, tile_pairs = -(-m // world), skip["density"], 128 * 128
            phase_ms = k_density if k_density > 0 else query_avg
            kname = f"pairwise_tc_kernel<{'Laplace' if job == 'laplace' else 'Gauss'}> (density pass)"
        exps = rows_rank * n
        exec_tiles = max(st["tiles_total"] - st["tiles_skipped"], 0) if st["spatial_order"] \
            else st["tiles_total"] or -(-rows_rank // 128) * -(-n // (tile_pairs // 128))
        exec_exps = exec_tiles * tile_pairs
        achieved = exec_exps / (phase_ms / 1e3) / 1e9      # Gexp/s executed (MUFU)
        algorithmic = exps / (phase_ms / 1e3) / 1e9        # Gpairs/s of the pass's result
        peak = 148 * MUFU_EX2_PER_CLK_SM * max_mhz * 1e6 / 1e9
        # score: 2 GEMMs x 2d flop per pair; density: 1 GEMM
        tflops = (4 if sd else 2) * d * exps / (phase_ms / 1e3) / 1e12
        prof = os.path.join(ROOT, "profiles", "ncu_score_pass.json" if args.workload == 5
                            else f"ncu_workload{args.workload}.json")
        traffic = None
        if os.path.exists(prof):
            with open(prof) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        d2h = m * 8 + (n * d * 8 if sd else 0)
        line = {
            "metric": metric_of(args.workload), "value": qps, "unit": "queries/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_step,
            "wall_s": wall, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": qps / (N_QUERY / PAPER_WALL_S) if args.workload == 5 else None,
            "vs_baseline_note": ("paper's 2.3 s on one RTX A6000 (PAPER.md:30), same workload"
                                 if args.workload == 5 else "no published number for this config"),
            "dtype": "f32 (fp16 hi/lo split tensor-core operands, f32 accumulate, f64 finalize)",
            "data": "synthetic: reference 16-D Gaussian mixture (configs/mixture-16d-default.json),"
                    " reference RNG + runtime-sweep seeds, "
                    + ("SD-KDE rate bandwidth" if sd else "Silverman bandwidth"),
            "config": workload_config(n, m, d, h, args.workload),
            "parallelism": (f"dp{world}: score rows sharded, 1 NCCL allgather of debiased samples, "
                            f"queries sharded" if sd else f"dp{world}: queries sharded, samples replicated"),
            "phases_ms": {"score_pass": score_avg, "density_pass": query_avg},
            "kernels_ms": {"score": k_score, "check": k_check, "density": k_density,
                           "note": "CUDA events bracketing each pass kernel on the engine's "
                                   "stream (phases include the planning kernels around them)"},
            # the reference's own performance model of this run:
            # paper-model pipeline FLOPs (4d+12+d/4+3/2) k^2 (perfmodel.cpp:62-67) and
            # the runtime sweep's model_flops (sweep.cpp:74-90), with the utilization
            # the reference's sweep would print against the B200 FP32 preset
            "perf_model": {
                "paper_flops": (4 * d + 12 + d / 4 + 1.5) * n * n,
                "model_flops": (4 * d + 12) * n * n + (2 * d + 12) * n * m,
                "utilization_vs_b200_fp32": ((4 * d + 12) * n * n + (2 * d + 12) * n * m)
                / wall / 74.4e12,
                "exp_count": float(n) * n + float(n) * m},
            "clocks": clocks,
            "e2e": {"value": m / e2e_s, "unit": "queries/s", "wall_s": e2e_s,
                    "host_buffers": "pinned",
                    "h2d_bytes_per_step": (n + m) * d * 8,
                    "d2h_bytes_per_step": d2h, "outputs_finite": out_ok},
            "e2e_pageable": {"value": m / e2e_pg_s, "unit": "queries/s", "wall_s": e2e_pg_s,
                             "host_buffers": "pageable (numpy)",
                             "h2d_bytes_per_step": (n + m) * d * 8,
                             "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "roofline": {"bound": "mufu",
                         "kernel": kname,
                         "achieved": achieved, "peak": peak, "unit": "Gexp/s (executed)",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": f"nominal 16 ex2/clk/SM x 148 SMs x sm_max_mhz "
                                        f"{max_mhz:.0f} ({src} MEASURED_PEAKS)",
                         "frac_at_observed_clock": exec_exps / (phase_ms / 1e3) /
                         (148 * MUFU_EX2_PER_CLK_SM * sm_mhz * 1e6),
                         "algorithmic": {
                             "pairs_per_s_G": algorithmic, "pairs": exps,
                             "vs_full_mufu_roof": algorithmic / peak,
                             "note": "every (row, column) pair of the result per second of the "
                                     "dominant kernel; above 1 because tile pairs whose every pair "
                                     "contributes exactly zero (score: fp16 P representation; "
                                     "density: below 2^-24 of the row's mass, else recomputed) "
                                     "are proven (box bound) or checked (GEMM1 max) and skipped"},
                         "tile_skipping": skip,
                         "tensor": {"achieved_tflops": tflops,
                                    "peak_tflops": peaks.get("bf16_tflops"),
                                    "frac": tflops / peaks.get("bf16_tflops", 1590.0),
                                    "note": "algorithmic 2x(2d) flop/pair vs dense bf16 peak"}},
        }
        if world == 1 and not args.no_cpu_baseline:
            kind, orc = oracle_handle()
            smp, full, info = cpu_oracle_sample(orc, kind, X, Y, h, job=job)
            line["cpu_baseline"] = dict(info, value=m / full, unit="queries/s",
                                        wall_s=full, reference_flash_engine=REF_FLASH_NOTE)
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()
    return 0


def run_dry(args, rank, world):
    """--dry-run: the launcher and the rank protocol (process group, barrier,
    max-over-ranks, one JSON line from rank 0) without a GPU (gloo), for the
    CPU tests of the N-rank launch."""
    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        dist.barrier()
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"metric": metric_of(args.workload), "dry_run": True, "n_gpus": world,
                          "max_over_ranks": float(t.item()), "steps": args.steps,
                          "warmup": args.warmup}), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(argv, n):
    """bench.py --gpus N outside torchrun: one process per GPU via torchrun
    (the same launch the driver uses), rank 0's JSON line passes through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__)] + argv
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", type=int, default=5, choices=sorted(WORKLOADS),
                    help="BASELINE.json config (default 5, the headline)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(sys.argv[1:], args.gpus)
    rank, world, _ = env_rank()
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; reporting n_gpus={world}",
              file=sys.stderr)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
