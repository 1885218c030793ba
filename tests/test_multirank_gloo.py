"""Multi-rank protocol of the engine, exercised on CPU with torch.distributed
(gloo, world_size 2).

The device program per rank (csrc/fkde_gpu.cu: score_program / query_program)
is: score pass on the rank's row shard -> in-place allgather of the debiased
samples -> density pass on the rank's query shard -> in-place allgather of
the densities.  Here the per-shard compute is the CPU oracle (a test double:
the GPU kernels are covered by tests/test_gpu_parity.py) and the partition is
the engine's own (fkde_gpu_shard_range: row shards tile-aligned for the score
pass, equal-size allgather slices), so the test pins the sharding + gather
layout: the gathered result must equal the single-process oracle bitwise,
the analogue of the reference's partition-invariance test
(proj/tests/test_engine.cpp:245-262).
"""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, n, m, d, h, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist
    import oracle as O
    from paper_2602_10378_b200 import _native as N

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = O.get("port")
    X = P.random_gaussian(n, d, 11, 1.3)
    Y = P.random_gaussian(m, d, 12, 1.3)

    # score pass on this rank's row shard (tile-aligned, as the engine does)
    b, rows, chunk = N.shard_range(n, world, rank, 128)
    xsd = np.zeros((chunk * world, d))
    if rows:
        s = P.score_naive(X, X, h, rows=(b, b + rows))
        xsd[b:b + rows] = X[b:b + rows] + (0.5 * h * h) * s
    t = torch.from_numpy(xsd)
    parts = list(t.view(world, chunk, d).unbind(0))
    dist.all_gather(parts, parts[rank].clone())
    xsd_full = torch.cat(parts).numpy()[:n]

    # density pass on this rank's query shard
    qb, qrows, qchunk = N.shard_range(m, world, rank, 1)
    dens = np.zeros(qchunk * world)
    if qrows:
        dens[qb:qb + qrows] = P.kde_naive(xsd_full, Y, h, rows=(qb, qb + qrows))
    t = torch.from_numpy(dens)
    parts = list(t.view(world, qchunk).unbind(0))
    dist.all_gather(parts, parts[rank].clone())
    full = torch.cat(parts).numpy()[:m]
    np.save(os.path.join(out_dir, f"rank{rank}_dens.npy"), full)
    np.save(os.path.join(out_dir, f"rank{rank}_xsd.npy"), xsd_full)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,m", [(300, 77), (1000, 129), (129, 1)])
def test_two_rank_sdkde_protocol_matches_single_process(tmp_path, port, n, m):
    import torch.multiprocessing as mp
    d, h, world = 3, 0.8, 2
    mp.start_processes(_rank_main, args=(world, _free_port(), n, m, d, h, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    X = port.random_gaussian(n, d, 11, 1.3)
    Y = port.random_gaussian(m, d, 12, 1.3)
    ref_vals, ref_deb = port.sdkde_naive(X, Y, h)
    for r in range(world):
        dens = np.load(tmp_path / f"rank{r}_dens.npy")
        xsd = np.load(tmp_path / f"rank{r}_xsd.npy")
        assert np.array_equal(xsd, ref_deb)        # every rank holds all debiased samples
        assert np.array_equal(dens, ref_vals)      # every rank holds all densities
