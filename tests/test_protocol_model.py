"""Model check of the score kernel's barrier protocol (tools/sim_score_protocol.py):
no deadlock and no parity-wait aliasing under random warp interleavings, for the
drain intervals and unit shapes the engine can produce (1-tile units, odd lengths,
units shorter than the epilogue phase count)."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import sim_score_protocol as sim  # noqa: E402

SHAPES = [[7, 6], [1, 2, 3], [2, 2, 1, 5], [1] * 7, [4, 1, 1, 4], [3, 3, 3, 3], [9], [11, 10, 1]]


@pytest.mark.parametrize("SB,NP", [(3, 2), (3, 3), (4, 2), (4, 3), (6, 2), (6, 3)])
@pytest.mark.parametrize("F", [1, 2, 4, 8])
def test_protocol_is_deadlock_and_alias_free(SB, NP, F):
    # SB = S/P buffers (384 TMEM columns / column-tile width 128, 96, 64)
    for lens in SHAPES:
        for seed in range(12):
            assert sim.run(NP, F, lens, seed, SB) == "OK", (SB, NP, F, lens, seed)
