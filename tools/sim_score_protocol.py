"""Model check of the score kernel's mbarrier protocol (csrc/pairwise_tc.cuh,
pairwise_tc_kernel<kModeScore>) for one CTA.

Actors: the GEMM1 issuer, the GEMM2 issuer, the 4 O-drain warps (one per TMEM
lane quadrant) and the 4*NP epilogue warps, each a
generator yielding the waits of the kernel in program order; arrivals and
tensor-core commits are applied when the actor resumes (the tensor core is
in-order, so a commit after an MMA completes when the actor issues it).  A
random scheduler interleaves ready actors.  Every parity wait also carries the
completion count it semantically needs: passing a parity wait on an older phase
(aliasing) is reported as an error, as is a deadlock.

    python tools/sim_score_protocol.py NP F 7,6,1 [seed] [SB]
"""
import random
import sys



class _Bar:
    def __init__(self, name, count):
        self.name, self.count, self.pending, self.phase = name, count, count, 0

    def arrive(self):
        self.pending -= 1
        if self.pending == 0:
            self.phase += 1
            self.pending = self.count

    def done(self, parity, need):
        ok = (self.phase & 1) != parity
        if ok and need is not None and self.phase < need:
            raise RuntimeError(f"ALIAS {self.name} phase {self.phase} need {need}")
        return ok


def run(NP, F, lens, seed=0, SB=4):
    """SB: S/P TMEM buffers (384 / column-tile width)."""
    lf = F.bit_length() - 1
    fmask = F - 1
    bars = {}

    def B(name, i, count):
        if (name, i) not in bars:
            bars[(name, i)] = _Bar((name, i), count)
        return bars[(name, i)]

    sfull = lambda i: B("s_full", i, 1)
    sfree = lambda i: B("s_free", i, 1)
    pfull = lambda i: B("p_full", i, 4)
    ofull = lambda i: B("o_full", i, 1)
    oempty = lambda i: B("o_empty", i, 4)

    def g1():
        it = 0
        for L in lens:
            for _ in range(L):
                sb, ph = it % SB, (it // SB) & 1
                yield (sfree(sb), ph ^ 1, it // SB)
                sfull(sb).arrive()
                it += 1

    def g2():
        it = itu = 0
        for L in lens:
            for rel in range(L):
                sb, ph = it % SB, (it // SB) & 1
                first = (rel & fmask) == 0
                last = (rel & fmask) == fmask or rel == L - 1
                ob = itu & 1
                yield (pfull(sb), ph, it // SB + 1)
                if first:
                    yield (oempty(ob), ((itu >> 1) & 1) ^ 1, itu >> 1)
                sfree(sb).arrive()
                if last:
                    ofull(ob).arrive()
                    itu += 1
                it += 1

    def drainer(q):
        itu = 0
        for L in lens:
            for _ in range((L + fmask) >> lf):
                g = itu
                yield (ofull(g & 1), (g >> 1) & 1, (g >> 1) + 1)
                oempty(g & 1).arrive()
                itu += 1

    def epi(par, q):
        its = 0
        for L in lens:
            rel = (par - its % NP) % NP
            sidx = its + rel
            sb, ph = sidx % SB, (sidx // SB) & 1
            while rel < L:
                yield (sfull(sb), ph, (its + rel) // SB + 1)
                pfull(sb).arrive()
                sb += NP
                if sb >= SB:
                    sb -= SB
                    ph ^= 1
                rel += NP
            its += L

    rng = random.Random(seed)
    actors = [g1(), g2()] + [drainer(q) for q in range(4)] + \
        [epi(p, q) for p in range(NP) for q in range(4)]
    cur = [None] * len(actors)
    done = [False] * len(actors)
    try:
        while True:
            for i, a in enumerate(actors):
                if not done[i] and cur[i] is None:
                    try:
                        cur[i] = next(a)
                    except StopIteration:
                        done[i] = True
            if all(done):
                return "OK"
            ready = [i for i in range(len(actors)) if not done[i] and cur[i][0].done(*cur[i][1:])]
            if not ready:
                return "DEADLOCK"
            cur[rng.choice(ready)] = None
    except RuntimeError as e:
        return str(e)


if __name__ == "__main__":
    print(run(int(sys.argv[1]), int(sys.argv[2]), [int(x) for x in sys.argv[3].split(",")],
              int(sys.argv[4]) if len(sys.argv) > 4 else 0, int(sys.argv[5]) if len(sys.argv) > 5 else 4))
