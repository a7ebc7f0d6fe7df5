"""Host model of flux_ring_kernel's warp schedule (paper_2207_01173_b200/csrc/flux_ring.cuh).

Each warp is a generator that yields wait predicates; a random scheduler advances warps whose
predicate holds, as the SM's warp schedulers would.  The model follows the kernel's order exactly
(produce the warp's rows -- recycle wait, publish -- then wait for rows bb..bb+4, read them, release
them) and records what every consumer actually read, so a test can check (1) termination for any
interleaving (no deadlock) and (2) that each face row read exactly rows bb..bb+4 of its own strip
(no slot overwritten while still in use).
"""
from __future__ import annotations

import random


def strip_lengths(n1t: int, n2c: int, L: int, n2: int, nf: int, block: int, G: int):
    out = []
    s = block
    total = n1t * n2c * nf
    while s < total:
        i2 = (s // n1t) % n2c
        out.append(min(L, n2 - i2 * L))
        s += G
    return out


def row_consumers(l2: int, Ls: int) -> int:
    lo, hi = max(0, l2 - 4), min(l2, Ls - 1)
    return max(0, hi - lo + 1)


def prologue_rows(bb: int, L: int):
    """stream rows l2 < 4 produced by face row bb (l2 % L == bb)."""
    return [l2 for l2 in range(4) if l2 % L == bb]


def simulate(NW: int, RING: int, L: int, Ls_list, seed: int = 0, max_steps: int = 10_000_000):
    rnd = random.Random(seed)
    L4 = L + 4
    seq = [0] * RING
    done = [0] * RING
    data = [None] * RING  # (strip, l2) held by the slot
    nface_rows = len(Ls_list) * L
    reads = {}

    def produce(j, l2, real):
        R = j * L4 + l2
        sl = R % RING
        if R >= RING:
            Rp = R - RING
            jp, l2p = divmod(Rp, L4)
            need = row_consumers(l2p, Ls_list[jp])
            # the slot must hold the previous occupant (its producer ran) and be released by its
            # consumers: producers of one slot then run in stream order
            yield lambda: seq[sl] == Rp + 1 and done[sl] >= need
            assert done[sl] == need, (R, done[sl], need)
            done[sl] = 0
        if real:
            data[sl] = (j, l2)
        yield None
        seq[sl] = R + 1

    def warp(w):
        F = w
        while F < nface_rows:
            j, bb = divmod(F, L)
            Ls = Ls_list[j]
            for l2 in prologue_rows(bb, L):
                yield from produce(j, l2, True)
            yield from produce(j, bb + 4, bb < Ls)
            if bb < Ls:
                R0 = j * L4 + bb
                for r in range(5):
                    sl = (R0 + r) % RING
                    yield (lambda sl=sl, v=R0 + r + 1: seq[sl] == v)
                got = []
                for r in range(5):
                    got.append(data[(R0 + r) % RING])
                    yield None  # reads interleave with other warps
                # the reads must still be valid when the last one is done
                reads[(j, bb)] = got
                for r in range(5):
                    done[(R0 + r) % RING] += 1
            F += NW

    gens = {w: warp(w) for w in range(NW)}
    pending = {w: None for w in gens}
    steps = 0
    while gens:
        ready = [w for w in gens if pending[w] is None or pending[w]()]
        if not ready:
            raise RuntimeError(f"deadlock after {steps} steps: waiting warps {sorted(gens)}")
        w = rnd.choice(ready)
        try:
            pending[w] = next(gens[w])
        except StopIteration:
            del gens[w]
        steps += 1
        if steps > max_steps:
            raise RuntimeError("no termination")
    for j, Ls in enumerate(Ls_list):
        for bb in range(Ls):
            assert reads[(j, bb)] == [(j, bb + r) for r in range(5)], (j, bb, reads[(j, bb)])
    return steps
