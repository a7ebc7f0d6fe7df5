"""The warp schedule of flux_ring_kernel (host model, tests/ring_schedule.py): for the kernel's
(NW, RING) in fp64 and fp32 and strip lengths from 1 row (thin slabs) to 2.5 rings, ragged strip
ends and several strips per block, every random interleaving terminates (no deadlock) and every face
row reads exactly rows bb..bb+4 of its own strip (no ring slot is recycled while in use)."""
import pytest

from tests.ring_schedule import simulate, strip_lengths

CFG = {"fp64": (16, 24), "fp32": (24, 32)}


@pytest.mark.parametrize("prec", sorted(CFG))
@pytest.mark.parametrize("n2,L", [(1, 1), (3, 3), (5, 5), (11, 11), (16, 16), (37, 37), (70, 35), (130, 65), (60, 64)])
def test_ring_schedule_terminates_and_reads_its_rows(prec, n2, L):
    NW, RING = CFG[prec]
    n2c = -(-n2 // L)
    Ls = strip_lengths(n1t=2, n2c=n2c, L=L, n2=n2, nf=3, block=0, G=1)
    for seed in range(6):
        simulate(NW, RING, L, Ls, seed=seed)


def test_ring_schedule_detects_a_short_ring():
    """the model is sharp: a ring smaller than a face row's five rows plus the producer lead hangs"""
    with pytest.raises(RuntimeError):
        simulate(16, 4, 16, [16, 16], seed=0)
