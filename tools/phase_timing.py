"""Debug: cycles per flux-kernel phase (build with -DHGKS_PHASE_TIMING into libhgks_timing.so)."""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.getcwd())
os.environ.setdefault("HGKS_LIB", os.path.join(os.getcwd(), "paper_2207_01173_b200", "libhgks_timing.so"))
from paper_2207_01173_b200 import hgks as H  # noqa: E402
from paper_2207_01173_b200 import inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
q, dx = inputs.tgv(n)
L = H.lib()
L.hgks_debug_phase_cycles.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 4)()
with H.Solver((n, n, n), (-math.pi,) * 3, (math.pi,) * 3, mu=1 / 1600, cfl=0.4) as s:
    s.set_state(q)
    s.step(1)
    L.hgks_debug_phase_cycles(buf, 1)
    s.step(2)
    L.hgks_debug_phase_cycles(buf, 1)
tot = buf[0] + buf[1] + buf[2]
print(f"blocks {buf[3]}  per-block cycles: A(copy+wait) {buf[0] / buf[3]:.0f}  B {buf[1] / buf[3]:.0f}  C {buf[2] / buf[3]:.0f}"
      f"  shares A {buf[0] / tot:.3f} B {buf[1] / tot:.3f} C {buf[2] / tot:.3f}")
