"""C-ABI library checks that need no GPU: the library loads, exports every symbol declared in
include/*.h, validates parameters before touching a device, and its host-side decomposition logic
(slab split, halo plan) is right."""
import re

import pytest

from paper_2207_01173_b200 import hgks as H


def _declared_functions():
    names = set()
    for hdr in ("include/hgks.h", "include/hgks_test.h"):
        src = open(hdr).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(hgks_[a-z0-9_]+)\s*\(", src, re.M):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    lib = H.lib()
    declared = _declared_functions()
    assert {"hgks_create", "hgks_set_state", "hgks_step", "hgks_get_state", "hgks_destroy"} <= declared
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert set(H.EXPORTED) == declared


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", H.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_slab_decomposition():
    for nz, nr in [(256, 1), (256, 8), (130, 4), (17, 5)]:
        spans = [H.hgks_slab_of(nz, r, nr) for r in range(nr)]
        assert spans[0][0] == 0
        for (z0, n), (z1, _) in zip(spans, spans[1:]):
            assert z0 + n == z1
        assert spans[-1][0] + spans[-1][1] == nz
        assert max(n for _, n in spans) - min(n for _, n in spans) <= 1
    with pytest.raises(H.HgksError):
        H.hgks_slab_of(3, 0, 4)


def test_halo_plan_ring_and_offsets():
    nx, ny, nzl = 7, 5, 4
    plane = 5 * (ny + 6) * (nx + 6)
    p = H.hgks_make_halo_plan(nx, ny, nzl, 0, 3)
    assert (p["up"], p["down"]) == (1, 2)
    assert p["count"] == 3 * plane
    # ghosted z index g = k + 3: sends start at interior planes nzl-3 and 0, receives at ghosts
    assert p["send_up"] == (nzl - 3 + 3) * plane and p["recv_down"] == 0
    assert p["send_down"] == 3 * plane and p["recv_up"] == (nzl + 3) * plane
    p1 = H.hgks_make_halo_plan(nx, ny, nzl, 0, 1)
    assert (p1["up"], p1["down"]) == (0, 0)


def test_create_validates_before_device():
    bad = [dict(n=(4, 8, 8)), dict(gamma=2.0), dict(prandtl=0.0), dict(cfl=0.0, dt_fixed=0.0),
           dict(bc=(0, 0, 1)), dict(stretch=(0, 0, 1), stretch_b=(0, 0, 2.0)), dict(stretch=(1, 0, 0)),
           dict(bc=(0, 1, 0), T_wall=0.0),
           dict(nranks=2, rank=0), dict(n=(8, 8, 5), nranks=2, rank=1, nccl_id=b"x" * 128),
           dict(nranks=2, rank=0, nccl_id=b"x" * 128, group_key=7),  # NCCL and loopback are exclusive
           dict(n=(8, 8, 60), nranks=17, rank=0, group_key=7),       # loopback group: <= 16 ranks
           dict(bc=(1, 1, 0), T_wall=1.0)]                            # walls on x AND y (duct corners)
    for kw in bad:
        args = dict(n=(8, 8, 8), lo=(0, 0, 0), hi=(1, 1, 1))
        args.update(kw)
        n = args.pop("n")
        with pytest.raises(H.HgksError) as e:
            H.hgks_create(H.make_params(n, args.pop("lo"), args.pop("hi"), **args))
        assert e.value.code == H.HGKS_EINVAL, kw


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(H.HgksError) as e:
        H.hgks_create(H.make_params((8, 8, 8), (0, 0, 0), (1, 1, 1)))
    assert e.value.code == H.HGKS_ECUDA
