"""The counting build of the oracle (oracle/flopcount.cpp) runs and its counts hang together: the
operator per face is the four Gauss-point fluxes plus the reconstruction, per cell-update is two
operator evaluations (stages) plus the Eq. (7) update, and the GPU's executed flops per face
(profiles/flux_flops.json, ncu) are a fraction of the method as the oracle computes it."""
import json
import os

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_flopcount_consistent():
    c = O.flopcount()
    gp = c["gp_flux_per_gauss_point"]["flops"]
    face = c["operator_per_face_per_stage"]["flops"]
    cell = c["operator_per_cell_per_stage"]["flops"]
    assert gp > 1000 and face > 4 * gp  # 2x2 Gauss points per face (O-8) + tangential reconstruction
    assert abs(cell - 3 * face) <= 1e-6 * cell  # periodic: one face per cell per direction
    upd = c["s2o4_update_per_cell"]["flops"]
    assert abs(c["flops_per_cell_update"] - (2 * cell + upd)) <= 1e-6 * c["flops_per_cell_update"]
    assert c["gp_flux_per_gauss_point"]["erfc"] == 2 and c["gp_flux_per_gauss_point"]["exp"] >= 2
    ftab = json.load(open(os.path.join(ROOT, "profiles", "flux_flops.json")))
    assert ftab["fp64_flop_per_face_stage1"] < face  # the GPU's reduced algebra executes fewer flops
