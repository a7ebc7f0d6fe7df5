"""ctypes wrapper of the plain CPU fp64 oracle (oracle/hgks_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The product path
(``paper_2207_01173_b200``) never imports it; the two share no code.

Arrays use the ABI layout [5][nz][ny][nx] (x fastest), float64, C-contiguous.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "hgks_oracle.c")

_dp = C.POINTER(C.c_double)


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, OpenMP, strict IEEE: no -ffast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
        os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "hgks_oracle.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-fopenmp", "-fPIC", "-shared",
             "-fno-fast-math", "-ffp-contract=off", "-o", LIB, SRC, "-lm"]
        )
    return LIB


FLOPCOUNT_SRC = os.path.join(HERE, "flopcount.cpp")
FLOPCOUNT_BIN = os.path.join(HERE, "flopcount")


def build_flopcount(force: bool = False) -> str:
    """g++ the counting build of the oracle (oracle/flopcount.cpp: hgks_oracle.c with a counting double)."""
    if force or not os.path.exists(FLOPCOUNT_BIN) or os.path.getmtime(FLOPCOUNT_BIN) < max(
        os.path.getmtime(FLOPCOUNT_SRC), os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "hgks_oracle.h"))
    ):
        subprocess.check_call(["g++", "-O1", "-std=c++17", "-w", "-o", FLOPCOUNT_BIN, FLOPCOUNT_SRC])
    return FLOPCOUNT_BIN


def flopcount() -> dict:
    """The oracle's arithmetic counted on TGV 16^3 (flops per Gauss point, face, cell-update)."""
    import json
    return json.loads(subprocess.check_output([build_flopcount()]))


class Gas(C.Structure):
    _fields_ = [("gamma", C.c_double), ("K", C.c_double), ("prandtl", C.c_double),
                ("mu_law", C.c_int), ("mu_ref", C.c_double), ("T_ref", C.c_double),
                ("omega", C.c_double), ("T_wall", C.c_double)]


class Grid(C.Structure):
    _fields_ = [("n", C.c_int * 3), ("dx", C.c_double * 3), ("bc", C.c_int * 3),
                ("stretch", C.c_int * 3), ("lo", C.c_double * 3), ("hi", C.c_double * 3),
                ("stretch_b", C.c_double * 3)]


class Forcing(C.Structure):
    _fields_ = [("mode", C.c_int), ("force", C.c_double), ("target", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        L.or_K.restype = C.c_double
        L.or_K.argtypes = [C.c_double]
        L.or_moments_u.argtypes = [C.c_double, C.c_double, C.c_int, _dp]
        L.or_psi_moment.argtypes = [C.c_double] * 5 + [C.c_int] * 5 + [_dp]
        L.or_cons_to_maxw.argtypes = [_dp, C.c_double, _dp]
        L.or_slope_solve.argtypes = [_dp, C.c_double, _dp, _dp]
        L.or_time_integrals.argtypes = [C.c_double, C.c_double, _dp]
        L.or_gp_flux.argtypes = [C.POINTER(Gas), _dp, _dp, _dp, _dp, _dp, C.c_double, _dp, _dp, _dp]
        L.or_set_num_threads.argtypes = [C.c_int]
        L.or_weno5z_right.restype = C.c_double
        L.or_weno5z_right.argtypes = [_dp]
        L.or_weno5z_left.restype = C.c_double
        L.or_weno5z_left.argtypes = [_dp]
        L.or_face_gauss_points.argtypes = [_dp, C.c_double, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.or_fill_ghosts.argtypes = [C.POINTER(Gas), C.POINTER(Grid), _dp]
        L.or_axis_face.restype = C.c_double
        L.or_axis_face.argtypes = [C.POINTER(Grid), C.c_int, C.c_int]
        L.or_axis_metric.restype = C.c_double
        L.or_axis_metric.argtypes = [C.POINTER(Grid), C.c_int, C.c_double]
        L.or_operator.argtypes = [C.POINTER(Gas), C.POINTER(Grid), _dp, C.c_double, _dp, _dp]
        L.or_s2o4_stage1.argtypes = [C.c_long, _dp, _dp, _dp, C.c_double, _dp]
        L.or_s2o4_final.argtypes = [C.c_long, _dp, _dp, _dp, _dp, C.c_double, _dp]
        L.or_cfl_dt.restype = C.c_double
        L.or_cfl_dt.argtypes = [C.POINTER(Gas), C.POINTER(Grid), _dp, C.c_double]
        L.or_run.argtypes = [C.POINTER(Gas), C.POINTER(Grid), _dp, C.c_int, C.c_double,
                             C.c_double, _dp]
        L.or_run_forced.argtypes = [C.POINTER(Gas), C.POINTER(Grid), _dp, C.c_int, C.c_double, C.c_double,
                                    C.POINTER(Forcing), _dp, _dp]
        L.or_plane_stats.argtypes = [C.POINTER(Gas), C.POINTER(Grid), _dp, _dp]
        L.or_diagnostics.argtypes = [C.POINTER(Gas), C.POINTER(Grid), _dp, C.c_double, _dp]
        L.or_num_threads.restype = C.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _arr(x, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


def K_of(gamma: float) -> float:
    return lib().or_K(gamma)


def make_gas(gamma=1.4, mu=0.0, prandtl=1.0, mu_law=0, T_ref=1.0, omega=0.0, T_wall=1.0) -> Gas:
    return Gas(gamma, K_of(gamma), prandtl, mu_law, mu, T_ref, omega, T_wall)


def make_grid(n, dx, bc=(0, 0, 0), stretch=(0, 0, 0), lo=(0.0, 0.0, 0.0), hi=None, stretch_b=(0.0, 0.0, 0.0)) -> Grid:
    """n cells; dx widths of uniform axes; bc 0 periodic / 1 isothermal wall; stretch 1 = tanh
    on [lo, hi] with b = stretch_b."""
    g = Grid()
    for d in range(3):
        g.n[d] = int(n[d])
        g.dx[d] = float(dx[d])
        g.bc[d] = int(bc[d])
        g.stretch[d] = int(stretch[d])
        g.lo[d] = float(lo[d])
        g.hi[d] = float(hi[d]) if hi is not None else float(lo[d]) + n[d] * float(dx[d])
        g.stretch_b[d] = float(stretch_b[d])
    return g


def axis_faces(grid: Grid, d: int) -> np.ndarray:
    return np.array([lib().or_axis_face(C.byref(grid), d, j) for j in range(grid.n[d] + 1)])


def axis_metric(grid: Grid, d: int, zeta: float) -> float:
    return lib().or_axis_metric(C.byref(grid), d, zeta)


def moments_u(U, lam, which):
    m = np.zeros(9)
    lib().or_moments_u(U, lam, which, _p(m))
    return m


def psi_moment(U, V, W, lam, K, which, a, b, c, d):
    out = np.zeros(5)
    lib().or_psi_moment(U, V, W, lam, K, which, a, b, c, d, _p(out))
    return out


def cons_to_maxw(q, K):
    q = _arr(q)
    mx = np.zeros(5)
    rc = lib().or_cons_to_maxw(_p(q), K, _p(mx))
    return None if rc else mx


def slope_solve(mx, K, b):
    mx, b = _arr(mx), _arr(b)
    a = np.zeros(5)
    assert lib().or_slope_solve(_p(mx), K, _p(b), _p(a)) == 0
    return a


def time_integrals(T, tau):
    g = np.zeros(6)
    lib().or_time_integrals(T, tau, _p(g))
    return g


def gp_flux(gas: Gas, Wl, dWl, Wr, dWr, dW0, dt):
    Wl, Wr = _arr(Wl, (5,)), _arr(Wr, (5,))
    dWl, dWr, dW0 = _arr(dWl, (3, 5)), _arr(dWr, (3, 5)), _arr(dW0, (3, 5))
    F, dF, tau = np.zeros(5), np.zeros(5), np.zeros(1)
    rc = lib().or_gp_flux(C.byref(gas), _p(Wl), _p(dWl), _p(Wr), _p(dWr), _p(dW0), dt, _p(F),
                          _p(dF), _p(tau))
    if rc:
        raise ValueError("invalid Gauss-point state")
    return F, dF, float(tau[0])


def weno5z(q, side="right"):
    q = _arr(q, (5,))
    f = lib().or_weno5z_right if side == "right" else lib().or_weno5z_left
    return f(_p(q))


def face_gauss_points(cells, h=None, J=None):
    """cells: [6 normal][5 t1][5 t2][5 comp] -> dict of GP inputs.  Uniform widths h = (hn, h1, h2)
    or metrics J = (Jn, [Jt1_m0, Jt1_m1], [Jt2_n0, Jt2_n1])."""
    cells = _arr(cells, (6, 5, 5, 5))
    if J is None:
        J = (1.0 / h[0], [1.0 / h[1]] * 2, [1.0 / h[2]] * 2)
    Jt1, Jt2 = _arr(J[1], (2,)), _arr(J[2], (2,))
    Wl, Wr = np.zeros((4, 5)), np.zeros((4, 5))
    dWl, dWr, dW0 = np.zeros((4, 3, 5)), np.zeros((4, 3, 5)), np.zeros((4, 3, 5))
    lib().or_face_gauss_points(_p(cells), float(J[0]), _p(Jt1), _p(Jt2), _p(Wl), _p(Wr), _p(dWl),
                               _p(dWr), _p(dW0))
    return dict(Wl=Wl, Wr=Wr, dWl=dWl, dWr=dWr, dW0=dW0)


def _grid_of(q, dx, grid):
    _, nz, ny, nx = q.shape
    return grid if grid is not None else make_grid((nx, ny, nz), dx)


def ghosted(q: np.ndarray, ng: int = 3, gas: Gas | None = None, grid: Grid | None = None) -> np.ndarray:
    """[5][nz][ny][nx] -> [5][nz+6][ny+6][nx+6] with ghosts filled by the oracle (periodic unless
    grid says walls)."""
    q = _arr(q)
    _, nz, ny, nx = q.shape
    qg = np.zeros((5, nz + 2 * ng, ny + 2 * ng, nx + 2 * ng))
    qg[:, ng:-ng, ng:-ng, ng:-ng] = q
    gr = grid if grid is not None else make_grid((nx, ny, nz), (1, 1, 1))
    lib().or_fill_ghosts(C.byref(gas if gas is not None else make_gas()), C.byref(gr), _p(qg))
    return qg


def operator(gas: Gas, q: np.ndarray, dx, dt: float, qg: np.ndarray | None = None, grid: Grid | None = None):
    """L(Q), d_t L(Q) for a state (periodic unless grid has walls) or a pre-ghosted block qg."""
    q = _arr(q)
    gr = _grid_of(q, dx, grid)
    if qg is None:
        qg = ghosted(q, gas=gas, grid=gr)
    qg = _arr(qg)
    L, dL = np.zeros_like(q), np.zeros_like(q)
    rc = lib().or_operator(C.byref(gas), C.byref(gr), _p(qg), dt, _p(L), _p(dL))
    if rc:
        raise ValueError("invalid state inside operator")
    return L, dL


def s2o4_stage1(q, L, dL, dt):
    q, L, dL = _arr(q), _arr(L), _arr(dL)
    qs = np.zeros_like(q)
    lib().or_s2o4_stage1(q.size, _p(q), _p(L), _p(dL), dt, _p(qs))
    return qs


def s2o4_final(q, L, dL, dLs, dt):
    q, L, dL, dLs = _arr(q), _arr(L), _arr(dL), _arr(dLs)
    qn = np.zeros_like(q)
    lib().or_s2o4_final(q.size, _p(q), _p(L), _p(dL), _p(dLs), dt, _p(qn))
    return qn


def cfl_dt(gas: Gas, q: np.ndarray, dx, cfl: float = 0.4, grid: Grid | None = None) -> float:
    q = _arr(q)
    return lib().or_cfl_dt(C.byref(gas), C.byref(_grid_of(q, dx, grid)), _p(q), cfl)


def run(gas: Gas, q: np.ndarray, dx, nsteps: int, dt_fixed: float = 0.0, cfl: float = 0.4,
        grid: Grid | None = None):
    """Advance a state nsteps full S2O4 steps (periodic unless grid has walls); returns
    (q_new, dt_history)."""
    q = _arr(q).copy()
    hist = np.zeros(max(nsteps, 1))
    rc = lib().or_run(C.byref(gas), C.byref(_grid_of(q, dx, grid)), _p(q), nsteps, dt_fixed,
                      cfl, _p(hist))
    if rc:
        raise ValueError("oracle run hit an invalid state")
    return q, hist[:nsteps]


DIAG_NAMES = ("E_k", "enstrophy", "eps_s", "eps_d", "mass", "mom_x", "mom_y", "mom_z", "energy", "volume",
              "p_dil")


def diagnostics(gas: Gas, q: np.ndarray | None = None, dx=None, rho0: float = 1.0, qg: np.ndarray | None = None,
                grid: Grid | None = None) -> np.ndarray:
    """Volume diagnostics (or_diagnostics) of a state (ghosts filled by the oracle) or of a
    pre-ghosted block qg (ghosts as given).  Returns the OR_NDIAG vector in DIAG_NAMES order."""
    if qg is None:
        q = _arr(q)
        gr = _grid_of(q, dx, grid)
        qg = ghosted(q, gas=gas, grid=gr)
    else:
        qg = _arr(qg)
        gr = grid if grid is not None else make_grid(tuple(s - 6 for s in qg.shape[:0:-1]), dx)
    out = np.zeros(len(DIAG_NAMES))
    lib().or_diagnostics(C.byref(gas), C.byref(gr), _p(qg), rho0, _p(out))
    return out


def run_forced(gas: Gas, q: np.ndarray, dx, nsteps: int, mode: int, force: float = 0.0, target: float = 0.0,
               dt_fixed: float = 0.0, cfl: float = 0.4, grid: Grid | None = None):
    """or_run_forced: returns (q_new, dt_history, force_history)."""
    q = _arr(q).copy()
    hist = np.zeros(max(nsteps, 1))
    fh = np.zeros(max(nsteps, 1))
    fc = Forcing(mode, force, target)
    rc = lib().or_run_forced(C.byref(gas), C.byref(_grid_of(q, dx, grid)), _p(q), nsteps, dt_fixed, cfl,
                             C.byref(fc), _p(hist), _p(fh))
    if rc:
        raise ValueError("oracle run hit an invalid state")
    return q, hist[:nsteps], fh[:nsteps]


STAT_NAMES = ("rho", "U", "V", "W", "UU", "VV", "WW", "UV", "rhoU", "rhoV", "rhoUV", "c", "M", "MM", "T", "p")


def plane_stats(gas: Gas, q: np.ndarray, dx=None, grid: Grid | None = None) -> np.ndarray:
    """or_plane_stats: [ny][16] x-z plane means in STAT_NAMES order."""
    q = _arr(q)
    gr = _grid_of(q, dx, grid)
    out = np.zeros((q.shape[2], len(STAT_NAMES)))
    lib().or_plane_stats(C.byref(gas), C.byref(gr), _p(q), _p(out))
    return out


def num_threads() -> int:
    return lib().or_num_threads()


def set_num_threads(n: int) -> None:
    """Host threads of the OpenMP loops (n <= 0: all cores)."""
    lib().or_set_num_threads(int(n))
