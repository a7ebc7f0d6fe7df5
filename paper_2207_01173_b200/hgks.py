"""Thin ctypes binding of libhgks.so (include/hgks.h).  Argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; this module never computes
physics.  There is no fallback: if libhgks.so is missing or cannot be loaded, importing the
binding's functions raises.

Names mirror the C ABI: hgks_create, hgks_local_extent, hgks_set_state, hgks_step,
hgks_get_state, hgks_destroy, hgks_last_error, plus a small ``Solver`` convenience wrapper.
States use the ABI layout [5][nz_local][ny][nx] float64 (numpy host arrays, or torch CUDA
tensors passed by device pointer).

Multi-rank: one process per GPU with an NCCL unique id (``hgks_get_nccl_id`` on rank 0, broadcast,
``make_params(..., rank, nranks, nccl_id=...)``), or the in-process loopback group for tests on one
device (``run_loopback_group`` with ``group_key``).  Environment: ``HGKS_GRAPHS=0`` disables the
CUDA-graph replay of step pairs (single-rank contexts); ``HGKS_LIB`` points at another build.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HGKS_LIB") or os.path.join(PKG, "libhgks.so")

HGKS_OK, HGKS_EINVAL, HGKS_ECUDA, HGKS_ENCCL, HGKS_ESTATE, HGKS_ENOMEM = 0, -1, -2, -3, -4, -5
HGKS_FP64, HGKS_FP32 = 0, 1
HGKS_PERIODIC, HGKS_WALL_ISOTHERMAL = 0, 1
HGKS_UNIFORM, HGKS_TANH = 0, 1
HGKS_MU_CONST, HGKS_MU_POWER = 0, 1
HGKS_FORCE_NONE, HGKS_FORCE_CONST, HGKS_FORCE_BULK = 0, 1, 2
KERNEL_CLASSES = ("flux_x", "flux_y", "flux_z", "update", "ghost", "halo", "dt", "recon")
EXPORTED = ("hgks_create", "hgks_local_extent", "hgks_set_state", "hgks_step", "hgks_get_state",
            "hgks_destroy", "hgks_last_error", "hgks_nccl_id_bytes", "hgks_get_nccl_id",
            "hgks_slab_of", "hgks_make_halo_plan", "hgks_profile_enable", "hgks_profile_read",
            "hgks_diagnostics", "hgks_history_enable", "hgks_history_read", "hgks_plane_stats", "hgks_get_forcing",
            "hgks_upload_state", "hgks_commit_state", "hgks_download_state", "hgks_io_wait",
            "hgks_test_gp_flux", "hgks_test_operator", "hgks_test_face_flux")
STAT_NAMES = ("rho", "U", "V", "W", "UU", "VV", "WW", "UV", "rhoU", "rhoV", "rhoUV", "c", "M", "MM", "T", "p")
DIAG_NAMES = ("E_k", "enstrophy", "eps_s", "eps_d", "mass", "mom_x", "mom_y", "mom_z", "energy", "volume",
              "p_dil")


class HgksError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"hgks error {code}: {msg}")
        self.code = code


class Params(C.Structure):
    _fields_ = [("n", C.c_int32 * 3), ("lo", C.c_double * 3), ("hi", C.c_double * 3),
                ("bc", C.c_int * 3), ("stretch", C.c_int * 3), ("stretch_b", C.c_double * 3),
                ("gamma", C.c_double), ("prandtl", C.c_double),
                ("mu_law", C.c_int), ("mu_ref", C.c_double), ("T_ref", C.c_double),
                ("omega", C.c_double), ("T_wall", C.c_double), ("cfl", C.c_double), ("dt_fixed", C.c_double),
                ("precision", C.c_int), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("device", C.c_int32), ("nccl_id", C.c_void_p), ("stream", C.c_void_p),
                ("force_mode", C.c_int), ("force", C.c_double), ("force_target", C.c_double),
                ("group_key", C.c_int64)]


class HaloPlan(C.Structure):
    _fields_ = [("up", C.c_int32), ("down", C.c_int32), ("send_up", C.c_int64),
                ("recv_down", C.c_int64), ("send_down", C.c_int64), ("recv_up", C.c_int64),
                ("count", C.c_int64)]


_lib = None
_dp = C.POINTER(C.c_double)


def lib():
    """Load libhgks.so (fails loudly when it is missing: there is no CPU path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.hgks_create.argtypes = [C.POINTER(Params), C.POINTER(vp)]
        L.hgks_local_extent.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.hgks_set_state.argtypes = [vp, vp, C.c_int]
        L.hgks_step.argtypes = [vp, C.c_int32, C.c_double, _dp, _dp]
        L.hgks_get_state.argtypes = [vp, vp, C.c_int]
        L.hgks_upload_state.argtypes = [vp, vp]
        L.hgks_commit_state.argtypes = [vp]
        L.hgks_download_state.argtypes = [vp, vp]
        L.hgks_io_wait.argtypes = [vp]
        L.hgks_destroy.argtypes = [vp]
        L.hgks_last_error.restype = C.c_char_p
        L.hgks_last_error.argtypes = [vp]
        L.hgks_nccl_id_bytes.restype = C.c_size_t
        L.hgks_get_nccl_id.argtypes = [vp]
        L.hgks_slab_of.argtypes = [C.c_int32] * 3 + [C.POINTER(C.c_int32)] * 2
        L.hgks_make_halo_plan.argtypes = [C.c_int32] * 5 + [C.POINTER(HaloPlan)]
        L.hgks_diagnostics.argtypes = [vp, C.c_double, _dp]
        L.hgks_get_forcing.argtypes = [vp, _dp, _dp, _dp]
        L.hgks_history_enable.argtypes = [vp, C.c_int32, C.c_double]
        L.hgks_history_read.argtypes = [vp, _dp, C.c_int32, C.POINTER(C.c_int32)]
        L.hgks_plane_stats.argtypes = [vp, _dp]
        L.hgks_profile_enable.argtypes = [vp, C.c_int]
        L.hgks_profile_read.argtypes = [vp, _dp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.hgks_test_gp_flux.argtypes = [C.c_int, C.c_double, C.c_int, C.c_double, C.c_double,
                                        C.c_double, C.c_double, C.c_double, _dp, C.c_int64, _dp]
        L.hgks_test_operator.argtypes = [vp, C.c_double, _dp, _dp]
        L.hgks_test_face_flux.argtypes = [vp, C.c_int, _dp]
        _lib = L
    return _lib


def _check(rc: int, ctx=None):
    if rc != HGKS_OK:
        msg = lib().hgks_last_error(ctx).decode(errors="replace")
        raise HgksError(rc, msg)


def hgks_last_error(ctx=None) -> str:
    return lib().hgks_last_error(ctx).decode(errors="replace")


def hgks_slab_of(nz: int, rank: int, nranks: int):
    z0, nl = C.c_int32(), C.c_int32()
    _check(lib().hgks_slab_of(nz, rank, nranks, C.byref(z0), C.byref(nl)))
    return z0.value, nl.value


def hgks_make_halo_plan(nx: int, ny: int, nz_local: int, rank: int, nranks: int) -> dict:
    p = HaloPlan()
    _check(lib().hgks_make_halo_plan(nx, ny, nz_local, rank, nranks, C.byref(p)))
    return {k: getattr(p, k) for k, _ in HaloPlan._fields_}


def hgks_get_nccl_id() -> bytes:
    n = lib().hgks_nccl_id_bytes()
    buf = C.create_string_buffer(n)
    _check(lib().hgks_get_nccl_id(buf))
    return buf.raw


def make_params(n, lo, hi, gamma=1.4, mu=0.0, prandtl=1.0, mu_law=HGKS_MU_CONST, T_ref=1.0,
                omega=0.0, cfl=0.4, dt_fixed=0.0, precision=HGKS_FP64, rank=0, nranks=1,
                device=0, nccl_id=None, stream=None, bc=(HGKS_PERIODIC,) * 3,
                stretch=(HGKS_UNIFORM,) * 3, stretch_b=(0.0, 0.0, 0.0), T_wall=1.0,
                force_mode=HGKS_FORCE_NONE, force=0.0, force_target=0.0, group_key=0):
    p = Params()
    for d in range(3):
        p.n[d] = int(n[d])
        p.lo[d] = float(lo[d])
        p.hi[d] = float(hi[d])
        p.bc[d] = int(bc[d])
        p.stretch[d] = int(stretch[d])
        p.stretch_b[d] = float(stretch_b[d])
    p.gamma, p.prandtl, p.mu_law = gamma, prandtl, mu_law
    p.mu_ref, p.T_ref, p.omega, p.T_wall = mu, T_ref, omega, T_wall
    p.cfl, p.dt_fixed, p.precision = cfl, dt_fixed, precision
    p.rank, p.nranks, p.device = rank, nranks, device
    p._id_buf = C.create_string_buffer(nccl_id, len(nccl_id)) if nccl_id is not None else None
    p.nccl_id = C.cast(p._id_buf, C.c_void_p) if nccl_id is not None else None
    p.stream = stream
    p.force_mode, p.force, p.force_target = int(force_mode), float(force), float(force_target)
    p.group_key = int(group_key)
    return p


def hgks_create(params: Params):
    ctx = C.c_void_p()
    _check(lib().hgks_create(C.byref(params), C.byref(ctx)))
    return ctx


def hgks_destroy(ctx) -> None:
    _check(lib().hgks_destroy(ctx))


def hgks_local_extent(ctx):
    z0, nl = C.c_int32(), C.c_int32()
    _check(lib().hgks_local_extent(ctx, C.byref(z0), C.byref(nl)), ctx)
    return z0.value, nl.value


def _ptr(q):
    """(pointer, on_device) of a float64 C-contiguous numpy array or torch CUDA tensor."""
    if isinstance(q, np.ndarray):
        if q.dtype != np.float64 or not q.flags.c_contiguous:
            raise TypeError("state must be C-contiguous float64")
        return q.ctypes.data, 0
    import torch  # noqa: PLC0415 (torch only for device memory)
    if not isinstance(q, torch.Tensor) or q.dtype != torch.float64 or not q.is_contiguous():
        raise TypeError("state must be a contiguous float64 torch tensor or numpy array")
    if q.is_cuda:
        # the library's stream does not know the tensor's producer: finish pending torch work first
        torch.cuda.current_stream(q.device).synchronize()
    return q.data_ptr(), int(q.is_cuda)


def hgks_set_state(ctx, q) -> None:
    p, dev = _ptr(q)
    _check(lib().hgks_set_state(ctx, p, dev), ctx)


def hgks_get_state(ctx, q) -> None:
    p, dev = _ptr(q)
    _check(lib().hgks_get_state(ctx, p, dev), ctx)


def _host_ptr(q) -> int:
    """Address of a C-contiguous float64 HOST buffer (numpy array or CPU torch tensor, ideally pinned)."""
    if isinstance(q, np.ndarray):
        if q.dtype != np.float64 or not q.flags["C_CONTIGUOUS"]:
            raise TypeError("state must be C-contiguous float64")
        return q.ctypes.data
    import torch  # noqa: PLC0415
    if not isinstance(q, torch.Tensor) or q.dtype != torch.float64 or not q.is_contiguous() or q.is_cuda:
        raise TypeError("asynchronous I/O needs a contiguous float64 host tensor (pinned for overlap)")
    return q.data_ptr()


def hgks_upload_state(ctx, q) -> None:
    """Enqueue the H2D copy of host state q (keep q alive until the next hgks_commit_state)."""
    _check(lib().hgks_upload_state(ctx, _host_ptr(q)), ctx)


def hgks_commit_state(ctx) -> None:
    """Make the last upload the current state (= hgks_set_state of it)."""
    _check(lib().hgks_commit_state(ctx), ctx)


def hgks_download_state(ctx, q) -> None:
    """Enqueue the D2H copy of the current state into host buffer q (valid after hgks_io_wait)."""
    _check(lib().hgks_download_state(ctx, _host_ptr(q)), ctx)


def hgks_io_wait(ctx) -> None:
    _check(lib().hgks_io_wait(ctx), ctx)


def hgks_step(ctx, nsteps: int, t: float = 0.0, t_end: float = 0.0):
    """Advance up to nsteps steps; returns (t_reached, dt_last)."""
    tt, dtl = C.c_double(t), C.c_double(0.0)
    _check(lib().hgks_step(ctx, nsteps, t_end, C.byref(tt), C.byref(dtl)), ctx)
    return tt.value, dtl.value


def hgks_diagnostics(ctx, rho0: float = 1.0) -> np.ndarray:
    """Global volume diagnostics of the current state (collective), in DIAG_NAMES order."""
    out = np.zeros(len(DIAG_NAMES))
    _check(lib().hgks_diagnostics(ctx, rho0, out.ctypes.data_as(_dp)), ctx)
    return out


HIST_COLS = 2 + len(DIAG_NAMES)  # t, dt, DIAG_NAMES


def hgks_history_enable(ctx, capacity: int, rho0: float = 1.0) -> None:
    """Record the volume diagnostics of the start state of every following step (fused into the
    stage-1 update; capacity rows on the device; 0 disables)."""
    _check(lib().hgks_history_enable(ctx, int(capacity), float(rho0)), ctx)


def hgks_history_read(ctx, max_rows: int) -> np.ndarray:
    """[rows][HIST_COLS] = (t, dt, DIAG_NAMES...) of the steps since the last read (collective)."""
    out = np.zeros((max(max_rows, 1), HIST_COLS))
    n = C.c_int32()
    _check(lib().hgks_history_read(ctx, out.ctypes.data_as(_dp), int(max_rows), C.byref(n)), ctx)
    return out[:n.value]


def hgks_plane_stats(ctx, ny: int) -> np.ndarray:
    """[ny][16] x-z plane means of the current state (STAT_NAMES order); collective."""
    out = np.zeros((ny, len(STAT_NAMES)))
    _check(lib().hgks_plane_stats(ctx, out.ctypes.data_as(_dp)), ctx)
    return out


def hgks_get_forcing(ctx):
    """(f of the last committed step, bulk momentum m, bulk density rho_b) of the current state."""
    f, m, r = C.c_double(), C.c_double(), C.c_double()
    _check(lib().hgks_get_forcing(ctx, C.byref(f), C.byref(m), C.byref(r)), ctx)
    return f.value, m.value, r.value


def hgks_profile_enable(ctx, enable: bool = True) -> None:
    _check(lib().hgks_profile_enable(ctx, int(enable)), ctx)


def hgks_profile_read(ctx):
    ms = (C.c_double * len(KERNEL_CLASSES))()
    launches = (C.c_int64 * len(KERNEL_CLASSES))()
    total = C.c_int64()
    _check(lib().hgks_profile_read(ctx, ms, launches, C.byref(total)), ctx)
    return ({k: ms[i] for i, k in enumerate(KERNEL_CLASSES)},
            {k: launches[i] for i, k in enumerate(KERNEL_CLASSES)}, total.value)


def hgks_test_gp_flux(records: np.ndarray, dt: float, gamma=1.4, mu=0.0, precision=HGKS_FP64,
                      mu_law=HGKS_MU_CONST, T_ref=1.0, omega=0.0, prandtl=1.0) -> np.ndarray:
    """records [n,55] (Wl, Wr, dWl[3], dWr[3], dW0[3]) -> [n,11] (F, dF, tau)."""
    rec = np.ascontiguousarray(records, dtype=np.float64).reshape(-1, 55)
    out = np.zeros((rec.shape[0], 11))
    _check(lib().hgks_test_gp_flux(precision, gamma, mu_law, mu, T_ref, omega, prandtl, dt,
                                   rec.ctypes.data_as(_dp), rec.shape[0], out.ctypes.data_as(_dp)))
    return out


def hgks_test_operator(ctx, dt: float, shape):
    L, dL = np.zeros(shape), np.zeros(shape)
    _check(lib().hgks_test_operator(ctx, dt, L.ctypes.data_as(_dp), dL.ctypes.data_as(_dp)), ctx)
    return L, dL


def hgks_test_face_flux(ctx, d: int, n) -> np.ndarray:
    """[10][nz'][ny'][nx'] face fluxes of direction d after the last sweep (n = local (nx,ny,nz))."""
    dims = [n[2], n[1], n[0]]
    dims[2 - d] += 1
    out = np.zeros((10, *dims))
    _check(lib().hgks_test_face_flux(ctx, d, out.ctypes.data_as(_dp)), ctx)
    return out


def run_loopback_group(nranks: int, fn, key: int | None = None):
    """Run fn(rank, nranks, group_key) on nranks host threads (one loopback-group rank each; every
    rank's hgks_* calls must come from its own thread, ctypes releases the GIL).  Returns the list
    of results by rank; re-raises the first exception."""
    import threading
    key = key if key is not None else next(_group_keys)
    out, err = [None] * nranks, []

    def work(r):
        try:
            out[r] = fn(r, nranks, key)
        except BaseException as e:  # noqa: BLE001 (propagated below)
            err.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if err:
        raise err[0]
    return out


def _keys():
    import itertools
    return itertools.count(os.getpid() * 1000 + 1)


_group_keys = _keys()


class Solver:
    """Convenience owner of one context: create / set_state / step / get_state / destroy."""

    def __init__(self, n, lo, hi, **kw):
        self.params = make_params(n, lo, hi, **kw)
        self.ctx = hgks_create(self.params)
        self.n = tuple(int(x) for x in n)
        self.z0, self.nz_local = hgks_local_extent(self.ctx)
        self.t = 0.0

    @property
    def local_shape(self):
        return (5, self.nz_local, self.n[1], self.n[0])

    def set_state(self, q, t: float = 0.0):
        hgks_set_state(self.ctx, q)
        self.t = t

    def step(self, nsteps: int = 1, t_end: float = 0.0):
        self.t, dt = hgks_step(self.ctx, nsteps, self.t, t_end)
        return dt

    def plane_stats(self) -> np.ndarray:
        return hgks_plane_stats(self.ctx, self.n[1])

    def diagnostics(self, rho0: float = 1.0) -> dict:
        return dict(zip(DIAG_NAMES, hgks_diagnostics(self.ctx, rho0)))

    def get_state(self, out=None):
        if out is None:
            out = np.zeros(self.local_shape)
        hgks_get_state(self.ctx, out)
        return out

    # asynchronous host I/O overlapped with the steps (hgks.h: hgks_upload_state .. hgks_io_wait)
    def upload_state(self, q):
        hgks_upload_state(self.ctx, q)

    def commit_state(self, t: float = 0.0):
        hgks_commit_state(self.ctx)
        self.t = t

    def download_state(self, out):
        hgks_download_state(self.ctx, out)

    def io_wait(self):
        hgks_io_wait(self.ctx)

    def close(self):
        if self.ctx:
            hgks_destroy(self.ctx)
            self.ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
