/*
 * hgks.h — C ABI of the B200-native HGKS S2O4 step library (libhgks.so).
 *
 * Method: one full two-stage fourth-order (S2O4) step of the high-order gas-kinetic scheme of
 * arXiv 2207.01173 §2 on a structured 3D grid of cell-averaged conservative variables
 *   Q = (rho, rhoU, rhoV, rhoW, rhoE)
 * advanced by Eq. (7)
 *   Q*      = Q^n + dt/2 L(Q^n) + dt^2/8 d_t L(Q^n)
 *   Q^{n+1} = Q^n + dt L(Q^n) + dt^2/6 (d_t L(Q^n) + 2 d_t L(Q*))
 * with L = -(1/|Omega|) sum_faces F (Eqs. (3)-(4)), face fluxes from 2x2 Gauss points
 * of the BGK time-dependent distribution Eq. (6), linearised in time by
 * the two-window solve Eq. (8), fifth-order WENO reconstruction, and the
 * CFL time step of Alg. 1.  The readings of every point the paper leaves open are
 * listed in DESIGN.md ("Readings"), numbered as in SURVEY.md §8(c) (O-1 .. O-26).
 *
 * Conventions
 *   - Every call is collective over the nranks of one context (same order on every rank).
 *   - Return codes: HGKS_OK (0) or a negative hgks_status; a message is kept per context
 *     (hgks_last_error(ctx)) or per thread when ctx is NULL.
 *   - The ABI is always fp64 and uses the layout [5][nz_local][ny][nx] (x fastest, variable
 *     outermost) for states; fp32 contexts round on set_state and widen on get_state.
 *   - The library owns all device memory, its streams (unless one is passed in) and the NCCL
 *     communicator; callers own every pointer they pass and keep ownership after the call.
 *   - There is no CPU fallback: every compute step runs in sm_100a kernels; without a usable
 *     CUDA device hgks_create fails with HGKS_ECUDA.
 */
#ifndef HGKS_H
#define HGKS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hgks_ctx hgks_ctx; /* opaque: device buffers, streams, NCCL comm, status */

typedef enum {
  HGKS_OK = 0,
  HGKS_EINVAL = -1, /* bad argument / parameter combination                                  */
  HGKS_ECUDA = -2,  /* CUDA runtime error (context must then be destroyed)                     */
  HGKS_ENCCL = -3,  /* NCCL error (context must then be destroyed)                             */
  HGKS_ESTATE = -4, /* rho<=0, p<=0 or non-finite state; first bad global cell in last_error  */
  HGKS_ENOMEM = -5  /* device allocation failed                                                */
} hgks_status;

typedef enum { HGKS_FP64 = 0, HGKS_FP32 = 1 } hgks_precision;      /* P:1091-1093 FP32/FP64 builds */
typedef enum { HGKS_PERIODIC = 0, HGKS_WALL_ISOTHERMAL = 1 } hgks_bc;
typedef enum { HGKS_UNIFORM = 0, HGKS_TANH = 1 } hgks_stretch;       /* P:945-956 channel mesh        */
typedef enum { HGKS_MU_CONST = 0, HGKS_MU_POWER = 1 } hgks_mu_law;
/* streamwise (x) body force, "the constant moment flux in the streamwise direction is
 * used to determine the external force"; discrete form = readings O-26 / O-27:
 *   O-26 a uniform acceleration f, constant over a step, is the source S = (0, rho f, 0, 0, rho U f)
 *        of L, with d_t S = (0, f L_rho, 0, 0, f L_rhoU); in stage 2, L(Q*) in that product is its
 *        Taylor value L(Q^n) + dt/2 d_t L(Q^n) (stage 2 evaluates no flux);
 *   O-27 HGKS_FORCE_BULK chooses f every step (dead-beat on the bulk momentum
 *        m = (1/Omega) sum rho U dV, rho_b = (1/Omega) sum rho dV, target m_b):
 *          f^n = f^{n-1} + [ (m_b - m^n)/dt^n - (m^n - m^{n-1})/dt^{n-1} ] / rho_b^n,
 *        first step after set_state: f^0 = force + (m_b - m^0)/(dt^0 rho_b^0).                     */
typedef enum { HGKS_FORCE_NONE = 0, HGKS_FORCE_CONST = 1, HGKS_FORCE_BULK = 2 } hgks_force_mode;

typedef struct {
  int32_t n[3];          /* GLOBAL interior cells (nx, ny, nz); each >= 5; nz/nranks >= 3           */
  double lo[3], hi[3];   /* box [lo_d, hi_d]                                                        */
  hgks_bc bc[3];         /* per axis (both ends).  Walls: x or y only (z is the slab axis).  A wall
                            axis gets isothermal no-slip mirror ghosts (reading O-17):
                            U_g = -U_m, T_g = 2 T_wall - T_m, p_g = p_m                              */
  hgks_stretch stretch[3]; /* HGKS_UNIFORM: dx = (hi-lo)/n.  HGKS_TANH (reading O-18):
                            faces x_j = (lo+hi)/2 + (hi-lo)/2 tanh(b(2j/n - 1))/tanh(b); the
                            reconstruction runs in the uniform cell-index coordinate and derivatives
                            use the analytic metric of the map; x or y only                        */
  double stretch_b[3];   /* b of HGKS_TANH axes (the paper's b_g = 2)                              */
  double gamma;          /* 1 < gamma <= 5/3 ; K = (5 - 3 gamma)/(gamma - 1)              */
  double prandtl;        /* Pr > 0; Pr != 1 adds (1/Pr - 1) q to the energy flux,
                            q the heat flux of the interface distribution relative to U0 (O-12)   */
  hgks_mu_law mu_law;    /* mu = mu_ref (const) or mu_ref (T/T_ref)^omega with T = p/rho          */
  double mu_ref, T_ref, omega;
  double T_wall;         /* wall temperature (T = p/rho units) of HGKS_WALL_ISOTHERMAL axes        */
  double cfl;            /* > 0: adaptive dt = cfl / max_cells max_d (|U_d| + c)/dx_d (O-13)       */
  double dt_fixed;       /* > 0: fixed dt, overrides cfl (parity / timing runs)                    */
  hgks_precision precision;
  int32_t rank, nranks;  /* slab decomposition along z (outermost storage axis)                   */
  int32_t device;        /* CUDA device ordinal used by this context                              */
  const void* nccl_id;   /* 128-byte ncclUniqueId identical on all ranks; required for NCCL ranks
                            (nranks > 1, group_key == 0).  With nranks == 1 it is optional: non-NULL
                            creates a one-member communicator, and the periodic z wrap then runs as
                            an NCCL self send/recv and every reduction as an NCCL allreduce (the same
                            calls as P > 1, so the NCCL path can be exercised on one GPU); NULL uses
                            device copies                                                         */
  void* stream;          /* cudaStream_t for all work; NULL => the library creates one            */
  hgks_force_mode force_mode; /* streamwise body force (see hgks_force_mode); NONE for TGV           */
  double force;          /* CONST: the acceleration f; BULK: f before the first step (f_init)      */
  double force_target;   /* BULK: target bulk momentum m_b (e.g. rho_b U_b = 1 for the channel)    */
  int64_t group_key;     /* nranks > 1 without NCCL: != 0 joins the in-process LOOPBACK group of
                            that key (nccl_id must be NULL).  The nranks contexts of the group live
                            in ONE process, each driven by its own host thread, and may share one
                            device (ranks on different devices get peer access enabled): halos move by device-to-device copies ordered with CUDA events,
                            reductions run in a fixed rank order on the device, and the collective
                            calls synchronise the threads with a host barrier (120 s timeout ->
                            HGKS_ENCCL).  Same kernels, slab split and halo plan as the NCCL path:
                            it exists so the decomposition can be verified on a single GPU
                            (decomposition invariance, SURVEY O-P15).  nranks <= 16.  0: unused.  */
} hgks_params;

/* Validate p, allocate device memory, create streams and (nranks > 1) the NCCL communicator, or
 * join the loopback group (group_key; returns once all nranks members have joined).
 * Defines: the problem of P:185-204 (conservative variables, gamma, K = (5-3gamma)/(gamma-1) P:202),
 * tau = mu/p with mu(T) (power law and Pr), the CFL time step (Alg. 1
 * P:419-421), and one domain per process/GPU ("the computational domain is divided into N parts ...
 * N GPUs are used"; here along z).  Own stream (stream == NULL): a blocking stream that
 * orders with the legacy default stream.  Walls on both x and y are rejected (HGKS_EINVAL).
 * *out receives the context, or NULL on failure.  Errors: EINVAL, ECUDA, ENCCL (NCCL init failure
 * or loopback group timeout / inconsistent nranks), ENOMEM. */
int hgks_create(const hgks_params* p, hgks_ctx** out);

/* This rank's slab: global z planes [z_begin, z_begin + nz_local) -- the "i-th decomposed
 * computational domain" of process P_i.  Planes are split as evenly as possible, lower
 * ranks taking the remainder (see hgks_slab_of).  c, z_begin, nz_local non-NULL (HGKS_EINVAL). */
int hgks_local_extent(const hgks_ctx* c, int32_t* z_begin, int32_t* nz_local);

/* Initial data of this rank's domain (the paper's P_0 distributes the divided initial data to each
 * process; here every rank passes its own part).  Cell averages Q = (rho, rhoU, rhoV,
 * rhoW, rhoE) of Eq. (2).
 * Copy in this rank's slab q[5][nz_local][ny][nx] (fp64; host pointer, or device pointer when
 * on_device != 0; a device buffer must be complete -- the Python binding synchronises torch's
 * current stream first), check validity (rho > 0, p > 0, finite; HGKS_ESTATE names the first bad
 * global cell) and, in CFL mode, compute the first step's global max wave speed.  q is not
 * retained. */
int hgks_set_state(hgks_ctx* c, const double* q, int on_device);

/* Advance up to nsteps S2O4 steps.  dt per step is dt_fixed, or the CFL value from
 * the global max wave speed (one 8-byte NCCL max-allreduce per step).  Each stage's z halo (Alg. 2,
 * P:497-521) runs on a high-priority communication stream while the x-direction reconstruction of
 * the interior z planes proceeds; only the ghost-plane lines wait for it.  If t_end > 0 the last dt
 * is clamped so t does not pass t_end and the call stops there.  *t_inout is read (start time)
 * and written (time reached); *dt_last (may be NULL) receives the last dt taken.  All steps are
 * enqueued without host round trips; the call reads one status word at the end.
 * On HGKS_ESTATE the state is rolled back to the last good Q^n and *t_inout is that step's start
 * time. */
int hgks_step(hgks_ctx* c, int32_t nsteps, double t_end, double* t_inout, double* dt_last);
/* (multi-rank NCCL contexts: the final wait polls ncclCommGetAsyncError; an asynchronous NCCL error,
 * or no progress for HGKS_NCCL_TIMEOUT_S seconds (environment, default 300), aborts both
 * communicators and returns HGKS_ENCCL -- the context must then be destroyed.) */

/* Output of this rank's domain (P_0 collects from every process; here each rank reads
 * its own part).  Copy out this rank's slab in the set_state layout (fp64; host or device pointer;
 * the library owns nothing of q).  Errors: HGKS_EINVAL (NULL, no state yet), HGKS_ECUDA, HGKS_ENCCL
 * (a failed peer, see hgks_step).  Synchronises. */
int hgks_get_state(hgks_ctx* c, double* q, int on_device);

/* Asynchronous host I/O: the per-rank input / output of the run overlapped with the step.
 * The copies run on a dedicated I/O stream of the context (the GPU's copy engines), so an upload of the
 * next input and the download of the last result proceed while hgks_step computes.  Buffers (two fp64
 * states) and the stream are allocated on the first call.  q must be PAGE-LOCKED host memory (pinned;
 * pageable memory works but the copy is then synchronous) in the hgks_set_state layout, and must stay
 * valid and untouched until the copy is known complete (below).  All four are collective like every call.
 *   hgks_upload_state(c, q)   enqueue the host-to-device copy of q into the upload buffer; returns at once.
 *                             q may be reused after the next hgks_commit_state returns.
 *   hgks_commit_state(c)      make the last upload the current state: exactly hgks_set_state of it
 *                             (validity check, first wave speed; synchronises the compute stream; same
 *                             errors).  HGKS_EINVAL without a pending upload.
 *   hgks_download_state(c, q) snapshot the current state (ordered after every enqueued step) into the
 *                             download buffer and enqueue its device-to-host copy to q; returns at once.
 *                             q holds the state once hgks_io_wait returns; a following hgks_step overlaps
 *                             the copy.  HGKS_EINVAL without a state.
 *   hgks_io_wait(c)           wait for every upload and download enqueued so far (HGKS_ECUDA on failure).
 * A time-marching driver that reads every step's state out and feeds new inputs in thus pays the PCIe
 * transfers only where they exceed the step (bench.py's e2e loop). */
int hgks_upload_state(hgks_ctx* c, const double* q);
int hgks_commit_state(hgks_ctx* c);
int hgks_download_state(hgks_ctx* c, double* q);
int hgks_io_wait(hgks_ctx* c);

/* Release everything owned by c (device buffers, streams, events, NCCL communicators; the end of
 * the run of Fig. 3's code frame).  NULL-safe.  Collective like every call: a loopback-group rank
 * waits (host barrier) until every rank of the group has entered hgks_destroy, so no rank frees
 * buffers or events a peer is still using. */
int hgks_destroy(hgks_ctx* c);

/* Last error message of c (or of the calling thread when c == NULL); never NULL. */
const char* hgks_last_error(const hgks_ctx* c);

/* ---- diagnostics ---------------------------------------------------- */

/* Volume integrals of the current state over the WHOLE domain (collective: every rank calls it,
 * every rank receives the global values).  P:889-903 define E_k and eps_com; O-24/O-25:
 *   out[HGKS_DIAG_EK]        E_k   = 1/(rho0 Omega) sum 1/2 rho |U|^2 dV
 *   out[HGKS_DIAG_ENSTROPHY] zeta  = 1/(rho0 Omega) sum 1/2 rho |omega|^2 dV, omega = curl U
 *   out[HGKS_DIAG_EPS_S]     mu/(rho0 Omega) sum |omega|^2 dV          (eps_com, first term)
 *   out[HGKS_DIAG_EPS_D]     4/3 mu/(rho0 Omega) sum (div U)^2 dV      (eps_com, second term)
 *   out[HGKS_DIAG_MASS..ENERGY]  sum rho dV, sum rho U dV (x, y, z), sum rho E dV
 *   out[HGKS_DIAG_VOLUME]    Omega = sum dV
 *   out[HGKS_DIAG_PDIL]      Pi = 1/(rho0 Omega) sum p div U dV  (pressure-dilatation; with the two
 *                            eps_com terms it closes dE_k/dt = Pi - eps_s - eps_d)
 * mu = params.mu_ref.  Velocity derivatives: fourth-order central difference in the cell index
 * times d(index)/dx at the cell centre, ghosts as the step fills them (periodic, wall mirror,
 * halo).  Computed in fp64 for either precision by a fixed-order (deterministic) two-pass
 * reduction, then an NCCL sum over ranks.  rho0 > 0.  Synchronises the stream.
 * Errors: HGKS_EINVAL (NULL, no state, rho0 <= 0), HGKS_ECUDA, HGKS_ENCCL. */
#define HGKS_DIAG_COUNT 11
typedef enum {
  HGKS_DIAG_EK = 0, HGKS_DIAG_ENSTROPHY = 1, HGKS_DIAG_EPS_S = 2, HGKS_DIAG_EPS_D = 3,
  HGKS_DIAG_MASS = 4, HGKS_DIAG_MOM_X = 5, HGKS_DIAG_MOM_Y = 6, HGKS_DIAG_MOM_Z = 7,
  HGKS_DIAG_ENERGY = 8, HGKS_DIAG_VOLUME = 9, HGKS_DIAG_PDIL = 10
} hgks_diag;
int hgks_diagnostics(hgks_ctx* c, double rho0, double out[HGKS_DIAG_COUNT]);

/* Per-step diagnostic history (time histories of E_k, eps_com, enstrophy, Figs 7-8):
 * with capacity > 0 every following hgks_step computes the volume diagnostics of hgks_diagnostics
 * for the state at the START of each step, fused into that step's stage-1 update kernel (Q^n with the
 * ghosts its halo has just filled; fixed-order per-block sums, two fixed-order reduction kernels,
 * fp64 for either precision; no host round trip).  capacity = rows held on the device (each row is
 * read once); rho0 > 0 normalises as hgks_diagnostics.  capacity 0 disables (the default).  Frees
 * and re-allocates the history buffers; the rows pending are discarded.
 * Errors: HGKS_EINVAL (capacity < 0, rho0 <= 0), HGKS_ENOMEM, HGKS_ECUDA. */
#define HGKS_HIST_COLS (2 + HGKS_DIAG_COUNT) /* t, dt, then the hgks_diag order */
int hgks_history_enable(hgks_ctx* c, int32_t capacity, double rho0);

/* Read and clear the rows recorded since the last read: out[r * HGKS_HIST_COLS + k], k = 0: t of the
 * step's start state, 1: the step's dt, 2..: hgks_diagnostics of that state.  *rows = rows written
 * (<= max_rows, else HGKS_EINVAL and nothing is consumed).  Collective: one NCCL sum of all rows.
 * hgks_step refuses (HGKS_EINVAL) a call that could overflow the capacity.  Synchronises. */
int hgks_history_read(hgks_ctx* c, double* out, int32_t max_rows, int32_t* rows);

/* x-z plane means of the current state for every GLOBAL y index j (channel statistics, P:1186-1238;
 * the paper's <.> averages over time and the X and Z directions, P:1190-1191 -- time averaging is
 * left to the caller, who samples this every few steps).  out[j * HGKS_STAT_COUNT + s], j < ny,
 * s in hgks_stat order; c = sqrt(gamma p / rho), M = |U| / c, T = p / rho (reading O-28).  fp64 for
 * either precision; one block per plane with a fixed summation order, then an NCCL sum over the z
 * slabs.  Collective; synchronises.  Errors: HGKS_EINVAL (NULL, no state), ECUDA, ENCCL. */
#define HGKS_STAT_COUNT 16
typedef enum {
  HGKS_STAT_RHO = 0, HGKS_STAT_U, HGKS_STAT_V, HGKS_STAT_W, HGKS_STAT_UU, HGKS_STAT_VV, HGKS_STAT_WW,
  HGKS_STAT_UV, HGKS_STAT_RHOU, HGKS_STAT_RHOV, HGKS_STAT_RHOUV, HGKS_STAT_C, HGKS_STAT_M,
  HGKS_STAT_MM, HGKS_STAT_T, HGKS_STAT_P
} hgks_stat;
int hgks_plane_stats(hgks_ctx* c, double* out);

/* Streamwise force state (collective, synchronises): *force = f applied in the last committed step
 * (the params' force before the first step); *bulk_momentum, *bulk_density = m and rho_b of the
 * current state (HGKS_FORCE_BULK; 0 otherwise).  Any output pointer may be NULL. */
int hgks_get_forcing(hgks_ctx* c, double* force, double* bulk_momentum, double* bulk_density);

/* ---- small helpers (host logic, no device work) ----------------------------------------- */

/* Size of the opaque NCCL unique id (128) and generator for rank 0 (broadcast it yourself). */
size_t hgks_nccl_id_bytes(void);
int hgks_get_nccl_id(void* out);

/* Slab of `rank` among `nranks` for nz planes: [*z_begin, *z_begin + *nz_local). */
int hgks_slab_of(int32_t nz, int32_t rank, int32_t nranks, int32_t* z_begin, int32_t* nz_local);

/* Halo plan of the z decomposition (periodic ring): neighbours, and the element offsets (in the
 * ghosted fp32/fp64 device layout [nz_local+6][5][ny+6][nx+6]) of the 3-plane chunks sent to and
 * received from each neighbour.  count = elements per chunk.  Used by hgks_step's NCCL exchange
 * and exported so the host logic can be exercised without a GPU. */
typedef struct {
  int32_t up, down;                 /* neighbour ranks (rank+1, rank-1 mod nranks)          */
  int64_t send_up, recv_down;       /* top interior planes -> up ; bottom ghosts <- down    */
  int64_t send_down, recv_up;       /* bottom interior planes -> down ; top ghosts <- up    */
  int64_t count;                    /* elements in one 3-plane chunk                        */
} hgks_halo_plan;
int hgks_make_halo_plan(int32_t nx, int32_t ny, int32_t nz_local, int32_t rank, int32_t nranks,
                        hgks_halo_plan* out);

/* ---- instrumentation (bench.py roofline / launch accounting) ----------------------------- */

/* Kernel classes timed with CUDA events when profiling is enabled (FLUX_*: the fused
 * tangential-reconstruction + Gauss-point flux sweep of one direction; RECON: the normal
 * reconstruction sweeps of all three directions). */
typedef enum {
  HGKS_K_FLUX_X = 0, HGKS_K_FLUX_Y = 1, HGKS_K_FLUX_Z = 2, HGKS_K_UPDATE = 3,
  HGKS_K_GHOST = 4, HGKS_K_HALO = 5, HGKS_K_DT = 6, HGKS_K_RECON = 7, HGKS_K_COUNT = 8
} hgks_kernel_class;

/* enable != 0: bracket every launch of each class with CUDA events on the compute stream.
 * Resets the accumulators. */
int hgks_profile_enable(hgks_ctx* c, int enable);
/* Synchronise and read: ms[k] = summed event time of class k, launches[k] = launches of class k
 * since the last enable/reset; total_launches = all kernels this library launched since then. */
int hgks_profile_read(hgks_ctx* c, double ms[HGKS_K_COUNT], int64_t launches[HGKS_K_COUNT],
                      int64_t* total_launches);

#ifdef __cplusplus
}
#endif
#endif /* HGKS_H */
