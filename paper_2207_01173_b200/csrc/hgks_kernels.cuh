// hgks_kernels.cuh — sm_100a kernels of one S2O4 stage (product path).
//
//   recon_kernel<T, 0/2>,       normal reconstruction (A2): one thread per (face line, component,
//   recon_yz_kernel<T>          march segment), WENO5-Z edges once per cell, six face fields per face
//                               written to the face-field array of the sweep
//   flux_kernel<T, DIR, STAGE>  fused per tile of TT1 x TT2 faces (FluxCfg: fp64 4x8, fp32 8x8),
//                               marching up to 16 normal faces: 16-byte
//                               cp.async copy of the face fields (A) -> tangential pass t1 (B, A3) ->
//                               per-Gauss-point thread: tangential pass t2 + BGK flux (C, A4-A6) ->
//                               4-point face quadrature by warp shuffles (A7) -> face-flux array
//   update_kernel<T, STAGE>     flux divergence L, d_t L (Eqs. (3)-(4)) + Eq. (7) stage update,
//                               stage-2 epilogue: validity flags + CFL wave-speed max (A0, A8)
//   ghost_wall_kernel<T>,       isothermal-wall mirror ghosts (O-17) and periodic x/y ghost bands
//   ghost_xy_kernel<T>          (A1, O-16); the z halo is a copy / NCCL / loopback exchange (hgks.cu)
//   cfl_kernel<T> / dt_kernel   initial wave-speed max, per-step dt + commit logic (A0)
//
// Layout of a ghosted state (elements of T): [nz_l+6][5][ny+6][nx+6], x fastest.
// A face-flux array of direction d: [10][fz][fy][fx] with f_a = n_a + (a == d); components
// 0..4 = F^n, 5..9 = d_t F^n (per unit face area, i.e. 1/4 sum over the 2x2 Gauss points).
#pragma once
#include "gks_device.cuh"

#ifdef HGKS_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[4];  // debug builds: cycles per flux phase
#endif
namespace hgks {

// device control block (one per context)
struct Ctl {
  double t, dt, dt_last;
  double t_end;                 // <= 0: none
  double dt_fixed, cfl;
  unsigned long long smax_cur;  // bits of the max wave speed of the current state
  unsigned long long red[2];    // [0] smax of the newest state, [1] error flag (allreduced, max)
  unsigned long long bad_cell;  // min linear global index of an invalid cell (ULLONG_MAX: none)
  int halt;                     // 0 running, 1 invalid state, 2 reached t_end
  int pending;                  // 1: a step has run and awaits commit
  long long steps_done;         // committed steps in the current hgks_step call
  // streamwise body force (O-26, O-27; hgks_force_mode)
  int force_mode;               // 0 none, 1 constant f, 2 dead-beat on the bulk momentum
  int hist;                     // mode 2: 1 once a step has been committed since set_state
  double force;                 // f of the step in flight
  double f_init, force_target, volume;
  double m_cur, rho_cur;        // bulk momentum / density of the committed state
  double m_prev, dt_prev, f_prev;  // controller memory: previous step's m, dt and f
  double bulk_new[2];           // (sum rho dV, sum rho U dV) of the newest state (allreduced)
  int hist_n, hist_cap;         // per-step diagnostic history: rows written / capacity
  double idt;                   // 1 / dt of the step in flight (one IEEE division per step, not per Gauss point)
};

template <typename T>
struct Geo {
  int n[3];        // local interior cells (nx, ny, nz_local)
  int px, py;      // pitches: nx+6, ny+6
  long long plane; // 5*py*px: stride of one z plane
  long long vs;    // py*px: stride of one variable
  T h[3];          // cell widths of uniform axes
  T ih[3];         // 1/h of uniform axes
  int z0;          // global z of local plane 0
  int ny_g, nx_g;  // global sizes (for linear cell ids)
  // metric tables of every axis (local indices; O-18): J = d(cell index)/dx at the faces
  // jf[d][0..n_d], at the Gauss abscissae jg[d][m * n_d + j] (m = 0: -sqrt(3)/6), and the
  // reciprocal cell widths iw[d][0..n_d-1].  Uniform axes hold 1/h.
  const T* jf[3];
  const T* jg[3];
  const T* iw[3];
  int wall[3];     // 1: isothermal no-slip walls at both ends of the axis (O-17)
  T T_wall;
};

constexpr int DIAG_TPB = 256;  // block size of the fixed-order reductions (update, diagnostics)

// fp64 cell-centre metric J = d(index)/dx and cell widths of every axis (local cell index)
struct DiagGeo {
  const double* jc[3];
  const double* w[3];
};

// sum v[0..N) over the block (fixed tree order); result valid in thread 0
template <int N>
__device__ __forceinline__ void block_sum_fixed(double (&v)[N], double* sh) {
  const int t = threadIdx.x;
#pragma unroll
  for (int n = 0; n < N; ++n) sh[n * DIAG_TPB + t] = v[n];
  __syncthreads();
  for (int s = DIAG_TPB / 2; s > 0; s >>= 1) {
    if (t < s) {
#pragma unroll
      for (int n = 0; n < N; ++n) sh[n * DIAG_TPB + t] += sh[n * DIAG_TPB + t + s];
    }
    __syncthreads();
  }
#pragma unroll
  for (int n = 0; n < N; ++n) v[n] = sh[n * DIAG_TPB];
}

template <typename T>
__device__ __forceinline__ long long qidx(const Geo<T>& g, int v, int i, int j, int k) {
  return (long long)(k + 3) * g.plane + (long long)v * g.vs + (long long)(j + 3) * g.px + (i + 3);
}

// ---- volume diagnostics of one cell (readings O-24, O-25, O-29) --
// acc += (1/2 rho|U|^2, 1/2 rho|omega|^2, |omega|^2, (div U)^2, rho, rho U, rho V, rho W, rho E, 1,
//         p div U) dV, velocity derivatives by 4th-order central differences of the cell-average
// velocities in the cell index times J = d(index)/dx at the cell centre (ghosts as filled).  fp64 for
// either precision.  Used by diag_kernel (on demand) and by the stage-1 update (per-step history).
constexpr int NDIAG = 11;  // HGKS_DIAG_COUNT

// velocity (U, V, W) of one cell in fp64: one reciprocal of rho (MUFU seed + Newton, ~1 ulp) per cell
// instead of three IEEE divisions
template <typename T>
__device__ __forceinline__ void vel_of(const T* __restrict__ q, const Geo<T>& g, int i, int j, int k, double (&u)[3]) {
  const double ir = rcp((double)q[qidx(g, 0, i, j, k)]);
#pragma unroll
  for (int c = 0; c < 3; ++c) u[c] = (double)q[qidx(g, 1 + c, i, j, k)] * ir;
}

// the per-cell integrands from the cell's state and velocity gradient
__device__ __forceinline__ void diag_terms(double rho, const double (&u)[3], const double (&m)[3], const double (&grad)[3][3],
                                           double rhoE, double vol, double gamma, double (&acc)[NDIAG]) {
  const double o0 = grad[2][1] - grad[1][2], o1 = grad[0][2] - grad[2][0], o2 = grad[1][0] - grad[0][1];
  const double om2 = o0 * o0 + o1 * o1 + o2 * o2;
  const double dv = grad[0][0] + grad[1][1] + grad[2][2];
  const double u2 = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
  acc[0] += 0.5 * rho * u2 * vol;
  acc[1] += 0.5 * rho * om2 * vol;
  acc[2] += om2 * vol;
  acc[3] += dv * dv * vol;
  acc[4] += rho * vol;
  acc[5] += m[0] * vol;
  acc[6] += m[1] * vol;
  acc[7] += m[2] * vol;
  acc[8] += rhoE * vol;
  acc[9] += vol;
  const double p = (gamma - 1.0) * (rhoE - 0.5 * rho * u2);
  acc[10] += p * dv * vol;  // pressure-dilatation (O-29)
}

template <typename T>
__device__ __forceinline__ void diag_cell(const T* __restrict__ q, const Geo<T>& g, const DiagGeo& dg, double gamma, int i,
                                          int j, int k, double (&acc)[NDIAG]) {
  const int ijk[3] = {i, j, k};
  const double vol = dg.w[0][i] * dg.w[1][j] * dg.w[2][k];
  const double rho = (double)q[qidx(g, 0, i, j, k)];
  double u[3], m[3];
  const double ir = rcp(rho);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    m[c] = (double)q[qidx(g, 1 + c, i, j, k)];
    u[c] = m[c] * ir;
  }
  double grad[3][3];  // grad[c][d] = d u_c / d x_d (O-25)
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double J12 = dg.jc[d][ijk[d]] * (1.0 / 12.0);
    const int di = d == 0, dj = d == 1, dk = d == 2;
    double up1[3], um1[3], up2[3], um2[3];
    vel_of(q, g, i + di, j + dj, k + dk, up1);
    vel_of(q, g, i - di, j - dj, k - dk, um1);
    vel_of(q, g, i + 2 * di, j + 2 * dj, k + 2 * dk, up2);
    vel_of(q, g, i - 2 * di, j - 2 * dj, k - 2 * dk, um2);
#pragma unroll
    for (int c = 0; c < 3; ++c) grad[c][d] = J12 * (8.0 * (up1[c] - um1[c]) - (up2[c] - um2[c]));
  }
  diag_terms(rho, u, m, grad, (double)q[qidx(g, 4, i, j, k)], vol, gamma, acc);
}

// sum v[0..N) over a DIAG_TPB block in a fixed order (warp butterflies, then the warps in order);
// result valid in thread 0.  sh: >= N * (DIAG_TPB / 32) doubles.
template <int N>
__device__ __forceinline__ void block_sum_warps(double (&v)[N], double* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int n = 0; n < N; ++n) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[n] += __shfl_xor_sync(0xffffffffu, v[n], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int n = 0; n < N; ++n) sh[n * (DIAG_TPB / 32) + w] = v[n];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int n = 0; n < N; ++n) {
      double s = 0.0;
      for (int k = 0; k < DIAG_TPB / 32; ++k) s += sh[n * (DIAG_TPB / 32) + k];
      v[n] = s;
    }
  }
}

#ifndef HGKS_FLUX_TPB
#define HGKS_FLUX_TPB 16  // max consecutive normal faces per flux block (host lowers it for small grids)
#endif
// Tile shape and residency per precision (measured at TGV 256^3):
//   fp64: 4 x 8 faces (t1 x t2, 128 threads), 3 blocks per SM, no spills.  The t1 pass (phase B) runs
//         over the TT1 x (TT2 + 4) (face, row) pairs, so the short side goes along t1: 4 x 12 = 48 pairs
//         per component instead of 8 x 8 = 64 for the 8 x 4 tile (round 2a), 2 passes of 128 threads
//         instead of 2.5
//   fp32: 8 x 8 faces (256 threads), 3 blocks per SM, 80 registers (8 x 4 at 6 blocks: -10 %)
#ifndef HGKS_TT1_64
#define HGKS_TT1_64 4
#endif
#ifndef HGKS_TT1_32
#define HGKS_TT1_32 8
#endif
#ifndef HGKS_VEC32
#define HGKS_VEC32 1  // fp32: vectorised sB layout (FluxCfg::VEC): +3.2 % fp32 at 256^3
#endif
#ifndef HGKS_TT2_64
#define HGKS_TT2_64 8
#endif
#ifndef HGKS_FLUX_MINB
#define HGKS_FLUX_MINB 3
#endif
#ifndef HGKS_TT2_32
#define HGKS_TT2_32 8
#endif
#ifndef HGKS_FLUX_MINB32
#define HGKS_FLUX_MINB32 3
#endif
constexpr int NB = 9;  // t1-pass outputs per (row, m, comp): V1 of 6 fields, D1 of Ql, Qr, C
template <typename T>
struct FluxCfg {
  static constexpr int TT1 = sizeof(T) == 8 ? HGKS_TT1_64 : HGKS_TT1_32;        // faces per tile along t1
  static constexpr int TL1 = TT1 + 4;                                         // lines (+-2 halo) along t1
  static constexpr int TT2 = sizeof(T) == 8 ? HGKS_TT2_64 : HGKS_TT2_32;      // faces per tile along t2
  static constexpr int TL2 = TT2 + 4;                                         // lines along t2
  static constexpr int NT = TT1 * TT2 * 4;                                    // threads: one per Gauss point
  static constexpr int MINB = sizeof(T) == 8 ? HGKS_FLUX_MINB : HGKS_FLUX_MINB32;
  // sA row pitch: TT1 = 4 -> 12 (phase-B half-warps read 4 rows of 4 lines: rows 12 apart hit 4
  // disjoint 4-slot groups of a 16-slot wavefront); TT1 = 8 -> TL1 = 12.  (fp32 with items (a, l2, c)
  // and a conflict-free pitch of 24 measured 6 % slower: 35 KB instead of 18 KB of sA per block.)
  static constexpr int TL1P = 12;
  static constexpr int SA_C = TL2 * TL1P + 8;  // one (field, component) plane of sA
  // sB: the t1-pass outputs, word (row, comp c, slot k, m, a) at row RS + c CS + k KS + MA(m, a).
  //   TT1 = 8: [row][c][k][m][a] (SB_RC = 152 words per (row, c), padded): a phase-C half-warp reads the
  //            16 (m, a) words of one row; a phase-B warp stores (a, c) words of one row, c CS = 0, 24,
  //            16, 8 (mod 32 4-byte banks) -- both conflict-free
  //   TT1 = 4: [k][c][row][a][m]: a phase-C half-warp reads the 8 (a, m) words of two consecutive rows
  //            b, b+1 = 16 consecutive words; a phase-B thread stores its (m = 0, m = 1) pair as one
  //            16-byte word pair, a warp's 8 rows x 4 a = 64 consecutive words -- both conflict-free
  //   VEC (fp32, HGKS_VEC32): [row][k][comps 0-3 of the 16 (m, a) as float4 | comp 4 of the 16 (m, a)],
  //            so phase C reads the five components of one (row, slot) with one 16-byte and one 4-byte
  //            load (2 instead of 5 issue slots; fp32 is issue-bound)
  static constexpr bool VEC = sizeof(T) == 4 && HGKS_VEC32 && TT1 == 8;
  static constexpr int SB_K = 2 * TT1;
  static constexpr int SB_RC = NB * SB_K + 8;  // TT1 = 8 layout only
  static constexpr int VK = 5 * 2 * TT1;       // VEC: words per (row, k)
  static constexpr int RS = VEC ? NB * VK : (TT1 == 8 ? 5 * SB_RC : 2 * TT1);
  static constexpr int CS = TT1 == 8 ? SB_RC : TL2 * 2 * TT1;
  static constexpr int KS = VEC ? VK : (TT1 == 8 ? SB_K : 5 * TL2 * 2 * TT1);
  static constexpr int SB_WORDS = VEC ? TL2 * RS : (TT1 == 8 ? TL2 * 5 * SB_RC : NB * KS);
  // VEC: offset of component c of (m, a) within a (row, k) block
  __device__ static constexpr int VOFF(int c, int ma) { return c < 4 ? 4 * ma + c : 8 * TT1 + ma; }
  __device__ static constexpr int MA(int m, int a) { return TT1 == 8 ? m * TT1 + a : 2 * a + m; }
  static constexpr int BPW = 16 / (2 * TT1);  // t2 faces per warp (lane = 16 n + 2 TT1 bl + TT1 m + a)
  static_assert(TT1 == 4 || TT1 == 8, "lane layout");
};

template <typename T>
constexpr size_t flux_smem_bytes() {
  return sizeof(T) * (6 * 5 * FluxCfg<T>::SA_C + FluxCfg<T>::SB_WORDS);
}

#ifndef HGKS_CP16_32
#define HGKS_CP16_32 0  // 16-byte face-field copies for fp32 (4 lines per chunk): measured neutral
#endif
#ifndef HGKS_CP16
#define HGKS_CP16 1  // 16-byte face-field copies (fp64): +7 % fp64 step rate (x, z sweeps); no gain fp32
#endif

// ---- normal reconstruction (A2): face fields of every face-line of one direction -------------
// Face-field array of direction DIR (elements of T): ff[field][comp][fn][line], fields
//   0 Ql, 1 Qr, 2 dQl/dn, 3 dQr/dn, 4 C, 5 D   (normal_fields, O-3 / O-6)
// for faces fn = 0..n_DIR (face fn between cells fn-1 and fn) and tangential lines
// (t1, t2) in [-2, n_t1+2) x [-2, n_t2+2) (the +-2 halo the tangential stencils need), line index
// with the x-most tangent fastest: DIR 0 (t1 = y, t2 = z) and DIR 2 (t1 = x, t2 = y): t1 fastest;
// DIR 1 (t1 = z, t2 = x): t2 fastest.
// Pitch of the t1 axis in the face-field line index: n_t1 + 4 lines rounded up to 16 bytes, so a
// tile row of lines starts 16-byte aligned and the flux kernel's copy moves 16-byte chunks (2 fp64
// / 4 fp32 lines).  The pad lines are never written by the reconstruction and only ever feed
// faces outside the domain.
__host__ __device__ constexpr int ff_pitch(int n_t1, int esz) {
  return (n_t1 + 4 + (16 / esz) - 1) / (16 / esz) * (16 / esz);
}

// line index of tangential line (t1, t2), t1 fastest, for every direction
template <typename T, int DIR>
struct FFLayout {
  int n1, n2, nf;   // tangential cells, faces along the normal
  int p;            // pitch of t1
  long long nl;     // lines per face plane (including pad lines)
  __device__ __forceinline__ long long line(int t1, int t2) const { return (long long)(t2 + 2) * p + (t1 + 2); }
  __device__ __forceinline__ long long at(int f, int c, int fn, long long l) const {
    return ((long long)(f * 5 + c) * nf + fn) * nl + l;
  }
};

template <typename T, int DIR>
__device__ __forceinline__ FFLayout<T, DIR> ff_layout(const Geo<T>& g) {
  constexpr int A1 = (DIR + 1) % 3, A2 = (DIR + 2) % 3;
  FFLayout<T, DIR> L;
  L.n1 = g.n[A1];
  L.n2 = g.n[A2];
  L.nf = g.n[DIR] + 1;
  L.p = ff_pitch(L.n1, (int)sizeof(T));
  L.nl = (long long)L.p * (L.n2 + 4);
  return L;
}

#ifndef HGKS_RECON_MINB
#define HGKS_RECON_MINB 8  // min blocks per SM of the reconstruction kernels (64 registers: 6.64 -> 6.15 ms/step on one box)
#endif
#ifndef HGKS_RC_PF
#define HGKS_RC_PF 1  // cells of the reconstruction march prefetched ahead (1: one, the loop's own)
#endif
constexpr int RC_PF = HGKS_RC_PF;

// Subset of the face lines of one sweep: lines lbeg + j for j in [0, lcnt), where j >= gap_at
// skips ahead by gap (two disjoint ranges in one launch: the ghost-plane lines of the x sweep).
struct LineRange {
  long long lbeg, lcnt, gap_at, gap;
};

// One thread per (line, component): marches along the normal with a 6-cell register ring, so
// every cell's WENO edge pair is computed exactly once.  x and z sweeps (t1 = y / x is also the
// fastest axis of the state, so reads and writes are coalesced); the y sweep is recon_yz_kernel.
template <typename T, int DIR>
__global__ void __launch_bounds__(128, HGKS_RECON_MINB) recon_kernel(const T* __restrict__ q, T* __restrict__ ff, Geo<T> g,
                                                    const Ctl* __restrict__ ctl, LineRange lr, int nseg) {
  if (ctl->halt) return;
  constexpr int A1 = (DIR + 1) % 3, A2 = (DIR + 2) % 3;
  const FFLayout<T, DIR> L = ff_layout<T, DIR>(g);
  const long long e0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e0 >= 5 * lr.lcnt * nseg) return;
  const int seg = (int)(e0 / (5 * lr.lcnt));  // segment of the march (outermost: lines stay coalesced)
  const long long e = e0 - seg * 5 * lr.lcnt;
  const int c = (int)(e / lr.lcnt);
  const long long j = e % lr.lcnt;
  const long long l = lr.lbeg + j + (j >= lr.gap_at ? lr.gap : 0);
  static_assert(DIR != 1, "the y sweep is recon_yz_kernel");
  const int t2 = (int)(l / L.p) - 2, t1 = (int)(l % L.p) - 2;
  if (t1 >= L.n1 + 2) return;  // pad line
  const long long sN = (DIR == 0) ? 1 : (DIR == 1 ? g.px : g.plane);
  const long long s1 = (A1 == 0) ? 1 : (A1 == 1 ? g.px : g.plane);
  const long long s2 = (A2 == 0) ? 1 : (A2 == 1 ? g.px : g.plane);
  const int gv = (c == 0) ? 0 : (c == 4 ? 4 : (c == 1 ? 1 + DIR : (c == 2 ? 1 + A1 : 1 + A2)));
  // cell -3 along the normal at (t1, t2)
  const T* p = q + 3LL * (g.plane + g.px + 1) + (long long)gv * g.vs - 3 * sN + t1 * s1 + t2 * s2;
  const T* jfn = g.jf[DIR];
  // every cell's WENO pair is evaluated at the same call site (the loop body), so all faces see
  // bitwise-identical arithmetic (uniform flow stays exactly uniform, O-P1)
  // faces [fs, fe) of this segment: the march starts one cell early (cell fs-1, whose right edge is
  // Q^l of face fs) from the window Qbar_{fs-3..fs}; the cells' WENO pairs are the same bits whatever
  // the segmentation
  const int nf = L.nf;
  const int fs = (int)(((long long)seg * nf) / nseg), fe = (int)(((long long)(seg + 1) * nf) / nseg);
  T s1v = p[fs * sN], s2v = p[(fs + 1) * sN], s3 = p[(fs + 2) * sN], s4 = p[(fs + 3) * sN], s5;
  T Ap = T(0), Bp = T(0);
  // software prefetch: the next RC_PF cells of the march are in flight while cell fn is reconstructed
  // (window index fn + 5 of the march ends at fe + 4, the last ghost layer)
  T pf[RC_PF];
#pragma unroll
  for (int k = 0; k < RC_PF; ++k) pf[k] = (fs + 4 + k <= fe + 4) ? p[(fs + 4 + k) * sN] : T(0);  // edges of cell fn-1
  for (int fn = fs - 1; fn < fe; ++fn) {
    s5 = pf[0];  // Qbar_{fn+2}; window s1..s5 = Qbar_{fn-2..fn+2}
#pragma unroll
    for (int k = 0; k + 1 < RC_PF; ++k) pf[k] = pf[k + 1];
    pf[RC_PF - 1] = (fn + 5 + RC_PF <= fe + 4) ? p[(fn + 5 + RC_PF) * sN] : T(0);
    T Ac, Bc;
    weno5z_cell(s1v, s2v, s3, s4, s5, Ac, Bc);  // cell fn
    if (fn >= fs) {
      const T ih = jfn[fn];  // metric of the face (O-18; 1/h on uniform axes)
      ff[L.at(0, c, fn, l)] = Bp;
      ff[L.at(1, c, fn, l)] = Ac;
      ff[L.at(2, c, fn, l)] = (T(2) * Ap + T(4) * Bp - T(6) * s2v) * ih;
      ff[L.at(3, c, fn, l)] = (T(-4) * Ac - T(2) * Bc + T(6) * s3) * ih;
      ff[L.at(4, c, fn, l)] = (-s1v + T(7) * s2v + T(7) * s3 - s4) * T(1.0 / 12.0);
      ff[L.at(5, c, fn, l)] = (s1v - T(15) * s2v + T(15) * s3 - s4) * (T(1.0 / 12.0) * ih);
    }
    s1v = s2v;
    s2v = s3;
    s3 = s4;
    s4 = s5;
    Ap = Ac;
    Bp = Bc;
  }
}

// y sweep (normal y, t1 = z, t2 = x).  The face-field lines are t1-fastest in every direction (so
// the flux kernel copies 16-byte chunks), here z-fastest while the state is x-fastest: lanes run
// along z (stores coalesced) and the 4 warps of a block take 4 consecutive x, so the strided state
// reads of one warp share their 32-byte sectors with the other three warps (served from L1).
// Measured against a shared-memory transpose (32 x by 8/16/24 z per block): the transpose blocks
// hold shared memory and barriers, and slow the concurrent x-sweep flux kernel more than they gain.
constexpr int RZ_Z = 32, RZ_X = 4;
// Lines (z, x) with z from the range zr (lbeg + j, j in [0, lcnt), skipping gap after gap_at: the
// interior z lines run while the z halo is in flight, the 4 ghost-plane z lines after it).
template <typename T>
__global__ void __launch_bounds__(RZ_Z * RZ_X, HGKS_RECON_MINB) recon_yz_kernel(const T* __restrict__ q, T* __restrict__ ff, Geo<T> g,
                                                                const Ctl* __restrict__ ctl, LineRange zr, int nseg) {
  if (ctl->halt) return;
  const FFLayout<T, 1> L = ff_layout<T, 1>(g);
  const int tz = threadIdx.x % RZ_Z, tx = threadIdx.x / RZ_Z;
  const int c = blockIdx.z % 5, seg = blockIdx.z / 5;
  const long long jz = (long long)blockIdx.x * RZ_Z + tz;
  const int x = blockIdx.y * RZ_X + tx - 2;
  if (jz >= zr.lcnt || x >= g.n[0] + 2) return;
  const int z = (int)(zr.lbeg + jz + (jz >= zr.gap_at ? zr.gap : 0));
  const int gv = (c == 0) ? 0 : (c == 4 ? 4 : (c == 1 ? 2 : (c == 2 ? 3 : 1)));  // (V, W, U) frame (O-23)
  const long long sN = g.px;
  const T* p = q + 3LL * (g.plane + g.px + 1) + (long long)gv * g.vs - 3 * sN + (long long)z * g.plane + x;
  const T* jfn = g.jf[1];
  const long long l = L.line(z, x);
  const int nf = L.nf;
  const int fs = (int)(((long long)seg * nf) / nseg), fe = (int)(((long long)(seg + 1) * nf) / nseg);
  T s1v = p[fs * sN], s2v = p[(fs + 1) * sN], s3 = p[(fs + 2) * sN], s4 = p[(fs + 3) * sN], s5;
  T Ap = T(0), Bp = T(0);
  // software prefetch: the next RC_PF cells of the march are in flight while cell fn is reconstructed
  // (window index fn + 5 of the march ends at fe + 4, the last ghost layer)
  T pf[RC_PF];
#pragma unroll
  for (int k = 0; k < RC_PF; ++k) pf[k] = (fs + 4 + k <= fe + 4) ? p[(fs + 4 + k) * sN] : T(0);
  for (int fn = fs - 1; fn < fe; ++fn) {
    s5 = pf[0];
#pragma unroll
    for (int k = 0; k + 1 < RC_PF; ++k) pf[k] = pf[k + 1];
    pf[RC_PF - 1] = (fn + 5 + RC_PF <= fe + 4) ? p[(fn + 5 + RC_PF) * sN] : T(0);
    T Ac, Bc;
    weno5z_cell(s1v, s2v, s3, s4, s5, Ac, Bc);
    if (fn >= fs) {
      const T ih = jfn[fn];
      ff[L.at(0, c, fn, l)] = Bp;
      ff[L.at(1, c, fn, l)] = Ac;
      ff[L.at(2, c, fn, l)] = (T(2) * Ap + T(4) * Bp - T(6) * s2v) * ih;
      ff[L.at(3, c, fn, l)] = (T(-4) * Ac - T(2) * Bc + T(6) * s3) * ih;
      ff[L.at(4, c, fn, l)] = (-s1v + T(7) * s2v + T(7) * s3 - s4) * T(1.0 / 12.0);
      ff[L.at(5, c, fn, l)] = (s1v - T(15) * s2v + T(15) * s3 - s4) * (T(1.0 / 12.0) * ih);
    }
    s1v = s2v;
    s2v = s3;
    s3 = s4;
    s4 = s5;
    Ap = Ac;
    Bp = Bc;
  }
}

// Fused flux sweep of one direction for one tile of TT1 x TT2 faces at normal face index fn:
//   A  copy of the face fields (A2, from recon_kernel) of the (TT1+4) x (TT2+4) lines -> sA
//   B  t1 pass (A3): values at the two t1 Gauss abscissae of all 6 fields and t1-derivatives of
//      Ql, Qr, C on every row -> sB[l2][comp][slot][m][a]
//   C  one thread per Gauss point: t2 pass, loaded lazily one derivative direction at a time,
//      feeding the BGK flux (A4-A6); 4-point quadrature by warp shuffles (A7)
// Lane layout in phase C: lane = 16 n + 2 TT1 bl + TT1 m + a (a = t1 face in tile, (m, n) the Gauss
// point, t2 face b = BPW w + bl), so every half-warp reads 2 TT1 consecutive (m, a) words of sB from
// each of its 16 / (2 TT1) rows, in disjoint bank groups.
// VAR: bit 0 = PRF (Pr != 1 heat-flux fix, O-12), bit 1 = power-law viscosity
template <typename T, int DIR, int STAGE, int VAR>
__global__ void __launch_bounds__(FluxCfg<T>::NT, FluxCfg<T>::MINB)
    flux_kernel(const T* __restrict__ ff, T* __restrict__ flux, Geo<T> g, GasK<T> gas, const Ctl* __restrict__ ctl,
                int jofs) {
  if (ctl->halt) return;
  constexpr int A1 = (DIR + 1) % 3, A2 = (DIR + 2) % 3;  // tangent axes t1, t2 (O-23)
  using Cfg = FluxCfg<T>;
  constexpr int TT1 = Cfg::TT1, TL1 = Cfg::TL1, TL1P = Cfg::TL1P, TT2 = Cfg::TT2, TL2 = Cfg::TL2;
  constexpr int NTHREADS_FLUX = Cfg::NT, SA_C = Cfg::SA_C, RS = Cfg::RS, CS = Cfg::CS, KS = Cfg::KS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sA = reinterpret_cast<T*>(smem_raw);  // [6][5][SA_C]
  T* sB = sA + 6 * 5 * SA_C;               // t1-pass outputs (FluxCfg: RS, CS, KS, MA)

  const int n1 = g.n[A1], n2 = g.n[A2];
  // jofs: first t2 tile of this launch (the x sweep's tiles run in parts as their face-field lines land)
  const int t10 = blockIdx.x * TT1, t20 = (blockIdx.y + jofs) * TT2;
  // fpb consecutive normal faces per block: the face fields of face fn+1 are copied
  // (cp.async) into sA while face fn is in phase C, so only the first copy's latency is exposed
  // gridDim.z blocks share the n+1 normal faces as evenly as possible (fpb or fpb - 1 each)
  const int nf_all = g.n[DIR] + 1;
  const int fn0 = (int)(((long long)blockIdx.z * nf_all) / gridDim.z);
  const int nfn = (int)(((long long)(blockIdx.z + 1) * nf_all) / gridDim.z) - fn0;
  auto issue_A = [&](int fn) {
    const FFLayout<T, DIR> L = ff_layout<T, DIR>(g);
    const long long fstride = (long long)L.nf * L.nl;  // next (field, component)
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(sA);
    const T* fbase = ff + (long long)fn * L.nl;
    constexpr int VEC = 16 / (int)sizeof(T);  // lines per 16-byte chunk
    constexpr int NCH = TL1 / VEC;            // chunks per tile row
    // t1 is the contiguous axis of the array and every tile row of TL1 lines starts 16-byte aligned
    // (ff_pitch, t10 % 4 == 0): 16-byte copies.  Tiles whose rows would run past line n1+1 (ragged
    // edge) copy single lines, clamped.
    if ((sizeof(T) == 8 ? HGKS_CP16 : HGKS_CP16_32) && t10 + TL1 - 2 <= n1 + 2) {
      // item = (chunk, row l2, fc group): FS groups of 30/FS (field, component) planes each
      constexpr int NRC = TL2 * NCH;
      constexpr int FSM = NTHREADS_FLUX / NRC;
      constexpr int FS = FSM >= 6 ? 6 : (FSM >= 5 ? 5 : (FSM >= 3 ? 3 : (FSM >= 2 ? 2 : 1)));
      constexpr int FPG = 30 / FS;
      static_assert(30 % FS == 0, "fc groups");
      const int j = threadIdx.x;
      if (j < NRC * FS) {
        const int ch = j % NCH, l2 = (j / NCH) % TL2, fg = j / NRC;
        const int t2 = min(t20 + l2 - 2, n2 + 1);
        const T* src = fbase + (long long)(fg * FPG) * fstride + L.line(t10 - 2 + ch * VEC, t2);
        unsigned dst = sbase + (unsigned)(((fg * FPG) * SA_C + l2 * TL1P + ch * VEC) * (int)sizeof(T));
#pragma unroll
        for (int f = 0; f < FPG; ++f) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
          src += fstride;
          dst += SA_C * sizeof(T);
        }
      }
    } else {
      constexpr int NLINE = TL1 * TL2;
      constexpr int NPASS = (NLINE + NTHREADS_FLUX - 1) / NTHREADS_FLUX;
#pragma unroll
      for (int pass = 0; pass < NPASS; ++pass) {
        const int j = threadIdx.x + pass * NTHREADS_FLUX;
        if (j < NLINE) {
          const int l1 = j % TL1, l2 = j / TL1;
          const int t1 = min(t10 + l1 - 2, n1 + 1), t2 = min(t20 + l2 - 2, n2 + 1);  // ragged tiles: clamp
          const T* src = fbase + L.line(t1, t2);
          unsigned dst = sbase + (unsigned)((l2 * TL1P + l1) * sizeof(T));
#pragma unroll
          for (int fc = 0; fc < 30; ++fc) {
            if (sizeof(T) == 8)
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
            else
              asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
            src += fstride;
            dst += SA_C * sizeof(T);
          }
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue_A(fn0);
#ifndef HGKS_HOIST_C
#define HGKS_HOIST_C 1  // phase-C thread constants (lane roles, metrics, dt) loaded once per block, not per face
#endif
#if HGKS_HOIST_C
  // lane = 16 n + 2 TT1 bl + TT1 m + a; t2 face b = BPW warp + bl
  const int lane = threadIdx.x & 31;
  const int a = lane % TT1, m = (lane / TT1) & 1, nn = lane >> 4;
  const int b = (threadIdx.x >> 5) * Cfg::BPW + ((lane & 15) / (2 * TT1));
  const T ih1 = g.jg[A1][m * n1 + min(t10 + a, n1 - 1)], ih2 = g.jg[A2][nn * n2 + min(t20 + b, n2 - 1)];
  const T dt = T(ctl->dt), idt = T(ctl->idt);
#endif
#ifdef HGKS_PHASE_TIMING
  long long tA = 0, tB = 0, tC = 0;
#endif
  for (int it = 0; it < nfn; ++it) {
    const int fn = fn0 + it;  // face fn: cells fn-1 | fn
#ifdef HGKS_PHASE_TIMING
    long long tp0 = clock64();
#endif
#ifndef HGKS_DEBUG_SKIP_AB
#define HGKS_DEBUG_SKIP_AB 0  // timing experiment only: phases A/B run for the first face alone
#endif
    const bool do_ab = !HGKS_DEBUG_SKIP_AB || it == 0;
    if (do_ab) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();  // sA(fn) landed; every thread is done with sB of the previous face
    }
#ifdef HGKS_PHASE_TIMING
    long long tp1 = clock64();
#endif

  // ---- phase B: t1 pass on every row l2: value (6 fields) and t1-derivative (Ql, Qr, C) -----
  // One item = (a, c, l2) computes both Gauss abscissae m = 0, 1 from the same 30 loads: point
  // m = 1 uses the mirrored weights wv[1][r] = wv[0][4-r], wd[1][r] = -wd[0][4-r].
  // Item order: TT1 = 8: (a, c, l2), a half-warp reads 2 components of one row; TT1 = 4: (a, l2, c),
  // a half-warp reads 4 rows (TL1P apart) of one component -- conflict-free (TT1 = 8 except where a
  // warp straddles two rows).
  for (int w = threadIdx.x; do_ab && w < TT1 * 5 * TL2; w += NTHREADS_FLUX) {
    const int a = w % TT1;
    const int c = TT1 == 8 ? (w / TT1) % 5 : w / (TT1 * TL2);
    const int l2 = TT1 == 8 ? w / (TT1 * 5) : (w / TT1) % TL2;
    T o0[NB], o1[NB];
    const T* src = sA + c * SA_C + l2 * TL1P + a;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      o0[k] = T(0);
      o1[k] = T(0);
    }
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const T wv0 = hgks::wv0<T>(r), wd0 = hgks::wd0<T>(r);          // m = 0 weights of tap r
      const T wv1 = hgks::wv0<T>(4 - r), wd1 = -hgks::wd0<T>(4 - r);  // m = 1 weights of tap r
#pragma unroll
      for (int ff = 0; ff < 6; ++ff) {
        const T x = src[ff * 5 * SA_C + r];
        o0[ff] += wv0 * x;
        o1[ff] += wv1 * x;
        if (ff == 0) { o0[6] += wd0 * x; o1[6] += wd1 * x; }
        if (ff == 1) { o0[7] += wd0 * x; o1[7] += wd1 * x; }
        if (ff == 4) { o0[8] += wd0 * x; o1[8] += wd1 * x; }
      }
    }
    T* dst = sB + l2 * RS + (Cfg::VEC ? 0 : c * CS + Cfg::MA(0, a));
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      if constexpr (Cfg::VEC) {
        dst[k * KS + Cfg::VOFF(c, Cfg::MA(0, a))] = o0[k];
        dst[k * KS + Cfg::VOFF(c, Cfg::MA(1, a))] = o1[k];
      } else if constexpr (TT1 == 4 && sizeof(T) == 8) {  // (m = 0, m = 1) adjacent: one 16-byte store
        *reinterpret_cast<double2*>(dst + k * KS) = make_double2((double)o0[k], (double)o1[k]);
      } else if constexpr (TT1 == 4) {
        *reinterpret_cast<float2*>(dst + k * KS) = make_float2((float)o0[k], (float)o1[k]);
      } else {
        dst[k * KS] = o0[k];
        dst[k * KS + Cfg::MA(1, 0)] = o1[k];
      }
    }
  }
  if (do_ab) {
  __syncthreads();  // sB complete; sA free for the next face
  if (it + 1 < nfn && !HGKS_DEBUG_SKIP_AB) issue_A(fn + 1);
  }
#ifdef HGKS_PHASE_TIMING
  long long tp2 = clock64();
#endif

  // ---- phase C: one thread per Gauss point ----------------------------------------------------
  // lane = 16 n + 2 TT1 bl + TT1 m + a; t2 face b = BPW warp + bl
#if !HGKS_HOIST_C
  const int lane = threadIdx.x & 31;
  const int a = lane % TT1, m = (lane / TT1) & 1, nn = lane >> 4;
  const int b = (threadIdx.x >> 5) * Cfg::BPW + ((lane & 15) / (2 * TT1));
  const T ih1 = g.jg[A1][m * n1 + min(t10 + a, n1 - 1)], ih2 = g.jg[A2][nn * n2 + min(t20 + b, n2 - 1)];
#endif
  const T sgn = nn ? T(-1) : T(1);
  // t2 pass of slot k, component c, over rows b..b+4: value (wv) or derivative (wd) at this Gauss
  // point.  n = 1 uses the mirrored weights wv[1][r] = wv[0][4-r], wd[1][r] = -wd[0][4-r]:
  //  * fp64: mirror the ROW order instead (weights stay immediates); lanes n = 0 / 1 sit in different
  //    half-warps, so the two row streams never share a bank within a 128-byte wavefront;
  //  * fp32: a whole warp is one wavefront, so keep the row order (n = 0 and n = 1 lanes read the
  //    same word: broadcast) and hold the 10 mirrored weights in registers.
  // The empty asm with a memory clobber keeps ptxas from hoisting these shared loads ahead of
  // earlier flux work (register pressure: they would be spilled).
#ifndef HGKS_ROW_MIRROR64
#define HGKS_ROW_MIRROR64 1
#endif
  constexpr bool kRowMirror = sizeof(T) == 8 && HGKS_ROW_MIRROR64;
  const T* row0 = sB + Cfg::MA(m, a) + (b + (kRowMirror && nn ? 4 : 0)) * RS;
  const int rstep = (kRowMirror && nn) ? -RS : RS;
  T wvl[5], wdl[5];
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    wvl[r] = (!kRowMirror && nn) ? T(kWV0(4 - r)) : T(kWV0(r));
    wdl[r] = (!kRowMirror && nn) ? -T(kWD0(4 - r)) : T(kWD0(r));
  }
#ifndef HGKS_TV_FENCE
#define HGKS_TV_FENCE 1  // keep the t2-pass loads from being hoisted (register pressure)
#endif
#ifndef HGKS_TV_SPLIT
#define HGKS_TV_SPLIT 0  // 1: each 5-tap sum as two partial chains (shorter dependency latency)
#endif
  auto tv = [&](int c, int k) {
    if (HGKS_TV_FENCE) asm volatile("" ::: "memory");
    if (HGKS_TV_SPLIT) {
      const T* p = row0 + c * CS + k * KS;
      const T a0 = (kRowMirror ? wv0<T>(0) : wvl[0]) * p[0] + (kRowMirror ? wv0<T>(2) : wvl[2]) * p[2 * rstep] +
                   (kRowMirror ? wv0<T>(4) : wvl[4]) * p[4 * rstep];
      const T a1 = (kRowMirror ? wv0<T>(1) : wvl[1]) * p[rstep] + (kRowMirror ? wv0<T>(3) : wvl[3]) * p[3 * rstep];
      return a0 + a1;
    }
    T v = T(0);
#pragma unroll
    for (int r = 0; r < 5; ++r) v += (kRowMirror ? wv0<T>(r) : wvl[r]) * row0[r * rstep + c * CS + k * KS];
    return v;
  };
  // row mirror: the derivative of a mirrored row stream carries the sign sgn, folded into ih2s (every
  // t2 derivative is multiplied by the metric ih2)
  const T ih2s = kRowMirror ? sgn * ih2 : ih2;
  auto td = [&](int c, int k) {
    if (HGKS_TV_FENCE) asm volatile("" ::: "memory");
    T v = T(0);
#pragma unroll
    for (int r = 0; r < 5; ++r) v += (kRowMirror ? wd0<T>(r) : wdl[r]) * row0[r * rstep + c * CS + k * KS];
    return v;
  };
#if !HGKS_HOIST_C
  const T dt = T(ctl->dt), idt = T(ctl->idt);
#endif
  constexpr bool PRF = VAR & 1;
  GpFlux<T, STAGE == 1, PRF, (VAR >> 1) & 1> gf;
  // value and t2-derivative of Ql, Qr from the same five row loads (the t2 derivatives are held
  // until the side passes: 10 more live registers, 50 fewer shared loads per Gauss point)
  auto tvd = [&](int c, int k, T& v, T& d) {
    if (HGKS_TV_FENCE) asm volatile("" ::: "memory");
    v = T(0);
    d = T(0);
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const T x = row0[r * rstep + c * CS + k * KS];
      v += (kRowMirror ? wv0<T>(r) : wvl[r]) * x;
      d += (kRowMirror ? wd0<T>(r) : wdl[r]) * x;
    }
  };
  T d2l[5], d2r[5];
  if constexpr (Cfg::VEC) {
    // five components of slot k per row: one float4 + one float load (VOFF layout); weights w[r]
    const T* rv = sB + b * RS + 4 * Cfg::MA(m, a);
    const T* rs = sB + b * RS + 8 * TT1 + Cfg::MA(m, a);
    auto pass5 = [&](int k, const T (&w)[5], T (&o)[5]) {
      if (HGKS_TV_FENCE) asm volatile("" ::: "memory");
#pragma unroll
      for (int r = 0; r < 5; ++r) {
        const float4 x = *reinterpret_cast<const float4*>(rv + r * rstep + k * KS);
        const T x4 = rs[r * rstep + k * KS];
        o[0] = r ? o[0] + w[r] * x.x : w[r] * x.x;
        o[1] = r ? o[1] + w[r] * x.y : w[r] * x.y;
        o[2] = r ? o[2] + w[r] * x.z : w[r] * x.z;
        o[3] = r ? o[3] + w[r] * x.w : w[r] * x.w;
        o[4] = r ? o[4] + w[r] * x4 : w[r] * x4;
      }
    };
    auto pass5vd = [&](int k, T (&v)[5], T (&d)[5]) {
      if (HGKS_TV_FENCE) asm volatile("" ::: "memory");
#pragma unroll
      for (int r = 0; r < 5; ++r) {
        const float4 x = *reinterpret_cast<const float4*>(rv + r * rstep + k * KS);
        const T x4 = rs[r * rstep + k * KS];
        const T xs[5] = {x.x, x.y, x.z, x.w, x4};
#pragma unroll
        for (int c = 0; c < 5; ++c) {
          v[c] = r ? v[c] + wvl[r] * xs[c] : wvl[r] * xs[c];
          d[c] = r ? d[c] + wdl[r] * xs[c] : wdl[r] * xs[c];
        }
      }
    };
    {
      T Wl[5], Wr[5];
      pass5vd(0, Wl, d2l);
      pass5vd(1, Wr, d2r);
      gf.begin(gas, Wl, Wr, dt, idt);
    }
    gf.template add_side<+1>([&](int i, T (&d)[5]) {
      if (i == 0) pass5(2, wvl, d);
      if (i == 1) { pass5(6, wvl, d); for (int c = 0; c < 5; ++c) d[c] *= ih1; }
      if (i == 2) for (int c = 0; c < 5; ++c) d[c] = d2l[c] * ih2s;
    });
    gf.template add_side<-1>([&](int i, T (&d)[5]) {
      if (i == 0) pass5(3, wvl, d);
      if (i == 1) { pass5(7, wvl, d); for (int c = 0; c < 5; ++c) d[c] *= ih1; }
      if (i == 2) for (int c = 0; c < 5; ++c) d[c] = d2r[c] * ih2s;
    });
    gf.add_equilibrium([&](int i, T (&d)[5]) {
      if (i == 0) pass5(5, wvl, d);
      if (i == 1) { pass5(8, wvl, d); for (int c = 0; c < 5; ++c) d[c] *= ih1; }
      if (i == 2) { pass5(4, wdl, d); for (int c = 0; c < 5; ++c) d[c] *= ih2s; }
    });
  } else {
  {
    T Wl[5], Wr[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      tvd(c, 0, Wl[c], d2l[c]);
      tvd(c, 1, Wr[c], d2r[c]);
    }
    gf.begin(gas, Wl, Wr, dt, idt);
  }
  gf.template add_side<+1>([&](int i, T (&d)[5]) {
#pragma unroll
    for (int c = 0; c < 5; ++c) d[c] = i == 0 ? tv(c, 2) : (i == 1 ? tv(c, 6) * ih1 : d2l[c] * ih2s);
  });
  gf.template add_side<-1>([&](int i, T (&d)[5]) {
#pragma unroll
    for (int c = 0; c < 5; ++c) d[c] = i == 0 ? tv(c, 3) : (i == 1 ? tv(c, 7) * ih1 : d2r[c] * ih2s);
  });
  gf.add_equilibrium([&](int i, T (&d)[5]) {
#pragma unroll
    for (int c = 0; c < 5; ++c) d[c] = i == 0 ? tv(c, 5) : (i == 1 ? tv(c, 8) * ih1 : td(c, 4) * ih2s);
  });
  }
  T F[5], dF[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    F[k] = gf.F[k];
    dF[k] = gf.dF[k];
  }
  // 2x2 Gauss quadrature, omega_mn = 1/4 (O-8): the face's Gauss points sit at lanes l, l ^ TT1 (m),
  // l ^ 16 (n), l ^ TT1 ^ 16
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    if (STAGE == 1) {
      F[k] += __shfl_xor_sync(0xffffffffu, F[k], TT1);
      F[k] += __shfl_xor_sync(0xffffffffu, F[k], 16);
    }
    dF[k] += __shfl_xor_sync(0xffffffffu, dF[k], TT1);
    dF[k] += __shfl_xor_sync(0xffffffffu, dF[k], 16);
  }
  const int f1 = t10 + a, f2 = t20 + b;
  if (m == 0 && nn == 0 && f1 < n1 && f2 < n2) {
    int cd[3];
    cd[DIR] = fn;
    cd[A1] = f1;
    cd[A2] = f2;
    const int fx = g.n[0] + (DIR == 0), fy = g.n[1] + (DIR == 1), fz = g.n[2] + (DIR == 2);
    const long long nface = (long long)fx * fy * fz;
    const long long id = ((long long)cd[2] * fy + cd[1]) * fx + cd[0];
    const int gc[5] = {0, 1 + DIR, 1 + A1, 1 + A2, 4};
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      if (STAGE == 1) flux[gc[k] * nface + id] = T(0.25) * F[k];
      flux[(5 + gc[k]) * nface + id] = T(0.25) * dF[k];
    }
  }
#ifdef HGKS_PHASE_TIMING
  long long tp3 = clock64();
  tA += tp1 - tp0;
  tB += tp2 - tp1;
  tC += tp3 - tp2;
#endif
  }  // faces of this block
#ifdef HGKS_PHASE_TIMING
  if (threadIdx.x == 0) {
    atomicAdd(&g_phase_cycles[0], (unsigned long long)tA);
    atomicAdd(&g_phase_cycles[1], (unsigned long long)tB);
    atomicAdd(&g_phase_cycles[2], (unsigned long long)tC);
    atomicAdd(&g_phase_cycles[3], (unsigned long long)nfn);
  }
#endif
}

// ---- ghost layers along x and y over the interior z planes (A1; O-16, O-17) ---------------------
// 1. wall axes (isothermal no-slip mirror: U_g = -U_m, T_g = 2 T_wall - T_m, p_g = p_m, rho_g = p_g/T_g)
//    over the interior of the other in-plane axis; 2. periodic axes over the full extended plane
//    (a ghost cell copies the cell whose periodic coordinates are wrapped), which fills corners.
template <typename T>
__global__ void ghost_wall_kernel(T* __restrict__ q, Geo<T> g, double gamma, const Ctl* __restrict__ ctl) {
  if (ctl->halt) return;
  const int nx = g.n[0], ny = g.n[1];
  // items: (k, axis-position along the other in-plane axis, layer m, side); axes handled: x, y
  for (int ax = 0; ax < 2; ++ax) {
    if (!g.wall[ax]) continue;
    const int n_ax = g.n[ax], n_ot = g.n[1 - ax];
    const long long total = (long long)g.n[2] * n_ot * 3 * 2;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
      const int side = (int)(e % 2);
      const int m = (int)((e / 2) % 3);
      const int o = (int)((e / 6) % n_ot);
      const int k = (int)(e / (6LL * n_ot));
      const int im = side ? n_ax - 1 - m : m, ig = side ? n_ax + m : -1 - m;
      int ci, cj, gi, gj;
      if (ax == 0) { ci = im; gi = ig; cj = gj = o; } else { cj = im; gj = ig; ci = gi = o; }
      const double rho = (double)q[qidx(g, 0, ci, cj, k)];
      const double U = (double)q[qidx(g, 1, ci, cj, k)] / rho, V = (double)q[qidx(g, 2, ci, cj, k)] / rho,
                   W = (double)q[qidx(g, 3, ci, cj, k)] / rho;
      const double p = (gamma - 1.0) * ((double)q[qidx(g, 4, ci, cj, k)] - 0.5 * rho * (U * U + V * V + W * W));
      const double Tg = 2.0 * (double)g.T_wall - p / rho;
      const double rg = p / Tg;
      q[qidx(g, 0, gi, gj, k)] = T(rg);
      q[qidx(g, 1, gi, gj, k)] = T(-rg * U);
      q[qidx(g, 2, gi, gj, k)] = T(-rg * V);
      q[qidx(g, 3, gi, gj, k)] = T(-rg * W);
      q[qidx(g, 4, gi, gj, k)] = T(p / (gamma - 1.0) + 0.5 * rg * (U * U + V * V + W * W));
    }
    (void)nx;
    (void)ny;
  }
}

template <typename T>
__global__ void ghost_xy_kernel(T* __restrict__ q, Geo<T> g, const Ctl* __restrict__ ctl) {
  if (ctl->halt) return;
  // only the ghost cells of each (plane, variable): the 3-deep bands j < 0, j >= ny over the full
  // extended x range (6 px cells), then the x bands i < 0, i >= nx of the interior rows (6 ny)
  const int nx = g.n[0], ny = g.n[1];
  const long long per = 6LL * g.px + 6LL * ny;
  const long long total = (long long)g.n[2] * 5 * per;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const long long r = e % per;
    const long long kv = e / per;
    const int v = (int)(kv % 5);
    const int k = (int)(kv / 5);
    int i, j;
    if (r < 6LL * g.px) {
      const int jj = (int)(r / g.px);
      j = jj < 3 ? jj - 3 : ny + jj - 3;
      i = (int)(r % g.px) - 3;
    } else {
      const int rr = (int)(r - 6LL * g.px);
      const int ii = rr % 6;
      j = rr / 6;
      i = ii < 3 ? ii - 3 : nx + ii - 3;
    }
    // source: wrap the periodic in-plane axes only (wall ghosts come from ghost_wall_kernel)
    const int si = g.wall[0] ? i : (i + nx) % nx, sj = g.wall[1] ? j : (j + ny) % ny;  // n >= 5 > 3
    if (si == i && sj == j) continue;  // a pure wall ghost
    q[qidx(g, v, i, j, k)] = q[qidx(g, v, si, sj, k)];
  }
}

// max over d of (|U_d| + c)/dx_d for one cell (O-13); c = sqrt(gamma p / rho)
template <typename T>
__device__ __forceinline__ double wave_speed(const T (&c5)[5], const Geo<T>& g, int i, int j, int k, double gamma,
                                             bool& ok) {
  double rho = (double)c5[0];
  double U = (double)c5[1] / rho, V = (double)c5[2] / rho, W = (double)c5[3] / rho;
  double p = (gamma - 1.0) * ((double)c5[4] - 0.5 * rho * (U * U + V * V + W * W));
  ok = (rho > 0.0) && (p > 0.0) && isfinite(rho) && isfinite(p) && isfinite(U) && isfinite(V) && isfinite(W);
  double c = sqrt(gamma * p / rho);
  double sx = (fabs(U) + c) * (double)g.iw[0][i], sy = (fabs(V) + c) * (double)g.iw[1][j],
         sz = (fabs(W) + c) * (double)g.iw[2][k];
  return fmax(sx, fmax(sy, sz));
}

// Block max of s, then ONE atomicMax per block on the bit pattern (which orders non-negative doubles).
// Every thread of the block must call it.  (One atomic per warp -- 524k atomics on one address per
// stage-2 update at 256^3 -- serialised in the L2 atomic unit.)
__device__ __forceinline__ void block_max_commit(double s, unsigned long long* dst) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
  __shared__ double wmax[32];
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    for (int w = 1; w < nw; ++w) s = fmax(s, wmax[w]);
    if (s > 0.0) atomicMax(dst, (unsigned long long)__double_as_longlong(s));
  }
}

// ---- flux divergence + S2O4 stage update (Eqs. (3)-(4), (7)) ----------------------------------
// STAGE 1: Qs = Q + dt/2 L + dt^2/8 dL ;  R = Q + dt L + dt^2/6 dL
// STAGE 2: R  = R + dt^2/3 dL(Q*)  (= Q^{n+1}); epilogue: validity + wave speed into ctl->red
// Body force (O-26; ctl->force_mode != 0): stage 1 adds S = (0, rho f, 0, 0, rho U f) to L and
// f (L_rho, L_rhoU) to dL of (Q^n); stage 2 adds f (Lt_rho, Lt_rhoU) to dL(Q*) with
// Lt = L + dt/2 dL of Q^n, recovered from the two stage-1 outputs: with a = Q* - Q^n and
// b = R - Q^n (a = dt L/2 + dt^2 dL/8, b = dt L + dt^2 dL/6), Lt = (8a - 3b)/dt.  Mode 2 also
// sums (rho dV, rho U dV) of Q^{n+1} per block (fixed order) into bulk[2 * blockIdx.x + {0, 1}].
// DIAG (stage 1 only; the per-step history of hgks_history_enable, NEXT-2): the volume diagnostics
// of Q^n -- whose ghosts the stage-1 halo has just filled -- summed per block (fixed order) into
// dpart[NDIAG * block]; hist_reduce_kernel / hist_final_kernel finish the sum.  Stage 2 cannot see
// the gradients of Q^{n+1} (its neighbours are written by other blocks of the same launch), so the
// history holds the state at the START of every step; the final state is one hgks_diagnostics call.
constexpr int UPD_X = 64, UPD_Y = DIAG_TPB / UPD_X;  // update_kernel block shape (DIAG_TPB threads)
// stage-1 update with the per-step history: block shape of its own (HGKS_UPDD_X = 32 -> 32 x 8 cells, a
// 36 x 12 velocity tile instead of 68 x 8, measured 0.565 vs 0.525 ms/step of history at 256^3: kept 64)
#ifndef HGKS_UPD2_MINB
#define HGKS_UPD2_MINB 1  // min blocks per SM of the stage-2 update (occupancy experiment)
#endif
#ifndef HGKS_UPD1_MINB
#define HGKS_UPD1_MINB 2  // min blocks per SM of the stage-1 update without the history (128 registers: 1.88 -> 1.66 ms/step)
#endif
#ifndef HGKS_UPDD_X
#define HGKS_UPDD_X 64
#endif
constexpr int UPDD_X = HGKS_UPDD_X, UPDD_Y = DIAG_TPB / UPDD_X;
template <typename T, int STAGE, bool DIAG = false>
__global__ void __launch_bounds__(DIAG_TPB, (STAGE == 2 && !DIAG) ? HGKS_UPD2_MINB : (DIAG ? 1 : HGKS_UPD1_MINB)) update_kernel(const T* __restrict__ Q, T* __restrict__ Qs, T* __restrict__ R,
                              const T* __restrict__ FX, const T* __restrict__ FY, const T* __restrict__ FZ,
                              Geo<T> g, DiagGeo dg, double gamma, Ctl* __restrict__ ctl, double* __restrict__ bulk,
                              double* __restrict__ dpart = nullptr) {
  if (ctl->halt) return;
  const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
  // block = UPD_X x UPD_Y cells of one z plane (grid: x tiles, y tiles, z): no index divisions
  constexpr int UX = DIAG ? UPDD_X : UPD_X, UY = DIAG ? UPDD_Y : UPD_Y;
  const int i = blockIdx.x * UX + (threadIdx.x % UX);
  const int j = blockIdx.y * UY + (threadIdx.x / UX);
  const int k = blockIdx.z;
  const double dt = ctl->dt;
  const int fmode = ctl->force_mode;
  double smax = 0.0, bsum[2] = {0.0, 0.0};
  if (i < nx && j < ny) {
    const long long nfx = (long long)(nx + 1) * ny * nz, nfy = (long long)nx * (ny + 1) * nz, nfz = (long long)nx * ny * (nz + 1);
    const long long ix = ((long long)k * ny + j) * (nx + 1) + i;
    const long long iy = ((long long)k * (ny + 1) + j) * nx + i;
    const long long iz = ((long long)k * ny + j) * nx + i;
    const long long oy = nx, oz = (long long)nx * ny;
    const T ihx = g.iw[0][i], ihy = g.iw[1][j], ihz = g.iw[2][k];
    const T tdt = T(dt);
    T dL[5], L[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) {
      dL[c] = -((FX[(5 + c) * nfx + ix + 1] - FX[(5 + c) * nfx + ix]) * ihx +
                (FY[(5 + c) * nfy + iy + oy] - FY[(5 + c) * nfy + iy]) * ihy +
                (FZ[(5 + c) * nfz + iz + oz] - FZ[(5 + c) * nfz + iz]) * ihz);
      if (STAGE == 1)
        L[c] = -((FX[c * nfx + ix + 1] - FX[c * nfx + ix]) * ihx + (FY[c * nfy + iy + oy] - FY[c * nfy + iy]) * ihy +
                 (FZ[c * nfz + iz + oz] - FZ[c * nfz + iz]) * ihz);
    }
    if (STAGE == 1) {
      T q[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) q[c] = Q[qidx(g, c, i, j, k)];
      if (fmode) {  // O-26
        const T f = T(ctl->force);
        L[1] += q[0] * f;
        L[4] += q[1] * f;
        dL[1] += f * L[0];
        dL[4] += f * L[1];
      }
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const long long qi = qidx(g, c, i, j, k);
        Qs[qi] = q[c] + T(0.5) * tdt * L[c] + T(0.125) * tdt * tdt * dL[c];
        R[qi] = q[c] + tdt * L[c] + (T(1) / T(6)) * tdt * tdt * dL[c];
      }
    } else {
      // R of all five components loaded before the first store: the in-place update R[qi] = ... would
      // otherwise order each component's load after the previous component's store (R may alias
      // itself), five dependent DRAM round trips per thread (ncu: long-scoreboard 13 stalls per issue)
      T r5[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) r5[c] = R[qidx(g, c, i, j, k)];
      if (fmode) {  // O-26: Lt = L + dt/2 dL of Q^n = (8a - 3b)/dt
        const double f = ctl->force;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const long long qi = qidx(g, c, i, j, k);
          const double qn = (double)Q[qi], a = (double)Qs[qi] - qn, b = (double)r5[c] - qn;
          dL[c == 0 ? 1 : 4] += T(f * (8.0 * a - 3.0 * b) / dt);
        }
      }
      T out[5];
#pragma unroll
      for (int c = 0; c < 5; ++c) {
        const long long qi = qidx(g, c, i, j, k);
        const T v = r5[c] + (T(1) / T(3)) * tdt * tdt * dL[c];
        R[qi] = v;
        out[c] = v;
      }
      bool ok;
      smax = wave_speed(out, g, i, j, k, gamma, ok);
      if (!ok) {
        smax = 0.0;
        unsigned long long gid = ((unsigned long long)(k + g.z0) * g.ny_g + j) * g.nx_g + i;
        atomicMin(&ctl->bad_cell, gid);
        ctl->red[1] = 1ull;  // benign race: every writer stores 1
      }
      if (fmode == 2) {
        const double vol = dg.w[0][i] * dg.w[1][j] * dg.w[2][k];
        bsum[0] = (double)out[0] * vol;
        bsum[1] = (double)out[1] * vol;
      }
    }
  }
  if (STAGE == 1 && DIAG) {
    double acc[NDIAG];
#pragma unroll
    for (int n = 0; n < NDIAG; ++n) acc[n] = 0.0;
    // velocities of the block's 64 x 4 cells and their +-2 x/y halo, one reciprocal each, staged in
    // shared memory; the z neighbours (other planes) come from global memory
    constexpr int TX = UX + 4, TY = UY + 4;
    __shared__ double su[3][TY][TX];
    for (int e = threadIdx.x; e < TX * TY; e += DIAG_TPB) {
      const int lx = e % TX, ly = e / TX;
      const int gi = blockIdx.x * UX + lx - 2, gj = blockIdx.y * UY + ly - 2;
      if (gi <= nx + 2 && gj <= ny + 2) {
        double uu[3];
        vel_of(Q, g, gi, gj, k, uu);
#pragma unroll
        for (int c = 0; c < 3; ++c) su[c][ly][lx] = uu[c];
      }
    }
    __syncthreads();
    if (i < nx && j < ny) {
      const int lx = threadIdx.x % UX + 2, ly = threadIdx.x / UX + 2;
      const double vol = dg.w[0][i] * dg.w[1][j] * dg.w[2][k];
      const double rho = (double)Q[qidx(g, 0, i, j, k)];
      double u[3], m[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        m[c] = (double)Q[qidx(g, 1 + c, i, j, k)];
        u[c] = su[c][ly][lx];
      }
      double grad[3][3];  // grad[c][d] = d u_c / d x_d (O-25), as diag_cell
      double up1[3], um1[3], up2[3], um2[3];
      vel_of(Q, g, i, j, k + 1, up1);
      vel_of(Q, g, i, j, k - 1, um1);
      vel_of(Q, g, i, j, k + 2, up2);
      vel_of(Q, g, i, j, k - 2, um2);
      const double Jx = dg.jc[0][i] * (1.0 / 12.0), Jy = dg.jc[1][j] * (1.0 / 12.0), Jz = dg.jc[2][k] * (1.0 / 12.0);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        grad[c][0] = Jx * (8.0 * (su[c][ly][lx + 1] - su[c][ly][lx - 1]) - (su[c][ly][lx + 2] - su[c][ly][lx - 2]));
        grad[c][1] = Jy * (8.0 * (su[c][ly + 1][lx] - su[c][ly - 1][lx]) - (su[c][ly + 2][lx] - su[c][ly - 2][lx]));
        grad[c][2] = Jz * (8.0 * (up1[c] - um1[c]) - (up2[c] - um2[c]));
      }
      diag_terms(rho, u, m, grad, (double)Q[qidx(g, 4, i, j, k)], vol, gamma, acc);
    }
    __shared__ double shd[NDIAG * (DIAG_TPB / 32)];
    block_sum_warps(acc, shd);
    if (threadIdx.x == 0) {
      const long long bid = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
#pragma unroll
      for (int n = 0; n < NDIAG; ++n) dpart[bid * NDIAG + n] = acc[n];
    }
  }
  if (STAGE == 2) {
    block_max_commit(smax, &ctl->red[0]);
    if (fmode == 2) {  // uniform branch: every thread of the block takes it
      __shared__ double sh[2 * DIAG_TPB];
      block_sum_fixed(bsum, sh);
      if (threadIdx.x == 0) {
        const long long bid = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        bulk[2 * bid] = bsum[0];
        bulk[2 * bid + 1] = bsum[1];
      }
    }
  }
}

// ---- per-step diagnostic history (NEXT-2) -------------------------------------------------------
// hist_reduce_kernel: HIST_RB blocks, block b sums the update-block partials [b*per, (b+1)*per) in a
// fixed order into dpart2[b]; hist_final_kernel (one block) sums dpart2 in order into row
// ctl->hist_n of hist[cap][NDIAG] and records (t, dt) of the step in hist_td[cap][2].
constexpr int HIST_RB = 148;
__global__ void __launch_bounds__(DIAG_TPB) hist_reduce_kernel(const double* __restrict__ dpart, long long nblocks,
                                                               double* __restrict__ dpart2, const Ctl* __restrict__ ctl) {
  if (ctl->halt) return;
  __shared__ double sh[NDIAG * (DIAG_TPB / 32)];
  const long long per = (nblocks + gridDim.x - 1) / gridDim.x;
  const long long b0 = blockIdx.x * per, b1 = min(nblocks, b0 + per);
  double acc[NDIAG];
#pragma unroll
  for (int n = 0; n < NDIAG; ++n) acc[n] = 0.0;
  for (long long b = b0 + threadIdx.x; b < b1; b += DIAG_TPB) {
#pragma unroll
    for (int n = 0; n < NDIAG; ++n) acc[n] += dpart[b * NDIAG + n];
  }
  block_sum_warps(acc, sh);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int n = 0; n < NDIAG; ++n) dpart2[blockIdx.x * NDIAG + n] = acc[n];
  }
}

__global__ void __launch_bounds__(DIAG_TPB) hist_final_kernel(const double* __restrict__ dpart2, double* __restrict__ hist,
                                                              double* __restrict__ hist_td, Ctl* __restrict__ ctl) {
  if (ctl->halt) return;
  __shared__ double sh[NDIAG * (DIAG_TPB / 32)];
  double acc[NDIAG];
#pragma unroll
  for (int n = 0; n < NDIAG; ++n) acc[n] = 0.0;
  for (int b = threadIdx.x; b < HIST_RB; b += DIAG_TPB) {
#pragma unroll
    for (int n = 0; n < NDIAG; ++n) acc[n] += dpart2[b * NDIAG + n];
  }
  block_sum_warps(acc, sh);
  if (threadIdx.x == 0) {
    const int row = ctl->hist_n;
    if (row < ctl->hist_cap) {
#pragma unroll
      for (int n = 0; n < NDIAG; ++n) hist[(long long)row * NDIAG + n] = acc[n];
      hist_td[2 * row] = ctl->t;
      hist_td[2 * row + 1] = ctl->dt;
      ctl->hist_n = row + 1;
    }
  }
}

// ---- wave-speed max / validity of the current state (set_state) ------------------------------
template <typename T>
__global__ void cfl_kernel(const T* __restrict__ Q, Geo<T> g, double gamma, Ctl* __restrict__ ctl) {
  const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const long long ncell = (long long)nx * ny * nz;
  double smax = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < ncell + 0; e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % nx), j = (int)((e / nx) % ny), k = (int)(e / ((long long)nx * ny));
    T c5[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) c5[c] = Q[qidx(g, c, i, j, k)];
    bool ok;
    double s = wave_speed(c5, g, i, j, k, gamma, ok);
    if (!ok) {
      unsigned long long gid = ((unsigned long long)(k + g.z0) * g.ny_g + j) * g.nx_g + i;
      atomicMin(&ctl->bad_cell, gid);
      ctl->red[1] = 1ull;
    } else {
      smax = fmax(smax, s);
    }
  }
  block_max_commit(smax, &ctl->red[0]);
}

// ---- per-step control (A0): commit the previous step, then choose dt ------------------------
__device__ __forceinline__ void commit_pending(Ctl* c) {
  if (!c->pending) return;
  c->pending = 0;
  if (c->red[1]) {  // the step produced an invalid state somewhere (global after allreduce)
    c->halt = 1;
    return;
  }
  c->t += c->dt;
  c->dt_last = c->dt;
  c->steps_done += 1;
  c->smax_cur = c->red[0];
  c->f_prev = c->force;
  if (c->force_mode == 2) {
    c->m_prev = c->m_cur;
    c->dt_prev = c->dt;
    c->m_cur = c->bulk_new[1] / c->volume;
    c->rho_cur = c->bulk_new[0] / c->volume;
    c->hist = 1;
  }
}

__global__ void dt_kernel(Ctl* c) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (c->halt) return;
  commit_pending(c);
  if (c->halt) return;
  double dt = c->dt_fixed > 0.0 ? c->dt_fixed : c->cfl / __longlong_as_double((long long)c->smax_cur);
  if (c->t_end > 0.0) {
    double rem = c->t_end - c->t;
    if (rem <= 1e-14 * c->t_end) {
      c->halt = 2;
      return;
    }
    if (dt > rem) dt = rem;
  }
  c->dt = dt;
  c->idt = 1.0 / dt;
  if (c->force_mode == 1) {
    c->force = c->f_init;
  } else if (c->force_mode == 2) {  // O-27
    c->force = c->hist ? c->f_prev + ((c->force_target - c->m_cur) / dt - (c->m_cur - c->m_prev) / c->dt_prev) / c->rho_cur
                       : c->f_prev + (c->force_target - c->m_cur) / (dt * c->rho_cur);
  }
  c->red[0] = 0ull;
  c->red[1] = 0ull;
  c->pending = 1;
}

__global__ void commit_kernel(Ctl* c) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (c->halt) return;
  commit_pending(c);
}

// ---- layout conversion: ABI [5][nz][ny][nx] fp64 <-> ghosted [nz+6][5][ny+6][nx+6] T ----------
template <typename T>
__global__ void pack_kernel(const double* __restrict__ in, T* __restrict__ Q, Geo<T> g) {
  const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const long long ncell = (long long)nx * ny * nz;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < 5 * ncell; e += (long long)gridDim.x * blockDim.x) {
    const long long s = e % ncell;
    const int v = (int)(e / ncell);
    const int i = (int)(s % nx), j = (int)((s / nx) % ny), k = (int)(s / ((long long)nx * ny));
    Q[qidx(g, v, i, j, k)] = T(in[e]);
  }
}

template <typename T>
__global__ void unpack_kernel(const T* __restrict__ Q, double* __restrict__ out, Geo<T> g) {
  const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const long long ncell = (long long)nx * ny * nz;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < 5 * ncell; e += (long long)gridDim.x * blockDim.x) {
    const long long s = e % ncell;
    const int v = (int)(e / ncell);
    const int i = (int)(s % nx), j = (int)((s / nx) % ny), k = (int)(s / ((long long)nx * ny));
    out[e] = (double)Q[qidx(g, v, i, j, k)];
  }
}

// L and d_t L from the face arrays (test entry hgks_test_operator), ABI layout, fp64
template <typename T>
__global__ void operator_out_kernel(const T* __restrict__ FX, const T* __restrict__ FY, const T* __restrict__ FZ,
                                    Geo<T> g, double* __restrict__ L, double* __restrict__ dL) {
  const int nx = g.n[0], ny = g.n[1], nz = g.n[2];
  const long long ncell = (long long)nx * ny * nz;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= ncell) return;
  const int i = (int)(e % nx), j = (int)((e / nx) % ny), k = (int)(e / ((long long)nx * ny));
  const long long nfx = (long long)(nx + 1) * ny * nz, nfy = (long long)nx * (ny + 1) * nz, nfz = (long long)nx * ny * (nz + 1);
  const long long ix = ((long long)k * ny + j) * (nx + 1) + i;
  const long long iy = ((long long)k * (ny + 1) + j) * nx + i;
  const long long iz = ((long long)k * ny + j) * nx + i;
  const long long oy = nx, oz = (long long)nx * ny;
  for (int c = 0; c < 10; ++c) {
    const T v = -((FX[c * nfx + ix + 1] - FX[c * nfx + ix]) * g.iw[0][i] + (FY[c * nfy + iy + oy] - FY[c * nfy + iy]) * g.iw[1][j] +
                  (FZ[c * nfz + iz + oz] - FZ[c * nfz + iz]) * g.iw[2][k]);
    if (c < 5) L[c * ncell + e] = (double)v;
    else dL[(c - 5) * ncell + e] = (double)v;
  }
}

// batched Gauss-point flux (test entry hgks_test_gp_flux)
template <typename T, bool PRF>
__global__ void gp_flux_test_kernel(const double* __restrict__ in, double* __restrict__ out, long long n, GasK<T> gas, T dt) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= n) return;
  const double* r = in + 55 * e;
  T Wl[5], Wr[5], dWl[3][5], dWr[3][5], dW0[3][5];
  for (int k = 0; k < 5; ++k) {
    Wl[k] = T(r[k]);
    Wr[k] = T(r[5 + k]);
    for (int i = 0; i < 3; ++i) {
      dWl[i][k] = T(r[10 + 5 * i + k]);
      dWr[i][k] = T(r[25 + 5 * i + k]);
      dW0[i][k] = T(r[40 + 5 * i + k]);
    }
  }
  T F[5], dF[5], tau;
  gp_flux<T, true, PRF>(gas, Wl, Wr, dWl, dWr, dW0, dt, F, dF, tau);
  double* o = out + 11 * e;
  for (int k = 0; k < 5; ++k) {
    o[k] = (double)F[k];
    o[5 + k] = (double)dF[k];
  }
  o[10] = (double)tau;
}

}  // namespace hgks
