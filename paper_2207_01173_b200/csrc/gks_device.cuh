// gks_device.cuh — device-side building blocks of the HGKS S2O4 stage for sm_100a.
//
// Product code (no oracle dependency).  Templated on the working precision T (float/double):
// the paper compiles the whole code in either precision.
//
//   weno5z_cell   WENO5-Z edge values of one cell (readings O-1, O-2)
//   normal_fields six face fields of one line (O-3 slopes, O-6 C and D)
//   gp_flux       BGK time-dependent Gauss-point flux, Eq. (6), linearised by the
//                 closed-form two-window coefficients of Eq. (8)
//
// Differences from the oracle (by design, same mathematics): WENO smoothness indicators shared
// between the two edges of a cell, closed-form 5x5 compatibility inverse (A.4) instead of
// Gaussian elimination, closed-form Gamma / Gamma' time coefficients (cancellation free)
// instead of integrating both windows and solving the 2x2 system, and the three Maxwellians
// (g0, g_l on u>0, g_r on u<0) processed one after another so only one moment table is live.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace hgks {

// ---------------------------------------------------------------------------------------------
// precision-generic math
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ double m_sqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float m_sqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ double m_exp(double x) { return exp(x); }
__device__ __forceinline__ float m_exp(float x) { return expf(x); }
__device__ __forceinline__ double m_erfc(double x) { return erfc(x); }
__device__ __forceinline__ float m_erfc(float x) { return erfcf(x); }
__device__ __forceinline__ double m_pow(double x, double y) { return pow(x, y); }
__device__ __forceinline__ float m_pow(float x, float y) { return powf(x, y); }
__device__ __forceinline__ double m_abs(double x) { return fabs(x); }
__device__ __forceinline__ float m_abs(float x) { return fabsf(x); }

template <typename T>
struct GasK {
  T K;       // internal degrees of freedom, computed in fp64 on the host (O-20)
  T gamma;
  T mu_ref, T_ref, omega;
  int mu_law;  // 0 const, 1 power law
};

// ---------------------------------------------------------------------------------------------
// WENO5-Z (Borges et al.; O-1): linear weights (1/10, 6/10, 3/10), tau5 = |beta0 - beta2|,
// alpha_k = d_k (1 + (tau5/(beta_k + eps))^2), eps = 1e-16.  Both edges of the middle cell of
// s[0..4] = Qbar_{i-2..i+2}; the left edge is the mirror image, which reuses the same betas.
// ---------------------------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void weno5z_cell(T s0, T s1, T s2, T s3, T s4, T& left, T& right) {
  const T eps = T(1e-16);
  const T c13 = T(13.0 / 12.0);
  T d0 = s0 - T(2) * s1 + s2, e0 = s0 - T(4) * s1 + T(3) * s2;
  T d1 = s1 - T(2) * s2 + s3, e1 = s1 - s3;
  T d2 = s2 - T(2) * s3 + s4, e2 = T(3) * s2 - T(4) * s3 + s4;
  T b0 = c13 * d0 * d0 + T(0.25) * e0 * e0;
  T b1 = c13 * d1 * d1 + T(0.25) * e1 * e1;
  T b2 = c13 * d2 * d2 + T(0.25) * e2 * e2;
  T t5 = m_abs(b0 - b2);
  T r0 = t5 / (b0 + eps), r1 = t5 / (b1 + eps), r2 = t5 / (b2 + eps);
  T q0 = T(1) + r0 * r0, q1 = T(1) + r1 * r1, q2 = T(1) + r2 * r2;
  const T sixth = T(1.0 / 6.0);
  {  // right edge x_{i+1/2}
    T a0 = T(0.1) * q0, a1 = T(0.6) * q1, a2 = T(0.3) * q2;
    T p0 = (T(2) * s0 - T(7) * s1 + T(11) * s2) * sixth;
    T p1 = (-s1 + T(5) * s2 + T(2) * s3) * sixth;
    T p2 = (T(2) * s2 + T(5) * s3 - s4) * sixth;
    right = (a0 * p0 + a1 * p1 + a2 * p2) / (a0 + a1 + a2);
  }
  {  // left edge x_{i-1/2}: stencil reversed, beta0 <-> beta2
    T a0 = T(0.1) * q2, a1 = T(0.6) * q1, a2 = T(0.3) * q0;
    T p0 = (T(2) * s4 - T(7) * s3 + T(11) * s2) * sixth;
    T p1 = (-s3 + T(5) * s2 + T(2) * s1) * sixth;
    T p2 = (T(2) * s2 + T(5) * s1 - s0) * sixth;
    left = (a0 * p0 + a1 * p1 + a2 * p2) / (a0 + a1 + a2);
  }
}

// Six face fields of the face between cells i and i+1 from s[0..5] = Qbar_{i-2..i+3}:
//   f[0] = Q^l (right edge of cell i), f[1] = Q^r (left edge of cell i+1),
//   f[2] = dQ^l/dn, f[3] = dQ^r/dn (in-cell parabola through both edges and the mean, O-3),
//   f[4] = C (4-point face value, O-6), f[5] = D (4-point face derivative, O-6).
template <typename T>
__device__ __forceinline__ void normal_fields(const T (&s)[6], T inv_h, T (&f)[6]) {
  T Ai, Bi, Aj, Bj;
  weno5z_cell(s[0], s[1], s[2], s[3], s[4], Ai, Bi);
  weno5z_cell(s[1], s[2], s[3], s[4], s[5], Aj, Bj);
  f[0] = Bi;
  f[1] = Aj;
  f[2] = (T(2) * Ai + T(4) * Bi - T(6) * s[2]) * inv_h;
  f[3] = (T(-4) * Aj - T(2) * Bj + T(6) * s[3]) * inv_h;
  f[4] = (-s[1] + T(7) * s[2] + T(7) * s[3] - s[4]) * T(1.0 / 12.0);
  f[5] = (s[1] - T(15) * s[2] + T(15) * s[3] - s[4]) * (T(1.0 / 12.0) * inv_h);
}

// Tangential weights of the linear degree-4 reconstruction (O-4) at the 2-point Gauss abscissae
// -+sqrt(3)/6 (O-8), from the 5 face-averaged values j-2..j+2 (sympy-derived):
// value weights WV[m][r], derivative weights WD[m][r] (per unit cell width).
#define HGKS_S3 1.7320508075688772935274463415059
__device__ __constant__ static const double kWV[2][5] = {
    {-7.0 * HGKS_S3 / 432.0 - 1.0 / 4320.0, 1.0 / 1080.0 + 25.0 * HGKS_S3 / 216.0, 719.0 / 720.0,
     1.0 / 1080.0 - 25.0 * HGKS_S3 / 216.0, -1.0 / 4320.0 + 7.0 * HGKS_S3 / 432.0},
    {-1.0 / 4320.0 + 7.0 * HGKS_S3 / 432.0, 1.0 / 1080.0 - 25.0 * HGKS_S3 / 216.0, 719.0 / 720.0,
     1.0 / 1080.0 + 25.0 * HGKS_S3 / 216.0, -7.0 * HGKS_S3 / 432.0 - 1.0 / 4320.0}};
__device__ __constant__ static const double kWD[2][5] = {
    {HGKS_S3 / 54.0 + 1.0 / 12.0, -2.0 / 3.0 - 13.0 * HGKS_S3 / 54.0, 4.0 * HGKS_S3 / 9.0,
     2.0 / 3.0 - 13.0 * HGKS_S3 / 54.0, -1.0 / 12.0 + HGKS_S3 / 54.0},
    {1.0 / 12.0 - HGKS_S3 / 54.0, -2.0 / 3.0 + 13.0 * HGKS_S3 / 54.0, -4.0 * HGKS_S3 / 9.0,
     2.0 / 3.0 + 13.0 * HGKS_S3 / 54.0, -1.0 / 12.0 - HGKS_S3 / 54.0}};

// ---------------------------------------------------------------------------------------------
// Kinetic part.  Moments <u^a v^b w^c (alpha.psi) psi> of one Maxwellian, with
// psi = (1, u, v, w, (u^2+v^2+w^2+xi^2)/2).  Tables: u[0..6], v[0..5], w[0..5],
// x1 = <xi^2>, x2 = <xi^4>.  All indices are compile-time so the tables stay in registers.
// ---------------------------------------------------------------------------------------------
template <typename T>
struct Tab {
  T u[7], v[6], w[6];
  T x1, x2;
};

template <int N, typename T>
__device__ __forceinline__ void recur(T* m, T U, T th) {  // m[n+2] = U m[n+1] + (n+1) th m[n]
#pragma unroll
  for (int n = 0; n + 2 < N; ++n) m[n + 2] = U * m[n + 1] + T(n + 1) * th * m[n];
}

// S(a,b,c) = <u^a v^b w^c (alpha.psi)>
template <int a, int b, int c, typename T>
__device__ __forceinline__ T S_(const Tab<T>& t, const T (&al)[5]) {
  const T uvw = t.u[a] * t.v[b] * t.w[c];
  return al[0] * uvw + al[1] * (t.u[a + 1] * t.v[b] * t.w[c]) + al[2] * (t.u[a] * t.v[b + 1] * t.w[c]) +
         al[3] * (t.u[a] * t.v[b] * t.w[c + 1]) +
         T(0.5) * al[4] *
             (t.u[a + 2] * t.v[b] * t.w[c] + t.u[a] * t.v[b + 2] * t.w[c] + t.u[a] * t.v[b] * t.w[c + 2] +
              uvw * t.x1);
}
// Sx(a,b,c) = <u^a v^b w^c xi^2 (alpha.psi)>
template <int a, int b, int c, typename T>
__device__ __forceinline__ T Sx_(const Tab<T>& t, const T (&al)[5]) {
  const T uvw = t.u[a] * t.v[b] * t.w[c];
  return t.x1 * (al[0] * uvw + al[1] * (t.u[a + 1] * t.v[b] * t.w[c]) + al[2] * (t.u[a] * t.v[b + 1] * t.w[c]) +
                 al[3] * (t.u[a] * t.v[b] * t.w[c + 1]) +
                 T(0.5) * al[4] * (t.u[a + 2] * t.v[b] * t.w[c] + t.u[a] * t.v[b + 2] * t.w[c] + t.u[a] * t.v[b] * t.w[c + 2])) +
         T(0.5) * al[4] * uvw * t.x2;
}
// out += <u^a v^b w^c (alpha.psi) psi>
template <int a, int b, int c, typename T>
__device__ __forceinline__ void polypsi_acc(const Tab<T>& t, const T (&al)[5], T (&out)[5]) {
  out[0] += S_<a, b, c>(t, al);
  out[1] += S_<a + 1, b, c>(t, al);
  out[2] += S_<a, b + 1, c>(t, al);
  out[3] += S_<a, b, c + 1>(t, al);
  out[4] += T(0.5) * (S_<a + 2, b, c>(t, al) + S_<a, b + 2, c>(t, al) + S_<a, b, c + 2>(t, al) + Sx_<a, b, c>(t, al));
}

// Closed-form inverse of the compatibility matrix: solves <(a.psi) psi> = b for
// the Maxwellian (U, V, W, lambda).  Sq = U^2+V^2+W^2+(K+3)/(2 lambda), tl = 2 lambda,
// c5 = 4 lambda^2/(K+3).
template <typename T>
__device__ __forceinline__ void minv(T U, T V, T W, T Sq, T tl, T c5, const T (&b)[5], T (&a)[5]) {
  T R4 = T(2) * b[4] - Sq * b[0];
  T R1 = b[1] - U * b[0], R2 = b[2] - V * b[0], R3 = b[3] - W * b[0];
  a[4] = c5 * (R4 - T(2) * (U * R1 + V * R2 + W * R3));
  a[3] = tl * R3 - W * a[4];
  a[2] = tl * R2 - V * a[4];
  a[1] = tl * R1 - U * a[4];
  a[0] = b[0] - U * a[1] - V * a[2] - W * a[3] - T(0.5) * a[4] * Sq;
}

// Contribution of one Maxwellian g (density rho, velocity U,V,W, lambda) with conservative
// derivatives dW[i] (i: normal, t1, t2) to the flux:
//   F  += rho (Ga Z + Gb X + Gc Y),   dF += rho (Gpa Z + Gpb X + Gpc Y)
// with Z = <u psi>, X = <u^2 a1.psi psi> + <u v a2.psi psi> + <u w a3.psi psi>, Y = <u A.psi psi>
// over the u-range WHICH (0: full, +1: u>0, -1: u<0) — the g0 terms (Ga..Gc = Gamma_1..3) and
// the g_l / g_r terms (Gamma_4..6) of Eq. (6).  Slopes a_i from <a_i> = dW_i/rho (O-7) and A from
// <u a1.psi + v a2.psi + w a3.psi + A.psi> = 0 on the FULL space.
// h0, h1: half-space <u^0>, <u^1> of this Maxwellian (unused when WHICH == 0).
template <typename T, int WHICH, bool NEED_F>
__device__ __forceinline__ void maxwellian_contrib(T K, T rho, T U, T V, T W, T lam, const T (&dW)[3][5],
                                                   T h0, T h1, T Ga, T Gb, T Gc, T Gpa, T Gpb, T Gpc,
                                                   T (&F)[5], T (&dF)[5]) {
  Tab<T> t;
  const T th = T(0.5) / lam;  // 1/(2 lambda)
  t.u[0] = T(1); t.u[1] = U; recur<7>(t.u, U, th);
  t.v[0] = T(1); t.v[1] = V; recur<6>(t.v, V, th);
  t.w[0] = T(1); t.w[1] = W; recur<6>(t.w, W, th);
  t.x1 = K * th;
  t.x2 = K * (K + T(2)) * th * th;
  const T Sq = U * U + V * V + W * W + (K + T(3)) * th;
  const T tl = T(2) * lam;
  const T c5 = T(4) * lam * lam / (K + T(3));
  const T irho = T(1) / rho;

  T a[3][5];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    T b[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) b[k] = dW[i][k] * irho;
    minv(U, V, W, Sq, tl, c5, b, a[i]);
  }
  T A[5];
  {
    T R[5] = {T(0), T(0), T(0), T(0), T(0)};
    polypsi_acc<1, 0, 0>(t, a[0], R);
    polypsi_acc<0, 1, 0>(t, a[1], R);
    polypsi_acc<0, 0, 1>(t, a[2], R);
#pragma unroll
    for (int k = 0; k < 5; ++k) R[k] = -R[k];
    minv(U, V, W, Sq, tl, c5, R, A);
  }
  if (WHICH != 0) {  // switch the u-table to the half space
    t.u[0] = h0;
    t.u[1] = h1;
    recur<7>(t.u, U, th);
  }
  T X[5] = {T(0), T(0), T(0), T(0), T(0)};
  polypsi_acc<2, 0, 0>(t, a[0], X);
  polypsi_acc<1, 1, 0>(t, a[1], X);
  polypsi_acc<1, 0, 1>(t, a[2], X);
  T Y[5] = {T(0), T(0), T(0), T(0), T(0)};
  polypsi_acc<1, 0, 0>(t, A, Y);
  T Z[5];
  Z[0] = t.u[1];
  Z[1] = t.u[2];
  Z[2] = t.u[1] * t.v[1];
  Z[3] = t.u[1] * t.w[1];
  Z[4] = T(0.5) * (t.u[3] + t.u[1] * (t.v[2] + t.w[2] + t.x1));
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    if (NEED_F) F[k] += rho * (Ga * Z[k] + Gb * X[k] + Gc * Y[k]);
    dF[k] += rho * (Gpa * Z[k] + Gpb * X[k] + Gpc * Y[k]);
  }
}

// Gauss-point flux in the local frame (u along the face normal).  Inputs as in the oracle:
// Wl, Wr conservative states; dWl/dWr/dW0 [i][k] derivatives along (normal, t1, t2).
// Returns F^n (if NEED_F) and d_t F^n, and tau.  Invalid input propagates as NaN.
template <typename T, bool NEED_F>
__device__ __forceinline__ void gp_flux(const GasK<T>& g, const T (&Wl)[5], const T (&Wr)[5],
                                        const T (&dWl)[3][5], const T (&dWr)[3][5], const T (&dW0)[3][5],
                                        T dt, T (&F)[5], T (&dF)[5], T& tau) {
  const T K = g.K;
  const T isqpi = T(0.56418958354775628694807945156077);  // 1/sqrt(pi)
  // left / right Maxwellians (A.1)
  T rl = Wl[0], irl = T(1) / rl;
  T Ul = Wl[1] * irl, Vl = Wl[2] * irl, Wl3 = Wl[3] * irl;
  T laml = (K + T(3)) * rl / (T(4) * (Wl[4] - T(0.5) * rl * (Ul * Ul + Vl * Vl + Wl3 * Wl3)));
  T rr = Wr[0], irr = T(1) / rr;
  T Ur = Wr[1] * irr, Vr = Wr[2] * irr, Wr3 = Wr[3] * irr;
  T lamr = (K + T(3)) * rr / (T(4) * (Wr[4] - T(0.5) * rr * (Ur * Ur + Vr * Vr + Wr3 * Wr3)));
  // half-space seeds (A.2): <u^0>_{>0}, <u^1>_{>0} of g_l; <u^0>_{<0}, <u^1>_{<0} of g_r
  T sl = m_sqrt(laml), sr = m_sqrt(lamr);
  T hl0 = T(0.5) * m_erfc(-sl * Ul);
  T hl1 = Ul * hl0 + T(0.5) * isqpi * m_exp(-laml * Ul * Ul) / sl;
  T hr0 = T(0.5) * m_erfc(sr * Ur);
  T hr1 = Ur * hr0 - T(0.5) * isqpi * m_exp(-lamr * Ur * Ur) / sr;
  // Q0 = int_{u>0} psi g_l + int_{u<0} psi g_r
  T thl = T(0.5) / laml, thr = T(0.5) / lamr;
  T hl2 = Ul * hl1 + thl * hl0, hr2 = Ur * hr1 + thr * hr0;
  T Q0[5];
  Q0[0] = rl * hl0 + rr * hr0;
  Q0[1] = rl * hl1 + rr * hr1;
  Q0[2] = rl * hl0 * Vl + rr * hr0 * Vr;
  Q0[3] = rl * hl0 * Wl3 + rr * hr0 * Wr3;
  Q0[4] = T(0.5) * (rl * (hl2 + hl0 * (Vl * Vl + Wl3 * Wl3 + (K + T(2)) * thl)) +
                    rr * (hr2 + hr0 * (Vr * Vr + Wr3 * Wr3 + (K + T(2)) * thr)));
  T r0 = Q0[0], ir0 = T(1) / r0;
  T U0 = Q0[1] * ir0, V0 = Q0[2] * ir0, W0 = Q0[3] * ir0;
  T lam0 = (K + T(3)) * r0 / (T(4) * (Q0[4] - T(0.5) * r0 * (U0 * U0 + V0 * V0 + W0 * W0)));
  // tau = mu/p0 (O-9)
  T T0 = T(0.5) / lam0;
  T p0 = r0 * T0;
  T mu = (g.mu_law == 1) ? g.mu_ref * m_pow(T0 / g.T_ref, g.omega) : g.mu_ref;
  tau = mu / p0;
  // closed-form time coefficients, h = exp(-dt/(2 tau)); tau = 0 -> h = 0 (O-10)
  T h = m_exp(-dt / (T(2) * tau));
  T om = T(1) - h, idt = T(1) / dt;
  T c13 = om * (T(3) - h) * idt;
  T tt = tau * tau;
  T G1 = T(1) - tau * c13;
  T G2 = -tau * (T(1) + T(2) * h - h * h) + T(2) * tt * c13;
  T G3 = -tau + tt * c13;
  T G4 = tau * c13;
  T G5 = tau * h * (T(2) - h) - T(2) * tt * c13;
  T G6 = -tt * c13;
  T idt2 = idt * idt;
  T Gp1 = T(4) * tau * om * om * idt2;
  T Gp2 = T(4) * tau * om * (dt * h - T(2) * tau * om) * idt2;
  T Gp3 = T(1) - T(4) * tt * om * om * idt2;
  T Gp4 = -Gp1, Gp5 = -Gp2, Gp6 = tau * Gp1;

#pragma unroll
  for (int k = 0; k < 5; ++k) {
    F[k] = T(0);
    dF[k] = T(0);
  }
  maxwellian_contrib<T, 0, NEED_F>(K, r0, U0, V0, W0, lam0, dW0, T(0), T(0), G1, G2, G3, Gp1, Gp2, Gp3, F, dF);
  maxwellian_contrib<T, 1, NEED_F>(K, rl, Ul, Vl, Wl3, laml, dWl, hl0, hl1, G4, G5, G6, Gp4, Gp5, Gp6, F, dF);
  maxwellian_contrib<T, -1, NEED_F>(K, rr, Ur, Vr, Wr3, lamr, dWr, hr0, hr1, G4, G5, G6, Gp4, Gp5, Gp6, F, dF);
}

}  // namespace hgks
