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
#ifndef HGKS_RSQRT_NR
#define HGKS_RSQRT_NR 1
#endif
__host__ __device__ __forceinline__ double m_sqrt(double x) { return sqrt(x); }
__host__ __device__ __forceinline__ float m_sqrt(float x) { return sqrtf(x); }
// 1/sqrt(x) for the normal positive operands of the scheme (2 theta): MUFU seed + two Newton steps, no
// slow-path branch (libdevice rsqrt branches to a special-case path, splitting the Gauss-point code into
// basic blocks the scheduler cannot interleave across).  Host builds use the library.
__host__ __device__ __forceinline__ double m_rsqrt(double x) {
#ifdef __CUDA_ARCH__
  if (HGKS_RSQRT_NR) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x * y, y, 1.0);  // 1 - x y^2
    y = fma(0.5 * y, e, y);
    e = fma(-x * y, y, 1.0);
    return fma(0.5 * y, e, y);
  }
#endif
  return rsqrt(x);
}
__host__ __device__ __forceinline__ float m_rsqrt(float x) { return rsqrtf(x); }
__host__ __device__ __forceinline__ double m_exp(double x) { return exp(x); }
__host__ __device__ __forceinline__ float m_exp(float x) { return expf(x); }
__host__ __device__ __forceinline__ double m_erfc(double x) { return erfc(x); }
#ifndef HGKS_FAST_ERFC
#define HGKS_FAST_ERFC 1
#endif
#ifndef HGKS_ERFC_2CHAIN
#define HGKS_ERFC_2CHAIN 0
#endif
// erfc(x)/2.  For |x| < 0.75 (every low-Mach state: x = sqrt(lambda) U) the Maclaurin series of
// erf (14 terms, truncation < 1e-19; measured max relative error 8e-16 for erfc(-x)/2, 2e-15 for
// erfc(x)/2 at x = 0.75) replaces the general-range libdevice erfc (~145 instructions).
// 64-bit constants live in constant memory on the device: DFMA takes a c[][] operand directly,
// while a 64-bit literal costs two uniform-register moves (UMOV) at every use.
#define HGKS_ERFC_COEFS -5.9477940136376354e-12, 8.35070279514724e-11, -1.0892221037148573e-09, 1.3122532963802806e-08, -1.4503852223150468e-07, 1.4589169000933706e-06, -1.3227513227513228e-05, 0.00010683760683760684, -0.0007575757575757576, 0.004629629629629629, -0.023809523809523808, 0.1, -0.3333333333333333, 1.0
#ifdef __CUDACC__
__constant__ double c_erfc_series[14] = {HGKS_ERFC_COEFS};
#endif
__host__ __device__ __forceinline__ double erfc_series_coef(int i) {
#ifdef __CUDA_ARCH__
  return c_erfc_series[i];
#else
  constexpr double k[14] = {HGKS_ERFC_COEFS};
  return k[i];
#endif
}
__host__ __device__ __forceinline__ double half_erfc(double x) {
  if (HGKS_FAST_ERFC && fabs(x) < 0.75) {
    const double z = x * x;
    double s;
    if (HGKS_ERFC_2CHAIN) {
      // two interleaved Horner chains in w = z^2 (even / odd powers of z), joined by one FMA: dependency
      // depth 8 instead of 13 for one more multiply
      const double w = z * z;
      double a = erfc_series_coef(1), b = erfc_series_coef(0);
#pragma unroll
      for (int i = 1; i < 7; ++i) {
        a = fma(a, w, erfc_series_coef(2 * i + 1));
        b = fma(b, w, erfc_series_coef(2 * i));
      }
      s = fma(b, z, a);
    } else {
      s = erfc_series_coef(0);
#pragma unroll
      for (int i = 1; i < 14; ++i) s = fma(s, z, erfc_series_coef(i));
    }
    return fma(-0.56418958354775628694807945156077 * x, s, 0.5);  // 1/2 - x s / sqrt(pi)
  }
  return 0.5 * erfc(x);
}
// erfc(x)/2 and exp(-x^2) together (the two transcendental factors of the half-space moments t0, t1 of one
// side, A.2).  |x| < 0.75: the erf series above and the Taylor series of e^{-z}, z = x^2 (18 terms,
// truncation < 3e-19 relative at z = 0.5625), each as two Horner chains in w = z^2, so four independent
// dependency chains of depth <= 9 replace the 13-deep erf chain plus libdevice exp; else erfc and exp.
#ifndef HGKS_SERIES_EXP
#define HGKS_SERIES_EXP 2
#endif
#ifndef HGKS_H0_FAST
#define HGKS_H0_FAST 1
#endif
#ifndef HGKS_SERIES_SHORT
#define HGKS_SERIES_SHORT 1
#endif
#ifndef HGKS_LATE_GAMMA
#define HGKS_LATE_GAMMA 1
#endif
#define HGKS_INVFACT 1.0, 1.0, 0.5, 0.16666666666666666, 0.041666666666666664, 0.008333333333333333, 0.001388888888888889, 0.0001984126984126984, 2.48015873015873e-05, 2.7557319223985893e-06, 2.755731922398589e-07, 2.505210838544172e-08, 2.08767569878681e-09, 1.6059043836821613e-10, 1.1470745597729725e-11, 7.647163731819816e-13, 4.779477332387385e-14, 2.8114572543455206e-15
#ifdef __CUDACC__
__constant__ double c_invfact[18] = {HGKS_INVFACT};
#endif
__host__ __device__ __forceinline__ double invfact(int n) {
#ifdef __CUDA_ARCH__
  return c_invfact[n];
#else
  constexpr double k[18] = {HGKS_INVFACT};
  return k[n];
#endif
}
__host__ __device__ __forceinline__ void half_erfc_exp(double x, double& he, double& ex) {
  if (fabs(x) < 0.75) {
    const double z = x * x, w = z * z;
    double a = erfc_series_coef(1), b = erfc_series_coef(0);
    double e = invfact(16), o = invfact(17);  // e^{-z} = E(w) - z O(w), E = sum w^j/(2j)!, O = sum w^j/(2j+1)!
#pragma unroll
    for (int i = 1; i < 7; ++i) {
      a = fma(a, w, erfc_series_coef(2 * i + 1));
      b = fma(b, w, erfc_series_coef(2 * i));
    }
#pragma unroll
    for (int j = 7; j >= 0; --j) {
      e = fma(e, w, invfact(2 * j));
      o = fma(o, w, invfact(2 * j + 1));
    }
    he = fma(-0.56418958354775628694807945156077 * x, fma(b, z, a), 0.5);
    ex = fma(-z, o, e);
    return;
  }
  he = 0.5 * erfc(x);
  ex = exp(-x * x);
}
#ifndef HGKS_FAST_ERFC32
#define HGKS_FAST_ERFC32 1
#endif
// fp32: the same Maclaurin series, its last 10 terms (truncation < 1e-9 at |x| = 0.75, below fp32
// rounding), for |x| < 0.75; erfcf elsewhere
__host__ __device__ __forceinline__ float half_erfc(float x) {
  if (HGKS_FAST_ERFC32 && fabsf(x) < 0.75f) {
    constexpr double k[14] = {HGKS_ERFC_COEFS};
    const float z = x * x;
    float s = (float)k[4];
#pragma unroll
    for (int i = 5; i < 14; ++i) s = fmaf(s, z, (float)k[i]);
    return fmaf(-0.564189583547756f * x, s, 0.5f);
  }
  return 0.5f * erfcf(x);
}
__host__ __device__ __forceinline__ float m_erfc(float x) { return erfcf(x); }
// both sides at once, one branch: with both |x| < 0.75 the eight Horner chains share one basic block, so
// the scheduler interleaves the left and right series (two separate calls leave a branch between them)
__host__ __device__ __forceinline__ void half_erfc_exp2(double xl, double xr, double& hel, double& exl, double& her,
                                                        double& exr) {
#ifdef __CUDA_ARCH__
  // low-Mach tier, warp-uniform: every lane with |x| < 0.25 (z <= 1/16; x = sqrt(lambda) U is < 0.1 on the
  // Ma 0.1 TGV): 9 terms of the erf series (next term < 3e-18 relative) and 10 of the exp series
  // (< 3e-19) instead of 14 and 18
  if (HGKS_SERIES_SHORT && __all_sync(__activemask(), fabs(xl) < 0.25 && fabs(xr) < 0.25)) {
    const double zl = xl * xl, wl = zl * zl, zr = xr * xr, wr = zr * zr;
    // erf: s = A(w) + z B(w), A = b0 + b2 w + b4 w^2 + b6 w^3 + b8 w^4, B = b1 + b3 w + b5 w^2 + b7 w^3,
    // b_k = erfc_series_coef(13 - k)
    double al = erfc_series_coef(5), bl = erfc_series_coef(6), ar = al, br = bl;
#pragma unroll
    for (int j = 3; j >= 0; --j) {
      al = fma(al, wl, erfc_series_coef(13 - 2 * j));
      ar = fma(ar, wr, erfc_series_coef(13 - 2 * j));
      if (j > 0) {
        bl = fma(bl, wl, erfc_series_coef(14 - 2 * j));
        br = fma(br, wr, erfc_series_coef(14 - 2 * j));
      }
    }
    // exp(-z) = E(w) - z O(w), E = sum_{j<=4} w^j/(2j)!, O = sum_{j<=4} w^j/(2j+1)!
    double el = invfact(8), ol = invfact(9), er = el, orr = ol;
#pragma unroll
    for (int j = 3; j >= 0; --j) {
      el = fma(el, wl, invfact(2 * j));
      ol = fma(ol, wl, invfact(2 * j + 1));
      er = fma(er, wr, invfact(2 * j));
      orr = fma(orr, wr, invfact(2 * j + 1));
    }
    hel = fma(-0.56418958354775628694807945156077 * xl, fma(bl, zl, al), 0.5);
    exl = fma(-zl, ol, el);
    her = fma(-0.56418958354775628694807945156077 * xr, fma(br, zr, ar), 0.5);
    exr = fma(-zr, orr, er);
    return;
  }
#endif
  if (fabs(xl) < 0.75 && fabs(xr) < 0.75) {
    const double zl = xl * xl, wl = zl * zl, zr = xr * xr, wr = zr * zr;
    double al = erfc_series_coef(1), bl = erfc_series_coef(0), ar = al, br = bl;
    double el = invfact(16), ol = invfact(17), er = el, orr = ol;
#pragma unroll
    for (int i = 1; i < 7; ++i) {
      al = fma(al, wl, erfc_series_coef(2 * i + 1));
      bl = fma(bl, wl, erfc_series_coef(2 * i));
      ar = fma(ar, wr, erfc_series_coef(2 * i + 1));
      br = fma(br, wr, erfc_series_coef(2 * i));
    }
#pragma unroll
    for (int j = 7; j >= 0; --j) {
      el = fma(el, wl, invfact(2 * j));
      ol = fma(ol, wl, invfact(2 * j + 1));
      er = fma(er, wr, invfact(2 * j));
      orr = fma(orr, wr, invfact(2 * j + 1));
    }
    hel = fma(-0.56418958354775628694807945156077 * xl, fma(bl, zl, al), 0.5);
    exl = fma(-zl, ol, el);
    her = fma(-0.56418958354775628694807945156077 * xr, fma(br, zr, ar), 0.5);
    exr = fma(-zr, orr, er);
    return;
  }
  half_erfc_exp(xl, hel, exl);
  half_erfc_exp(xr, her, exr);
}
__host__ __device__ __forceinline__ void half_erfc_exp(float x, float& he, float& ex) {
  he = half_erfc(x);
  ex = expf(-x * x);
}
__host__ __device__ __forceinline__ double m_pow(double x, double y) { return pow(x, y); }
__host__ __device__ __forceinline__ float m_pow(float x, float y) { return powf(x, y); }
__host__ __device__ __forceinline__ double m_abs(double x) { return fabs(x); }
__host__ __device__ __forceinline__ float m_abs(float x) { return fabsf(x); }

// Reciprocal / quotient without the IEEE slow path: MUFU seed (rcp.approx) refined by Newton steps
// (two for fp64: 23 -> 46 -> full 53 bits; the residual-corrected quotient is within 1 ulp of the
// IEEE result for the normal-range operands the scheme produces).  Host builds use plain division.
__host__ __device__ __forceinline__ double rcp(double x) {
#ifdef __CUDA_ARCH__
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
#else
  return 1.0 / x;
#endif
}
__host__ __device__ __forceinline__ float rcp(float x) {
#ifdef __CUDA_ARCH__
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return fmaf(y, fmaf(-x, y, 1.0f), y);
#else
  return 1.0f / x;
#endif
}
template <typename T>
__host__ __device__ __forceinline__ T qdiv(T a, T b) {  // a / b, residual-corrected
  const T y = rcp(b);
  const T q = a * y;
  return q + y * (a - b * q);
}

template <typename T>
struct GasK {
  T K;       // internal degrees of freedom, computed in fp64 on the host (O-20)
  T gamma;
  T mu_ref, T_ref, omega;
  int mu_law;  // 0 const, 1 power law
  T prf;       // 1/Pr - 1 (heat-flux fix, O-12; used by GpFlux<.., PRF = true>)
  T ik3;       // 1/(K+3), host-computed
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
  const T d0 = s0 - T(2) * s1 + s2, e0 = s0 - T(4) * s1 + T(3) * s2;
  const T d1 = s1 - T(2) * s2 + s3, e1 = s1 - s3;
  const T d2 = s2 - T(2) * s3 + s4, e2 = T(3) * s2 - T(4) * s3 + s4;
  const T D0 = c13 * d0 * d0 + T(0.25) * e0 * e0 + eps;  // beta_k + eps
  const T D1 = c13 * d1 * d1 + T(0.25) * e1 * e1 + eps;
  const T D2 = c13 * d2 * d2 + T(0.25) * e2 * e2 + eps;
  const T t5 = m_abs(D0 - D2);
  const T sixth = T(1.0 / 6.0);
  const T p0 = (T(2) * s0 - T(7) * s1 + T(11) * s2) * sixth;  // right-edge candidates
  const T p1 = (-s1 + T(5) * s2 + T(2) * s3) * sixth;
  const T p2 = (T(2) * s2 + T(5) * s3 - s4) * sixth;
  const T m0 = (T(2) * s4 - T(7) * s3 + T(11) * s2) * sixth;  // left-edge candidates (mirror)
  const T m1 = (-s3 + T(5) * s2 + T(2) * s1) * sixth;
  const T m2 = (T(2) * s2 + T(5) * s1 - s0) * sixth;
  if (sizeof(T) == 8) {
    // alpha_k = d_k (1 + (tau5/D_k)^2) = d_k (D_k^2 + tau5^2)/D_k^2: scale every alpha by
    // D0^2 D1^2 D2^2 (in fp64 range: 1e-96 <= product <= 1e18) so each edge needs one quotient
    const T D0s = D0 * D0, D1s = D1 * D1, D2s = D2 * D2, ts = t5 * t5;
    const T n0 = (D0s + ts) * (D1s * D2s), n1 = (D1s + ts) * (D0s * D2s), n2 = (D2s + ts) * (D0s * D1s);
    const T a0 = T(0.1) * n0, a1 = T(0.6) * n1, a2 = T(0.3) * n2;   // right edge weights (1,6,3)/10
    right = qdiv(a0 * p0 + a1 * p1 + a2 * p2, a0 + a1 + a2);
    const T b0 = T(0.1) * n2, b1 = T(0.6) * n1, b2 = T(0.3) * n0;   // left edge: beta0 <-> beta2
    left = qdiv(b0 * m0 + b1 * m1 + b2 * m2, b0 + b1 + b2);
  } else {
    const T r0 = t5 * rcp(D0), r1 = t5 * rcp(D1), r2 = t5 * rcp(D2);
    const T q0 = T(1) + r0 * r0, q1 = T(1) + r1 * r1, q2 = T(1) + r2 * r2;
    const T a0 = T(0.1) * q0, a1 = T(0.6) * q1, a2 = T(0.3) * q2;
    right = qdiv(a0 * p0 + a1 * p1 + a2 * p2, a0 + a1 + a2);
    const T b0 = T(0.1) * q2, b1 = T(0.6) * q1, b2 = T(0.3) * q0;
    left = qdiv(b0 * m0 + b1 * m1 + b2 * m2, b0 + b1 + b2);
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
// point -sqrt(3)/6 (m = 0); the point +sqrt(3)/6 uses the mirror image (see the kernels)
__host__ __device__ constexpr double kWV0(int r) {
  return r == 0 ? -7.0 * HGKS_S3 / 432.0 - 1.0 / 4320.0
       : r == 1 ? 1.0 / 1080.0 + 25.0 * HGKS_S3 / 216.0
       : r == 2 ? 719.0 / 720.0
       : r == 3 ? 1.0 / 1080.0 - 25.0 * HGKS_S3 / 216.0
                : -1.0 / 4320.0 + 7.0 * HGKS_S3 / 432.0;
}
__host__ __device__ constexpr double kWD0(int r) {
  return r == 0 ? HGKS_S3 / 54.0 + 1.0 / 12.0
       : r == 1 ? -2.0 / 3.0 - 13.0 * HGKS_S3 / 54.0
       : r == 2 ? 4.0 * HGKS_S3 / 9.0
       : r == 3 ? 2.0 / 3.0 - 13.0 * HGKS_S3 / 54.0
                : -1.0 / 12.0 + HGKS_S3 / 54.0;
}

// the quartic Gauss-point weights as device operands: constant memory for fp64 (see c_erfc_series),
// 32-bit literals for fp32
#ifdef __CUDACC__
__constant__ double c_wv0[5] = {kWV0(0), kWV0(1), kWV0(2), kWV0(3), kWV0(4)};
__constant__ double c_wd0[5] = {kWD0(0), kWD0(1), kWD0(2), kWD0(3), kWD0(4)};
template <class T>
__device__ __forceinline__ T wv0(int r) { return T(kWV0(r)); }
template <class T>
__device__ __forceinline__ T wd0(int r) { return T(kWD0(r)); }
template <>
__device__ __forceinline__ double wv0<double>(int r) { return c_wv0[r]; }
template <>
__device__ __forceinline__ double wd0<double>(int r) { return c_wd0[r]; }
#endif

// ---------------------------------------------------------------------------------------------
// Kinetic part (A4-A6).  Every Maxwellian is handled in a frame moving with it, where its
// velocity moments are those of an isotropic Gaussian (odd moments vanish), so each moment
// vector <u^a v^b w^c (alpha.psi) psi> collapses to a handful of terms; results are
// mapped back with the Galilean shift of psi = (1, u, v, w, (|u|^2 + xi^2)/2):
//   psi_lab = T(s) psi_frame,   T(s) x = (x1, x2 + s_u x1, x3 + s_v x1, x4 + s_w x1,
//                                          x5 + s.x_{2..4} + |s|^2 x1 / 2).
// theta = 1/(2 lambda) is the temperature; <c^2> = theta, <c^4> = 3 theta^2, <xi^2> = K theta,
// <xi^4> = K(K+2) theta^2.  g0 uses the fully co-moving frame; g_l / g_r (half spaces in u) use
// the frame moving with their tangential velocity only, with the half-space u-moments t_n.
// Identities used (derived in DESIGN.md "Kinetic algebra"; every one is exercised by the parity
// tests against the oracle's generic moment code):
//   compatibility inverse (isotropic):  a2..4 = b2..4/theta,  a5 = 2(b5 - (K+3)theta b1/2)/((K+3)theta^2),
//                                      a1 = b1 - (K+3)theta a5/2
//   Q_i(a) = <c_i (a.psi) psi> = theta a_{i+1} e_1 + theta(a1 + (K+5)theta a5/2) e_{i+1}
//            + (K+5)theta^2 a_{i+1}/2 e_5
// ---------------------------------------------------------------------------------------------
#define HD __host__ __device__ __forceinline__

// x <- T(su, sv, sw) x
template <typename T>
HD void shift_vec(T su, T sv, T sw, T (&x)[5]) {
  const T x1 = x[0];
  x[4] += su * x[1] + sv * x[2] + sw * x[3] + T(0.5) * (su * su + sv * sv + sw * sw) * x1;
  x[1] += su * x1;
  x[2] += sv * x1;
  x[3] += sw * x1;
}

// One direction of the compatibility solves of one Maxwellian in its fully co-moving
// frame: from the conservative derivative dW along local axis I, the spatial slope a_I
// (<a_I> = dW_I / rho, O-7) and the contribution s_I b_c + Q_I(a_I) to
// R = sum_i <u_i a_i.psi psi> (frame components), whose negative is M A.  Everything here is
// linear in dW, so the 1/rho of O-7 is left out: the slopes come out scaled by rho, which is exactly
// the factor rho of every slope term of the flux (callers scale only the Z term by rho).
#ifndef HGKS_CFORM
#define HGKS_CFORM 1
#endif
// HGKS_CFORM ("c-form"): the tangential-velocity slopes a_2..4 = c_2..4 / theta are almost always used
// as theta a_i (R, the P and G moments, H_n's theta t_n terms), so slope_dir<I, true> returns
// a_2..4 scaled by theta (= c_2..4, no multiply by 1/theta) and the callers fold the theta out of
// their moment factors: ~36 fewer FP64 instructions per Gauss point, same values up to rounding.
template <int I, bool CF = false, typename T>
HD void slope_dir(T K, T ik3, T U, T V, T W, T th, T it, const T (&dW)[5], T (&a)[5], T (&R)[5]) {
  const T hK3 = T(0.5) * (K + T(3)) * th;
  const T c5 = T(2) * it * it * ik3;
  const T hK5t = T(0.5) * (K + T(5)) * th;
  const T b1 = dW[0], b2 = dW[1], b3 = dW[2], b4 = dW[3], b5 = dW[4];
  // b_c = T(-s) b
  const T c5v = b5 - U * b2 - V * b3 - W * b4 + T(0.5) * (U * U + V * V + W * W) * b1;
  const T c2 = b2 - U * b1, c3 = b3 - V * b1, c4 = b4 - W * b1;
  const T a5 = c5 * (c5v - hK3 * b1);
  a[0] = b1 - hK3 * a5;
  a[1] = CF ? c2 : c2 * it;
  a[2] = CF ? c3 : c3 * it;
  a[3] = CF ? c4 : c4 * it;
  a[4] = a5;
  const T si = I == 0 ? U : (I == 1 ? V : W);
  const T ci = I == 0 ? c2 : (I == 1 ? c3 : c4);  // theta a_{1+I}
  R[0] += si * b1 + (CF ? ci : th * a[1 + I]);
  R[1] += si * c2;
  R[2] += si * c3;
  R[3] += si * c4;
  R[4] += si * c5v + hK5t * (CF ? ci : th * a[1 + I]);
  R[1 + I] += th * (a[0] + hK5t * a5);
}

// temporal slope A = M^-1 (-R) in the co-moving frame (CF: A_2..4 scaled by theta, i.e. -R_2..4)
template <bool CF = false, typename T>
HD void temporal_slope(T K, T ik3, T th, T it, const T (&R)[5], T (&A)[5]) {
  const T hK3 = T(0.5) * (K + T(3)) * th;
  const T c5 = T(2) * it * it * ik3;
  const T r1 = -R[0];
  A[4] = c5 * (-R[4] - hK3 * r1);
  A[0] = r1 - hK3 * A[4];
  A[1] = CF ? -R[1] : -R[1] * it;
  A[2] = CF ? -R[2] : -R[2] * it;
  A[3] = CF ? -R[3] : -R[3] * it;
}

// Gauss-point flux, Eq. (6), local frame (u = face normal), time-linearised by the
// closed-form two-window coefficients of Eq. (8).  Used in four calls so that the
// caller can supply the derivative inputs lazily, one direction at a time (a callable
// load(i, dW[5]) with i = 0 normal, 1 t1, 2 t2):
//   begin(Wl, Wr, dt)              g_l, g_r, Q0, g0, tau = mu/p0, h
//   add_side<+1>(load_l), add_side<-1>(load_r)   g_l H(u) and g_r (1 - H(u)) terms (Gamma_4..6)
//   add_equilibrium(load_0)        g0 terms of Eq. (6) (Gamma_1..3)
// Results: F (if NEED_F), dF, tau.  Invalid input propagates as NaN.
// MU: viscosity law known at compile time (0 constant, 1 power law) or -1 (GasK::mu_law at run time); a
// compile-time law keeps the uniform branch around pow() out of the Gauss-point code
template <typename T, bool NEED_F, bool PRF = false, int MU = -1>
struct GpFlux {
  T K;
  T rl, irl, Ul, Vl, Wl, thl, hl0, hl1;
  T rr, irr, Ur, Vr, Wr, thr, hr0, hr1;
  T r0, ir0, U0, V0, W0, th0;
  T h, idt, dt, prf, ik3;
#ifndef HGKS_GSHARE
#define HGKS_GSHARE 1
#endif
  // HGKS_GSHARE: the shared factors of the Gamma / Gamma' coefficients, computed once in begin()
  //   tc13 = tau (1-h)(3-h)/dt, ttc13 = tau tc13, hb = tau h (2-h), gp1 = 4 tau (1-h)^2/dt^2,
  //   gp2 = 4 tau (1-h)(dt h - 2 tau (1-h))/dt^2, tgp1 = tau gp1
  T tc13, ttc13, hb, gp1, gp2, tgp1;
  T F[5], dF[5], tau;

  HD void begin(const GasK<T>& g, const T (&WL)[5], const T (&WR)[5], T dt_, T idt_) {
    K = g.K;
    dt = dt_;
    idt = idt_;
    prf = g.prf;
    ik3 = g.ik3;
    const T isqpi = T(0.56418958354775628694807945156077);  // 1/sqrt(pi)
    const T k3 = T(4) * ik3;
    rl = WL[0];
    irl = rcp(rl);
    Ul = WL[1] * irl;
    Vl = WL[2] * irl;
    Wl = WL[3] * irl;
    // theta = 1/(2 lambda) = 2 (rhoE - rho|U|^2/2) / ((K+3) rho)   (A.1)
    thl = T(0.5) * k3 * (WL[4] * irl - T(0.5) * (Ul * Ul + Vl * Vl + Wl * Wl));
    rr = WR[0];
    irr = rcp(rr);
    Ur = WR[1] * irr;
    Vr = WR[2] * irr;
    Wr = WR[3] * irr;
    thr = T(0.5) * k3 * (WR[4] * irr - T(0.5) * (Ur * Ur + Vr * Vr + Wr * Wr));
    // half-space seeds (A.2): sqrt(lambda) = rsqrt(2 theta), 1/sqrt(lambda) = 2 theta rsqrt(2 theta)
    const T sl = m_rsqrt(T(2) * thl), sr = m_rsqrt(T(2) * thr);
    if constexpr (HGKS_SERIES_EXP && sizeof(T) == 8) {
      T el, er;
      if (HGKS_SERIES_EXP == 2) {
        half_erfc_exp2(-sl * Ul, sr * Ur, hl0, el, hr0, er);
      } else {
        half_erfc_exp(-sl * Ul, hl0, el);
        half_erfc_exp(sr * Ur, hr0, er);
      }
      hl1 = Ul * hl0 + isqpi * thl * sl * el;
      hr1 = Ur * hr0 - isqpi * thr * sr * er;
    } else {
      hl0 = half_erfc(-sl * Ul);
      hl1 = Ul * hl0 + isqpi * thl * sl * m_exp(-sl * sl * Ul * Ul);
      hr0 = half_erfc(sr * Ur);
      hr1 = Ur * hr0 - isqpi * thr * sr * m_exp(-sr * sr * Ur * Ur);
    }
    // Q0 = int_{u>0} psi g_l + int_{u<0} psi g_r
    const T hl2 = Ul * hl1 + thl * hl0, hr2 = Ur * hr1 + thr * hr0;
    const T q0 = rl * hl0 + rr * hr0;
    const T q1 = rl * hl1 + rr * hr1;
    const T q2 = rl * hl0 * Vl + rr * hr0 * Vr;
    const T q3 = rl * hl0 * Wl + rr * hr0 * Wr;
    const T q4 = T(0.5) * (rl * (hl2 + hl0 * (Vl * Vl + Wl * Wl + (K + T(2)) * thl)) +
                           rr * (hr2 + hr0 * (Vr * Vr + Wr * Wr + (K + T(2)) * thr)));
    r0 = q0;
    ir0 = rcp(r0);
    U0 = q1 * ir0;
    V0 = q2 * ir0;
    W0 = q3 * ir0;
    th0 = T(0.5) * k3 * (q4 * ir0 - T(0.5) * (U0 * U0 + V0 * V0 + W0 * W0));
    // tau = mu(T0)/p0 with T0 = theta0, p0 = rho0 theta0 (O-9)
    T mu;
    if constexpr (MU == 0) {
      mu = g.mu_ref;
    } else if constexpr (MU == 1) {
      mu = g.mu_ref * m_pow(th0 / g.T_ref, g.omega);
    } else {
      mu = (g.mu_law == 1) ? g.mu_ref * m_pow(th0 / g.T_ref, g.omega) : g.mu_ref;
    }
    tau = qdiv(mu * ir0, th0);
    if (!HGKS_LATE_GAMMA) finish_gamma();
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      F[k] = T(0);
      dF[k] = T(0);
    }
  }

  // h and the shared Gamma / Gamma' factors.  HGKS_LATE_GAMMA: called by add_side<+1> just before its
  // first use, so that the warp-uniform branch of the h exponential does not separate the tau chain of
  // begin() from the slope work of the first side (independent of tau) -- the scheduler can interleave
  // them within one basic block
  HD void finish_gamma() {
    // h = exp(-dt/(2 tau)); tau = 0 -> h = 0 (O-10)
    // (below 1e-20 -- dt/tau > 92, e.g. every low-Mach TGV face -- h changes no Gamma above rounding)
#ifdef __CUDA_ARCH__
    // warp-uniform skip: at low Mach every lane of a warp has dt/tau > 92 (h = 0), and the exp is
    // ~25 FP64 instructions per Gauss point.  HGKS_H0_FAST: the test needs no reciprocal of tau, and with
    // h = 0 the shared factors reduce to c13 = 3/dt, hb = 0, gp1 = 4 tau/dt^2, gp2 = -8 tau^2/dt^2
    const bool need_h = tau > T(0) && (HGKS_H0_FAST ? dt < T(92) * tau : -T(0.5) * dt * rcp(tau) > T(-46));
    const bool any_h = __any_sync(__activemask(), need_h);
    if (HGKS_H0_FAST && HGKS_GSHARE && !any_h) {
      h = T(0);
      const T idt2 = idt * idt;
      tc13 = T(3) * tau * idt;
      ttc13 = tau * tc13;
      hb = T(0);
      gp1 = T(4) * tau * idt2;
      gp2 = -T(8) * tau * tau * idt2;
      tgp1 = tau * gp1;
      return;
    }
    h = T(0);
    if (any_h) h = need_h ? m_exp(-T(0.5) * dt * rcp(tau)) : T(0);
#else
    const T harg = -T(0.5) * dt * rcp(tau);
    const bool need_h = tau > T(0) && harg > T(-46);
    h = need_h ? m_exp(harg) : T(0);
#endif
    if (HGKS_GSHARE) {
      const T om = T(1) - h;
      const T c13 = om * (T(3) - h) * idt;
      const T idt2 = idt * idt;
      tc13 = tau * c13;
      ttc13 = tau * tc13;
      hb = tau * h * (T(2) - h);
      gp1 = T(4) * tau * om * om * idt2;
      gp2 = T(4) * tau * om * (dt * h - T(2) * tau * om) * idt2;
      tgp1 = tau * gp1;
    }
  }

  // closed-form time coefficients: Gamma_1..3 (g0 terms) or Gamma_4..6 (g_l, g_r)
  HD void gammas(bool eq, T& ga, T& gb, T& gc, T& gpa, T& gpb, T& gpc) const {
    if (HGKS_GSHARE) {
      if (eq) {
        ga = T(1) - tc13;
        gb = -tau - hb + T(2) * ttc13;  // -tau (1 + 2h - h^2) + 2 tau^2 c13
        gc = -tau + ttc13;
        gpa = gp1;
        gpb = gp2;
        gpc = T(1) - tgp1;
      } else {
        ga = tc13;
        gb = hb - T(2) * ttc13;
        gc = -ttc13;
        gpa = -gp1;
        gpb = -gp2;
        gpc = tgp1;
      }
      return;
    }
    const T om = T(1) - h;
    const T c13 = om * (T(3) - h) * idt;
    const T tt = tau * tau;
    const T idt2 = idt * idt;
    const T gp1 = T(4) * tau * om * om * idt2;
    const T gp2 = T(4) * tau * om * (dt * h - T(2) * tau * om) * idt2;
    if (eq) {
      ga = T(1) - tau * c13;
      gb = -tau * (T(1) + T(2) * h - h * h) + T(2) * tt * c13;
      gc = -tau + tt * c13;
      gpa = gp1;
      gpb = gp2;
      gpc = T(1) - tau * gp1;
    } else {
      ga = tau * c13;
      gb = tau * h * (T(2) - h) - T(2) * tt * c13;
      gc = -tt * c13;
      gpa = -gp1;
      gpb = -gp2;
      gpc = tau * gp1;
    }
  }

  // F += T(s)(rho ga Z + gb X + gc Y), dF likewise with Gamma' (X, Y already carry rho); FIRST: the
  // first contribution (F, dF still zero) is assigned
  template <bool FIRST = false>
  HD void accumulate(bool eq, T rho, T su, T sv, T sw, const T (&Z)[5], const T (&X)[5], const T (&Y)[5]) {
    T ga, gb, gc, gpa, gpb, gpc;
    gammas(eq, ga, gb, gc, gpa, gpb, gpc);
    const T rpa = rho * gpa;
    T d[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) d[k] = rpa * Z[k] + gpb * X[k] + gpc * Y[k];
    shift_vec(su, sv, sw, d);
#pragma unroll
    for (int k = 0; k < 5; ++k) dF[k] = FIRST ? d[k] : dF[k] + d[k];
    if (NEED_F) {
      const T ra = rho * ga;
      T f[5];
#pragma unroll
      for (int k = 0; k < 5; ++k) f[k] = ra * Z[k] + gb * X[k] + gc * Y[k];
      shift_vec(su, sv, sw, f);
#pragma unroll
      for (int k = 0; k < 5; ++k) F[k] = FIRST ? f[k] : F[k] + f[k];
    }
  }

  // g0 terms: Z = <u psi>, X = sum_i <u u_i a_i.psi psi>, Y = <u A.psi psi> (full space), in the
  // co-moving frame: Z = U0 m0 + theta e2, Y = -U0 R + Q_x(A),
  // X = U0 R + sum_i (s_i Q_x(a_i) + P_xi(a_i)) with P_xi(a) = <c_x c_i (a.psi) psi>.
  template <class Load>
  HD void add_equilibrium(Load&& load) {
    const T th = th0, it = rcp(th0);
    const T hK3 = T(0.5) * (K + T(3)) * th;
    const T hK5t = T(0.5) * (K + T(5)) * th;
    const T t2 = th * th;
    constexpr bool CF = HGKS_CFORM;
    // CF: a_2..4 and A_2..4 come scaled by theta, so theta^2 a_i -> theta a_i, theta a_i -> a_i
    const T t2c = CF ? th : t2, thc = CF ? T(1) : th;
    T R[5] = {T(0), T(0), T(0), T(0), T(0)};
    T X[5] = {T(0), T(0), T(0), T(0), T(0)};
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      T dW[5], a[5];
      load(i, dW);
      if (i == 0) slope_dir<0, CF>(K, ik3, U0, V0, W0, th, it, dW, a, R);
      if (i == 1) slope_dir<1, CF>(K, ik3, U0, V0, W0, th, it, dW, a, R);
      if (i == 2) slope_dir<2, CF>(K, ik3, U0, V0, W0, th, it, dW, a, R);
      const T si = i == 0 ? U0 : (i == 1 ? V0 : W0);
      // s_i Q_x(a)
      X[0] += CF ? si * a[1] : si * th * a[1];
      X[1] += si * th * (a[0] + hK5t * a[4]);
      X[4] += CF ? si * hK5t * a[1] : si * hK5t * th * a[1];
      if (i == 0) {  // P_xx(a)
        X[0] += th * (a[0] + hK5t * a[4]);
        X[1] += T(3) * t2c * a[1];
        X[2] += t2c * a[2];
        X[3] += t2c * a[3];
        X[4] += hK5t * th * (a[0] + T(0.5) * (K + T(7)) * th * a[4]);
      } else if (i == 1) {  // P_xy(a)
        X[1] += t2c * a[2];
        X[2] += t2c * a[1];
      } else {  // P_xz(a)
        X[1] += t2c * a[3];
        X[3] += t2c * a[1];
      }
    }
    T A[5];
    temporal_slope<CF>(K, ik3, th, it, R, A);
    T Y[5];
    Y[0] = -U0 * R[0] + thc * A[1];
    Y[1] = -U0 * R[1] + th * (A[0] + hK5t * A[4]);
    Y[2] = -U0 * R[2];
    Y[3] = -U0 * R[3];
    Y[4] = -U0 * R[4] + hK5t * thc * A[1];
    if (PRF) {  // heat flux relative to U0 (O-12): energy component of <c_x ... psi_c>
      const T qx = X[4], qy = Y[4] + U0 * R[4];  // X[4] before the U0 R shift = X_c[4] - U0 R[4]
      T ga, gb, gc, gpa, gpb, gpc;
      gammas(true, ga, gb, gc, gpa, gpb, gpc);
      dF[4] += prf * (gpb * qx + gpc * qy);
      if (NEED_F) F[4] += prf * (gb * qx + gc * qy);
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) X[k] += U0 * R[k];
    T Z[5] = {U0, th, T(0), T(0), U0 * hK3};
    accumulate(true, r0, U0, V0, W0, Z, X, Y);
  }

  // g_l on u > 0 (SIDE = +1) or g_r on u < 0 (SIDE = -1): half-space u-moments t_n, frame moving
  // with the tangential velocity (V, W) only.
  template <int SIDE, class Load>
  HD void add_side(Load&& load) {
    const T rho = SIDE > 0 ? rl : rr;
    const T U = SIDE > 0 ? Ul : Ur, V = SIDE > 0 ? Vl : Vr, W = SIDE > 0 ? Wl : Wr;
    const T th = SIDE > 0 ? thl : thr, it = rcp(th);
    // half-space u-moments t_0..t_6 (A.2 recursion)
    T t[7];
    t[0] = SIDE > 0 ? hl0 : hr0;
    t[1] = SIDE > 0 ? hl1 : hr1;
#pragma unroll
    for (int n = 0; n + 2 < 7; ++n) t[n + 2] = U * t[n + 1] + T(n + 1) * th * t[n];
    const T k2 = (K + T(2)) * th, k4 = (K + T(4)) * th;
    const T hU2 = T(0.5) * U * U;
    auto e = [&](const T (&al)[5], int n) { return al[0] * t[n] + al[1] * t[n + 1] + T(0.5) * al[4] * (t[n + 2] + k2 * t[n]); };
    auto f = [&](const T (&al)[5], int n) { return al[0] * t[n] + al[1] * t[n + 1] + T(0.5) * al[4] * (t[n + 2] + k4 * t[n]); };
    // out += wgt H_n(al),  H_n(al) = <u^n (al.psi) psi>_t
    auto H = [&](const T (&al)[5], int n, T wgt, T (&out)[5]) {
      out[0] += wgt * e(al, n);
      out[1] += wgt * e(al, n + 1);
      out[2] += wgt * al[2] * th * t[n];
      out[3] += wgt * al[3] * th * t[n];
      out[4] += wgt * T(0.5) * (e(al, n + 2) + k2 * f(al, n));
    };
    // to the tangential frame: alpha_t = T(-U,0,0)^T alpha_c
    auto to_t = [&](T (&al)[5]) {
      al[0] += -U * al[1] + hU2 * al[4];
      al[1] += -U * al[4];
    };
    T R[5] = {T(0), T(0), T(0), T(0), T(0)};
    T X[5] = {T(0), T(0), T(0), T(0), T(0)};
#ifndef HGKS_HFAST
#define HGKS_HFAST 1
#endif
    // fp32 +0.9 %; fp64: 45 fewer FP64 instructions per Gauss point, +1.5 % at 256^3 with the 4 x 8
    // tile (round 1, at 2 blocks per SM with spills, it measured 0.6 % slower).  The Pr-fix variant
    // keeps the generic H (its heat-flux density terms reuse e, f).
#ifndef HGKS_HFAST64
#define HGKS_HFAST64 1
#endif
    constexpr bool kHfast = HGKS_HFAST && !PRF && (sizeof(T) == 4 || HGKS_HFAST64);
    // moment tables of this side: sn[n] = (t_{n+2} + k2 t_n)/2, tth[n] = theta t_n, so that
    //   e(al, n) = al0 t_n + al1 t_{n+1} + al4 sn[n],  f(al, n) = e(al, n) + al4 tth[n]
    // (k4 - k2 = 2 theta) and H_n(al) = (e_n, e_{n+1}, al2 tth_n, al3 tth_n, e_{n+2}/2 + (k2/2) f_n)
    T sn[5], tth[3];
#pragma unroll
    for (int n = 1; n <= 4; ++n) sn[n] = T(0.5) * (t[n + 2] + k2 * t[n]);
    tth[1] = th * t[1];
    tth[2] = th * t[2];
    const T hk2 = T(0.5) * k2;
    // CFS (c-form, HGKS_CFORM): al_2, al_3 of every Hf argument come scaled by theta, so their theta t_n
    // factors are t_n (al_0, al_1, al_4 are the true slopes: to_t needs al_1)
    constexpr bool CFS = HGKS_CFORM && kHfast;
    auto Hf = [&](const T (&al)[5], int n, T (&out)[5]) {  // out += H_n(al), n = 1 or 2
      const T en = al[0] * t[n] + al[1] * t[n + 1] + al[4] * sn[n];
      const T en1 = al[0] * t[n + 1] + al[1] * t[n + 2] + al[4] * sn[n + 1];
      const T en2 = al[0] * t[n + 2] + al[1] * t[n + 3] + al[4] * sn[n + 2];
      const T fn = en + al[4] * tth[n];
      out[0] += en;
      out[1] += en1;
      out[2] += al[2] * (CFS ? t[n] : tth[n]);
      out[3] += al[3] * (CFS ? t[n] : tth[n]);
      out[4] += T(0.5) * en2 + hk2 * fn;
    };
    const T r1 = sn[1] + tth[1];  // (t_3 + k4 t_1)/2
    const T g3 = th * r1;
    T ad[3][5];  // slopes kept for the heat-flux density moments (PRF only; dead otherwise)
    T Bt[5];     // V a_2 + W a_3 (tangential frame): the two n = 1 terms share one H_1 (linear in al)
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      T dW[5], a[5];
      load(i, dW);
      if (i == 0) slope_dir<0, CFS>(K, ik3, U, V, W, th, it, dW, a, R);
      if (i == 1) slope_dir<1, CFS>(K, ik3, U, V, W, th, it, dW, a, R);
      if (i == 2) slope_dir<2, CFS>(K, ik3, U, V, W, th, it, dW, a, R);
      if (CFS) a[1] *= it;
      to_t(a);
      if (PRF) {
#pragma unroll
        for (int k = 0; k < 5; ++k) ad[i][k] = a[k];
      }
      if (kHfast) {
        if (i == 0) {
          Hf(a, 2, X);
        } else {
          const T wt = i == 1 ? V : W;
#pragma unroll
          for (int k = 0; k < 5; ++k) Bt[k] = i == 1 ? wt * a[k] : Bt[k] + wt * a[k];
          const T ai = i == 1 ? a[2] : a[3];  // G_v(a) / G_w(a)
          X[0] += (CFS ? t[1] : tth[1]) * ai;
          X[1] += (CFS ? t[2] : tth[2]) * ai;
          X[1 + i] += th * (a[0] * t[1] + a[1] * t[2] + a[4] * r1);  // theta f(a, 1)
          X[4] += (CFS ? r1 : g3) * ai;
          if (i == 2) Hf(Bt, 1, X);
        }
      } else if (i == 0) {
        H(a, 2, T(1), X);
      } else if (i == 1) {  // V H_1(a) + G_v(a)
        H(a, 1, V, X);
        X[0] += th * t[1] * a[2];
        X[1] += th * t[2] * a[2];
        X[2] += th * f(a, 1);
        X[4] += g3 * a[2];
      } else {  // W H_1(a) + G_w(a)
        H(a, 1, W, X);
        X[0] += th * t[1] * a[3];
        X[1] += th * t[2] * a[3];
        X[3] += th * f(a, 1);
        X[4] += g3 * a[3];
      }
    }
    T A[5];
    temporal_slope<CFS>(K, ik3, th, it, R, A);
    if (CFS) A[1] *= it;
    to_t(A);
    T Y[5] = {T(0), T(0), T(0), T(0), T(0)};
    if (kHfast) Hf(A, 1, Y);
    else H(A, 1, T(1), Y);
    T Z[5] = {t[1], t[2], T(0), T(0), sn[1]};
    if (HGKS_LATE_GAMMA && SIDE > 0) finish_gamma();
    if (PRF) {
      // heat flux relative to U0 (O-12) from the flux vectors (Z, X, Y) and the density vectors
      // (Zd, Xd, Yd) = <psi>, sum_i <u_i a_i.psi psi>, <A.psi psi> of this side, all in its
      // tangential frame; d = U0 - (0, V, W) is the equilibrium velocity seen from that frame
      T Xd[5] = {T(0), T(0), T(0), T(0), T(0)}, Yd[5] = {T(0), T(0), T(0), T(0), T(0)};
      H(A, 0, T(1), Yd);
      H(ad[0], 1, T(1), Xd);
      H(ad[1], 0, V, Xd);
      H(ad[2], 0, W, Xd);
      const T g0 = T(0.5) * th * (t[2] + k4 * t[0]);
      Xd[0] += th * t[0] * (ad[1][2] + ad[2][3]);
      Xd[1] += th * t[1] * (ad[1][2] + ad[2][3]);
      Xd[2] += th * f(ad[1], 0);
      Xd[3] += th * f(ad[2], 0);
      Xd[4] += g0 * (ad[1][2] + ad[2][3]);
      const T Zd[5] = {t[0], t[1], T(0), T(0), T(0.5) * (t[2] + k2 * t[0])};
      const T dx = U0, dy = V0 - V, dz = W0 - W, d2 = T(0.5) * (dx * dx + dy * dy + dz * dz);
      auto heat = [&](T a, T b, T c) {
        T Fv[5], Wv[5];
#pragma unroll
        for (int k = 0; k < 5; ++k) {  // X, Y, Xd, Yd carry rho (slopes scaled by rho)
          Fv[k] = rho * a * Z[k] + b * X[k] + c * Y[k];
          Wv[k] = rho * a * Zd[k] + b * Xd[k] + c * Yd[k];
        }
        return Fv[4] - (dx * Fv[1] + dy * Fv[2] + dz * Fv[3]) + d2 * Fv[0] -
               dx * (Wv[4] - (dx * Wv[1] + dy * Wv[2] + dz * Wv[3]) + d2 * Wv[0]);
      };
      T ga, gb, gc, gpa, gpb, gpc;
      gammas(false, ga, gb, gc, gpa, gpb, gpc);
      dF[4] += prf * heat(gpa, gpb, gpc);
      if (NEED_F) F[4] += prf * heat(ga, gb, gc);
    }
    accumulate<SIDE == 1 && !PRF>(false, rho, T(0), V, W, Z, X, Y);  // g_l side is the first term
  }
};

// One-call form (tests and the batched test entry point).
template <typename T, bool NEED_F, bool PRF = false>
HD void gp_flux(const GasK<T>& g, const T (&Wl)[5], const T (&Wr)[5], const T (&dWl)[3][5], const T (&dWr)[3][5],
                const T (&dW0)[3][5], T dt, T (&F)[5], T (&dF)[5], T& tau) {
  GpFlux<T, NEED_F, PRF> gf;
  gf.begin(g, Wl, Wr, dt, T(1) / dt);
  gf.template add_side<+1>([&](int i, T (&d)[5]) { for (int k = 0; k < 5; ++k) d[k] = dWl[i][k]; });
  gf.template add_side<-1>([&](int i, T (&d)[5]) { for (int k = 0; k < 5; ++k) d[k] = dWr[i][k]; });
  gf.add_equilibrium([&](int i, T (&d)[5]) { for (int k = 0; k < 5; ++k) d[k] = dW0[i][k]; });
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    F[k] = gf.F[k];
    dF[k] = gf.dF[k];
  }
  tau = gf.tau;
}

}  // namespace hgks
