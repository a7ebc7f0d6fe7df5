/*
 * hgks_oracle.c — plain, slow, fp64 CPU oracle of the HGKS S2O4 step (arXiv 2207.01173 §2).
 *
 * TEST INFRASTRUCTURE ONLY (see hgks_oracle.h).  Written from PAPER.md P:185-365 and the
 * readings O-1..O-26 of SURVEY.md §8(c) (restated in DESIGN.md).  It follows the paper's
 * order: reconstruction -> Gauss-point distribution (Eq. 6) -> time integrals over the two
 * windows -> 2x2 linear solve (Eq. 8) -> face quadrature -> L, d_t L -> Eq. (7).
 * Deliberately plain: whole-array passes, every intermediate stored, generic moment
 * function, Gaussian elimination for every compatibility solve, no fusion or reordering.
 *
 * Parity status: every function is pinned by tests/test_oracle_*.py (see the header).
 */
#include "hgks_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* host threading only (bench.py's single-thread / all-core cpu_baseline): n <= 0 restores all cores */
void or_set_num_threads(int n) {
#ifdef _OPENMP
  static int all = 0;
  if (all == 0) all = omp_get_max_threads();
  omp_set_num_threads(n > 0 ? n : all);
#else
  (void)n;
#endif
}

/* ------------------------------------------------------------------------------------------
 * A.1 gas model.  K = (5 - 3 gamma)/(gamma - 1)  (O-20: evaluated in fp64 as written)
 * ---------------------------------------------------------------------------------------- */
double or_K(double gamma) { return (5.0 - 3.0 * gamma) / (gamma - 1.0); }

/* q = (rho, rhoU, rhoV, rhoW, rhoE) -> (rho, U, V, W, lambda), lambda = (K+3) rho / (4 rho e)
 * with rho e = rhoE - rho|U|^2/2 (A.1). */
int or_cons_to_maxw(const double q[5], double K, double mx[5]) {
  double rho = q[0];
  if (!(rho > 0.0) || !isfinite(rho)) return -1;
  double U = q[1] / rho, V = q[2] / rho, W = q[3] / rho;
  double rhoe = q[4] - 0.5 * rho * (U * U + V * V + W * W);
  if (!(rhoe > 0.0) || !isfinite(rhoe)) return -1;
  mx[0] = rho;
  mx[1] = U;
  mx[2] = V;
  mx[3] = W;
  mx[4] = (K + 3.0) * rho / (4.0 * rhoe);
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * A.2 moments of the Maxwellian g = rho (lambda/pi)^{(K+3)/2} exp(-lambda(|u-U|^2 + xi^2)),
 * normalised by rho.  Full space: <u^0> = 1, <u^1> = U, <u^{n+2}> = U <u^{n+1}> + (n+1)/(2 lambda) <u^n>.
 * Half spaces: <u^0>_{>0} = erfc(-sqrt(lambda) U)/2, <u^1>_{>0} = U <u^0>_{>0} + e^{-lambda U^2}/(2 sqrt(pi lambda)),
 * <u^0>_{<0} = erfc(sqrt(lambda) U)/2, <u^1>_{<0} = U <u^0>_{<0} - e^{-lambda U^2}/(2 sqrt(pi lambda)),
 * then the same recursion.  (The paper defers these to [GKS-Xu1/2].)
 * ---------------------------------------------------------------------------------------- */
void or_moments_u(double U, double lam, int which, double m[OR_NM]) {
  if (which == 0) {
    m[0] = 1.0;
    m[1] = U;
  } else {
    double s = (which > 0) ? -1.0 : 1.0;
    double e = exp(-lam * U * U) / (2.0 * sqrt(M_PI * lam));
    m[0] = 0.5 * erfc(s * sqrt(lam) * U);
    m[1] = U * m[0] - s * e;
  }
  for (int n = 0; n + 2 < OR_NM; ++n) m[n + 2] = U * m[n + 1] + (n + 1) / (2.0 * lam) * m[n];
}

/* moment tables of one Maxwellian: u-table (full or half), full v and w tables, xi^0, xi^2, xi^4 */
typedef struct {
  double u[OR_NM], v[OR_NM], w[OR_NM], xi[3];
} or_mom;

static void mom_build(const double mx[5], double K, int which, or_mom* t) {
  or_moments_u(mx[1], mx[4], which, t->u);
  or_moments_u(mx[2], mx[4], 0, t->v);
  or_moments_u(mx[3], mx[4], 0, t->w);
  t->xi[0] = 1.0;                                          /* <xi^0>                      */
  t->xi[1] = K / (2.0 * mx[4]);                            /* <xi^2> = K/(2 lambda)       */
  t->xi[2] = K * (K + 2.0) / (4.0 * mx[4] * mx[4]);        /* <xi^4> = K(K+2)/(4 lambda^2) */
}

/* <u^a v^b w^c xi^{2d}> = <u^a><v^b><w^c><xi^{2d}> (product moments factorise, A.2) */
static double mom_G(const or_mom* t, int a, int b, int c, int d) {
  return t->u[a] * t->v[b] * t->w[c] * t->xi[d];
}

/* <u^a v^b w^c xi^{2d} psi>, psi = (1, u, v, w, (u^2+v^2+w^2+xi^2)/2) */
static void mom_psi(const or_mom* t, int a, int b, int c, int d, double out[5]) {
  out[0] = mom_G(t, a, b, c, d);
  out[1] = mom_G(t, a + 1, b, c, d);
  out[2] = mom_G(t, a, b + 1, c, d);
  out[3] = mom_G(t, a, b, c + 1, d);
  out[4] = 0.5 * (mom_G(t, a + 2, b, c, d) + mom_G(t, a, b + 2, c, d) + mom_G(t, a, b, c + 2, d) +
                  mom_G(t, a, b, c, d + 1));
}

/* <u^a v^b w^c (alpha . psi) psi>, alpha . psi = al1 + al2 u + al3 v + al4 w + al5 (u^2+v^2+w^2+xi^2)/2 */
static void mom_poly_psi(const or_mom* t, int a, int b, int c, const double al[5], double out[5]) {
  double p0[5], pu[5], pv[5], pw[5], puu[5], pvv[5], pww[5], pxx[5];
  mom_psi(t, a, b, c, 0, p0);
  mom_psi(t, a + 1, b, c, 0, pu);
  mom_psi(t, a, b + 1, c, 0, pv);
  mom_psi(t, a, b, c + 1, 0, pw);
  mom_psi(t, a + 2, b, c, 0, puu);
  mom_psi(t, a, b + 2, c, 0, pvv);
  mom_psi(t, a, b, c + 2, 0, pww);
  mom_psi(t, a, b, c, 1, pxx);
  for (int k = 0; k < 5; ++k)
    out[k] = al[0] * p0[k] + al[1] * pu[k] + al[2] * pv[k] + al[3] * pw[k] +
             0.5 * al[4] * (puu[k] + pvv[k] + pww[k] + pxx[k]);
}

void or_psi_moment(double U, double V, double W, double lam, double K, int which, int a, int b,
                   int c, int d, double out[5]) {
  double mx[5] = {1.0, U, V, W, lam};
  or_mom t;
  mom_build(mx, K, which, &t);
  mom_psi(&t, a, b, c, d, out);
}

/* ------------------------------------------------------------------------------------------
 * A.3 compatibility solves: <a_i> = dQ/dx_i / rho (O-7), <a1 u + a2 v + a3 w + A> = 0.
 * The 5x5 system M a = b with M_{kn} = <psi_n psi_k> is assembled column by column from the
 * moment function and solved by Gaussian elimination with partial pivoting.
 * ---------------------------------------------------------------------------------------- */
static int gauss_solve(int n, double* A /* n x n row-major, destroyed */, double* x /* rhs in, sol out */) {
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (fabs(A[r * n + col]) > fabs(A[piv * n + col])) piv = r;
    if (A[piv * n + col] == 0.0) return -1;
    if (piv != col) {
      for (int k = 0; k < n; ++k) {
        double tmp = A[col * n + k];
        A[col * n + k] = A[piv * n + k];
        A[piv * n + k] = tmp;
      }
      double tmp = x[col];
      x[col] = x[piv];
      x[piv] = tmp;
    }
    for (int r = col + 1; r < n; ++r) {
      double f = A[r * n + col] / A[col * n + col];
      for (int k = col; k < n; ++k) A[r * n + k] -= f * A[col * n + k];
      x[r] -= f * x[col];
    }
  }
  for (int r = n - 1; r >= 0; --r) {
    double s = x[r];
    for (int k = r + 1; k < n; ++k) s -= A[r * n + k] * x[k];
    x[r] = s / A[r * n + r];
  }
  return 0;
}

static void mom_matrix(const or_mom* full, double M[25]) {
  for (int n = 0; n < 5; ++n) {
    double e[5] = {0, 0, 0, 0, 0}, col[5];
    e[n] = 1.0;
    mom_poly_psi(full, 0, 0, 0, e, col);
    for (int k = 0; k < 5; ++k) M[k * 5 + n] = col[k];
  }
}

static int solve_with(const or_mom* full, const double b[5], double a[5]) {
  double M[25];
  mom_matrix(full, M);
  for (int k = 0; k < 5; ++k) a[k] = b[k];
  return gauss_solve(5, M, a);
}

int or_slope_solve(const double mx[5], double K, const double b[5], double a[5]) {
  or_mom t;
  mom_build(mx, K, 0, &t);
  return solve_with(&t, b, a);
}

/* spatial slopes a_1..a_3 and temporal slope A of one Maxwellian:
 *   <a_i> = dW_i / rho ;   <u a_1.psi + v a_2.psi + w a_3.psi + A.psi> = 0 (full-space moments) */
static int kinetic_slopes(const or_mom* full, double rho, const double dW[3][5], double a[3][5],
                          double A[5]) {
  for (int i = 0; i < 3; ++i) {
    double b[5];
    for (int k = 0; k < 5; ++k) b[k] = dW[i][k] / rho;
    if (solve_with(full, b, a[i])) return -1;
  }
  double t1[5], t2[5], t3[5], rhs[5];
  mom_poly_psi(full, 1, 0, 0, a[0], t1);
  mom_poly_psi(full, 0, 1, 0, a[1], t2);
  mom_poly_psi(full, 0, 0, 1, a[2], t3);
  for (int k = 0; k < 5; ++k) rhs[k] = -(t1[k] + t2[k] + t3[k]);
  return solve_with(full, rhs, A);
}

/* ------------------------------------------------------------------------------------------
 * A.6 time integrals over [0,T] of the six time functions of Eq. (6), e = exp(-T/tau):
 *   g0:            1 - e^{-t/tau}                 -> gamma1 = T - tau(1-e)
 *   (abar.u) g0:   (t+tau) e^{-t/tau} - tau      -> gamma2 = 2 tau^2 (1-e) - tau T (1+e)
 *   Abar g0:       t - tau + tau e^{-t/tau}      -> gamma3 = T^2/2 - tau T + tau^2 (1-e)
 *   g_{l,r}:       e^{-t/tau}                    -> gamma4 = tau (1-e)
 *   (a.u) g_{l,r}: -(t+tau) e^{-t/tau}           -> gamma5 = tau T e - 2 tau^2 (1-e)
 *   A g_{l,r}:     -tau e^{-t/tau}               -> gamma6 = -tau^2 (1-e)
 * ---------------------------------------------------------------------------------------- */
void or_time_integrals(double T, double tau, double g[6]) {
  double e = exp(-T / tau); /* tau = 0 (Euler, O-10): exp(-inf) = 0 */
  g[0] = T - tau * (1.0 - e);
  g[1] = 2.0 * tau * tau * (1.0 - e) - tau * T * (1.0 + e);
  g[2] = 0.5 * T * T - tau * T + tau * tau * (1.0 - e);
  g[3] = tau * (1.0 - e);
  g[4] = tau * T * e - 2.0 * tau * tau * (1.0 - e);
  g[5] = -tau * tau * (1.0 - e);
}

/* ------------------------------------------------------------------------------------------
 * Axis geometry (P:219-223 uniform; P:945-956 tanh-stretched channel, O-18)
 * ---------------------------------------------------------------------------------------- */
double or_axis_face(const or_grid* gr, int d, int j) {
  if (gr->stretch[d] == 0) return gr->lo[d] + j * gr->dx[d];
  double b = gr->stretch_b[d], s = (double)j / gr->n[d];
  return 0.5 * (gr->lo[d] + gr->hi[d]) + 0.5 * (gr->hi[d] - gr->lo[d]) * tanh(b * (2.0 * s - 1.0)) / tanh(b);
}

/* J = d zeta / dx with zeta the cell-index coordinate (x(zeta) = or_axis_face at integer zeta) */
double or_axis_metric(const or_grid* gr, int d, double zeta) {
  if (gr->stretch[d] == 0) return 1.0 / gr->dx[d];
  double b = gr->stretch_b[d], n = gr->n[d];
  double ch = cosh(b * (2.0 * zeta / n - 1.0));
  double dxdz = 0.5 * (gr->hi[d] - gr->lo[d]) / tanh(b) * b * (2.0 / n) / (ch * ch);
  return 1.0 / dxdz;
}

static double cell_width(const or_grid* gr, int d, int j) {
  if (gr->stretch[d] == 0) return gr->dx[d];
  return or_axis_face(gr, d, j + 1) - or_axis_face(gr, d, j);
}

/* viscosity law (O-9) at temperature T = p/rho */
static double mu_of(const or_gas* g, double T) {
  if (g->mu_law == 1) return g->mu_ref * pow(T / g->T_ref, g->omega);
  return g->mu_ref;
}

/* ------------------------------------------------------------------------------------------
 * Gauss-point flux, Eq. (6), local frame.
 * ---------------------------------------------------------------------------------------- */
int or_gp_flux(const or_gas* g, const double Wl[5], const double dWl[3][5], const double Wr[5],
               const double dWr[3][5], const double dW0[3][5], double dt, double F[5],
               double dF[5], double* tau_out) {
  const double K = g->K;
  double ml[5], mr[5], m0[5];
  if (or_cons_to_maxw(Wl, K, ml) || or_cons_to_maxw(Wr, K, mr)) return -1;

  /* half-space tables of g_l (u>0) and g_r (u<0), full tables of each */
  or_mom tl_pos, tr_neg, tl_full, tr_full, t0;
  mom_build(ml, K, +1, &tl_pos);
  mom_build(mr, K, -1, &tr_neg);
  mom_build(ml, K, 0, &tl_full);
  mom_build(mr, K, 0, &tr_full);

  /* Q0 = int_{u>0} psi g_l + int_{u<0} psi g_r */
  double Q0[5], pl[5], pr[5];
  mom_psi(&tl_pos, 0, 0, 0, 0, pl);
  mom_psi(&tr_neg, 0, 0, 0, 0, pr);
  for (int k = 0; k < 5; ++k) Q0[k] = ml[0] * pl[k] + mr[0] * pr[k];
  if (or_cons_to_maxw(Q0, K, m0)) return -1;
  mom_build(m0, K, 0, &t0);

  /* tau = mu / p with p from Q0 (O-9) */
  double p0 = m0[0] / (2.0 * m0[4]);
  double T0 = 1.0 / (2.0 * m0[4]);
  double tau = mu_of(g, T0) / p0;
  if (tau_out) *tau_out = tau;

  /* slopes */
  double al[3][5], Al[5], ar[3][5], Ar[5], ab[3][5], Ab[5];
  if (kinetic_slopes(&tl_full, ml[0], dWl, al, Al)) return -1;
  if (kinetic_slopes(&tr_full, mr[0], dWr, ar, Ar)) return -1;
  if (kinetic_slopes(&t0, m0[0], dW0, ab, Ab)) return -1;

  /* moment vectors of the six terms of Eq. (6) (A.7); flux = int u psi f dXi */
  double Mk[6][5], tmp[5], t1[5], t2[5], t3[5];
  mom_psi(&t0, 1, 0, 0, 0, tmp);
  for (int k = 0; k < 5; ++k) Mk[0][k] = m0[0] * tmp[k];
  mom_poly_psi(&t0, 2, 0, 0, ab[0], t1);
  mom_poly_psi(&t0, 1, 1, 0, ab[1], t2);
  mom_poly_psi(&t0, 1, 0, 1, ab[2], t3);
  for (int k = 0; k < 5; ++k) Mk[1][k] = m0[0] * (t1[k] + t2[k] + t3[k]);
  mom_poly_psi(&t0, 1, 0, 0, Ab, tmp);
  for (int k = 0; k < 5; ++k) Mk[2][k] = m0[0] * tmp[k];

  double l4[5], r4[5];
  mom_psi(&tl_pos, 1, 0, 0, 0, l4);
  mom_psi(&tr_neg, 1, 0, 0, 0, r4);
  for (int k = 0; k < 5; ++k) Mk[3][k] = ml[0] * l4[k] + mr[0] * r4[k];

  double l5[5], r5[5];
  mom_poly_psi(&tl_pos, 2, 0, 0, al[0], t1);
  mom_poly_psi(&tl_pos, 1, 1, 0, al[1], t2);
  mom_poly_psi(&tl_pos, 1, 0, 1, al[2], t3);
  for (int k = 0; k < 5; ++k) l5[k] = t1[k] + t2[k] + t3[k];
  mom_poly_psi(&tr_neg, 2, 0, 0, ar[0], t1);
  mom_poly_psi(&tr_neg, 1, 1, 0, ar[1], t2);
  mom_poly_psi(&tr_neg, 1, 0, 1, ar[2], t3);
  for (int k = 0; k < 5; ++k) r5[k] = t1[k] + t2[k] + t3[k];
  for (int k = 0; k < 5; ++k) Mk[4][k] = ml[0] * l5[k] + mr[0] * r5[k];

  double l6[5], r6[5];
  mom_poly_psi(&tl_pos, 1, 0, 0, Al, l6);
  mom_poly_psi(&tr_neg, 1, 0, 0, Ar, r6);
  for (int k = 0; k < 5; ++k) Mk[5][k] = ml[0] * l6[k] + mr[0] * r6[k];

  /* integrate over the two windows [0, dt] and [0, dt/2] */
  double gf[6], gh[6];
  or_time_integrals(dt, tau, gf);
  or_time_integrals(0.5 * dt, tau, gh);
  double Ifull[5], Ihalf[5];
  for (int k = 0; k < 5; ++k) {
    Ifull[k] = 0.0;
    Ihalf[k] = 0.0;
    for (int j = 0; j < 6; ++j) {
      Ifull[k] += gf[j] * Mk[j][k];
      Ihalf[k] += gh[j] * Mk[j][k];
    }
  }

  /* Eq. (8): [dt, dt^2/2 ; dt/2, dt^2/8] [F ; dF] = [Ifull ; Ihalf]  (Cramer's rule) */
  double a11 = dt, a12 = 0.5 * dt * dt, a21 = 0.5 * dt, a22 = 0.125 * dt * dt;
  double det = a11 * a22 - a12 * a21;
  for (int k = 0; k < 5; ++k) {
    F[k] = (Ifull[k] * a22 - a12 * Ihalf[k]) / det;
    dF[k] = (a11 * Ihalf[k] - a21 * Ifull[k]) / det;
  }

  /* Pr != 1 (reading O-12): add (1/Pr - 1) q to the energy flux, q the heat flux
   * int (u - U0) (|u - U0|^2 + xi^2)/2 f dXi of the interface distribution of Eq. (6) relative to
   * the interface equilibrium velocity U0, linearised in time like the flux.  With F = int u psi f
   * and Wd = int psi f (density moments of the same six terms):
   *   q = F5 - U0.F_m + |U0|^2 F1/2 - U0 (Wd5 - U0.Wd_m + |U0|^2 Wd1/2). */
  if (g->prandtl != 1.0) {
    double Dk[6][5];
    mom_psi(&t0, 0, 0, 0, 0, tmp);
    for (int k = 0; k < 5; ++k) Dk[0][k] = m0[0] * tmp[k];
    mom_poly_psi(&t0, 1, 0, 0, ab[0], t1);
    mom_poly_psi(&t0, 0, 1, 0, ab[1], t2);
    mom_poly_psi(&t0, 0, 0, 1, ab[2], t3);
    for (int k = 0; k < 5; ++k) Dk[1][k] = m0[0] * (t1[k] + t2[k] + t3[k]);
    mom_poly_psi(&t0, 0, 0, 0, Ab, tmp);
    for (int k = 0; k < 5; ++k) Dk[2][k] = m0[0] * tmp[k];
    for (int k = 0; k < 5; ++k) Dk[3][k] = ml[0] * pl[k] + mr[0] * pr[k];
    double d5l[5], d5r[5];
    mom_poly_psi(&tl_pos, 1, 0, 0, al[0], t1);
    mom_poly_psi(&tl_pos, 0, 1, 0, al[1], t2);
    mom_poly_psi(&tl_pos, 0, 0, 1, al[2], t3);
    for (int k = 0; k < 5; ++k) d5l[k] = t1[k] + t2[k] + t3[k];
    mom_poly_psi(&tr_neg, 1, 0, 0, ar[0], t1);
    mom_poly_psi(&tr_neg, 0, 1, 0, ar[1], t2);
    mom_poly_psi(&tr_neg, 0, 0, 1, ar[2], t3);
    for (int k = 0; k < 5; ++k) d5r[k] = t1[k] + t2[k] + t3[k];
    for (int k = 0; k < 5; ++k) Dk[4][k] = ml[0] * d5l[k] + mr[0] * d5r[k];
    double d6l[5], d6r[5];
    mom_poly_psi(&tl_pos, 0, 0, 0, Al, d6l);
    mom_poly_psi(&tr_neg, 0, 0, 0, Ar, d6r);
    for (int k = 0; k < 5; ++k) Dk[5][k] = ml[0] * d6l[k] + mr[0] * d6r[k];
    double Jf[5], Jh[5], Wn[5], dWn[5];
    for (int k = 0; k < 5; ++k) {
      Jf[k] = 0.0;
      Jh[k] = 0.0;
      for (int j = 0; j < 6; ++j) {
        Jf[k] += gf[j] * Dk[j][k];
        Jh[k] += gh[j] * Dk[j][k];
      }
      Wn[k] = (Jf[k] * a22 - a12 * Jh[k]) / det;
      dWn[k] = (a11 * Jh[k] - a21 * Jf[k]) / det;
    }
    double U0 = m0[1], V0 = m0[2], W0 = m0[3], u2 = 0.5 * (U0 * U0 + V0 * V0 + W0 * W0);
    double q = F[4] - (U0 * F[1] + V0 * F[2] + W0 * F[3]) + u2 * F[0] -
               U0 * (Wn[4] - (U0 * Wn[1] + V0 * Wn[2] + W0 * Wn[3]) + u2 * Wn[0]);
    double dq = dF[4] - (U0 * dF[1] + V0 * dF[2] + W0 * dF[3]) + u2 * dF[0] -
                U0 * (dWn[4] - (U0 * dWn[1] + V0 * dWn[2] + W0 * dWn[3]) + u2 * dWn[0]);
    F[4] += (1.0 / g->prandtl - 1.0) * q;
    dF[4] += (1.0 / g->prandtl - 1.0) * dq;
  }
  for (int k = 0; k < 5; ++k)
    if (!isfinite(F[k]) || !isfinite(dF[k])) return -1;
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * Reconstruction (readings O-1..O-4, O-6; formula sheet A.9)
 * ---------------------------------------------------------------------------------------- */

/* WENO5-Z: candidates p0, p1, p2 at x_{i+1/2}, linear weights (1/10, 6/10, 3/10), Jiang-Shu
 * smoothness indicators, tau5 = |beta0 - beta2|, alpha_k = d_k (1 + (tau5/(beta_k + eps))^2),
 * eps = 1e-16 (O-1). */
double or_weno5z_right(const double q[5]) {
  const double eps = 1e-16;
  double qm2 = q[0], qm1 = q[1], q0 = q[2], qp1 = q[3], qp2 = q[4];
  double p0 = (1.0 / 3.0) * qm2 - (7.0 / 6.0) * qm1 + (11.0 / 6.0) * q0;
  double p1 = -(1.0 / 6.0) * qm1 + (5.0 / 6.0) * q0 + (1.0 / 3.0) * qp1;
  double p2 = (1.0 / 3.0) * q0 + (5.0 / 6.0) * qp1 - (1.0 / 6.0) * qp2;
  double b0 = (13.0 / 12.0) * pow(qm2 - 2.0 * qm1 + q0, 2) + 0.25 * pow(qm2 - 4.0 * qm1 + 3.0 * q0, 2);
  double b1 = (13.0 / 12.0) * pow(qm1 - 2.0 * q0 + qp1, 2) + 0.25 * pow(qm1 - qp1, 2);
  double b2 = (13.0 / 12.0) * pow(q0 - 2.0 * qp1 + qp2, 2) + 0.25 * pow(3.0 * q0 - 4.0 * qp1 + qp2, 2);
  double t5 = fabs(b0 - b2);
  double a0 = 0.1 * (1.0 + pow(t5 / (b0 + eps), 2));
  double a1 = 0.6 * (1.0 + pow(t5 / (b1 + eps), 2));
  double a2 = 0.3 * (1.0 + pow(t5 / (b2 + eps), 2));
  double s = a0 + a1 + a2;
  return (a0 / s) * p0 + (a1 / s) * p1 + (a2 / s) * p2;
}

/* left edge x_{i-1/2}: the mirror image (stencil reversed) */
double or_weno5z_left(const double q[5]) {
  double r[5] = {q[4], q[3], q[2], q[1], q[0]};
  return or_weno5z_right(r);
}

/* Weights of the linear degree-4 reconstruction through 5 cell averages (cells j-2..j+2 on
 * [m-1/2, m+1/2]) evaluated at x (value) and its x-derivative, obtained by DEFINITION: solve the
 * 5x5 cell-average system for the polynomial coefficients with each unit data vector.  (O-4) */
static void quartic_weights(double x, double wv[5], double wd[5]) {
  for (int s = 0; s < 5; ++s) {
    double A[25], c[5];
    for (int r = 0; r < 5; ++r) { /* row r: average over cell m = r-2 of x^p */
      double lo = (r - 2) - 0.5, hi = (r - 2) + 0.5;
      for (int p = 0; p < 5; ++p) A[r * 5 + p] = (pow(hi, p + 1) - pow(lo, p + 1)) / (p + 1);
      c[r] = (r == s) ? 1.0 : 0.0;
    }
    gauss_solve(5, A, c);
    double v = 0.0, d = 0.0;
    for (int p = 0; p < 5; ++p) {
      v += c[p] * pow(x, p);
      if (p > 0) d += p * c[p] * pow(x, p - 1);
    }
    wv[s] = v;
    wd[s] = d;
  }
}

/* 2x2 Gauss-Legendre abscissae -+ sqrt(3)/6 of the unit cell width, weights 1/4 (O-8) */
static double gauss_abscissa(int m) { return (m == 0 ? -1.0 : 1.0) * sqrt(3.0) / 6.0; }

void or_face_gauss_points(const double cells[6][5][5][5], double Jn, const double Jt1[2],
                          const double Jt2[2], double Wl[4][5], double Wr[4][5], double dWl[4][3][5],
                          double dWr[4][3][5], double dW0[4][3][5]) {
  /* normal pass on each of the 5x5 tangential lines: six face fields per component */
  double Ql[5][5][5], Qr[5][5][5], dQl[5][5][5], dQr[5][5][5], Cf[5][5][5], Df[5][5][5];
  for (int a = 0; a < 5; ++a)
    for (int b = 0; b < 5; ++b)
      for (int c = 0; c < 5; ++c) {
        double s[6];
        for (int n = 0; n < 6; ++n) s[n] = cells[n][a][b][c]; /* Qbar_{i-2..i+3} */
        double Ai = or_weno5z_left(&s[0]), Bi = or_weno5z_right(&s[0]), Mi = s[2];
        double Aj = or_weno5z_left(&s[1]), Bj = or_weno5z_right(&s[1]), Mj = s[3];
        Ql[a][b][c] = Bi;                                        /* left state  = cell i right edge   */
        Qr[a][b][c] = Aj;                                        /* right state = cell i+1 left edge  */
        dQl[a][b][c] = (2.0 * Ai + 4.0 * Bi - 6.0 * Mi) * Jn;  /* O-3 in-cell parabola slope        */
        dQr[a][b][c] = (-4.0 * Aj - 2.0 * Bj + 6.0 * Mj) * Jn;
        Cf[a][b][c] = (-s[1] + 7.0 * s[2] + 7.0 * s[3] - s[4]) / 12.0;        /* O-6 */
        Df[a][b][c] = (s[1] - 15.0 * s[2] + 15.0 * s[3] - s[4]) / 12.0 * Jn;
      }
  /* tangential pass (O-4): tensor-product quartic weights at the 2x2 Gauss points */
  double wv[2][5], wd[2][5];
  for (int m = 0; m < 2; ++m) quartic_weights(gauss_abscissa(m), wv[m], wd[m]);
  for (int m = 0; m < 2; ++m)
    for (int n = 0; n < 2; ++n) {
      int gp = 2 * m + n;
      for (int c = 0; c < 5; ++c) {
        double vQl = 0, vQr = 0, vdQl = 0, vdQr = 0, vD = 0;
        double d1Ql = 0, d2Ql = 0, d1Qr = 0, d2Qr = 0, d1C = 0, d2C = 0;
        for (int a = 0; a < 5; ++a)
          for (int b = 0; b < 5; ++b) {
            double w = wv[m][a] * wv[n][b];
            double w1 = wd[m][a] * wv[n][b];
            double w2 = wv[m][a] * wd[n][b];
            vQl += w * Ql[a][b][c];
            vQr += w * Qr[a][b][c];
            vdQl += w * dQl[a][b][c];
            vdQr += w * dQr[a][b][c];
            vD += w * Df[a][b][c];
            d1Ql += w1 * Ql[a][b][c];
            d2Ql += w2 * Ql[a][b][c];
            d1Qr += w1 * Qr[a][b][c];
            d2Qr += w2 * Qr[a][b][c];
            d1C += w1 * Cf[a][b][c];
            d2C += w2 * Cf[a][b][c];
          }
        Wl[gp][c] = vQl;
        Wr[gp][c] = vQr;
        dWl[gp][0][c] = vdQl;
        dWl[gp][1][c] = d1Ql * Jt1[m];
        dWl[gp][2][c] = d2Ql * Jt2[n];
        dWr[gp][0][c] = vdQr;
        dWr[gp][1][c] = d1Qr * Jt1[m];
        dWr[gp][2][c] = d2Qr * Jt2[n];
        dW0[gp][0][c] = vD;
        dW0[gp][1][c] = d1C * Jt1[m];
        dW0[gp][2][c] = d2C * Jt2[n];
      }
    }
}

/* ------------------------------------------------------------------------------------------
 * Ghosted block addressing: q[v][k][j][i] with (i,j,k) in [-3, n+3)
 * ---------------------------------------------------------------------------------------- */
static inline long gidx(const or_grid* gr, int v, int i, int j, int k) {
  long NX = gr->n[0] + 2 * OR_NG, NY = gr->n[1] + 2 * OR_NG, NZ = gr->n[2] + 2 * OR_NG;
  return (((long)v * NZ + (k + OR_NG)) * NY + (j + OR_NG)) * NX + (i + OR_NG);
}
static inline long cidx(const or_grid* gr, int v, int i, int j, int k) {
  return (((long)v * gr->n[2] + k) * gr->n[1] + j) * gr->n[0] + i;
}
static inline int wrap(int i, int n) {
  int r = i % n;
  return r < 0 ? r + n : r;
}

/* isothermal no-slip mirror (O-17): U_g = -U_m, T_g = 2 T_w - T_m, p_g = p_m, rho_g = p_g / T_g */
static void wall_mirror(const or_gas* g, const double m[5], double gq[5]) {
  double rho = m[0], U = m[1] / rho, V = m[2] / rho, W = m[3] / rho;
  double p = (g->gamma - 1.0) * (m[4] - 0.5 * rho * (U * U + V * V + W * W));
  double Tg = 2.0 * g->T_wall - p / rho;
  double rg = p / Tg;
  gq[0] = rg;
  gq[1] = -rg * U;
  gq[2] = -rg * V;
  gq[3] = -rg * W;
  gq[4] = p / (g->gamma - 1.0) + 0.5 * rg * (U * U + V * V + W * W);
}

void or_fill_ghosts(const or_gas* g, const or_grid* gr, double* q) {
  int n[3] = {gr->n[0], gr->n[1], gr->n[2]};
  /* 1. wall axes over the interior range of the other axes */
  for (int d = 0; d < 3; ++d) {
    if (gr->bc[d] != 1) continue;
    int a1 = (d + 1) % 3, a2 = (d + 2) % 3;
    /* interior of the other axes; their whole extended range when their ghosts are supplied (bc 2) */
    int lo1 = gr->bc[a1] == 2 ? -OR_NG : 0, hi1 = n[a1] + (gr->bc[a1] == 2 ? OR_NG : 0);
    int lo2 = gr->bc[a2] == 2 ? -OR_NG : 0, hi2 = n[a2] + (gr->bc[a2] == 2 ? OR_NG : 0);
    for (int i2 = lo2; i2 < hi2; ++i2)
      for (int i1 = lo1; i1 < hi1; ++i1)
        for (int m = 0; m < OR_NG; ++m)
          for (int side = 0; side < 2; ++side) {
            int pm[3], pg[3];
            pm[a1] = pg[a1] = i1;
            pm[a2] = pg[a2] = i2;
            pm[d] = side ? n[d] - 1 - m : m;
            pg[d] = side ? n[d] + m : -1 - m;
            double mv[5], gv[5];
            for (int v = 0; v < 5; ++v) mv[v] = q[gidx(gr, v, pm[0], pm[1], pm[2])];
            wall_mirror(g, mv, gv);
            for (int v = 0; v < 5; ++v) q[gidx(gr, v, pg[0], pg[1], pg[2])] = gv[v];
          }
  }
  /* 2. periodic axes over the full extended range: copy from the periodic image
   *    (bc 2 = ghosts supplied by the caller, e.g. a sub-block cut from a larger field: untouched) */
  for (int v = 0; v < 5; ++v)
    for (int k = -OR_NG; k < n[2] + OR_NG; ++k)
      for (int j = -OR_NG; j < n[1] + OR_NG; ++j)
        for (int i = -OR_NG; i < n[0] + OR_NG; ++i) {
          int c[3] = {i, j, k}, s[3] = {i, j, k}, moved = 0;
          for (int d = 0; d < 3; ++d)
            if (gr->bc[d] == 0) {
              s[d] = wrap(c[d], n[d]);
              moved |= s[d] != c[d];
            }
          if (moved) q[gidx(gr, v, c[0], c[1], c[2])] = q[gidx(gr, v, s[0], s[1], s[2])];
        }
}

/* ------------------------------------------------------------------------------------------
 * Operator L and d_t L (Eqs. (3)-(4); P:224-238 face quadrature)
 * ---------------------------------------------------------------------------------------- */
int or_operator(const or_gas* g, const or_grid* gr, const double* q, double dt, double* L,
                double* dL) {
  int nx = gr->n[0], ny = gr->n[1], nz = gr->n[2];
  long ncell = (long)nx * ny * nz;
  for (long s = 0; s < 5 * ncell; ++s) {
    L[s] = 0.0;
    dL[s] = 0.0;
  }
  int fail = 0;
  for (int d = 0; d < 3; ++d) {
    int t1 = (d + 1) % 3, t2 = (d + 2) % 3; /* O-23: local frame (n, t1, t2) */
    int nf[3] = {nx, ny, nz};
    nf[d] += 1; /* faces along d */
    long nface = (long)nf[0] * nf[1] * nf[2];
    double* Fd = (double*)malloc(sizeof(double) * 10 * nface);
#pragma omp parallel for collapse(2) schedule(dynamic) reduction(| : fail)
    for (int fk = 0; fk < nf[2]; ++fk)
      for (int fj = 0; fj < nf[1]; ++fj)
        for (int fi = 0; fi < nf[0]; ++fi) {
          int f[3] = {fi, fj, fk}; /* face f[d] lies between cells f[d]-1 and f[d] */
          double cells[6][5][5][5];
          for (int n = 0; n < 6; ++n)
            for (int a = 0; a < 5; ++a)
              for (int b = 0; b < 5; ++b) {
                int p[3];
                p[d] = f[d] - 3 + n;
                p[t1] = f[t1] - 2 + a;
                p[t2] = f[t2] - 2 + b;
                /* rotate momentum into the local frame: (rho, m_n, m_t1, m_t2, E) */
                cells[n][a][b][0] = q[gidx(gr, 0, p[0], p[1], p[2])];
                cells[n][a][b][1] = q[gidx(gr, 1 + d, p[0], p[1], p[2])];
                cells[n][a][b][2] = q[gidx(gr, 1 + t1, p[0], p[1], p[2])];
                cells[n][a][b][3] = q[gidx(gr, 1 + t2, p[0], p[1], p[2])];
                cells[n][a][b][4] = q[gidx(gr, 4, p[0], p[1], p[2])];
              }
          /* metrics (O-18): normal at the face, tangential at the Gauss abscissae */
          double s3 = sqrt(3.0) / 6.0;
          double Jn = or_axis_metric(gr, d, (double)f[d]);
          double Jt1[2] = {or_axis_metric(gr, t1, f[t1] + 0.5 - s3), or_axis_metric(gr, t1, f[t1] + 0.5 + s3)};
          double Jt2[2] = {or_axis_metric(gr, t2, f[t2] + 0.5 - s3), or_axis_metric(gr, t2, f[t2] + 0.5 + s3)};
          double Wl[4][5], Wr[4][5], dWl[4][3][5], dWr[4][3][5], dW0[4][3][5];
          or_face_gauss_points((const double(*)[5][5][5])cells, Jn, Jt1, Jt2, Wl, Wr, dWl, dWr, dW0);
          double Fs[5] = {0, 0, 0, 0, 0}, dFs[5] = {0, 0, 0, 0, 0};
          for (int gp = 0; gp < 4; ++gp) { /* (m, n) order, O-21 */
            double F[5], dF[5];
            if (or_gp_flux(g, Wl[gp], (const double(*)[5])dWl[gp], Wr[gp],
                           (const double(*)[5])dWr[gp], (const double(*)[5])dW0[gp], dt, F, dF,
                           NULL)) {
              fail |= 1;
              continue;
            }
            for (int c = 0; c < 5; ++c) {
              Fs[c] += 0.25 * F[c]; /* omega_mn = 1/4 */
              dFs[c] += 0.25 * dF[c];
            }
          }
          /* rotate back to global components, times the physical face area */
          double area = cell_width(gr, t1, f[t1]) * cell_width(gr, t2, f[t2]);
          int gc[5] = {0, 1 + d, 1 + t1, 1 + t2, 4};
          long fid = ((long)fk * nf[1] + fj) * nf[0] + fi;
          for (int c = 0; c < 5; ++c) {
            Fd[(long)gc[c] * nface + fid] = area * Fs[c];
            Fd[(long)(5 + gc[c]) * nface + fid] = area * dFs[c];
          }
        }
    /* accumulate -(F_{+} - F_{-}) / |Omega|, direction by direction (O-21) */
    for (int k = 0; k < nz; ++k)
      for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
          int lo[3] = {i, j, k}, hi[3] = {i, j, k};
          hi[d] += 1;
          double vol = cell_width(gr, 0, i) * cell_width(gr, 1, j) * cell_width(gr, 2, k);
          long flo = ((long)lo[2] * nf[1] + lo[1]) * nf[0] + lo[0];
          long fhi = ((long)hi[2] * nf[1] + hi[1]) * nf[0] + hi[0];
          for (int c = 0; c < 5; ++c) {
            long s = cidx(gr, c, i, j, k);
            L[s] += -(Fd[(long)c * nface + fhi] - Fd[(long)c * nface + flo]) / vol;
            dL[s] += -(Fd[(long)(5 + c) * nface + fhi] - Fd[(long)(5 + c) * nface + flo]) / vol;
          }
        }
    free(Fd);
  }
  return fail ? -1 : 0;
}

/* ------------------------------------------------------------------------------------------
 * Eq. (7) two-stage fourth-order update
 * ---------------------------------------------------------------------------------------- */
void or_s2o4_stage1(long n, const double* q, const double* L, const double* dL, double dt,
                    double* qs) {
  for (long s = 0; s < n; ++s) qs[s] = q[s] + 0.5 * dt * L[s] + (1.0 / 8.0) * dt * dt * dL[s];
}

void or_s2o4_final(long n, const double* q, const double* L, const double* dL, const double* dLs,
                   double dt, double* qn) {
  for (long s = 0; s < n; ++s)
    qn[s] = q[s] + dt * L[s] + (1.0 / 6.0) * dt * dt * (dL[s] + 2.0 * dLs[s]);
}

/* ------------------------------------------------------------------------------------------
 * CFL (O-13; pinned by Table 3)
 * ---------------------------------------------------------------------------------------- */
double or_cfl_dt(const or_gas* g, const or_grid* gr, const double* q, double cfl) {
  long ncell = (long)gr->n[0] * gr->n[1] * gr->n[2];
  double best = INFINITY;
  for (long s = 0; s < ncell; ++s) {
    double rho = q[s], U[3] = {q[ncell + s] / rho, q[2 * ncell + s] / rho, q[3 * ncell + s] / rho};
    double p = (g->gamma - 1.0) * (q[4 * ncell + s] - 0.5 * rho * (U[0] * U[0] + U[1] * U[1] + U[2] * U[2]));
    double c = sqrt(g->gamma * p / rho);
    int ijk[3] = {(int)(s % gr->n[0]), (int)((s / gr->n[0]) % gr->n[1]), (int)(s / ((long)gr->n[0] * gr->n[1]))};
    for (int d = 0; d < 3; ++d) {
      double v = cell_width(gr, d, ijk[d]) / (fabs(U[d]) + c);
      if (v < best) best = v;
    }
  }
  return cfl * best;
}

static int state_valid(const or_gas* g, long ncell, const double* q) {
  for (long s = 0; s < ncell; ++s) {
    double rho = q[s];
    double k = 0.5 * (q[ncell + s] * q[ncell + s] + q[2 * ncell + s] * q[2 * ncell + s] +
                      q[3 * ncell + s] * q[3 * ncell + s]) / rho;
    double p = (g->gamma - 1.0) * (q[4 * ncell + s] - k);
    if (!(rho > 0.0) || !(p > 0.0) || !isfinite(rho) || !isfinite(p)) return 0;
    for (int v = 1; v < 4; ++v)
      if (!isfinite(q[v * ncell + s])) return 0;
  }
  return 1;
}

static void to_ghosted(const or_grid* gr, const double* q, double* qg) {
  for (int v = 0; v < 5; ++v)
    for (int k = 0; k < gr->n[2]; ++k)
      for (int j = 0; j < gr->n[1]; ++j)
        for (int i = 0; i < gr->n[0]; ++i) qg[gidx(gr, v, i, j, k)] = q[cidx(gr, v, i, j, k)];
}

/* ------------------------------------------------------------------------------------------
 * Streamwise body force (channel; "the constant moment flux in the streamwise
 * direction is used to determine the external force").  The paper does not give the discrete
 * form; readings O-26 / O-27:
 *  O-26 a uniform acceleration f along x, constant over a step, enters as the source
 *       S(Q) = (0, rho f, 0, 0, rho U f) of L, and its time derivative through dS/dt = S'(Q) dQ/dt
 *       = (0, f L_rho, 0, 0, f L_rhoU) with L the source-inclusive operator.  Stage 2 evaluates no
 *       flux (only d_t L(Q*)), so L(Q*) in S'(Q*) L(Q*) is its Taylor value L(Q^n) + dt/2 d_t L(Q^n).
 *  O-27 mode 2 chooses f each step so that the bulk momentum m = (1/Omega) sum rho U dV returns to
 *       the target m_b in one step if the wall drag stays as in the previous step (dead-beat):
 *         f^n = f^{n-1} + [ (m_b - m^n)/dt^n - (m^n - m^{n-1})/dt^{n-1} ] / rho_b^n,
 *       rho_b = (1/Omega) sum rho dV, with f^{-1} = f_init and m^{-1} = m^0 (first step:
 *       f^0 = f_init + (m_b - m^0)/(dt^0 rho_b^0)).  Mode 1: f = f_init every step.
 * ---------------------------------------------------------------------------------------- */
static void bulk_of(const or_grid* gr, const double* q, double* m, double* rho_b) {
  long ncell = (long)gr->n[0] * gr->n[1] * gr->n[2];
  double sm = 0.0, sr = 0.0, vol = 0.0;
  for (int k = 0; k < gr->n[2]; ++k)
    for (int j = 0; j < gr->n[1]; ++j)
      for (int i = 0; i < gr->n[0]; ++i) {
        double dv = cell_width(gr, 0, i) * cell_width(gr, 1, j) * cell_width(gr, 2, k);
        sr += q[cidx(gr, 0, i, j, k)] * dv;
        sm += q[cidx(gr, 1, i, j, k)] * dv;
        vol += dv;
      }
  (void)ncell;
  *m = sm / vol;
  *rho_b = sr / vol;
}

/* O-26: add the source and its time derivative to (L, dL) of state q (all [5][ncell]) */
static void add_force(long ncell, const double* q, double f, double* L, double* dL) {
  for (long s = 0; s < ncell; ++s) {
    L[1 * ncell + s] += q[0 * ncell + s] * f;
    L[4 * ncell + s] += q[1 * ncell + s] * f;
    dL[1 * ncell + s] += f * L[0 * ncell + s];
    dL[4 * ncell + s] += f * L[1 * ncell + s];
  }
}

int or_run_forced(const or_gas* g, const or_grid* gr, double* q, int nsteps, double dt_fixed, double cfl,
                  const or_forcing* fc, double* dt_hist, double* f_hist) {
  long ncell = (long)gr->n[0] * gr->n[1] * gr->n[2];
  long ng = 5L * (gr->n[0] + 2 * OR_NG) * (gr->n[1] + 2 * OR_NG) * (gr->n[2] + 2 * OR_NG);
  double* qg = (double*)calloc(ng, sizeof(double));
  double* L = (double*)malloc(sizeof(double) * 5 * ncell);
  double* dL = (double*)malloc(sizeof(double) * 5 * ncell);
  double* Ls = (double*)malloc(sizeof(double) * 5 * ncell);
  double* dLs = (double*)malloc(sizeof(double) * 5 * ncell);
  double* qs = (double*)malloc(sizeof(double) * 5 * ncell);
  double* qn = (double*)malloc(sizeof(double) * 5 * ncell);
  int mode = fc ? fc->mode : 0;
  double f_prev = fc ? fc->force : 0.0, m_prev = 0.0, dt_prev = 0.0;
  int rc = 0;
  if (!state_valid(g, ncell, q)) rc = -1;
  for (int step = 0; step < nsteps && rc == 0; ++step) {
    double dt = dt_fixed > 0.0 ? dt_fixed : or_cfl_dt(g, gr, q, cfl);
    if (dt_hist) dt_hist[step] = dt;
    double f = 0.0;
    if (mode == 1) {
      f = fc->force;
    } else if (mode == 2) { /* O-27 */
      double m, rb;
      bulk_of(gr, q, &m, &rb);
      if (step == 0) f = f_prev + (fc->target - m) / (dt * rb);
      else f = f_prev + ((fc->target - m) / dt - (m - m_prev) / dt_prev) / rb;
      m_prev = m;
      dt_prev = dt;
      f_prev = f;
    }
    if (f_hist) f_hist[step] = f;
    /* stage 1 at Q^n */
    to_ghosted(gr, q, qg);
    or_fill_ghosts(g, gr, qg);
    if (or_operator(g, gr, qg, dt, L, dL)) { rc = -1; break; }
    if (mode) add_force(ncell, q, f, L, dL);
    or_s2o4_stage1(5 * ncell, q, L, dL, dt, qs);
    /* stage 2 at Q* (same dt and windows, O-11) */
    to_ghosted(gr, qs, qg);
    or_fill_ghosts(g, gr, qg);
    if (or_operator(g, gr, qg, dt, Ls, dLs)) { rc = -1; break; }
    if (mode) /* O-26: S'(Q*) L(Q*), L(Q*) ~ L(Q^n) + dt/2 d_t L(Q^n) */
      for (long s = 0; s < ncell; ++s) {
        dLs[1 * ncell + s] += f * (L[0 * ncell + s] + 0.5 * dt * dL[0 * ncell + s]);
        dLs[4 * ncell + s] += f * (L[1 * ncell + s] + 0.5 * dt * dL[1 * ncell + s]);
      }
    or_s2o4_final(5 * ncell, q, L, dL, dLs, dt, qn);
    if (!state_valid(g, ncell, qn)) { rc = -1; break; }
    memcpy(q, qn, sizeof(double) * 5 * ncell);
  }
  free(qg);
  free(L);
  free(dL);
  free(Ls);
  free(dLs);
  free(qs);
  free(qn);
  return rc;
}

int or_run(const or_gas* g, const or_grid* gr, double* q, int nsteps, double dt_fixed, double cfl,
           double* dt_hist) {
  return or_run_forced(g, gr, q, nsteps, dt_fixed, cfl, NULL, dt_hist, NULL);
}

/* ------------------------------------------------------------------------------------------
 * Volume diagnostics (readings O-24, O-25): on a ghosted block with ghosts filled.
 *   E_k   = 1/(rho0 Omega) sum 1/2 rho |U|^2 dV
 *   zeta  = 1/(rho0 Omega) sum 1/2 rho |omega|^2 dV, omega = curl U    (O-24)
 *   eps_s = mu/(rho0 Omega) sum omega.omega dV                         (first term)
 *   eps_d = 4/3 mu/(rho0 Omega) sum (div U)^2 dV                       (second term)
 * plus the conservation monitors sum rho dV, sum rho U dV (3), sum rho E dV and Omega, and
 *   Pi    = 1/(rho0 Omega) sum p div U dV                               (pressure-dilatation)
 * which closes the kinetic-energy budget of compressible decaying turbulence,
 * dE_k/dt = Pi - eps_s - eps_d (constant mu; the paper's eps_com = eps_s + eps_d).
 * Velocity derivatives at a cell centre (O-25): the fourth-order central difference in the cell
 * index of the cell-average velocities, times the metric J = d(index)/dx at the cell centre:
 *   du/dx_d (j) = J(j + 1/2) [8 (u_{j+1} - u_{j-1}) - (u_{j+2} - u_{j-2})] / 12.
 * mu is mu_ref (the paper's eps_com takes a constant mu).
 * ---------------------------------------------------------------------------------------- */
static double vel_at(const or_grid* gr, const double* qg, int c, int i, int j, int k) {
  return qg[gidx(gr, 1 + c, i, j, k)] / qg[gidx(gr, 0, i, j, k)];
}

void or_diagnostics(const or_gas* g, const or_grid* gr, const double* qg, double rho0, double out[OR_NDIAG]) {
  double acc[OR_NDIAG] = {0};
  for (int k = 0; k < gr->n[2]; ++k)
    for (int j = 0; j < gr->n[1]; ++j)
      for (int i = 0; i < gr->n[0]; ++i) {
        int ijk[3] = {i, j, k};
        double vol = cell_width(gr, 0, i) * cell_width(gr, 1, j) * cell_width(gr, 2, k);
        double rho = qg[gidx(gr, 0, i, j, k)];
        double u[3], grad[3][3]; /* grad[c][d] = d u_c / d x_d */
        for (int c = 0; c < 3; ++c) u[c] = qg[gidx(gr, 1 + c, i, j, k)] / rho;
        for (int d = 0; d < 3; ++d) {
          double J = or_axis_metric(gr, d, ijk[d] + 0.5);
          for (int c = 0; c < 3; ++c) {
            int a[3], b[3], a2[3], b2[3];
            for (int e = 0; e < 3; ++e) a[e] = b[e] = a2[e] = b2[e] = ijk[e];
            a[d] += 1;
            b[d] -= 1;
            a2[d] += 2;
            b2[d] -= 2;
            double d1 = vel_at(gr, qg, c, a[0], a[1], a[2]) - vel_at(gr, qg, c, b[0], b[1], b[2]);
            double d2 = vel_at(gr, qg, c, a2[0], a2[1], a2[2]) - vel_at(gr, qg, c, b2[0], b2[1], b2[2]);
            grad[c][d] = J * (8.0 * d1 - d2) / 12.0;
          }
        }
        double om[3] = {grad[2][1] - grad[1][2], grad[0][2] - grad[2][0], grad[1][0] - grad[0][1]};
        double om2 = om[0] * om[0] + om[1] * om[1] + om[2] * om[2];
        double dv = grad[0][0] + grad[1][1] + grad[2][2];
        acc[OR_DIAG_EK] += 0.5 * rho * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]) * vol;
        acc[OR_DIAG_ENSTROPHY] += 0.5 * rho * om2 * vol;
        acc[OR_DIAG_EPS_S] += om2 * vol;
        acc[OR_DIAG_EPS_D] += dv * dv * vol;
        acc[OR_DIAG_MASS] += rho * vol;
        for (int c = 0; c < 3; ++c) acc[OR_DIAG_MOM_X + c] += qg[gidx(gr, 1 + c, i, j, k)] * vol;
        acc[OR_DIAG_ENERGY] += qg[gidx(gr, 4, i, j, k)] * vol;
        acc[OR_DIAG_VOLUME] += vol;
        double p = (g->gamma - 1.0) * (qg[gidx(gr, 4, i, j, k)] - 0.5 * rho * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]));
        acc[OR_DIAG_PDIL] += p * dv * vol;
      }
  double omega = acc[OR_DIAG_VOLUME];
  for (int v = 0; v < OR_NDIAG; ++v) out[v] = acc[v];
  out[OR_DIAG_EK] = acc[OR_DIAG_EK] / (rho0 * omega);
  out[OR_DIAG_ENSTROPHY] = acc[OR_DIAG_ENSTROPHY] / (rho0 * omega);
  out[OR_DIAG_EPS_S] = g->mu_ref * acc[OR_DIAG_EPS_S] / (rho0 * omega);
  out[OR_DIAG_EPS_D] = 4.0 / 3.0 * g->mu_ref * acc[OR_DIAG_EPS_D] / (rho0 * omega);
  out[OR_DIAG_PDIL] = acc[OR_DIAG_PDIL] / (rho0 * omega);
}

/* ------------------------------------------------------------------------------------------
 * Plane statistics of the channel: raw moments of the state averaged over the x-z
 * plane of every y index j (the paper's <.> is the mean over time and the X and Z directions,
 * P:1190-1191; time averaging is done by the caller over samples).  Per plane, in this order:
 *   rho, U, V, W, U^2, V^2, W^2, UV, rho U, rho V, rho U V, c, M, M^2, T, p
 * with c = sqrt(gamma p / rho) the local sound speed, M = |U| / c, T = p / rho (O-28).
 * out[j * OR_NSTAT + s] = (1/(nx nz)) sum_{i,k} of moment s (x and z are uniform axes).
 * ---------------------------------------------------------------------------------------- */
void or_plane_stats(const or_gas* g, const or_grid* gr, const double* q, double* out) {
  int nx = gr->n[0], ny = gr->n[1], nz = gr->n[2];
  for (int j = 0; j < ny; ++j) {
    double acc[OR_NSTAT] = {0};
    for (int k = 0; k < nz; ++k)
      for (int i = 0; i < nx; ++i) {
        double rho = q[cidx(gr, 0, i, j, k)];
        double U = q[cidx(gr, 1, i, j, k)] / rho, V = q[cidx(gr, 2, i, j, k)] / rho, W = q[cidx(gr, 3, i, j, k)] / rho;
        double p = (g->gamma - 1.0) * (q[cidx(gr, 4, i, j, k)] - 0.5 * rho * (U * U + V * V + W * W));
        double c = sqrt(g->gamma * p / rho);
        double M = sqrt(U * U + V * V + W * W) / c;
        double v[OR_NSTAT] = {rho, U, V, W, U * U, V * V, W * W, U * V, rho * U, rho * V, rho * U * V,
                              c, M, M * M, p / rho, p};
        for (int s = 0; s < OR_NSTAT; ++s) acc[s] += v[s];
      }
    for (int s = 0; s < OR_NSTAT; ++s) out[(long)j * OR_NSTAT + s] = acc[s] / ((double)nx * nz);
  }
}
