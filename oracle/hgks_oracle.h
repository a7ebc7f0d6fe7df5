/*
 * hgks_oracle.h — plain CPU fp64 oracle for the HGKS S2O4 stage (arXiv 2207.01173 §2).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2207_01173_b200/, libhgks.so) never links, imports or executes it, and the two
 * share no code, header, table or constant generator.
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; O-n / A.n = SURVEY.md §8(c)
 * readings and Appendix A formula sheet (the readings are restated in DESIGN.md).
 *
 * Every function here is pinned by a `-m "not gpu"` test in tests/test_oracle_*.py
 * against something other than itself (quadrature, closed forms, paper tables,
 * invariants).  Pins are listed next to each declaration.
 */
#ifndef HGKS_ORACLE_H
#define HGKS_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

#define OR_NV 5      /* conservative variables (rho, rhoU, rhoV, rhoW, rhoE) */
#define OR_NG 3      /* ghost layers (O-16) */
#define OR_NM 9      /* velocity-moment tables hold orders 0..8 */

/* gas + transport model (P:202-204 gamma/K; P:270-273 tau=mu/p; P:971-973 power law, Pr) */
typedef struct {
  double gamma;   /* specific heat ratio                                         */
  double K;       /* internal DOF, or_K(gamma) (O-20)                      */
  double prandtl; /* Pr; 1 = no heat-flux fix (TGV); != 1: O-12 fix        */
  int    mu_law;  /* 0: mu = mu_ref ; 1: mu = mu_ref*(T/T_ref)^omega, T = p/rho     */
  double mu_ref, T_ref, omega;
  double T_wall;  /* isothermal wall temperature (p/rho units), O-17              */
} or_gas;

/* Geometry of a block that carries OR_NG ghost layers on every side.  Axis d is uniform
 * (stretch 0: width dx[d]) or tanh-stretched (stretch 1):
 *   x(s) = (lo+hi)/2 + (hi-lo)/2 * tanh(b (2 s - 1)) / tanh(b),  s = j / n[d] at face j,
 * i.e. uniform in the computational coordinate (the paper's eta / (3 pi) for the channel). */
typedef struct {
  int    n[3];          /* interior cells nx, ny, nz                                    */
  double dx[3];         /* cell widths of uniform axes                                  */
  int    bc[3];         /* 0 periodic, 1 isothermal no-slip walls at both ends (O-17),
                           2 ghosts supplied by the caller (sub-blocks in tests)          */
  int    stretch[3];    /* 0 uniform, 1 tanh                                            */
  double lo[3], hi[3];  /* box of stretched axes                                        */
  double stretch_b[3];  /* b_g of tanh axes (b_g = 2)                            */
} or_grid;

/* Face coordinate x_j (j = 0..n[d]), and the metric J = d(cell index)/dx at fractional cell-index
 * position zeta (zeta = j at face j, j + 1/2 at the centre of cell j) of axis d.  J = 1/dx on
 * uniform axes; the analytic derivative of the tanh map otherwise (O-18).  Pin: Tables 6-7. */
double or_axis_face(const or_grid* gr, int d, int j);
double or_axis_metric(const or_grid* gr, int d, double zeta);

double or_K(double gamma);

/* A.2: normalised Maxwellian u-moments <u^n>, n = 0..OR_NM-1.
 * which = 0 full space, +1 u>0 half space, -1 u<0 half space.
 * Pin: scipy quadrature (test_oracle_kinetic.py::test_moments_vs_quadrature). */
void or_moments_u(double U, double lam, int which, double m[OR_NM]);

/* <u^a v^b w^c xi^(2d) psi> (5-vector) for a Maxwellian (rho-normalised), u-table chosen by
 * which.  Pin: 5-D Gauss-Hermite quadrature. */
void or_psi_moment(double U, double V, double W, double lam, double K, int which,
                   int a, int b, int c, int d, double out[5]);

/* conservative -> Maxwellian parameters (rho,U,V,W,lambda); A.1.  returns 0, or -1 if invalid */
int or_cons_to_maxw(const double q[5], double K, double mx[5]);

/* A.3 compatibility solve <(a.psi) psi>_g = b (rho-normalised), by assembling the 5x5 moment
 * matrix from or_psi_moment and Gaussian elimination with partial pivoting.
 * Pin: quadrature residual (test_slope_solve_residual). */
int or_slope_solve(const double mx[5], double K, const double b[5], double a[5]);

/* time integrals gamma_1..gamma_6 of the six time functions of Eq. (6) over [0,T]
 * (A.6).  Pin: scipy.quad of the six kernels. */
void or_time_integrals(double T, double tau, double g[6]);

/* Gauss-point flux (A4-A6) in the local frame (u = face normal):
 *   Wl, Wr         left/right conservative states at the Gauss point
 *   dWl[i], dWr[i] their derivatives along local axis i (0 normal, 1 t1, 2 t2)
 *   dW0[i]         equilibrium derivatives (O-6)
 *   dt             step; the two windows are [0,dt/2] and [0,dt]
 * Outputs F^n, dF = d_t F^n (Eq. (8) two-window solve), and tau.  Returns 0 or -1 on an
 * invalid state.  Pins: Euler flux of a uniform state, Navier-Stokes limit (A.8),
 * brute-force velocity-space quadrature of Eq. (6) (test_gp_flux_vs_quadrature). */
int or_gp_flux(const or_gas* g, const double Wl[5], const double dWl[3][5],
               const double Wr[5], const double dWr[3][5], const double dW0[3][5], double dt,
               double F[5], double dF[5], double* tau);

/* WENO5-Z (O-1, A.9) value at the right edge of the middle cell of q[0..4] = Qbar_{i-2..i+2}.
 * Pins: constant/linear exactness, 5th-order convergence, linear-weight limit. */
double or_weno5z_right(const double q[5]);
double or_weno5z_left(const double q[5]);

/* Gauss-point inputs of one face from a 6 (normal) x 5 (t1) x 5 (t2) block of cell averages
 * cells[n][a][b] (n = i-2..i+3 normal, a = t1 offset -2..2, b = t2 offset -2..2).  Derivatives are
 * taken in cell-index units (reconstruction in the computational coordinate, O-18) and converted
 * with the metrics: Jn at the face (normal), Jt1[m], Jt2[n] at the Gauss abscissae.  For Gauss point
 * gp = 2*m + n (m index in t1, n in t2, point -sqrt(3)/6 first), component c:
 *   Wl[gp][c], Wr[gp][c], dWl[gp][i][c], dWr[gp][i][c], dW0[gp][i][c]   (i: normal, t1, t2)
 * Steps A2-A3 with readings O-3, O-4, O-6.  Pins: polynomial exactness, constants. */
void or_face_gauss_points(const double cells[6][5][5][5], double Jn, const double Jt1[2],
                          const double Jt2[2], double Wl[4][5], double Wr[4][5], double dWl[4][3][5],
                          double dWr[4][3][5], double dW0[4][3][5]);

/* Whole-grid ghost fill of q laid out [5][nz+6][ny+6][nx+6] (O-16, O-17): wall axes first over
 * the interior of the other axes (mirror: U_g = -U_m, T_g = 2 T_wall - T_m, p_g = p_m), then the
 * periodic axes over the full extended range (corners). */
void or_fill_ghosts(const or_gas* g, const or_grid* gr, double* q);

/* Operator L(Q) and d_t L(Q) (Eqs. (3)-(4)) on the interior of a ghosted
 * block q [5][nz+6][ny+6][nx+6] whose ghosts are already filled.  L, dL are [5][nz][ny][nx].
 * Returns 0, or -1 on an invalid Gauss-point state. */
int or_operator(const or_gas* g, const or_grid* gr, const double* q, double dt,
                double* L, double* dL);

/* S2O4 stage updates (Eq. (7)) on flat arrays of length n:
 *   stage 1: qs = q + dt/2 L + dt^2/8 dL
 *   final  : qn = q + dt L + dt^2/6 (dL + 2 dLs)
 * Pin: S:284 surrogate q' = q. */
void or_s2o4_stage1(long n, const double* q, const double* L, const double* dL, double dt,
                    double* qs);
void or_s2o4_final(long n, const double* q, const double* L, const double* dL,
                   const double* dLs, double dt, double* qn);

/* CFL time step (O-13): dt = cfl * min over cells, d of dx_d/(|U_d| + c), c = sqrt(gamma p/rho),
 * with the cell's own width dx_d on stretched axes, on an unghosted [5][nz][ny][nx] state.
 * Pin: Table 3. */
double or_cfl_dt(const or_gas* g, const or_grid* gr, const double* q, double cfl);

/* Full S2O4 steps on an unghosted [5][nz][ny][nx] state, in place (ghosts by or_fill_ghosts).
 * dt_fixed > 0 uses it; else CFL each step.  dt_hist (nsteps, may be NULL) receives the dt
 * used.  Returns 0, or -1 on an invalid state (q then holds the last good state). */
int or_run(const or_gas* g, const or_grid* gr, double* q, int nsteps, double dt_fixed,
           double cfl, double* dt_hist);

/* Streamwise body force (readings O-26 source, O-27 dead-beat bulk-momentum
 * controller, both restated at or_run_forced in hgks_oracle.c and in DESIGN.md).
 * mode 0 none, 1 constant acceleration f = force, 2 constant bulk momentum target (f_init = force).
 * f_hist[step] = f applied in that step.  Pins (test_oracle_forcing.py): uniform flow under a
 * constant acceleration is integrated exactly (U = U0 + f t, p unchanged); the dead-beat step
 * reaches the target in one step in a drag-free box with the closed-form f; laminar Poiseuille
 * balance f rho_b = tau_w / H (f = 3 mu U_b / (rho_b H^2)). */
typedef struct {
  int mode;
  double force;   /* mode 1: f ; mode 2: f_init */
  double target;  /* mode 2: bulk momentum m_b = (1/Omega) sum rho U dV */
} or_forcing;
int or_run_forced(const or_gas* g, const or_grid* gr, double* q, int nsteps, double dt_fixed, double cfl,
                  const or_forcing* fc, double* dt_hist, double* f_hist);

/* x-z plane means of 16 raw moments for every y index (channel statistics, O-28):
 * rho, U, V, W, U^2, V^2, W^2, UV, rho U, rho V, rho U V, c, M, M^2, T, p ; q unghosted
 * [5][nz][ny][nx]; out[ny][OR_NSTAT].  Pins (test_oracle_stats.py): plane means of fields built
 * from x/z harmonics, whose exact means follow from the discrete orthogonality of the harmonics. */
#define OR_NSTAT 16
void or_plane_stats(const or_gas* g, const or_grid* gr, const double* q, double* out);

/* Number of OpenMP threads the oracle uses (1 when built without OpenMP). */
/* Volume diagnostics of a ghosted block (ghosts filled): E_k, enstrophy (O-24),
 * the two terms of eps_com (mu = mu_ref), and conservation monitors; velocity
 * derivatives by O-25 (fourth-order central in the cell index times J at the cell centre).
 * Pins (test_oracle_diagnostics.py): TGV closed forms E_k = 1/8, zeta = 3/8 kappa(h)^2 with
 * kappa(h) = (8 sin h - sin 2h)/(6h) the exact symbol of the difference, div U = 0; a potential
 * flow (omega = 0, eps_d closed form); a linear shear on a tanh-stretched axis (metric); Omega;
 * the pressure-dilatation of a potential flow with a harmonic pressure (closed form). */
#define OR_NDIAG 11
enum { OR_DIAG_EK = 0, OR_DIAG_ENSTROPHY, OR_DIAG_EPS_S, OR_DIAG_EPS_D, OR_DIAG_MASS, OR_DIAG_MOM_X,
       OR_DIAG_MOM_Y, OR_DIAG_MOM_Z, OR_DIAG_ENERGY, OR_DIAG_VOLUME, OR_DIAG_PDIL };
void or_diagnostics(const or_gas* g, const or_grid* gr, const double* qg, double rho0, double out[OR_NDIAG]);

int or_num_threads(void);
void or_set_num_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
