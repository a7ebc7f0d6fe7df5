/*
 * hgks_test.h — test-only entry points of libhgks.so (not part of the user ABI in hgks.h).
 *
 * They run the SAME device code as hgks_step on small host-provided batches so the parity tests
 * can compare each step of the hot path with the oracle separately.  All arrays are host fp64;
 * computation happens on the current CUDA device in the requested precision.
 */
#ifndef HGKS_TEST_H
#define HGKS_TEST_H

#include "hgks.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Batched Gauss-point flux (steps A4-A6; Eq. (6) P:252-258 + Eq. (8)), local frame.
 *   in  : n records of 55 fp64 = Wl[5], Wr[5], dWl[3][5], dWr[3][5], dW0[3][5] (i: normal,t1,t2)
 *   out : n records of 11 fp64 = F[5], dF[5], tau
 *   gamma, mu_law/mu_ref/T_ref/omega, prandtl as in hgks_params; dt the step (windows [0,dt/2],
 *   [0,dt]).  Returns HGKS_OK or HGKS_ECUDA / HGKS_EINVAL. */
int hgks_test_gp_flux(int precision, double gamma, int mu_law, double mu_ref, double T_ref,
                      double omega, double prandtl, double dt, const double* in, int64_t n,
                      double* out);

/* Operator evaluation on the context's current state (after hgks_set_state): one ghost fill and
 * the three flux sweeps at time step dt, then L(Q) and d_t L(Q) (Eqs. (3)-(4), P:211-218,
 * P:355-358) written to host arrays L, dL in the set_state layout.  Used for per-stage parity. */
int hgks_test_operator(hgks_ctx* c, double dt, double* L, double* dL);

/* Face-flux array of direction dir (0 x, 1 y, 2 z) left by the last flux sweep (e.g. after
 * hgks_test_operator): out[10][nfaces] fp64 with components 0..4 = F^n, 5..9 = d_t F^n per unit
 * area, faces in natural [z][y][x] order with the normal extent n_dir + 1.  Synchronises. */
int hgks_test_face_flux(hgks_ctx* c, int dir, double* out);

#ifdef __cplusplus
}
#endif
#endif
