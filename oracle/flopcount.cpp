// flopcount.cpp — the ORACLE's arithmetic, counted (test/measurement infrastructure, not product).
//
// Compiles oracle/hgks_oracle.c unchanged as C++ with every `double` replaced by a counting type, so
// each floating-point operation the plain oracle performs -- i.e. the method of PAPER.md §2 in the
// paper's order (Eq. 6 moments, Gaussian-elimination compatibility solves, the two-window time
// integrals and the 2x2 solve of Eq. 8, generic WENO-Z, tangential weights solved per face) -- is
// counted.  bench.py / DESIGN.md §8 set this "algorithmic" count beside the flops the GPU kernels
// EXECUTE (ncu SASS counts), which come from a reduced algebra of the same mathematics.
//
// Build + run (host only):  g++ -O1 -std=c++17 -o /tmp/flopcount oracle/flopcount.cpp && /tmp/flopcount
// Prints one JSON object: counts per Gauss-point flux, per face (tangential reconstruction), per
// WENO edge, and per cell-update of the whole operator (both stages) on TGV 16^3.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cmath>

namespace fc {
struct Counters {
  long long add = 0, mul = 0, div = 0, sqrt_ = 0, exp_ = 0, erfc_ = 0, pow_ = 0, other = 0, cmp = 0;
};
static Counters C;

struct CD {
  double v;
  CD() = default;
  CD(double x) : v(x) {}  // NOLINT: implicit from literals, ints, longs
  explicit operator int() const { return (int)v; }
  explicit operator long() const { return (long)v; }
  explicit operator float() const { return (float)v; }
  CD& operator+=(CD o) { ++C.add; v += o.v; return *this; }
  CD& operator-=(CD o) { ++C.add; v -= o.v; return *this; }
  CD& operator*=(CD o) { ++C.mul; v *= o.v; return *this; }
  CD& operator/=(CD o) { ++C.div; v /= o.v; return *this; }
};
inline CD operator+(CD a, CD b) { ++C.add; return CD(a.v + b.v); }
inline CD operator-(CD a, CD b) { ++C.add; return CD(a.v - b.v); }
inline CD operator*(CD a, CD b) { ++C.mul; return CD(a.v * b.v); }
inline CD operator/(CD a, CD b) { ++C.div; return CD(a.v / b.v); }
inline CD operator-(CD a) { return CD(-a.v); }
inline CD operator+(CD a) { return a; }
inline bool operator<(CD a, CD b) { ++C.cmp; return a.v < b.v; }
inline bool operator>(CD a, CD b) { ++C.cmp; return a.v > b.v; }
inline bool operator<=(CD a, CD b) { ++C.cmp; return a.v <= b.v; }
inline bool operator>=(CD a, CD b) { ++C.cmp; return a.v >= b.v; }
inline bool operator==(CD a, CD b) { ++C.cmp; return a.v == b.v; }
inline bool operator!=(CD a, CD b) { ++C.cmp; return a.v != b.v; }
inline CD sqrt(CD a) { ++C.sqrt_; return CD(std::sqrt(a.v)); }
inline CD exp(CD a) { ++C.exp_; return CD(std::exp(a.v)); }
inline CD erfc(CD a) { ++C.erfc_; return CD(std::erfc(a.v)); }
inline CD pow(CD a, CD b) { ++C.pow_; return CD(std::pow(a.v, b.v)); }
inline CD fabs(CD a) { return CD(std::fabs(a.v)); }
inline CD tanh(CD a) { ++C.other; return CD(std::tanh(a.v)); }
inline CD cosh(CD a) { ++C.other; return CD(std::cosh(a.v)); }
inline CD fmax(CD a, CD b) { ++C.cmp; return CD(std::fmax(a.v, b.v)); }
inline CD fmin(CD a, CD b) { ++C.cmp; return CD(std::fmin(a.v, b.v)); }
inline bool isfinite(CD a) { return std::isfinite(a.v); }
}  // namespace fc

using fc::CD;
using fc::cosh;
using fc::erfc;
using fc::exp;
using fc::fabs;
using fc::fmax;
using fc::fmin;
using fc::isfinite;
using fc::pow;
using fc::sqrt;
using fc::tanh;
#undef isfinite
#define double CD
#include "hgks_oracle.c"
#undef double

static fc::Counters diff(const fc::Counters& b, const fc::Counters& a) {
  fc::Counters d;
  d.add = b.add - a.add, d.mul = b.mul - a.mul, d.div = b.div - a.div, d.sqrt_ = b.sqrt_ - a.sqrt_;
  d.exp_ = b.exp_ - a.exp_, d.erfc_ = b.erfc_ - a.erfc_, d.pow_ = b.pow_ - a.pow_, d.other = b.other - a.other;
  d.cmp = b.cmp - a.cmp;
  return d;
}
static void emit(const char* name, const fc::Counters& d, double per, bool comma) {
  const double flops = (double)(d.add + d.mul + d.div);
  printf("  \"%s\": {\"flops\": %.1f, \"add\": %.1f, \"mul\": %.1f, \"div\": %.1f, \"sqrt\": %.2f, \"exp\": %.2f, "
         "\"erfc\": %.2f, \"pow\": %.2f, \"cmp\": %.1f}%s\n",
         name, flops / per, d.add / per, d.mul / per, d.div / per, d.sqrt_ / per, d.exp_ / per, d.erfc_ / per,
         d.pow_ / per, d.cmp / per, comma ? "," : "");
}

int main() {
  const int n = 16;
  const double PI = 3.14159265358979323846;
  const double gamma = 1.4, c0 = 10.0, p0 = c0 * c0 / gamma, mu = 1.0 / 1600.0;
  or_gas g;
  g.gamma = gamma;
  g.K = or_K(gamma);
  g.prandtl = 1.0;
  g.mu_law = 0;
  g.mu_ref = mu;
  g.T_ref = 1.0;
  g.omega = 0.0;
  g.T_wall = 1.0;
  or_grid gr;
  memset((void*)&gr, 0, sizeof gr);
  const int NG = n + 6;
  for (int d = 0; d < 3; ++d) {
    gr.n[d] = n;
    gr.dx[d] = 2 * PI / n;
    gr.bc[d] = 0;
    gr.stretch[d] = 0;
    gr.lo[d] = -PI;
    gr.hi[d] = PI;
  }
  // TGV, cell-centre values; ghosted layout [5][n+6]^3
  const long gsz = 5L * NG * NG * NG, ncell = (long)n * n * n;
  CD* q = (CD*)calloc(gsz, sizeof(CD));
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const double x = -PI + (i + 0.5) * 2 * PI / n, y = -PI + (j + 0.5) * 2 * PI / n, z = -PI + (k + 0.5) * 2 * PI / n;
        const double U = std::sin(x) * std::cos(y) * std::cos(z), V = -std::cos(x) * std::sin(y) * std::cos(z), W = 0.0;
        const double p = p0 + (std::cos(2 * x) + std::cos(2 * y)) * (std::cos(2 * z) + 2) / 16.0;
        const double rho = p / p0;
        const double cons[5] = {rho, rho * U, rho * V, rho * W, p / (gamma - 1) + 0.5 * rho * (U * U + V * V + W * W)};
        for (int v = 0; v < 5; ++v) q[(((long)v * NG + k + 3) * NG + j + 3) * NG + i + 3] = CD(cons[v]);
      }
  or_fill_ghosts(&g, &gr, q);
  CD* L = (CD*)calloc(5 * ncell, sizeof(CD));
  CD* dL = (CD*)calloc(5 * ncell, sizeof(CD));
  const double dt = 7.0e-3;
  fc::Counters a = fc::C;
  or_operator(&g, &gr, q, dt, L, dL);
  fc::Counters op = diff(fc::C, a);
  // one Gauss-point flux on the TGV scales (a representative input: the operator's own mix)
  CD Wl[5], Wr[5], dWl[3][5], dWr[3][5], dW0[3][5], F[5], dF[5], tau;
  for (int k = 0; k < 5; ++k) {
    Wl[k] = q[(((long)k * NG + 5) * NG + 6) * NG + 7];
    Wr[k] = q[(((long)k * NG + 5) * NG + 6) * NG + 8];
    for (int d = 0; d < 3; ++d) dWl[d][k] = dWr[d][k] = dW0[d][k] = CD(0.01 * (k + 1) * (d + 1));
  }
  a = fc::C;
  or_gp_flux(&g, Wl, dWl, Wr, dWr, dW0, CD(dt), F, dF, &tau);
  fc::Counters gp = diff(fc::C, a);
  CD s5[5] = {CD(1.0), CD(1.1), CD(1.3), CD(1.2), CD(1.05)};
  a = fc::C;
  CD e = or_weno5z_right(s5);
  (void)e;
  fc::Counters we = diff(fc::C, a);
  // S2O4 update arithmetic per cell (Eq. 7): stage 1 + final
  a = fc::C;
  CD qs[5], qn[5], Lc[5], dLc[5], dLs[5];
  for (int k = 0; k < 5; ++k) Lc[k] = dLc[k] = dLs[k] = CD(0.1), qs[k] = CD(1.0);
  or_s2o4_stage1(5, qs, Lc, dLc, CD(dt), qn);
  or_s2o4_final(5, qs, Lc, dLc, dLs, CD(dt), qn);
  fc::Counters up = diff(fc::C, a);
  const double faces = 3.0 * ncell;  // periodic: one face per cell per direction
  printf("{\n  \"source\": \"oracle/flopcount.cpp: hgks_oracle.c compiled with a counting double (TGV 16^3, one operator evaluation)\",\n");
  emit("operator_per_cell_per_stage", op, (double)ncell, true);
  emit("operator_per_face_per_stage", op, faces, true);
  emit("gp_flux_per_gauss_point", gp, 1.0, true);
  emit("weno5z_per_edge", we, 1.0, true);
  emit("s2o4_update_per_cell", up, 5.0, true);
  const double per_cell_update = 2.0 * (double)(op.add + op.mul + op.div) / ncell + (double)(up.add + up.mul + up.div) / 5.0;
  printf("  \"flops_per_cell_update\": %.1f,\n  \"note\": \"flops = add + mul + div (sqrt, exp, erfc, pow counted "
         "separately, not as flops); per cell-update = 2 operator evaluations (stages) + the Eq. (7) updates\"\n}\n",
         per_cell_update);
  free(q);
  free(L);
  free(dL);
  return 0;
}
