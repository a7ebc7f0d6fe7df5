// Development aid (not part of the product or the tests): the device Gauss-point flux compiled
// for the HOST so the kinetic algebra can be checked against the oracle without a GPU.
//   nvcc -O2 -std=c++17 -Xcompiler -fPIC -shared -o /tmp/libhostflux.so tools/host_flux_check.cu
#include "../paper_2207_01173_b200/csrc/gks_device.cuh"
extern "C" void host_gp_flux(const double* in, long n, double gamma, double mu, double dt, double* out,
                             int mu_law, double T_ref, double omega, double prandtl) {
  hgks::GasK<double> g;
  g.K = (5.0 - 3.0 * gamma) / (gamma - 1.0);
  g.gamma = gamma; g.mu_ref = mu; g.T_ref = T_ref; g.omega = omega; g.mu_law = mu_law;
  g.prf = 1.0 / prandtl - 1.0;
  g.ik3 = 1.0 / (g.K + 3.0);
  for (long e = 0; e < n; ++e) {
    const double* r = in + 55 * e;
    double Wl[5], Wr[5], dWl[3][5], dWr[3][5], dW0[3][5];
    for (int k = 0; k < 5; ++k) {
      Wl[k] = r[k]; Wr[k] = r[5 + k];
      for (int i = 0; i < 3; ++i) { dWl[i][k] = r[10 + 5 * i + k]; dWr[i][k] = r[25 + 5 * i + k]; dW0[i][k] = r[40 + 5 * i + k]; }
    }
    double F[5], dF[5], tau;
    if (prandtl != 1.0) hgks::gp_flux<double, true, true>(g, Wl, Wr, dWl, dWr, dW0, dt, F, dF, tau);
    else hgks::gp_flux<double, true, false>(g, Wl, Wr, dWl, dWr, dW0, dt, F, dF, tau);
    for (int k = 0; k < 5; ++k) { out[11 * e + k] = F[k]; out[11 * e + 5 + k] = dF[k]; }
    out[11 * e + 10] = tau;
  }
}
