// wald.cu — edge significance under the empty-graph null (Theorem 5, P:768-; Corollary 10,
// P:877-885) and the critical magnitude used by the threshold mode of ggm_sparse_precision
// ("keep only the edges that are statistically significant (p = 0.05) after the
// Bonferroni correction").  Host-side scalars: the kernel only sees tau.
//
// Single modality (Cor. 10): z = sqrt(d_\l) · sigma² · psi / 2 ~ N(0, 1) under the null;
// p_raw = 2 (1 - Phi(|z|)); p_bonferroni = min(1, n_tests · p_raw).  The critical magnitude
// is the |psi| above which p_bonferroni < alpha:
//   tau = 2 · Phi^-1(1 - alpha / (2 n_tests)) / (sqrt(d_\l) · sigma²).
#include <cmath>
#include <cstdint>

#include "ggm_internal.h"

namespace {

// upper tail Q(z) = 1 - Phi(z) in double precision (erfc keeps relative accuracy far out)
double upper_tail(double z) { return 0.5 * std::erfc(z / std::sqrt(2.0)); }

// z with Q(z) = q for q in (0, 0.5]: Newton on log Q (its derivative -phi/Q), from the
// upper bound sqrt(-2 log q) of the root; converges in a handful of steps.
double inv_upper_tail(double q) {
  double z = std::sqrt(-2.0 * std::log(q));
  const double lq = std::log(q);
  for (int it = 0; it < 60; ++it) {
    const double Q = upper_tail(z);
    const double phi = std::exp(-0.5 * z * z) / std::sqrt(2.0 * M_PI);
    const double step = (std::log(Q) - lq) / (phi / Q);  // g / (-g'), g = log Q - log q
    z += step;
    if (std::fabs(step) <= 1e-15 * std::fmax(1.0, std::fabs(z))) break;
  }
  return z;
}

}  // namespace

extern "C" ggm_status ggm_wald_edge(double psi, int64_t d_rest, double sigma2, int64_t n_tests,
                                    double* z, double* p_raw, double* p_bonferroni) {
  if (d_rest < 1 || !(sigma2 > 0.0) || n_tests < 1 || !std::isfinite(psi))
    return ggm::fail(GGM_ERR_INVALID_ARGUMENT, "wald: d_rest >= 1, sigma2 > 0, n_tests >= 1");
  const double zz = std::sqrt((double)d_rest) * sigma2 * psi / 2.0;
  const double pr = std::fmin(1.0, 2.0 * upper_tail(std::fabs(zz)));
  if (z) *z = zz;
  if (p_raw) *p_raw = pr;
  if (p_bonferroni) *p_bonferroni = std::fmin(1.0, (double)n_tests * pr);
  return GGM_OK;
}

extern "C" ggm_status ggm_wald_threshold(int64_t d_rest, double sigma2, double alpha,
                                         int64_t n_tests, double* tau) {
  if (d_rest < 1 || !(sigma2 > 0.0) || !(alpha > 0.0 && alpha < 1.0) || n_tests < 1 || !tau)
    return ggm::fail(GGM_ERR_INVALID_ARGUMENT,
                     "wald threshold: d_rest >= 1, sigma2 > 0, 0 < alpha < 1, n_tests >= 1");
  const double zc = inv_upper_tail(alpha / (2.0 * (double)n_tests));
  *tau = 2.0 * zc / (std::sqrt((double)d_rest) * sigma2);
  return GGM_OK;
}
