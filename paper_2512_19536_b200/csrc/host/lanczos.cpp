// Lanczos condition estimate from the PCG coefficients
// (/root/reference/proj/src/krylov.cpp:85-103): tridiagonal with
//   diag_k = 1/alpha_k + beta_{k-1}/alpha_{k-1}, offdiag_k = sqrt(beta_k)/alpha_k,
// extreme eigenvalues by Sturm-sequence bisection (the reference uses Eigen's
// tridiagonal QR; both are accurate to rounding). Host-side, O(m log) per
// bound, exactly as cheap as the reference's O(m^2).
#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>

namespace pdg {

namespace {
// number of eigenvalues < x
int sturm_count(const std::vector<double>& d, const std::vector<double>& e2, double x) {
  int count = 0;
  double q = d[0] - x;
  if (q < 0.0) ++count;
  for (std::size_t i = 1; i < d.size(); ++i) {
    const double prev = q == 0.0 ? std::numeric_limits<double>::min() * 1e3 : q;
    q = d[i] - x - e2[i - 1] / prev;
    if (q < 0.0) ++count;
  }
  return count;
}

double kth_eigenvalue(const std::vector<double>& d, const std::vector<double>& e2, double lo,
                      double hi, int k) {
  for (int it = 0; it < 300; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    if (sturm_count(d, e2, mid) > k) hi = mid;
    else lo = mid;
  }
  return 0.5 * (lo + hi);
}
}  // namespace

bool lanczos_condition(const double* alpha, const double* beta, int m, double* kappa) {
  if (m < 2) return false;
  std::vector<double> d(m), e(m - 1), e2(m - 1);
  d[0] = 1.0 / alpha[0];
  for (int k = 1; k < m; ++k) d[k] = 1.0 / alpha[k] + beta[k - 1] / alpha[k - 1];
  for (int k = 0; k + 1 < m; ++k) {
    e[k] = std::sqrt(beta[k]) / alpha[k];
    e2[k] = e[k] * e[k];
  }
  double lo = d[0], hi = d[0];
  for (int i = 0; i < m; ++i) {
    const double r = (i > 0 ? std::abs(e[i - 1]) : 0.0) + (i + 1 < m ? std::abs(e[i]) : 0.0);
    lo = std::min(lo, d[i] - r);
    hi = std::max(hi, d[i] + r);
  }
  const double pad = 1e-300 + 1e-15 * std::max(std::abs(lo), std::abs(hi));
  lo -= pad;
  hi += pad;
  if (!std::isfinite(lo) || !std::isfinite(hi)) return false;
  const double lmin = kth_eigenvalue(d, e2, lo, hi, 0);
  const double lmax = kth_eigenvalue(d, e2, lo, hi, m - 1);
  if (!(lmin > 0.0)) return false;  // numerically defective tridiagonal
  *kappa = lmax / lmin;
  return true;
}

}  // namespace pdg

extern "C" int pdg_condition_estimate(const double* alphas, const double* betas, int m, double* kappa) {
  return pdg::lanczos_condition(alphas, betas, m, kappa) ? 1 : 0;
}
