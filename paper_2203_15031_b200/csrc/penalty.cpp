// Penalty levels of §2.2 (host helpers; not on the device path).
//   lambda_univ = sqrt(2 log(p-1) / n)
//   lambda_ub   = A sqrt(4 log p / n)
//   lambda_pb   = A L_n(k/p), L_n(t) = Phi^{-1}(1-t)/sqrt(n),
//                 k the real root of k = L_1^4(k/p) + 2 L_1^2(k/p) (bisection)
// The upper-tail normal quantile is obtained by Newton iterations on
// Q(x) = erfc(x / sqrt 2) / 2 (std::erfc), safeguarded by a bracket.
#include <cmath>
#include <cstdint>
#include <limits>

#include "spmesl.h"

namespace {

double upper_tail(double x) { return 0.5 * std::erfc(x / std::sqrt(2.0)); }

// x with Q(x) = u, 0 < u < 1.
double inv_upper_tail(double u) {
  if (!(u > 0.0 && u < 1.0)) return std::numeric_limits<double>::quiet_NaN();
  if (u > 0.5) return -inv_upper_tail(1.0 - u);
  // bracket [0, hi] with Q(0) = 0.5 >= u > Q(hi)
  double lo = 0.0, hi = 1.0;
  while (upper_tail(hi) > u) { lo = hi; hi *= 2.0; }
  double x = 0.5 * (lo + hi);
  const double inv_sqrt_2pi = 0.3989422804014327;
  for (int it = 0; it < 200; ++it) {
    const double q = upper_tail(x);
    if (q > u) lo = x; else hi = x;
    const double pdf = inv_sqrt_2pi * std::exp(-0.5 * x * x);
    double xn = x + (q - u) / pdf;                      // Newton step on Q(x) - u
    if (!(xn > lo && xn < hi)) xn = 0.5 * (lo + hi);    // keep inside the bracket
    if (std::fabs(xn - x) <= 1e-15 * std::fmax(1.0, std::fabs(x))) { x = xn; break; }
    x = xn;
  }
  return x;
}

// L_1(t) = Phi^{-1}(1 - t) = x with Q(x) = t
double L1(double t) { return inv_upper_tail(t); }

}  // namespace

extern "C" {

double spmesl_lambda_univ(int64_t n, int64_t p) {
  if (n < 1 || p < 3) return std::numeric_limits<double>::quiet_NaN();
  return std::sqrt(2.0 * std::log((double)(p - 1)) / (double)n);
}

double spmesl_lambda_ub(int64_t n, int64_t p, double A) {
  if (n < 1 || p < 2 || !(A > 0.0)) return std::numeric_limits<double>::quiet_NaN();
  return A * std::sqrt(4.0 * std::log((double)p) / (double)n);
}

double spmesl_solve_k(int64_t p) {
  if (p < 3) return std::numeric_limits<double>::quiet_NaN();
  const double P = (double)p;
  auto f = [&](double k) {
    const double l = L1(k / P);
    return k - l * l * l * l - 2.0 * l * l;
  };
  double lo = 1e-9 * P, hi = 0.5 * P;   // f(lo) < 0 < f(hi) = p/2
  double flo = f(lo);
  if (!(flo < 0.0)) return std::numeric_limits<double>::quiet_NaN();
  for (int it = 0; it < 300; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (f(mid) < 0.0) lo = mid; else hi = mid;
    if (hi - lo <= 1e-13 * hi) break;
  }
  return 0.5 * (lo + hi);
}

double spmesl_lambda_pb(int64_t n, int64_t p, double A) {
  if (n < 1 || p < 3 || !(A > 0.0)) return std::numeric_limits<double>::quiet_NaN();
  const double k = spmesl_solve_k(p);
  return A * L1(k / (double)p) / std::sqrt((double)n);
}

}  // extern "C"
