// oracles.cuh — analytic oracles on the device.
//
// mittag_leffler_kernel: E_alpha(z) for a batch of (alpha, z) pairs, one
// thread each, with the reference's algorithm (verify.py:28-64): the power
// series sum_k z^k / Gamma(alpha k + 1) with terms evaluated in log space,
//     term_k = exp(k log|z| - lgamma(alpha k + 1)),  sign (-1)^k for z < 0,
// Kahan-compensated summation, stopping at the first k >= 5 with
// |term| < 1e-16 |total|, at most 20000 terms.  Status per pair:
//     0 ok, 1 invalid argument (ValueError: alpha not in (0, 1], |z| > 10 or
//     z not finite), 2 overflow (the reference returns +-inf: the sign of
//     the overflowing term), 3 no convergence (ArithmeticError).
// exp/lgamma are CUDA's, not glibc's, so values agree with the reference to
// the series' conditioning (sum |term_k| * a few ulp), which the tests state.
#pragma once

namespace fabm_oracle {

constexpr int kMlMaxTerms = 20000;

__global__ void mittag_leffler_kernel(const double* __restrict__ alpha, const double* __restrict__ z, long long n,
                                      double* __restrict__ out, int* __restrict__ code) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = alpha[i], x = z[i];
  if (!(a > 0.0 && a <= 1.0) || !isfinite(x) || fabs(x) > 10.0) {  // verify.py:40-43
    out[i] = nan("");
    code[i] = 1;
    return;
  }
  if (x == 0.0) {  // verify.py:44-45
    out[i] = 1.0;
    code[i] = 0;
    return;
  }
  const double log_az = log(fabs(x));
  const bool negative = x < 0.0;
  double total = 0.0, comp = 0.0;
  for (int k = 0; k < kMlMaxTerms; ++k) {
    double term = exp(static_cast<double>(k) * log_az - lgamma(a * static_cast<double>(k) + 1.0));
    if (isinf(term)) {  // math.exp raised OverflowError (verify.py:52-53)
      out[i] = (negative && (k & 1)) ? -INFINITY : INFINITY;
      code[i] = 2;
      return;
    }
    if (negative && (k & 1)) term = -term;
    const double y = __dsub_rn(term, comp);  // Kahan step, verify.py:56-59 (no contraction)
    const double t = __dadd_rn(total, y);
    comp = __dsub_rn(__dsub_rn(t, total), y);
    total = t;
    if (k >= 5 && fabs(term) < 1e-16 * fabs(total)) {
      out[i] = total;
      code[i] = 0;
      return;
    }
  }
  out[i] = total;
  code[i] = 3;
}

}  // namespace fabm_oracle
