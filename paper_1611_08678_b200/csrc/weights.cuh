// weights.cuh — device generation of the ABM quadrature weights.
//
// Reference: precompute_weights (core.py:134-154) evaluates
//   b_n = ((n+1)^a - n^a) / G(a+1)
//   a_n = ((n+2)^p - 2 (n+1)^p + n^p) / G(a+2),          p = a + 1
//   c_n = (n^p - (n-a)(n+1)^a) / G(a+2)
// with NumPy's vector pow.  Those differences cancel catastrophically for
// large n (a_n relative error 3.8e-5 at n=1e6).  Two modes:
//   FORMULA  — the same expressions (same operator order, no contraction)
//              with CUDA's pow; for cross-checking the reference formula.
//   ACCURATE — cancellation-free forms, one thread per n:
//     b_n = n^a expm1(a log1p(1/n)) / G1                         (n >= 1)
//     a_n = 2 x^(a-1) sum_{k>=1} C(p,2k) x^(2-2k) / G2,  x = n+1 (n >= 1)
//           (all series terms positive for 0 < a <= 1)
//     c_n = n^(a-1) sum_{k>=2} [a C(a,k-1) - C(a,k)] n^(2-k) / G2 (n >= 2)
//     b_0 = 1/G1, a_0 = 2 expm1(a ln 2)/G2, c_0 = a/G2,
//     c_1 = (a - (1-a) expm1(a ln 2)) / G2
//   Checked against 60-digit mpmath in tests/test_weights_accuracy.py.
#pragma once
#include "device_common.cuh"

namespace fabm {

constexpr double kLn2 = 0.69314718055994530942;

__device__ __forceinline__ double weight_b_accurate(double al, double g1, long long n) {
  if (n == 0) return 1.0 / g1;
  const double x = static_cast<double>(n);
  return pow(x, al) * expm1(al * log1p(1.0 / x)) / g1;
}

__device__ __forceinline__ double weight_a_accurate(double al, double g2, long long n) {
  if (n == 0) return 2.0 * expm1(al * kLn2) / g2;
  const double p = al + 1.0;
  const double x = static_cast<double>(n + 1);
  const double u2 = 1.0 / (x * x);
  double coef = 0.5 * p * (p - 1.0);  // C(p, 2)
  double s = coef, upow = 1.0;
  for (int k = 1; k < 400; ++k) {
    // C(p, 2k+2) = C(p, 2k) (p-2k)(p-2k-1) / ((2k+1)(2k+2))
    coef *= (p - 2.0 * k) * (p - 2.0 * k - 1.0) / ((2.0 * k + 1.0) * (2.0 * k + 2.0));
    upow *= u2;
    const double term = coef * upow;
    s += term;
    if (fabs(term) <= 1e-18 * fabs(s)) break;
  }
  return 2.0 * pow(x, al - 1.0) * s / g2;
}

__device__ __forceinline__ double weight_c_accurate(double al, double g2, long long n) {
  if (n == 0) return al / g2;
  if (n == 1) return (al - (1.0 - al) * expm1(al * kLn2)) / g2;
  const double x = static_cast<double>(n);
  const double v = 1.0 / x;
  // C(a,1) = a, C(a,2) = a(a-1)/2 ; D_k = a C(a,k-1) - C(a,k)
  double cprev = al;                       // C(a, k-1) at k = 2
  double ccur = 0.5 * al * (al - 1.0);     // C(a, k)   at k = 2
  double s = al * cprev - ccur, vpow = 1.0;
  for (int k = 3; k < 600; ++k) {
    cprev = ccur;
    ccur = cprev * (al - k + 1.0) / k;
    vpow *= v;
    const double term = (al * cprev - ccur) * vpow;
    s += term;
    if (fabs(term) <= 1e-18 * fabs(s)) break;
  }
  return pow(x, al - 1.0) * s / g2;
}

// the reference expressions, operator by operator (core.py:149-151)
__device__ __forceinline__ void weights_formula(double al, double g1, double g2, long long n,
                                                double& b, double& a, double& c) {
  const double x = static_cast<double>(n);
  const double p = al + 1.0;
  b = __ddiv_rn(sub_rn(pow(x + 1.0, al), pow(x, al)), g1);
  a = __ddiv_rn(add_rn(sub_rn(pow(x + 2.0, p), mul_rn(2.0, pow(x + 1.0, p))), pow(x, p)), g2);
  c = __ddiv_rn(sub_rn(pow(x, p), mul_rn(sub_rn(x, al), pow(x + 1.0, al))), g2);
}

__global__ void weights_kernel(double al, double g1, double g2, long long len, int mode,
                               double* __restrict__ b, double* __restrict__ a, double* __restrict__ c) {
  for (long long n = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; n < len;
       n += static_cast<long long>(gridDim.x) * blockDim.x) {
    double vb, va, vc;
    if (mode == 1) {
      weights_formula(al, g1, g2, n, vb, va, vc);
    } else {
      vb = weight_b_accurate(al, g1, n);
      va = weight_a_accurate(al, g2, n);
      vc = weight_c_accurate(al, g2, n);
    }
    b[n] = vb;
    a[n] = va;
    c[n] = vc;
  }
}

// one weight table per trajectory: W[t] = {b[0..len), a[0..len), c[0..len)}
__global__ void weights_batch_kernel(const double* __restrict__ alphas, const double* __restrict__ g1,
                                     const double* __restrict__ g2, int T, long long len,
                                     double* __restrict__ W) {
  const long long total = static_cast<long long>(T) * len;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(q / len);
    const long long n = q % len;
    double* w = W + static_cast<long long>(t) * 3 * len;
    const double al = alphas[t];
    w[n] = weight_b_accurate(al, g1[t], n);
    w[len + n] = weight_a_accurate(al, g2[t], n);
    w[2 * len + n] = weight_c_accurate(al, g2[t], n);
  }
}

}  // namespace fabm
