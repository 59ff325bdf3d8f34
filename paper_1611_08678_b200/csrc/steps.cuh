// steps.cuh — the single-step public ops on the device.
//
// step_predictor / step_corrector (reference serial.py:74-111) recompute one
// step of the PECE scheme from a completed prefix f_0..f_n of a trajectory:
//   yP = y0 + h^a * sum_{k=0..n} b_{n-k} f_k                     (:74-83)
//   fP = f(t_{n+1}, y_pred)   (y_pred given, or yP)
//   y  = y0 + h^a * ((c_n f_0 + sum_{k=1..n} a_{n-k} f_k) + fP/Gamma(a+2))
//                                                                (:86-111)
// Here many steps n are evaluated at once, one warp per requested n: lanes
// stride over the history (coalesced rows of the compact f cache), each lane
// keeps FMA partial sums, a fixed xor-butterfly reduces them (deterministic),
// and lane 0 assembles the step with round-to-nearest operations in the
// reference's order (no contraction).  With every n requested this is the
// a-posteriori consistency check of a whole trajectory.
#pragma once
#include "device_common.cuh"

namespace fabm {

enum StepErr : int { STEP_OK = 0, STEP_PRED_NONFINITE = 1, STEP_RHS_NONFINITE = 2 };

struct StepParams {
  long long count;        // requested steps
  const long long* ns;    // [count] step indices n (0 <= n < N, validated on the host)
  const double* F;        // f cache rows 0.., compact (rows x D)
  const double* wb;       // b_j, a_j, c_j (j <= max n)
  const double* wa;
  const double* wc;
  const double* y0;       // [D]
  const double* ypred;    // [count x D] predicted states for the corrector, or null (use yP)
  double h, ha, ig;       // step, h^alpha, 1/Gamma(alpha+2)
  double params[kMaxParams];
  double* yp_out;         // [count x D] or null
  double* y_out;          // [count x D] or null
  int* err;               // [count]
};

template <int SYS, int D>
__global__ void __launch_bounds__(256) step_pc_kernel(StepParams P) {
  const long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= P.count) return;
  const long long n = P.ns[i];
  double sp[D], sc[D];
#pragma unroll
  for (int c = 0; c < D; ++c) { sp[c] = 0.0; sc[c] = 0.0; }
  for (long long k = lane; k <= n; k += 32) {
    const double wb = P.wb[n - k];
    const double wa = k >= 1 ? P.wa[n - k] : 0.0;  // the corrector interior starts at k = 1
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double f = P.F[k * D + c];
      sp[c] = fma(wb, f, sp[c]);
      sc[c] = fma(wa, f, sc[c]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      sp[c] += __shfl_xor_sync(0xffffffffu, sp[c], o);
      sc[c] += __shfl_xor_sync(0xffffffffu, sc[c], o);
    }
  if (lane != 0) return;
  double y0[D], yp[D], yq[D], fp[D], y[D];
#pragma unroll
  for (int c = 0; c < D; ++c) {
    y0[c] = P.y0[c];
    yp[c] = add_rn(y0[c], mul_rn(P.ha, sp[c]));  // problem.y0 + ha * S, serial.py:83
  }
  if (P.yp_out)
#pragma unroll
    for (int c = 0; c < D; ++c) P.yp_out[i * D + c] = yp[c];
  bool ok = true;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    yq[c] = P.ypred ? P.ypred[i * D + c] : yp[c];
    ok = ok && isfinite(yq[c]);
  }
  int err = ok ? STEP_OK : STEP_PRED_NONFINITE;  // serial.py:94-95
  if (ok) {
    const double t1 = mul_rn(static_cast<double>(n + 1), P.h);  // (n + 1) * h, serial.py:100
    Rhs<SYS, D>::eval(t1, yq, fp, P.params);
    err = all_finite<D>(fp) ? STEP_OK : STEP_RHS_NONFINITE;  // serial.py:104-105
  }
#pragma unroll
  for (int c = 0; c < D; ++c) {
    // acc = c_n f_0; acc += dot; acc += ig * fP; y0 + ha * acc   (serial.py:106-111)
    double acc = mul_rn(P.wc[n], P.F[c]);
    if (n >= 1) acc = add_rn(acc, sc[c]);
    acc = add_rn(acc, mul_rn(P.ig, err == STEP_OK ? fp[c] : 0.0));
    y[c] = err == STEP_OK ? add_rn(y0[c], mul_rn(P.ha, acc)) : __longlong_as_double(0x7ff8000000000000ll);
  }
  if (P.y_out)
#pragma unroll
    for (int c = 0; c < D; ++c) P.y_out[i * D + c] = y[c];
  P.err[i] = err;
}

}  // namespace fabm
