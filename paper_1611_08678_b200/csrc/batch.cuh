// batch.cuh — many independent trajectories (BASELINE config 4: the
// fractional financial system swept over 4096 orders alpha, N = 1e5).
//
// The reference integrates each problem with solve_serial (serial.py:114-176);
// a sweep is a loop of such calls.  Here one persistent kernel (one CTA per
// SM, 16 warps) integrates the whole sweep.  Work is cut into tickets taken
// from one global counter, in ROUNDS J = 0 .. nb-1 (block J = steps
// 128J .. 128J+127 of every trajectory):
//   * PULL units (t, J, s), s < S_J: the bulk of block J's 128 targets from
//     one segment of source blocks (pull_bounds: a body cut in pieces of G
//     blocks, then a short tail ending at block J-1) -- Toeplitz chunks on the
//     FP64 tensor cores (bulk_dmma.cuh) in ascending order -- into a partial
//     slot part[t][J mod 2][s];
//   * STEP units (t, J): the partials summed in slot order s = 0, 1, ..., then
//     the 128 steps of the block: all 32 lanes run the sequential chain
//     (serial.py:150-170) redundantly; lane l holds the sums of steps
//     JB+4l..JB+4l+3 and pushes every new f_k into them (in-block window).
// Within a round all pulls (s-major) precede all steps.  A tail pull waits
// for step (t, J-1), a body pull only for step (t, J-2) (earlier tickets, so
// their warps are running); a step waits for its round's pulls (earlier
// tickets too): no deadlock.
// Splitting the pull over S_J warps keeps each trajectory's critical path
// short (<= G chunks + 128 steps per round), so a few hundred trajectories
// per GPU -- the 8-GPU share of the config 4 sweep -- still fill the machine.
// The segment bounds depend only on J, so a trajectory's result is bitwise
// independent of its batch neighbours and of the launch.
#pragma once
#include "engine.cuh"

namespace fabm {

struct BatchParams {
  int T;                    // trajectories
  int nb;                   // blocks per trajectory
  long long N;              // steps
  long long WL;             // weight row length per trajectory (nb*B + 2B)
  double h;
  const double* ha;         // [T] h^alpha
  const double* ig;         // [T] 1/Gamma(alpha+2)
  const double* y0;         // [T][kMaxDim]
  const double* params;     // [T][kMaxParams]
  const double* W;          // [T][3][WL]: b, a, c
  double* F;                // [T][(nb+1)*B][DS]
  double* Y;                // [T][N+1][D] or null
  double* Fc;               // [T][N+1][D] or null
  double* ylast;            // [T][D]: y_N
  int* next_block;          // [T]: blocks completed (release)
  int* err_kind;            // [T]
  long long* err_step;      // [T]
  unsigned long long* ticket;
  unsigned long long timeout_ns;
  DevCtrl* ctrl;
  int G;                    // pull segment length (source blocks)
  int S_max;                // pull segments of the largest round
  const long long* round_start;  // [nb + 1]: first ticket of round J
  const long long* pull_cum;     // [nb]: pull units of the rounds j <= J with j = J (mod 2)
  double* part;             // [T][2][S_max][B * 2 * DS]: partial bulk sums by round parity (DMMA lane-major layout)
  int* pulls_done;          // [T][2]: completed pull units by round parity (cumulative)
};

// Round J's pull segments: the BODY [0, J - tl) in pieces of G source blocks,
// then the TAIL [J - tl, J), tl = min(J, kBatchTail).  Only the tail needs the
// block the previous step unit has just finished; the body pulls of round J
// run while the steps of round J-1 do (their slots are double-buffered by
// round parity), so a trajectory's critical path per round is a tail of
// <= kBatchTail chunks plus its 128 steps.  Bounds depend on J only.
#ifndef FABM_BATCH_TAIL
#define FABM_BATCH_TAIL 2
#endif
constexpr int kBatchTail = FABM_BATCH_TAIL;
__host__ __device__ __forceinline__ int batch_tail(int J) { return J < kBatchTail ? J : kBatchTail; }
__host__ __device__ __forceinline__ int pull_units(int J, int G) {
  const int tl = batch_tail(J);
  return (J - tl + G - 1) / G + (tl > 0 ? 1 : 0);
}
__host__ __device__ __forceinline__ void pull_bounds(int J, int s, int G, int& lo, int& hi) {
  const int tl = batch_tail(J);
  const int nbody = (J - tl + G - 1) / G;
  if (s < nbody) {
    lo = s * G;
    hi = (s + 1) * G < J - tl ? (s + 1) * G : J - tl;
  } else {
    lo = J - tl;
    hi = J;
  }
}

template <int D>
__device__ __forceinline__ double* part_slot(const BatchParams& P, int t, int parity, int s) {
  return P.part + ((static_cast<long long>(t) * 2 + parity) * P.S_max + s) * kB * 2 * Stride<D>::value;
}

// pull unit (t, J, s): sources [lo, hi) into the targets of block J
template <int D>
__device__ void batch_pull(const BatchParams& P, DmmaSmem<D>& A, int t, int J, int s, int lane) {
  constexpr int DS = Stride<D>::value;
  const double* wb = P.W + static_cast<long long>(t) * 3 * P.WL;
  const double* wa = wb + P.WL;
  const double* F = P.F + static_cast<long long>(t) * (P.nb + 1) * kB * DS;
  DmmaAcc<D> acc;
  dmma_zero<D>(acc);
  int lo, hi;
  pull_bounds(J, s, P.G, lo, hi);
  for (int I = lo; I < hi; ++I) dmma_chunk<D, true>(wb, wa, F, A, J * kB, I * kB, J * kB, lane, acc);
  dmma_spill<D>(part_slot<D>(P, t, J & 1, s), 0, lane, acc);
}

// spin until *flag >= want (acquire); false on abort or watchdog expiry
__device__ __forceinline__ bool batch_wait(const BatchParams& P, const int* flag, long long want, int lane) {
  int v = 0;
  const unsigned long long w0 = global_ns();
  for (;;) {
    if (lane == 0) v = ld_acquire_gpu(flag);
    v = __shfl_sync(0xffffffffu, v, 0);
    if (v >= want) break;
    if (*((volatile int*)&P.ctrl->abort)) return false;
    if (global_ns() - w0 > P.timeout_ns) {
      if (lane == 0) ctrl_abort(P.ctrl, ERR_TIMEOUT, KIND_NONE, -1, 0.0);
      return false;
    }
    __nanosleep(200);
  }
  __syncwarp();
  return true;
}

// step unit (t, J); false if the run was aborted while waiting for the pulls
template <int SYS, int D>
__device__ bool batch_unit(const BatchParams& P, DmmaSmem<D>& A, int t, int J, int lane) {
  constexpr int DS = Stride<D>::value;
  const long long N = P.N;
  const double* wb = P.W + static_cast<long long>(t) * 3 * P.WL;
  const double* wa = wb + P.WL;
  const double* wc = wa + P.WL;
  double* F = P.F + static_cast<long long>(t) * (P.nb + 1) * kB * DS;
  double* Y = P.Y ? P.Y + static_cast<long long>(t) * (N + 1) * D : nullptr;
  double* Fc = P.Fc ? P.Fc + static_cast<long long>(t) * (N + 1) * D : nullptr;
  const double* prm = P.params + static_cast<long long>(t) * kMaxParams;
  double params[kMaxParams];
#pragma unroll
  for (int i = 0; i < kMaxParams; ++i) params[i] = prm[i];
  double y0[D];
#pragma unroll
  for (int c = 0; c < D; ++c) y0[c] = P.y0[t * kMaxDim + c];
  const double ha = P.ha[t], ig = P.ig[t];
  const long long JB = static_cast<long long>(J) * kB;

  // ---- 1. the bulk of sources I < J: the round's partials summed in slot
  // order (each an ascending DMMA chain), re-dealt through shared memory from
  // the DMMA layout to the stepping layout (lane l: steps 4l..4l+3)
  double accP[kR][D], accC[kR][D];
  {
    // total = ((p_0 + p_1) + ...) + p_{S_J - 1} over the round's pull units
    DmmaAcc<D> acc;
    dmma_zero<D>(acc);
    const int np = pull_units(J, P.G);
    if (!batch_wait(P, &P.pulls_done[2 * t + (J & 1)], __ldg(P.pull_cum + J), lane)) return false;
    // no pull of a later round of this parity can have counted yet (it waits for this step)
    FABM_CHECK(P, lane != 0 || ld_relaxed_gpu(&P.pulls_done[2 * t + (J & 1)]) == __ldg(P.pull_cum + J));
    if (np > 0) dmma_reload<D>(part_slot<D>(P, t, J & 1, 0), 0, lane, acc);
    for (int sg = 1; sg < np; ++sg) {
      DmmaAcc<D> pa;
      dmma_reload<D>(part_slot<D>(P, t, J & 1, sg), 0, lane, pa);
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < D; ++c)
#pragma unroll
          for (int w = 0; w < 2; ++w)
#pragma unroll
            for (int e = 0; e < 2; ++e) acc[h][c][w][e] = add_rn(acc[h][c][w][e], pa[h][c][w][e]);
    }
    __syncwarp();
    double* rows = &A.f[0][0];  // [B][2][D]
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int tt = dmma_target(lane, h, e);
#pragma unroll
        for (int c = 0; c < D; ++c) {
          rows[(tt * 2 + 0) * D + c] = acc[h][c][0][e];
          rows[(tt * 2 + 1) * D + c] = acc[h][c][1][e];
        }
      }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < kR; ++r)
#pragma unroll
      for (int c = 0; c < D; ++c) {
        accP[r][c] = rows[((kR * lane + r) * 2 + 0) * D + c];
        accC[r][c] = rows[((kR * lane + r) * 2 + 1) * D + c];
      }
    __syncwarp();
  }

  // ---- 2. state at the block start: f_JB (and f_0), first-node terms
  double f0[D], fc[D];
  if (J == 0) {
    Rhs<SYS, D>::eval(0.0, y0, f0, params);
#pragma unroll
    for (int c = 0; c < D; ++c) fc[c] = f0[c];
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < D; ++c) {
        F[c] = f0[c];
        if (Y) Y[c] = y0[c];
        if (Fc) Fc[c] = f0[c];
      }
    }
    if (any_nonfinite<D>(f0)) {
      if (lane == 0) { P.err_kind[t] = KIND_INITIAL; P.err_step[t] = 0; }
      return true;
    }
  } else {
#pragma unroll
    for (int c = 0; c < D; ++c) { f0[c] = __ldcg(F + c); fc[c] = __ldcg(F + JB * DS + c); }
  }
  // in-block weights: tb[j + 128] = b_j for 1 <= j < B, 0 otherwise (A.w is free now)
  double* tb = &A.w[0][0];
  double* ta = &A.w[1][0];
  for (int i = lane; i < 2 * kB; i += 32) {
    const int j = i - kB;
    tb[i] = (j >= 1) ? __ldg(wb + j) : 0.0;
    ta[i] = (j >= 1) ? __ldg(wa + j) : 0.0;
  }
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const long long m = JB + kR * lane + r;
    // J >= 1: the bulk includes k = 0 in the a-sum -> (c_m - a_m) f0; J = 0:
    // the window excludes k = 0 from the a-sum -> c_m f0
    const double cf = m < N ? (J >= 1 ? __ldg(wc + m) - __ldg(wa + m) : __ldg(wc + m)) : 0.0;
#pragma unroll
    for (int c = 0; c < D; ++c) accC[r][c] = add_rn(accC[r][c], mul_rn(cf, f0[c]));
  }
  __syncwarp();
  // f_JB (the newest row when the block starts) enters the sums of the
  // block's later steps; k = 0 is not part of the corrector interior
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const double w1 = tb[kR * lane + r + kB];
    const double w2 = J == 0 ? 0.0 : ta[kR * lane + r + kB];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      accP[r][c] = fma(w1, fc[c], accP[r][c]);
      accC[r][c] = fma(w2, fc[c], accC[r][c]);
    }
  }
  const double b0 = __ldg(wb), a0 = __ldg(wa);

  // ---- 3. the sequential chain over the block
  const long long nend = (JB + kB < N) ? JB + kB : N;
  int ekind = KIND_NONE;
  long long estep = -1;
  for (long long n = JB; n < nend; ++n) {
    const int i = static_cast<int>(n - JB);
    const int owner = i >> 2, rr = i & 3;
    // pre-sums of step n from the owner lane (r is warp-uniform)
    double pP[D], pC[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double vp = accP[0][c], vc = accC[0][c];
#pragma unroll
      for (int r = 1; r < kR; ++r) {
        vp = rr == r ? accP[r][c] : vp;
        vc = rr == r ? accC[r][c] : vc;
      }
      pP[c] = __shfl_sync(0xffffffffu, vp, owner);
      pC[c] = __shfl_sync(0xffffffffu, vc, owner);
    }
    const double t1 = static_cast<double>(n + 1) * P.h;
    const double a0e = n >= 1 ? a0 : 0.0;
    double yP[D], fP[D], y1[D], f1[D];
#pragma unroll
    for (int c = 0; c < D; ++c) yP[c] = add_rn(mul_rn(fma(b0, fc[c], pP[c]), ha), y0[c]);
    Rhs<SYS, D>::eval(t1, yP, fP, params);
#pragma unroll
    for (int c = 0; c < D; ++c)
      y1[c] = add_rn(mul_rn(add_rn(fma(a0e, fc[c], pC[c]), mul_rn(ig, fP[c])), ha), y0[c]);
    Rhs<SYS, D>::eval(t1, y1, f1, params);
    const bool bp = any_nonfinite<D>(fP), bc = any_nonfinite<D>(f1);
    const int kind = bp ? KIND_PREDICTOR : (bc ? KIND_CORRECTOR : KIND_NONE);
    const bool first = (kind != KIND_NONE) & (ekind == KIND_NONE);
    ekind = first ? kind : ekind;
    estep = first ? n : estep;
    // rows y_{n+1}, f_{n+1}
    if (lane == ((i + 1) & 31)) {
      double* fd = F + (n + 1) * DS;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        fd[c] = f1[c];
        if (Y) Y[(n + 1) * D + c] = y1[c];
        if (Fc) Fc[(n + 1) * D + c] = f1[c];
        if (n + 1 == N) P.ylast[t * D + c] = y1[c];
      }
    }
    // push f_{n+1} into the steps m > n+1 of this block
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const int j = kR * lane + r - (i + 1);  // m - (n+1)
      const double w1 = tb[j + kB], w2 = ta[j + kB];
#pragma unroll
      for (int c = 0; c < D; ++c) {
        accP[r][c] = fma(w1, f1[c], accP[r][c]);
        accC[r][c] = fma(w2, f1[c], accC[r][c]);
      }
    }
#pragma unroll
    for (int c = 0; c < D; ++c) fc[c] = f1[c];
    if ((i & 7) == 7 && ekind != KIND_NONE) break;
  }
  if (ekind != KIND_NONE && lane == 0) {
    P.err_kind[t] = ekind;
    P.err_step[t] = estep;
  }
  return true;
}

template <int SYS, int D>
__global__ void __launch_bounds__(kThreads, 1) abm_batch_kernel(BatchParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  DmmaSmem<D>& A = reinterpret_cast<DmmaSmem<D>*>(smem_raw)[warp];
  const unsigned long long total = static_cast<unsigned long long>(P.round_start[P.nb]);
  for (;;) {
    unsigned long long u = 0;
    if (lane == 0) u = atomicAdd(P.ticket, 1ull);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= total) break;
    // round J: the last J with round_start[J] <= u
    int lo = 0, hi = P.nb - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (static_cast<unsigned long long>(__ldg(P.round_start + mid)) <= u) lo = mid; else hi = mid - 1;
    }
    const int J = lo;
    const int SJ = pull_units(J, P.G);
    const long long idx = static_cast<long long>(u) - __ldg(P.round_start + J);
    if (idx < static_cast<long long>(P.T) * SJ) {  // ---- pull unit (t, J, s)
      const int s = static_cast<int>(idx / P.T), t = static_cast<int>(idx % P.T);
      // its sources complete, and its parity's slots consumed by step (t, J-2)
      int lo, hi;
      pull_bounds(J, s, P.G, lo, hi);
      FABM_CHECK(P, s < P.S_max && 0 <= lo && lo < hi && hi <= J && t < P.T);
      if (!batch_wait(P, &P.next_block[t], hi > J - 1 ? hi : J - 1, lane)) return;
      if (*((volatile int*)&P.err_kind[t]) == KIND_NONE) batch_pull<D>(P, A, t, J, s, lane);
      __threadfence();
      __syncwarp();
      if (lane == 0) atomicAdd(&P.pulls_done[2 * t + (J & 1)], 1);
    } else {  // ---- step unit (t, J)
      const int t = static_cast<int>(idx - static_cast<long long>(P.T) * SJ);
      if (!batch_wait(P, &P.next_block[t], J, lane)) return;
      if (*((volatile int*)&P.err_kind[t]) == KIND_NONE) {
        if (!batch_unit<SYS, D>(P, A, t, J, lane)) return;
      } else if (!batch_wait(P, &P.pulls_done[2 * t + (J & 1)], __ldg(P.pull_cum + J), lane)) {
        return;  // a dead trajectory's pulls still finish before the slots are reused
      }
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release_gpu(&P.next_block[t], J + 1);
    }
  }
}

}  // namespace fabm
