// engine.cuh — the single-trajectory history engine (one cooperative kernel).
//
// Replaces the O(N^2) loop of solve_serial (reference serial.py:150-170):
//   P_n = sum_{k=0..n} b_{n-k} f_k                       (serial.py:153)
//   C_n = c_n f_0 + sum_{k=1..n} a_{n-k} f_k             (serial.py:160-163)
//   yP = P_n*h^a + y0; fP = f(t,yP); y = (C_n + fP/G2)*h^a + y0; f_{n+1} = f(t,y)
//
// Work split:
//   * CTA 0 is the STEPPER.  One leader thread runs the sequential chain of
//     every step; 384 helper threads each own one future step ("slot") and
//     push every newly published f_k into it (window k in [lo(m), m-G]);
//     an I/O warp streams y/f to HBM, publishes completed source blocks and
//     stages the bulk sums of the next target block into shared memory.
//   * CTAs 1.. are BULK agents (one per warp).  Agent a owns target blocks
//     J = L + a + i*A and accumulates the Toeplitz products T_{J-I} F_I of
//     every completed source block I <= J-L, in ascending I (deterministic),
//     earliest-deadline target first.  Tile = 128 targets x 128 sources,
//     register-blocked 4 targets x d components x {b,a} per lane, weights
//     staged in a mod-4 transposed smem layout (conflict-free sliding window).
// The only host interaction is the launch; there is no round trip per step.
#pragma once
#include "device_common.cuh"

namespace fabm {

// ------------------------------------------------------------ geometry
constexpr int kB = 128;                 // history block (targets = sources per tile)
constexpr int kL = 3;                   // stepper window, in blocks
constexpr int kSlots = kL * kB;         // 384 helper slots (12 helper warps)
constexpr int kG = 3;                   // newest terms added by the leader itself
constexpr int kThreads = 512;           // 16 warps per CTA (1 CTA per SM)
constexpr int kWarps = kThreads / 32;
constexpr int kRing = 64;               // published (y, f) ring in smem
constexpr int kNumBars = 64;            // publish mbarriers (step k -> bar k % 64)
constexpr int kHR = 8;                  // handoff ring
constexpr int kR = 4;                   // targets per lane in a bulk tile
constexpr int kWCols = 2 * kB / 4 + 2;  // transposed weight row length (+2 pad)
constexpr int kMaxOwn = 256;            // owned target blocks per agent

enum ErrCode : int { ERR_OK = 0, ERR_NONFINITE = 1, ERR_CONFIG = 2, ERR_TIMEOUT = 3 };
enum ErrKind : int { KIND_NONE = 0, KIND_INITIAL = 1, KIND_PREDICTOR = 2, KIND_CORRECTOR = 3 };

// device-side control block (global memory, zeroed before each run)
struct DevCtrl {
  int src_done;            // number of complete source blocks published (I/O warp)
  int pad0[31];
  int abort;               // set on error / timeout
  int err_code;
  int err_kind;
  int pad1;
  long long err_step;
  double err_t;
  unsigned long long leader_wait_ns;
  unsigned long long bulk_tiles;
  unsigned long long leader_throttle_ns;
  int pad2[16];
};

struct EngineParams {
  long long N;             // steps
  double h, ha, ig;        // step, h^alpha, 1/Gamma(alpha+2)
  const double* wb;        // b_j  (length >= nb*B + 2B)
  const double* wa;        // a_j
  const double* wc;        // c_j
  const double* y0;        // device y0 (d doubles)
  double* Y;               // states (N+1) x d
  double* F;               // f history (nb*B + B) x DS
  double* BK;              // bulk accumulators (nb*B) x 2 x DS
  int* ready;              // per target block: bulk complete
  DevCtrl* ctrl;
  double params[kMaxParams];
  int nb;                  // ceil(N / B)
  int n_agents;            // bulk agents = 16 * (gridDim.x - 1)
  unsigned long long timeout_ns;
};

__device__ __forceinline__ long long lo_of(long long m) {
  long long J = m / kB;
  long long lb = J - (kL - 1);
  return lb > 0 ? lb * kB : 0;
}

__device__ __forceinline__ void raise_abort(const EngineParams& P, int code, int kind, long long step, double t) {
  if (atomicCAS(&P.ctrl->err_code, 0, code) == 0) {
    P.ctrl->err_kind = kind;
    P.ctrl->err_step = step;
    P.ctrl->err_t = t;
  }
  __threadfence();
  atomicExch(&P.ctrl->abort, 1);
}

// ======================================================================
// STEPPER CTA
// ======================================================================
struct StepperSmem {
  double wb[kSlots];
  double wa[kSlots];
  double ringY[kRing][4];
  double ringF[kRing][4];
  double hP[kHR][4];
  double hC[kHR][4];
  double bulk[2][kB][2][4];
  uint64_t bars[kNumBars];
  int hflag[kHR];
  int hprog[kWarps];       // last step processed by each helper warp
  int bulk_flag;           // highest staged target block
  int io_done;             // steps written to HBM by the writer warp
  int io_block;            // complete source blocks written by the writer warp
  int abort;
};

__device__ __forceinline__ int slowest_consumer(StepperSmem& S) {
  int lo = ld_volatile_smem(&S.io_done);
#pragma unroll
  for (int w = 1; w < kWarps; ++w) {
    if ((w & 3) == 0) continue;
    const int p = ld_volatile_smem(&S.hprog[w]) + 1;
    lo = p < lo ? p : lo;
  }
  return lo;
}

// spin until the helpers handed off step m (flag == m); false on abort/timeout
__device__ __noinline__ bool leader_wait_handoff(const EngineParams& P, StepperSmem& S, long long m,
                                                 unsigned long long& waited) {
  const int slot = static_cast<int>(m % kHR);
  const unsigned long long w0 = global_ns();
  unsigned spins = 0;
  while (ld_acquire_cta_smem(&S.hflag[slot]) != static_cast<int>(m)) {
    if (((++spins) & 1023u) == 0) {
      if (ld_volatile_smem(&S.abort) || *((volatile int*)&P.ctrl->abort)) return false;
      if (global_ns() - w0 > P.timeout_ns) {
        raise_abort(P, ERR_TIMEOUT, KIND_NONE, m, 0.0);
        st_volatile_smem(&S.abort, 1);
        mbar_arrive(&S.bars[(m + 1) % kNumBars]);
        return false;
      }
    }
  }
  waited += global_ns() - w0;
  return true;
}

template <int SYS, int D>
__device__ void stepper_leader(const EngineParams& P, StepperSmem& S) {
  const long long N = P.N;
  const double h = P.h, ha = P.ha, ig = P.ig;
  double y0[D], fm1[D], fc[D];
#pragma unroll
  for (int c = 0; c < D; ++c) { y0[c] = P.y0[c]; fm1[c] = 0.0; }
  Rhs<SYS, D>::eval(0.0, y0, fc, P.params);
  const bool ok0 = all_finite<D>(fc);
#pragma unroll
  for (int c = 0; c < D; ++c) { S.ringY[0][c] = y0[c]; S.ringF[0][c] = fc[c]; }
  if (!ok0) {
    raise_abort(P, ERR_NONFINITE, KIND_INITIAL, 0, 0.0);
    st_volatile_smem(&S.abort, 1);
  }
  mbar_arrive(&S.bars[0]);
  if (!ok0) return;

  const double b0 = P.wb[0], b1 = P.wb[1], b2 = P.wb[2];
  const double a0 = P.wa[0], a1 = P.wa[1], a2 = P.wa[2];
  unsigned long long waited = 0, throttled = 0;

  // pre-sums of step n: everything but the f_n terms, i.e.
  //   preP = (H_P[n] + b2 f_{n-2}) + b1 f_{n-1},  preC likewise with a (k >= 1)
  // built one step ahead, off the critical path of the sequential chain.
  double preP[D], preC[D];
  if (!leader_wait_handoff(P, S, 0, waited)) return;
#pragma unroll
  for (int c = 0; c < D; ++c) { preP[c] = S.hP[0][c]; preC[c] = S.hC[0][c]; }

  for (long long n = 0; n < N; ++n) {
    // ---- speculative read of the handoff of step n+1 (normally long ready);
    // the data loads are issued after the flag load (in-order smem pipe)
    const long long m1 = n + 1;
    const int slot1 = static_cast<int>(m1 % kHR);
    const int fl = ld_acquire_cta_smem(&S.hflag[slot1]);
    double hp1[D], hc1[D];
#pragma unroll
    for (int c = 0; c < D; ++c) { hp1[c] = S.hP[slot1][c]; hc1[c] = S.hC[slot1][c]; }
    // coefficients of step m1 for its f_{m1-2} = f_{n-1} and f_{m1-1} = f_n terms
    const double nb2 = m1 >= 2 ? b2 : 0.0;
    const double na2 = m1 >= 3 ? a2 : 0.0, na1 = m1 >= 2 ? a1 : 0.0;
    double nP[D], nC[D];
#pragma unroll
    for (int c = 0; c < D; ++c) {
      nP[c] = fma(b1, fc[c], fma(nb2, fm1[c], hp1[c]));
      nC[c] = fma(na1, fc[c], fma(na2, fm1[c], hc1[c]));
    }

    // ---- the sequential chain of step n
    const double t1 = static_cast<double>(n + 1) * h;  // (n + 1) * h, serial.py:151
    const double a0e = n >= 1 ? a0 : 0.0;               // corrector interior starts at k = 1
    double yP[D], fP[D];
#pragma unroll
    for (int c = 0; c < D; ++c) yP[c] = add_rn(mul_rn(fma(b0, fc[c], preP[c]), ha), y0[c]);  // serial.py:153-155
    Rhs<SYS, D>::eval(t1, yP, fP, P.params);
    if (!all_finite<D>(fP)) {
      raise_abort(P, ERR_NONFINITE, KIND_PREDICTOR, n, t1);
      st_volatile_smem(&S.abort, 1);
      mbar_arrive(&S.bars[(n + 1) % kNumBars]);
      break;
    }
    double y1[D], f1[D];
#pragma unroll
    for (int c = 0; c < D; ++c)  // ((c_n f0 + C_n) + fP/G2) * h^a + y0, serial.py:160-165
      y1[c] = add_rn(mul_rn(add_rn(fma(a0e, fc[c], preC[c]), mul_rn(ig, fP[c])), ha), y0[c]);
    Rhs<SYS, D>::eval(t1, y1, f1, P.params);
    if (!all_finite<D>(f1)) {
      raise_abort(P, ERR_NONFINITE, KIND_CORRECTOR, n, t1);
      st_volatile_smem(&S.abort, 1);
      mbar_arrive(&S.bars[(n + 1) % kNumBars]);
      break;
    }
    // ---- publish (y_{n+1}, f_{n+1})
    const int ri = static_cast<int>((n + 1) % kRing);
#pragma unroll
    for (int c = 0; c < D; ++c) { S.ringY[ri][c] = y1[c]; S.ringF[ri][c] = f1[c]; }
    mbar_arrive(&S.bars[(n + 1) % kNumBars]);

    // ---- slow path: the handoff of step n+1 was not ready when read
    if (m1 < N && fl != static_cast<int>(m1)) {
      if (!leader_wait_handoff(P, S, m1, waited)) return;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        nP[c] = fma(b1, fc[c], fma(nb2, fm1[c], S.hP[slot1][c]));
        nC[c] = fma(na1, fc[c], fma(na2, fm1[c], S.hC[slot1][c]));
      }
    }
#pragma unroll
    for (int c = 0; c < D; ++c) { preP[c] = nP[c]; preC[c] = nC[c]; fm1[c] = fc[c]; fc[c] = f1[c]; }

    // ring back-pressure: the I/O warp and every helper warp must have
    // drained entry n+1-kRing (also keeps the mbarrier phases unaliased)
    if (((n + 1) & 7) == 0 && (n + 1) - slowest_consumer(S) > kRing - 24) {
      unsigned spins = 0;
      const unsigned long long w0 = global_ns();
      while ((n + 1) - slowest_consumer(S) > kRing - 24) {
        if (((++spins) & 1023u) == 0) {
          if (ld_volatile_smem(&S.abort) || *((volatile int*)&P.ctrl->abort)) return;
          if (global_ns() - w0 > P.timeout_ns) {
            raise_abort(P, ERR_TIMEOUT, KIND_NONE, n, 0.0);
            st_volatile_smem(&S.abort, 1);
            return;
          }
        }
      }
      throttled += global_ns() - w0;
    }
  }
  P.ctrl->leader_wait_ns = waited;
  P.ctrl->leader_throttle_ns = throttled;
}

template <int D>
__device__ void stepper_helper(const EngineParams& P, StepperSmem& S, int hid) {
  const long long N = P.N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long m = hid;
  double accP[D], accC[D], f0[D];
#pragma unroll
  for (int c = 0; c < D; ++c) { accP[c] = 0.0; accC[c] = 0.0; f0[c] = 0.0; }
  long long lo = lo_of(m);
  long long kh = m - kG > 0 ? m - kG : 0;
  double cm = m < N ? P.wc[m] : 0.0, am = m < N ? P.wa[m] : 0.0;

  for (long long k = 0; k <= N; ++k) {
    // wait for publication of step k
    uint64_t* bar = &S.bars[k % kNumBars];
    const uint32_t par = static_cast<uint32_t>((k / kNumBars) & 1);
    unsigned spins = 0;
    const unsigned long long w0 = global_ns();
    while (!mbar_try(bar, par)) {
      if (ld_volatile_smem(&S.abort)) return;
      if (((++spins) & 255u) == 0) {
        if (*((volatile int*)&P.ctrl->abort)) return;
        if (global_ns() - w0 > P.timeout_ns) return;
      }
    }
    const int ri = static_cast<int>(k % kRing);
    double fk[D];
#pragma unroll
    for (int c = 0; c < D; ++c) fk[c] = S.ringF[ri][c];
    if (k == 0) {
#pragma unroll
      for (int c = 0; c < D; ++c) f0[c] = fk[c];
    }
    if (m < N && k >= lo && k <= m - kG) {
      const int j = static_cast<int>(m - k);
      const double wb = S.wb[j];
      const double wa = k >= 1 ? S.wa[j] : 0.0;  // corrector interior excludes k = 0
#pragma unroll
      for (int c = 0; c < D; ++c) {
        accP[c] = fma(wb, fk[c], accP[c]);
        accC[c] = fma(wa, fk[c], accC[c]);
      }
    }
    if (m < N && k == kh) {
      const long long J = m / kB;
      double hp[D], hc[D];
      if (J >= kL) {
        // bulk sums (sources < lo) include k = 0 in the a-sum: fold (c_m - a_m) f0
        unsigned sp2 = 0;
        const unsigned long long w1 = global_ns();
        while (ld_acquire_cta_smem(&S.bulk_flag) < static_cast<int>(J)) {
          if (ld_volatile_smem(&S.abort)) return;
          if (((++sp2) & 255u) == 0) {
            if (*((volatile int*)&P.ctrl->abort)) return;
            if (global_ns() - w1 > P.timeout_ns) return;
          }
        }
        const int bsel = static_cast<int>(J & 1);
        const int r = static_cast<int>(m % kB);
        const double cma = cm - am;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          hp[c] = accP[c] + S.bulk[bsel][r][0][c];
          hc[c] = add_rn(accC[c] + S.bulk[bsel][r][1][c], mul_rn(cma, f0[c]));
        }
      } else {
#pragma unroll
        for (int c = 0; c < D; ++c) {
          hp[c] = accP[c];
          hc[c] = add_rn(accC[c], mul_rn(cm, f0[c]));
        }
      }
      const int slot = static_cast<int>(m % kHR);
#pragma unroll
      for (int c = 0; c < D; ++c) { S.hP[slot][c] = hp[c]; S.hC[slot][c] = hc[c]; }
      st_release_cta_smem(&S.hflag[slot], static_cast<int>(m));
      // reopen the slot for step m + kSlots
      m += kSlots;
#pragma unroll
      for (int c = 0; c < D; ++c) { accP[c] = 0.0; accC[c] = 0.0; }
      lo = lo_of(m);
      kh = m - kG;
      if (m < N) { cm = P.wc[m]; am = P.wa[m]; }
    }
    __syncwarp();
    if (lane == 0) st_volatile_smem(&S.hprog[warp], static_cast<int>(k));
  }
}

// Writer warp: streams published (y, f) from the smem ring to HBM in batches
// of 32 steps; after the last row of a source block it raises io_block (CTA
// scope, release).  It never touches slow global state, so it keeps pace.
template <int D>
__device__ void stepper_writer(const EngineParams& P, StepperSmem& S, int lane) {
  constexpr int DS = Stride<D>::value;
  const long long N = P.N;
  long long k0 = 0;
  while (k0 <= N) {
    const long long kend = (k0 + 31 < N) ? k0 + 31 : N;
    uint64_t* bar = &S.bars[kend % kNumBars];
    const uint32_t par = static_cast<uint32_t>((kend / kNumBars) & 1);
    unsigned spins = 0;
    const unsigned long long w0 = global_ns();
    while (!mbar_try(bar, par)) {
      if (ld_volatile_smem(&S.abort)) return;
      if (((++spins) & 255u) == 0) {
        if (*((volatile int*)&P.ctrl->abort)) return;
        if (global_ns() - w0 > P.timeout_ns) {
          if (lane == 0) raise_abort(P, ERR_TIMEOUT, KIND_NONE, k0, 0.0);
          st_volatile_smem(&S.abort, 1);
          return;
        }
      }
    }
    const long long k = k0 + lane;
    if (k <= kend) {
      const int ri = static_cast<int>(k % kRing);
      double* yd = P.Y + k * D;
      double* fd = P.F + k * DS;
#pragma unroll
      for (int c = 0; c < D; ++c) { yd[c] = S.ringY[ri][c]; fd[c] = S.ringF[ri][c]; }
    }
    __syncwarp();
    if (lane == 0) {
      st_volatile_smem(&S.io_done, static_cast<int>(kend + 1));
      if (((kend + 1) % kB) == 0) st_release_cta_smem(&S.io_block, static_cast<int>((kend + 1) / kB));
    }
    k0 = kend + 1;
  }
}

// Publisher warp: turns io_block (CTA scope) into src_done (GPU scope) for
// the bulk agents, and stages the bulk sums of each upcoming target block
// from HBM into shared memory for the helpers.  All slow global round trips
// of the stepper CTA live here, off the writer's and the leader's paths.
template <int D>
__device__ void stepper_publisher(const EngineParams& P, StepperSmem& S, int lane) {
  constexpr int DS = Stride<D>::value;
  const int nb = P.nb;
  const int last_block = static_cast<int>(P.N / kB);  // complete source blocks at the end
  int published = 0;
  int next_stage = kL;
  unsigned long long last_progress = global_ns();
  while (published < last_block || next_stage < nb) {
    bool progress = false;
    // (1) source blocks written by the writer warp -> GPU-scope publication
    int io_block = 0;
    if (lane == 0) io_block = ld_acquire_cta_smem(&S.io_block);
    io_block = __shfl_sync(0xffffffffu, io_block, 0);
    if (io_block > published) {
      if (lane == 0) {
        __threadfence();  // cumulative over the writer's rows (acquired above)
        st_release_gpu(&P.ctrl->src_done, io_block);
      }
      published = io_block;
      progress = true;
    }
    // (2) stage target block J once the helpers are done with buffer J&1
    // (the leader has published step (J-1)*B) and the agents flagged it
    if (next_stage < nb && ld_volatile_smem(&S.io_done) - 1 >= static_cast<long long>(next_stage - 1) * kB) {
      int rdy = 0;
      if (lane == 0) rdy = ld_acquire_gpu(&P.ready[next_stage]);
      rdy = __shfl_sync(0xffffffffu, rdy, 0);
      if (rdy) {
        __syncwarp();
        const int J = next_stage;
        const double* src = P.BK + static_cast<long long>(J) * kB * 2 * DS;
        double* dst = &S.bulk[J & 1][0][0][0];
        for (int i = lane; i < kB * 2 * D; i += 32) {
          const int row = i / (2 * D), rem = i % (2 * D), half = rem / D, c = rem % D;
          dst[(row * 2 + half) * 4 + c] = __ldcg(src + (row * 2 + half) * DS + c);
        }
        __syncwarp();
        if (lane == 0) st_release_cta_smem(&S.bulk_flag, J);
        ++next_stage;
        progress = true;
      }
    }
    if (progress) {
      last_progress = global_ns();
      continue;
    }
    if (ld_volatile_smem(&S.abort) || *((volatile int*)&P.ctrl->abort)) return;
    if (global_ns() - last_progress > P.timeout_ns) {
      if (lane == 0) raise_abort(P, ERR_TIMEOUT, KIND_NONE, -2, 0.0);
      st_volatile_smem(&S.abort, 1);
      return;
    }
    __nanosleep(128);
  }
}

template <int SYS, int D>
__device__ void stepper_cta(const EngineParams& P, StepperSmem& S) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < kSlots; i += kThreads) { S.wb[i] = P.wb[i]; S.wa[i] = P.wa[i]; }
  if (tid < kHR) S.hflag[tid] = -1;
  if (tid < kWarps) S.hprog[tid] = -1;
  if (tid == 0) {
    S.bulk_flag = kL - 1;
    S.io_done = 0;
    S.io_block = 0;
    S.abort = 0;
    for (int i = 0; i < kNumBars; ++i) mbar_init(&S.bars[i], 1);
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) stepper_leader<SYS, D>(P, S);
    return;
  }
  if (warp == 4) { stepper_writer<D>(P, S, lane); return; }
  if (warp == 8) { stepper_publisher<D>(P, S, lane); return; }
  if ((warp & 3) == 0) return;  // share the leader's SMSP: keep it quiet
  const int hid = (warp - (warp >> 2) - 1) * 32 + lane;
  stepper_helper<D>(P, S, hid);
}

// ======================================================================
// BULK AGENTS
// ======================================================================
struct AgentSmem {
  double w[2][4][kWCols];  // b, a in mod-4 transposed layout
  double f[kB][4];         // f tile of the source block (row stride 4)
  int own_next[kMaxOwn];   // next source block per owned target
};

template <int D>
__device__ __forceinline__ void agent_store_acc(const EngineParams& P, int J, int lane,
                                                const double (&accP)[kR][D], const double (&accC)[kR][D]) {
  constexpr int DS = Stride<D>::value;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    double* dst = P.BK + (static_cast<long long>(J) * kB + kR * lane + r) * 2 * DS;
#pragma unroll
    for (int c = 0; c < D; ++c) { dst[c] = accP[r][c]; dst[DS + c] = accC[r][c]; }
  }
}

template <int D>
__device__ __forceinline__ void agent_load_acc(const EngineParams& P, int J, int lane,
                                               double (&accP)[kR][D], double (&accC)[kR][D]) {
  constexpr int DS = Stride<D>::value;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const double* src = P.BK + (static_cast<long long>(J) * kB + kR * lane + r) * 2 * DS;
#pragma unroll
    for (int c = 0; c < D; ++c) { accP[r][c] = __ldcg(src + c); accC[r][c] = __ldcg(src + DS + c); }
  }
}

// acc[n] += sum_{k in block I} w[n - k] f_k for the lane's 4 targets of block J,
// ascending k.  Weight window u = 127 - s + r (jl = 4*lane + u), mod-4 transposed.
template <int D>
__device__ __forceinline__ void agent_tile(const EngineParams& P, AgentSmem& A, int I, int J, int lane,
                                           double (&accP)[kR][D], double (&accC)[kR][D]) {
  constexpr int DS = Stride<D>::value;
  __syncwarp();
  // ---- stage weights j in [Delta-127, Delta+127] (transposed) and the f tile
  const long long base = static_cast<long long>(J - I) * kB - (kB - 1);
  for (int jl = lane; jl < 2 * kB - 1; jl += 32) {
    const double vb = __ldg(P.wb + base + jl);
    const double va = __ldg(P.wa + base + jl);
    A.w[0][jl & 3][jl >> 2] = vb;
    A.w[1][jl & 3][jl >> 2] = va;
  }
  {
    const double* src = P.F + static_cast<long long>(I) * kB * DS;
    if constexpr (DS >= 2) {
      for (int i = lane; i < kB * DS / 2; i += 32) {
        const double2 v = __ldcg(reinterpret_cast<const double2*>(src) + i);
        const int row = (2 * i) / DS, c = (2 * i) % DS;
        A.f[row][c] = v.x;
        A.f[row][c + 1] = v.y;
      }
    } else {
      for (int i = lane; i < kB; i += 32) A.f[i][0] = __ldcg(src + i);
    }
  }
  __syncwarp();

  // ---- compute: groups of 4 sources; window W[i] <-> u = 124 - 4q + i
  double wb[7], wa[7];
#pragma unroll
  for (int i = 0; i < 3; ++i) {  // u = 128 + i  -> row i, col lane + 32
    wb[4 + i] = A.w[0][i][lane + 32];
    wa[4 + i] = A.w[1][i][lane + 32];
  }
#pragma unroll 2
  for (int q = 0; q < kB / 4; ++q) {
    const int col = lane + 31 - q;
#pragma unroll
    for (int i = 0; i < 4; ++i) { wb[i] = A.w[0][i][col]; wa[i] = A.w[1][i][col]; }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int s = 4 * q + t;
      double fk[D];
#pragma unroll
      for (int c = 0; c < D; ++c) fk[c] = A.f[s][c];
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        // u - (124 - 4q) = 3 + r - t
        const double bw = wb[3 + r - t], aw = wa[3 + r - t];
#pragma unroll
        for (int c = 0; c < D; ++c) {
          accP[r][c] = fma(bw, fk[c], accP[r][c]);
          accC[r][c] = fma(aw, fk[c], accC[r][c]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) { wb[4 + i] = wb[i]; wa[4 + i] = wa[i]; }
  }
}

template <int D>
__device__ void bulk_agent(const EngineParams& P, AgentSmem& A, int agent, int lane) {
  const int nb = P.nb;
  const int n_targets = nb - kL;  // targets J = L .. nb-1
  if (agent >= n_targets) return;
  const int nA = P.n_agents;
  const int nown = (n_targets - 1 - agent) / nA + 1;
  for (int i = lane; i < nown; i += 32) A.own_next[i] = 0;
  __syncwarp();
  double accP[kR][D], accC[kR][D];
#pragma unroll
  for (int r = 0; r < kR; ++r)
#pragma unroll
    for (int c = 0; c < D; ++c) { accP[r][c] = 0.0; accC[r][c] = 0.0; }
  int cur = -1, done = 0;
  unsigned long long tiles = 0;
  unsigned long long last_progress = global_ns();

  while (done < nown) {
    int M = 0, ab = 0;
    if (lane == 0) { M = ld_acquire_gpu(&P.ctrl->src_done); ab = ld_relaxed_gpu(&P.ctrl->abort); }
    M = __shfl_sync(0xffffffffu, M, 0);
    ab = __shfl_sync(0xffffffffu, ab, 0);
    if (ab) return;
    __syncwarp();
    // earliest-deadline owned target with available work
    int best = -1;
    for (int b0 = 0; b0 < nown; b0 += 32) {
      const int i = b0 + lane;
      bool pend = false;
      if (i < nown) {
        const int J = kL + agent + i * nA;
        const int nx = A.own_next[i];
        const int lim = min(M, J - kL + 1);
        pend = nx < lim;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, pend);
      if (bal) { best = b0 + __ffs(bal) - 1; break; }
    }
    if (best < 0) {
      __nanosleep(256);
      if (global_ns() - last_progress > P.timeout_ns) {
        if (lane == 0) raise_abort(P, ERR_TIMEOUT, KIND_NONE, -1, 0.0);
        return;
      }
      continue;
    }
    last_progress = global_ns();
    const int J = kL + agent + best * nA;
    if (cur != best) {
      if (cur >= 0) agent_store_acc<D>(P, kL + agent + cur * nA, lane, accP, accC);
      if (A.own_next[best] > 0) {
        agent_load_acc<D>(P, J, lane, accP, accC);
      } else {
#pragma unroll
        for (int r = 0; r < kR; ++r)
#pragma unroll
          for (int c = 0; c < D; ++c) { accP[r][c] = 0.0; accC[r][c] = 0.0; }
      }
      cur = best;
    }
    const int lim = min(M, J - kL + 1);
    int nx = A.own_next[best];
    while (nx < lim) {
      int M2 = 0;
      if (lane == 0) M2 = ld_relaxed_gpu(&P.ctrl->src_done);
      agent_tile<D>(P, A, nx, J, lane, accP, accC);
      ++nx;
      ++tiles;
      M2 = __shfl_sync(0xffffffffu, M2, 0);
      if (M2 != M) break;  // a newer source block arrived: re-run EDF selection
    }
    __syncwarp();
    if (lane == 0) A.own_next[best] = nx;
    __syncwarp();
    if (nx == J - kL + 1) {
      agent_store_acc<D>(P, J, lane, accP, accC);
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release_gpu(&P.ready[J], 1);
      cur = -1;
      ++done;
    }
  }
  if (lane == 0) atomicAdd(&P.ctrl->bulk_tiles, tiles);
}

// ======================================================================
template <int SYS, int D>
__global__ void __launch_bounds__(kThreads, 1) abm_engine_kernel(EngineParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  if (blockIdx.x == 0) {
    stepper_cta<SYS, D>(P, *reinterpret_cast<StepperSmem*>(smem_raw));
  } else {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    AgentSmem* A = reinterpret_cast<AgentSmem*>(smem_raw) + warp;
    bulk_agent<D>(P, *A, (blockIdx.x - 1) * kWarps + warp, lane);
  }
}

constexpr size_t engine_smem_bytes() {
  return sizeof(StepperSmem) > kWarps * sizeof(AgentSmem) ? sizeof(StepperSmem) : kWarps * sizeof(AgentSmem);
}

}  // namespace fabm
