// engine.cuh — the single-trajectory history engine (one cooperative kernel).
//
// Replaces the O(N^2) loop of solve_serial (reference serial.py:150-170):
//   P_n = sum_{k=0..n} b_{n-k} f_k                       (serial.py:153)
//   C_n = c_n f_0 + sum_{k=1..n} a_{n-k} f_k             (serial.py:160-163)
//   yP = P_n*h^a + y0; fP = f(t,yP); y = (C_n + fP/G2)*h^a + y0; f_{n+1} = f(t,y)
//
// Work split:
//   * CTA 0 is the STEPPER.  The leader warp (warp 0, alone on SMSP 0) runs
//     the sequential chain of every step on all 32 lanes and keeps the near
//     window (the last 32-64 steps) in registers; 8 helper warps own 512
//     future steps ("slots") and push every published f_k of the far window
//     into them, handing each step's far part to the leader ~30 steps ahead;
//     the writer warp streams (y, f) to HBM (and pinned host memory) and
//     checks every rhs output for non-finite values; the publisher warp
//     releases completed source blocks to the bulk agents and stages each
//     target block's bulk sums into shared memory.
//   * CTAs 1.. are BULK agents (one per warp, 16 per SM).  Agent a owns target
//     blocks J = L + a + i*A and accumulates the Toeplitz products T_{J-I} F_I
//     of every completed source block I <= J-L, in ascending I (deterministic),
//     earliest-deadline target first.  Tile = 128 targets x 128 sources on the
//     FP64 tensor cores (bulk_dmma.cuh: m8n8k4 DMMA, 8 diagonal shifts of one
//     weight fragment per instruction).
// The only host interaction is the launch; there is no round trip per step.
#pragma once
#include "device_common.cuh"

namespace fabm {

// ------------------------------------------------------------ geometry
constexpr int kB = 128;                 // history block (targets = sources per tile)
constexpr int kL = 4;                   // stepper window, in blocks (bulk slack: L-1 blocks)
constexpr int kSlots = kL * kB;         // 512 far-window slots
constexpr int kChunk = 32;              // near window: k in [32(c-1), m-1] for m in chunk c (leader warp)
constexpr int kGFar = 2 * kChunk + 1;   // sizing of the zero-padded weight tables
constexpr int kHelperWarps = 8;         // warps 1,2,3,5,6,7,9,10 (SMSPs 1-3)
constexpr int kWriterWarp = 13;         // SMSP 1
constexpr int kPublisherWarp = 14;      // SMSP 2
constexpr int kSlotsPerThread = kSlots / (kHelperWarps * 32);  // 2
constexpr int kBatch = 8;               // publishes consumed per helper wake-up
constexpr int kThreads = 512;           // 16 warps per CTA (1 CTA per SM)
constexpr int kWarps = kThreads / 32;
constexpr int kRing = 64;               // published (y, f) ring in smem
constexpr int kNumBars = 64;            // publish mbarriers (step group g -> bar g % 64)
constexpr int kHR = 128;                // far handoff ring (handoffs run ~60 steps ahead)
constexpr int kR = 4;                   // rows per lane in 128-row warp loops (batch stepping)
constexpr int kMaxOwn = 256;            // owned target blocks per agent
constexpr int kMaxShards = 8;           // GPUs of one node sharing a trajectory (config 5)

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
  unsigned long long bulk_claims;  // units taken by a claimer (not their owner)
  unsigned long long prof[8];  // FABM_PROFILE builds: leader phase cycles
  int check_line;          // FABM_CHECKED builds: source line of the first violated invariant
  int pad2[13];
  unsigned long long prof2[8];  // FABM_PROFILE builds: agent event counts / cycles (tools/prof_bulk.py)
};

// One shard = the bulk agents of one GPU.  Every shard holds a full copy of
// the f history (the stepper's writer fans rows out to all copies over
// NVLink) and its own control block (src_done is released into it by the
// stepper's publisher).  The bulk units' state -- claim words, partial
// slots, counters, cursors -- and the finished target sums (BK, ready) live
// in shard 0's arena.
struct ShardView {
  double* F;      // f history copy (same layout as EngineParams::F)
  DevCtrl* ctrl;  // src_done / abort polled by this shard's agents
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
  double* Fc;              // f_cache output, (N+1) x d compact
  double* Yh;              // optional: states / f_cache also streamed to mapped
  double* Fch;             //   pinned host memory (device aliases), or null
  double* BK;              // bulk accumulators (nb*B) x 2 x DS
  int* ready;              // per target block: bulk complete
  DevCtrl* ctrl;
  double params[kMaxParams];
  int nb;                  // ceil(N / B)
  int n_agents;            // bulk agents = 16 * (gridDim.x - 1)
  unsigned long long timeout_ns;
  unsigned long long* trace;  // FABM_PROFILE: per block {src published, ready, staged, first need}
  int debug;               // dev experiments: 1 = leader alone, 8 = no bulk agents (results invalid)
  // sharding (config 5).  n_shards = 1: everything local.  my_shard >= 0: this
  // launch hosts the agents of that shard (and the stepper if it is 0);
  // my_shard = -1: one-GPU emulation, agent CTA b belongs to shard (b-1) % n_shards
  int n_shards;
  int my_shard;
  int agent_cta_base;      // global index of this launch's first agent CTA
  int n_agent_ctas;        // agent CTAs over all shards
  const ShardView* shard;  // device table of n_shards views (global memory: indexed at run time)
  int has_stepper;         // CTA 0 of this launch is the stepper (every launch but a real shard > 0)
  // bulk units (shard 0's arena): per-unit claim words and partial-sum
  // slots, per-target counts of finished non-final units and of stage-2
  // arrivals, per-(class, column) claim cursors
  int k_max;               // highest segment class of this run
  long long n_units;       // allocated unit slots / claim words (FABM_CHECKED bounds)
  long long wlen;          // allocated weight entries
  long long f_rows;        // allocated f history rows (per shard copy)
  int* claim;
  int* tdone;
  int* tstage;
  int* col_next;           // [kMaxClasses][32]
  double* PK;
};

__device__ __forceinline__ long long lo_of(long long m) {
  long long J = m / kB;
  long long lb = J - (kL - 1);
  return lb > 0 ? lb * kB : 0;
}

__device__ __forceinline__ void ctrl_abort(DevCtrl* ctrl, int code, int kind, long long step, double t) {
  if (atomicCAS(&ctrl->err_code, 0, code) == 0) {
    ctrl->err_kind = kind;
    ctrl->err_step = step;
    ctrl->err_t = t;
  }
  __threadfence();
  atomicExch(&ctrl->abort, 1);
}
// cold path, out of line (keeps the stepper's hot loops small in the
// instruction cache; plain pointers, so P stays in the parameter space)
__device__ __noinline__ void raise_abort_cold(DevCtrl* ctrl, const ShardView* shard, int n_shards, int code, int kind,
                                              long long step, double t) {
  ctrl_abort(ctrl, code, kind, step, t);
  if (n_shards > 1) {  // stop every shard (peer control blocks)
    __threadfence_system();
    for (int s = 0; s < n_shards; ++s) atomicExch_system(&shard[s].ctrl->abort, 1);
  }
}
__device__ __forceinline__ void raise_abort(const EngineParams& P, int code, int kind, long long step, double t) {
  raise_abort_cold(P.ctrl, P.shard, P.n_shards, code, kind, step, t);
}

// FABM_CHECKED builds (tools/checked_sweep.sh): bounds and protocol
// invariants of the engine, the substitute for compute-sanitizer (closed on
// this GPU pool).  A violation records its source line and aborts the run;
// fabm_plan_run then reports it.  Compiled out otherwise.
#ifdef FABM_CHECKED
#define FABM_CHECK(P, cond)                                                      \
  do {                                                                           \
    if (!(cond)) {                                                               \
      atomicCAS(&(P).ctrl->check_line, 0, __LINE__);                            \
      atomicExch(&(P).ctrl->abort, 1);                                           \
    }                                                                            \
  } while (0)
#else
#define FABM_CHECK(P, cond) \
  do {                      \
  } while (0)
#endif

// ======================================================================
// STEPPER CTA
// ======================================================================
struct StepperSmem {
  double wb[kSlots + 2 * kGFar];   // b_j, a_j for j < kSlots (zero beyond)
  double wa[kSlots + 2 * kGFar];
  double ring[kRing][12];   // published step k: y_k at [0, d), f_k at [d, 2d), fP of step k-1 at [2d, 3d)
  double hbuf[kHR][8];      // far handoff of step m: P part at [0, d), C part at [d, 2d)
  double xfer[2][8];        // near pre-sum of the next step, owner lane -> leader warp
  double tb[4 * kChunk];    // near weights, tb[j + 2*kChunk - 1] = b_j for j >= 1, 0 for j <= 0
  double ta[4 * kChunk];
  double bulk[2][kB][2][4];
  double cfirst[2][kB];     // first-node coefficient of each staged step (c_m, or c_m - a_m)
  uint64_t bars[kNumBars];
  int hflag[kHR];
  int hprog[kWarps];        // last step processed by each helper warp
  int bulk_flag;            // highest staged block
  int io_done;              // steps written to HBM by the writer warp
  int io_block;             // complete source blocks written by the writer warp
  int abort;
};

// publication groups: row 0 alone, then rows 8q-7 .. 8q+... : group of row k
// is 0 for k = 0 and k/8 + 1 otherwise; a group's mbarrier completes when its
// last row (k = 7 mod 8) or row N is published.  Consumers only wait for
// rows that end a group (helper batches end at 7 mod 8 or N, writer batches
// at 31 mod 32 or N), and each group completes its barrier exactly once.
__device__ __forceinline__ int pub_group(long long k) { return k == 0 ? 0 : static_cast<int>(k >> 3) + 1; }

__device__ __forceinline__ int helper_index(int warp) { return warp - (warp >> 2) - 1; }

__device__ __forceinline__ int slowest_consumer(StepperSmem& S) {
  int lo = ld_volatile_smem(&S.io_done);
#pragma unroll
  for (int w = 1; w < kWarps; ++w) {
    if ((w & 3) == 0 || helper_index(w) >= kHelperWarps) continue;
    const int p = ld_volatile_smem(&S.hprog[w]) + 1;
    lo = p < lo ? p : lo;
  }
  return lo;
}


// 2d doubles as d 16-byte vectors (2d is even for every d)
template <int D>
__device__ __forceinline__ void st_pairs(double* dst, const double* v) {
#pragma unroll
  for (int i = 0; i < D; ++i) reinterpret_cast<double2*>(dst)[i] = make_double2(v[2 * i], v[2 * i + 1]);
}
template <int D>
__device__ __forceinline__ void ld_pairs(const double* src, double* v) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
    const double2 t = reinterpret_cast<const double2*>(src)[i];
    v[2 * i] = t.x;
    v[2 * i + 1] = t.y;
  }
}

// x*0 is +-0 for finite x and NaN otherwise: one NaN test covers a vector,
// exactly (no overflow false positives), without a branch per value
template <int D>
__device__ __forceinline__ bool any_nonfinite(const double* v) {
  double t = v[0] * 0.0;
#pragma unroll
  for (int i = 1; i < D; ++i) t = fma(v[i], 0.0, t);
  return t != t;
}

// ----------------------------------------------------------------------
// Leader warp (warp 0).  All 32 lanes run the sequential chain redundantly
// (bitwise identical values), so every lane holds f_{n+1} the moment it is
// computed and no broadcast is needed.  Lane l also keeps the NEAR window of
// two future steps m = l and m = l + 32 (mod 64): the terms w_{m-k} f_k for
// k in [m-64, m-1], pushed as soon as f_k exists.  The far remainder
// (bulk + far window + first-node term) arrives from the helper warps about
// 60 steps ahead of need, so the chain never waits on them in steady state.
// ----------------------------------------------------------------------
template <int D>
struct LeaderState {
  double y0[D], fc[D], preP[D], preC[D];
  // near sums (P | C) of this lane's step in the current chunk (A) and the
  // next chunk (B): lane l owns steps 32c + l
  double accA[2 * D], accB[2 * D];
  int cA;                // chunk index of A
};

// Cold paths of the leader's waits, out of line with plain arguments (the
// hot loop keeps only the test; its instruction footprint is what the
// stepper's SM fetches every block).  Return the time waited in ns, or
// kColdFailed on abort / timeout.
constexpr unsigned long long kColdFailed = ~0ull;
__device__ __noinline__ unsigned long long leader_wait_far_cold(const int* hflag, int m, bool live, int* sabort,
                                                                DevCtrl* ctrl, const ShardView* shard, int n_shards,
                                                                unsigned long long timeout_ns, int c0, int lane) {
  const unsigned long long w0 = global_ns();
  unsigned spins = 0;
  while (!__all_sync(0xffffffffu, !live || ld_volatile_smem(hflag) == m)) {
    if (((++spins) & 1023u) == 0) {
      if (ld_volatile_smem(sabort) || *((volatile int*)&ctrl->abort)) return kColdFailed;
      if (global_ns() - w0 > timeout_ns) {
        if (lane == 0) raise_abort_cold(ctrl, shard, n_shards, ERR_TIMEOUT, KIND_NONE, c0, 0.0);
        st_volatile_smem(sabort, 1);
        return kColdFailed;
      }
    }
  }
  return global_ns() - w0;
}

// near sums of step m1 (owner lane -> all lanes via smem) and its far handoff.
// ROT: a chunk rotation is possible at this step (the fast block path knows
// statically where the 32-step chunk boundaries can fall).
// The far handoffs of a whole 32-step chunk are folded into
// the lanes' near sums once, when the chunk becomes current (lane l: step
// c0 + l), instead of one handoff read and 2d adds per step on the chain.
// The helpers hand a chunk off ~30 steps before it starts, so this waits
// only when the bulk of the chunk's block is late.  false on abort/timeout.
template <int D>
__device__ __forceinline__ bool leader_absorb_far(const EngineParams& P, StepperSmem& S, LeaderState<D>& st, int c0,
                                               int lane, unsigned long long& waited) {
  const int m = c0 + lane;
  const bool live = m < static_cast<int>(P.N);  // the helpers hand off steps m < N
  const int slot = m & (kHR - 1);
  if (__builtin_expect(!__all_sync(0xffffffffu, !live || ld_volatile_smem(&S.hflag[slot]) == m), 0)) {
    const unsigned long long w = leader_wait_far_cold(&S.hflag[slot], m, live, &S.abort, P.ctrl, P.shard, P.n_shards,
                                                      P.timeout_ns, c0, lane);
    if (w == kColdFailed) return false;
    waited += w;
  }
  __threadfence_block();  // acquire: the helpers release hflag after writing hbuf
  if (live) {
    double fr[2 * D];
    ld_pairs<D>(&S.hbuf[slot][0], fr);
#pragma unroll
    for (int c = 0; c < 2 * D; ++c) st.accA[c] = st.accA[c] + fr[c];
  }
  return true;
}

// the pre-sums of step m1 (near + far): the owner lane's sums, to all lanes
// through shared memory
template <int D>
__device__ __forceinline__ void leader_gather(StepperSmem& S, const LeaderState<D>& st, int m1, int lane,
                                              double* nr) {
  const int owner = m1 & (kChunk - 1);
  double* xb = &S.xfer[m1 & 1][0];
  if (lane == owner) st_pairs<D>(xb, st.accA);
  __syncwarp();
  ld_pairs<D>(xb, nr);
}

// push f_k (k = m1, just computed) into the near sums of A and B; the padded
// weight tables give 0 for steps already consumed (j <= 0)
struct PushW {
  double bA, bB, aA, aB;
};
template <bool K0>
__device__ __forceinline__ PushW leader_push_weights(const StepperSmem& S, int cA, int m1, int lane) {
  const int jA = cA * kChunk + lane - m1;  // -31..31
  const int jB = jA + kChunk;              // 1..63
  PushW w;
  w.bA = S.tb[jA + 2 * kChunk - 1];
  w.bB = S.tb[jB + 2 * kChunk - 1];
  w.aA = K0 ? 0.0 : S.ta[jA + 2 * kChunk - 1];  // corrector interior excludes k = 0
  w.aB = K0 ? 0.0 : S.ta[jB + 2 * kChunk - 1];
  return w;
}
template <int D>
__device__ __forceinline__ void leader_push(LeaderState<D>& st, const PushW& w, const double* fk) {
#pragma unroll
  for (int c = 0; c < D; ++c) {
    st.accA[c] = fma(w.bA, fk[c], st.accA[c]);
    st.accA[D + c] = fma(w.aA, fk[c], st.accA[D + c]);
    st.accB[c] = fma(w.bB, fk[c], st.accB[c]);
    st.accB[D + c] = fma(w.aB, fk[c], st.accB[D + c]);
  }
}

// One step n of the sequential chain (serial.py:150-170).  Source order is
// the issue order the in-order warp needs: everything that does not depend on
// this step's f (the gather of step n+1, its pre-sums, the push weights) is
// issued before the chain so it completes under the chain's FP64 latencies.
//   ROT: a chunk rotation can happen at this step (the 16-step blocks know
//        statically where the 32-step chunk boundaries can fall).
template <int SYS, int D, bool ROT, int ARRIVE = 1>
__device__ __forceinline__ bool leader_step(const EngineParams& P, StepperSmem& S, LeaderState<D>& st,
                                            double b0, double a0e, int n, int lane, uint32_t bars_u32,
                                            unsigned long long& waited) {
  const int m1 = n + 1;
  if (ROT && (m1 & (kChunk - 1)) == 0 && m1 > 0) {  // warp-uniform: chunk rotation, far parts folded in
#pragma unroll
    for (int c = 0; c < 2 * D; ++c) { st.accA[c] = st.accB[c]; st.accB[c] = 0.0; }
    st.cA += 1;
    if (!leader_absorb_far<D>(P, S, st, m1, lane, waited)) return false;
  }
  double nr[2 * D];
  leader_gather<D>(S, st, m1, lane, nr);
  const PushW pw = leader_push_weights<false>(S, st.cA, m1, lane);
  const double t1 = static_cast<double>(m1) * P.h;  // (n + 1) * h, serial.py:151
  const double ha = P.ha;
  double yP[D], fP[D], v[2 * D];
#pragma unroll
  for (int c = 0; c < D; ++c) yP[c] = add_rn(mul_rn(fma(b0, st.fc[c], st.preP[c]), ha), st.y0[c]);
  Rhs<SYS, D>::eval(t1, yP, fP, P.params);
#pragma unroll
  for (int c = 0; c < D; ++c)  // ((c_n f0 + C_n) + fP/G2) * h^a + y0, serial.py:160-165
    v[c] = add_rn(mul_rn(add_rn(fma(a0e, st.fc[c], st.preC[c]), mul_rn(P.ig, fP[c])), ha), st.y0[c]);
  Rhs<SYS, D>::eval(t1, v, v + D, P.params);
  // publish (y_{n+1}, f_{n+1})
  const int ri = m1 & (kRing - 1);
  if (lane == 0) {
    st_pairs<D>(&S.ring[ri][0], v);
#pragma unroll
    for (int c = 0; c < D; ++c) S.ring[ri][2 * D + c] = fP[c];  // checked by the writer warp
  }
  // one release arrive per 8-step group (its last row, or row N), predicated:
  // the warp stays converged and 7 of 8 steps carry no fence
  if (ARRIVE == 1) {
    const bool group_end = ((m1 & 7) == 7) | (m1 == static_cast<int>(P.N));
    mbar_arrive_if_u32(bars_u32 + 8u * static_cast<uint32_t>(pub_group(m1) & (kNumBars - 1)), (lane == 0) & group_end);
  } else if (ARRIVE == 2) {  // the caller knows this row ends its publication group
    mbar_arrive_if_u32(bars_u32 + 8u * static_cast<uint32_t>(pub_group(m1) & (kNumBars - 1)), lane == 0);
  }
  leader_push<D>(st, pw, v + D);
#pragma unroll
  for (int c = 0; c < D; ++c) st.fc[c] = v[D + c];
  // non-finite rhs outputs are detected by the writer warp on the published
  // rows (fP and f of every step), off the chain's SMSP
  // pre-sums of step n+1: the owner's near sum (far part included at the
  // rotation), read now so the shared-memory loads complete under the chain
#pragma unroll
  for (int c = 0; c < D; ++c) {
    st.preP[c] = nr[c];
    st.preC[c] = nr[D + c];
  }
  return true;
}


// ring back-pressure wait (cold, out of line): until every consumer has
// drained entry n_next+1-kRing+32
__device__ __noinline__ unsigned long long leader_wait_ring_cold(StepperSmem* S, long long n_next, DevCtrl* ctrl,
                                                                 const ShardView* shard, int n_shards,
                                                                 unsigned long long timeout_ns, int lane) {
  unsigned spins = 0;
  const unsigned long long w0 = global_ns();
  while (n_next - slowest_consumer(*S) > kRing - 32) {
    if (((++spins) & 1023u) == 0) {
      if (ld_volatile_smem(&S->abort) || *((volatile int*)&ctrl->abort)) return kColdFailed;
      if (global_ns() - w0 > timeout_ns) {
        if (lane == 0) raise_abort_cold(ctrl, shard, n_shards, ERR_TIMEOUT, KIND_NONE, n_next, 0.0);
        st_volatile_smem(&S->abort, 1);
        return kColdFailed;
      }
    }
  }
  return global_ns() - w0;
}

template <int D>
__device__ __forceinline__ bool leader_check_block(const EngineParams& P, StepperSmem& S, const LeaderState<D>& st,
                                                   long long n_next, int lane, unsigned long long& throttled,
                                                   unsigned long long& lag_sum) {
  if (ld_volatile_smem(&S.abort)) return false;  // the writer found a non-finite rhs output (or a watchdog fired)
  // ring back-pressure: the writer warp and every helper warp must have
  // drained entry n+1-kRing (also keeps the mbarrier phases unaliased)
  const long long lag = n_next - slowest_consumer(S);
  lag_sum += static_cast<unsigned long long>(lag);
  if (__builtin_expect(lag > kRing - 32, 0)) {
    const unsigned long long w = leader_wait_ring_cold(&S, n_next, P.ctrl, P.shard, P.n_shards, P.timeout_ns, lane);
    if (w == kColdFailed) return false;
    throttled += w;
  }
  return true;
}

// 16 steps n .. n+15 (n % 16 == 0, n + 16 <= N): a 32-step chunk boundary
// (m1 % 32 == 0) can only be the last step, and only when LAST (the caller
// knows that row n+16 is not N otherwise); rows n+7 and n+15 end publication
// groups (arrive unconditionally), row n+16 when it is row N (predicated,
// LAST only); the other steps carry no arrive (an asm with a memory clobber)
// at all.  Blocks of 16 steps instead of 8 halve the loop's branch and
// instruction-fetch overhead: N=1e5 12.41 -> 11.47 ms, 243 -> 225 cycles/step
// (blocks of 32, as two halves with a check between: 12.16 ms -- not adopted)
constexpr int kLeaderBlock = 16;

template <int SYS, int D, bool LAST>
__device__ __forceinline__ bool leader_run16(const EngineParams& P, StepperSmem& S, LeaderState<D>& st, double b0,
                                             double a0, int n, int lane, uint32_t bars_u32,
                                             unsigned long long& waited) {
  constexpr int A0 = 0, A6 = 2, A7 = 1;
  if (!leader_step<SYS, D, false, A0>(P, S, st, b0, a0, n + 0, lane, bars_u32, waited)) return false;
  if (!leader_step<SYS, D, false, A0>(P, S, st, b0, a0, n + 1, lane, bars_u32, waited)) return false;
  if (!leader_step<SYS, D, false, A0>(P, S, st, b0, a0, n + 2, lane, bars_u32, waited)) return false;
  if (!leader_step<SYS, D, false, A0>(P, S, st, b0, a0, n + 3, lane, bars_u32, waited)) return false;
  if (!leader_step<SYS, D, false, A0>(P, S, st, b0, a0, n + 4, lane, bars_u32, waited)) return false;
  if (!leader_step<SYS, D, false, A0>(P, S, st, b0, a0, n + 5, lane, bars_u32, waited)) return false;
  if (!leader_step<SYS, D, false, A6>(P, S, st, b0, a0, n + 6, lane, bars_u32, waited)) return false;
  if (!leader_step<SYS, D, false, A0>(P, S, st, b0, a0, n + 7, lane, bars_u32, waited)) return false;
  if (!leader_step<SYS, D, false, A0>(P, S, st, b0, a0, n + 8, lane, bars_u32, waited)) return false;
  if (!leader_step<SYS, D, false, A0>(P, S, st, b0, a0, n + 9, lane, bars_u32, waited)) return false;
  if (!leader_step<SYS, D, false, A0>(P, S, st, b0, a0, n + 10, lane, bars_u32, waited)) return false;
  if (!leader_step<SYS, D, false, A0>(P, S, st, b0, a0, n + 11, lane, bars_u32, waited)) return false;
  if (!leader_step<SYS, D, false, A0>(P, S, st, b0, a0, n + 12, lane, bars_u32, waited)) return false;
  if (!leader_step<SYS, D, false, A0>(P, S, st, b0, a0, n + 13, lane, bars_u32, waited)) return false;
  if (!leader_step<SYS, D, false, A6>(P, S, st, b0, a0, n + 14, lane, bars_u32, waited)) return false;
  return leader_step<SYS, D, LAST, LAST ? A7 : A0>(P, S, st, b0, a0, n + 15, lane, bars_u32, waited);
}

template <int SYS, int D>
__device__ void stepper_leader(const EngineParams& P, StepperSmem& S, int lane) {
  const long long N = P.N;
  LeaderState<D> st;
  double f0[D];
#pragma unroll
  for (int c = 0; c < D; ++c) st.y0[c] = P.y0[c];
  Rhs<SYS, D>::eval(0.0, st.y0, f0, P.params);
  const bool bad0 = any_nonfinite<D>(f0);
  if (lane == 0) {
    double v0[2 * D];
#pragma unroll
    for (int c = 0; c < D; ++c) { v0[c] = st.y0[c]; v0[D + c] = f0[c]; }
    st_pairs<D>(&S.ring[0][0], v0);
    if (bad0) raise_abort(P, ERR_NONFINITE, KIND_INITIAL, 0, 0.0);
  }
  if (bad0) st_volatile_smem(&S.abort, 1);
  if (lane == 0) mbar_arrive(&S.bars[0]);
  if (bad0) return;

  const double b0 = P.wb[0], a0 = P.wa[0];
  unsigned long long waited = 0, throttled = 0;
  st.cA = 0;
#pragma unroll
  for (int c = 0; c < 2 * D; ++c) { st.accA[c] = 0.0; st.accB[c] = 0.0; }

  // step 0: its pre-sums are the far handoff alone (c_0 f_0); then f_0 enters
  // the near sums of steps 1..63
  if (!leader_absorb_far<D>(P, S, st, 0, lane, waited)) return;  // chunk 0: the first-node terms c_m f_0
  {
    double nr[2 * D];
    leader_gather<D>(S, st, 0, lane, nr);
#pragma unroll
    for (int c = 0; c < D; ++c) {
      st.preP[c] = nr[c];
      st.preC[c] = nr[D + c];
    }
  }
  leader_push<D>(st, leader_push_weights<true>(S, st.cA, 0, lane), f0);
#pragma unroll
  for (int c = 0; c < D; ++c) st.fc[c] = f0[c];

  const uint32_t bars_u32 = smem_u32(&S.bars[0]);
  const int N32 = static_cast<int>(N);
  const bool solo = (P.debug & 1) != 0;  // dev: leader ignores handoffs and back-pressure (results invalid)
  const long long c_loop = clock64();
  unsigned long long fast_blocks = 0, lag_sum = 0;
  int n = 0;
  // step 0 has no corrector interior (a0 term excluded); blocks start at kLeaderBlock
  if (!leader_step<SYS, D, true>(P, S, st, b0, 0.0, 0, lane, bars_u32, waited)) return;
  for (n = 1; n < kLeaderBlock && n < N32; ++n)
    if (!leader_step<SYS, D, true>(P, S, st, b0, a0, n, lane, bars_u32, waited)) return;
  if (!leader_check_block<D>(P, S, st, n, lane, throttled, lag_sum)) return;
  const int n_fast0 = n;
  while (n + kLeaderBlock <= N32) {
    if (!leader_run16<SYS, D, true>(P, S, st, b0, a0, n, lane, bars_u32, waited)) return;
    n += kLeaderBlock;
    // back-pressure / abort check every 16 steps (its 9 shared-memory loads
    // stall the in-order issue); the lag bound leaves room for 16 more steps
    if (!solo && !leader_check_block<D>(P, S, st, n, lane, throttled, lag_sum)) return;
  }
  fast_blocks = static_cast<unsigned long long>(n - n_fast0) / 8;  // (a counter in the loop costs a register)
#pragma unroll 1
  for (; n < N32; ++n)
    if (!leader_step<SYS, D, true>(P, S, st, b0, a0, n, lane, bars_u32, waited)) return;
  if (!solo && !leader_check_block<D>(P, S, st, n, lane, throttled, lag_sum)) return;
  if (lane == 0) {
    P.ctrl->prof[0] = static_cast<unsigned long long>(clock64() - c_loop);
    P.ctrl->prof[1] = fast_blocks;
    P.ctrl->prof[2] = lag_sum;
    P.ctrl->leader_wait_ns = waited;
    P.ctrl->leader_throttle_ns = throttled;
  }
}

// ----------------------------------------------------------------------
// Helper threads (warps 1,2,3,5,6,7): each owns kSlotsPerThread far slots m
// and pushes every published f_k with k in [lo(m), m-65] into them, in
// ascending k; after f_{m-65} it adds the staged bulk sum and the first-node
// term and hands the far part to the leader warp (~60 steps before it is
// needed), then re-opens the slot for step m + kSlots.  Wakes once per
// kBatch publishes.  The push is branch-free; only handoffs branch.
// ----------------------------------------------------------------------
template <int D>
__device__ __forceinline__ bool helper_handoff(const EngineParams& P, StepperSmem& S, int m, const double* f0,
                                               const double* accP, const double* accC) {
  // the publisher staged block J: its first-node coefficients and, for
  // J >= L, the bulk sums of the sources below lo (which include k = 0 in
  // the a-sum, hence the coefficient c_m - a_m there)
  const int J = m / kB;
#ifdef FABM_PROFILE
  if (P.trace && (m % kB) == 0) P.trace[4 * J + 3] = global_ns();
#endif
  if (ld_acquire_cta_smem(&S.bulk_flag) < J) {
    unsigned sp2 = 0;
    const unsigned long long w1 = global_ns();
    while (ld_acquire_cta_smem(&S.bulk_flag) < J) {
      if (ld_volatile_smem(&S.abort)) return false;
      if (((++sp2) & 255u) == 0) {
        if (*((volatile int*)&P.ctrl->abort)) return false;
        if (global_ns() - w1 > P.timeout_ns) return false;
      }
    }
  }
  const int bsel = J & 1;
  const int r = m % kB;
  const double cf = S.cfirst[bsel][r];
  double hv[2 * D];
  if (J >= kL) {
#pragma unroll
    for (int c = 0; c < D; ++c) {
      hv[c] = accP[c] + S.bulk[bsel][r][0][c];
      hv[D + c] = add_rn(accC[c] + S.bulk[bsel][r][1][c], mul_rn(cf, f0[c]));
    }
  } else {
#pragma unroll
    for (int c = 0; c < D; ++c) {
      hv[c] = accP[c];
      hv[D + c] = add_rn(accC[c], mul_rn(cf, f0[c]));
    }
  }
  const int slot = m % kHR;
  st_pairs<D>(&S.hbuf[slot][0], hv);
  st_release_cta_smem(&S.hflag[slot], m);
  return true;
}

// Push the published f_k, k in [k0, k0 + 8) (those <= kl), into this
// thread's far slots.  Batches are 8-aligned, and both ends of a slot's far
// window -- lo(m) (a multiple of 128) and kh(m) = 32(c-1) - 1 (== 7 mod 8) --
// are batch boundaries, so the window test is one predicate per slot per
// batch and the unrolled body is branch-free.
template <int D>
__device__ __forceinline__ void helper_batch(const StepperSmem& S, int k0, int kl, const int (&m)[kSlotsPerThread],
                                             const bool (&in)[kSlotsPerThread],
                                             double (&accP)[kSlotsPerThread][D],
                                             double (&accC)[kSlotsPerThread][D]) {
#pragma unroll
  for (int i = 0; i < kBatch; ++i) {
    const int k = k0 + i;
    const bool live = k <= kl;
    double fk[D];
    const double* row = &S.ring[k & (kRing - 1)][0];
#pragma unroll
    for (int c = 0; c < D; ++c) fk[c] = live ? row[D + c] : 0.0;  // entries past kl may be unwritten
#pragma unroll
    for (int s = 0; s < kSlotsPerThread; ++s) {
      const bool on = in[s] & live;
      const int jj = on ? m[s] - k : 0;
      const double wb = on ? S.wb[jj] : 0.0;
      const double wa = on ? S.wa[jj] : 0.0;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        accP[s][c] = fma(wb, fk[c], accP[s][c]);
        accC[s][c] = fma(wa, fk[c], accC[s][c]);
      }
    }
  }
}

template <int D>
__device__ void stepper_helper(const EngineParams& P, StepperSmem& S, int hid, int hwarp) {
  constexpr int NS = kSlotsPerThread;
  const int N = static_cast<int>(P.N);
  const int lane = threadIdx.x & 31;
  int m[NS], lo[NS];
  double accP[NS][D], accC[NS][D], f0[D];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    m[s] = hid + s * (kSlots / NS);
    lo[s] = static_cast<int>(lo_of(m[s]));
#pragma unroll
    for (int c = 0; c < D; ++c) { accP[s][c] = 0.0; accC[s][c] = 0.0; }
  }
  long long c_wait = 0, c_proc = 0;  // dev statistics (helper warp 1)

  // batches [0], [1, 7], [8, 15], [16, 23], ...: step 0 alone, since the
  // handoffs of chunks 0 and 1 need only f_0 and the leader waits for them
  for (int k0 = 0, kl = 0; k0 <= N; k0 = kl + 1, kl = (((k0 | (kBatch - 1)) < N) ? (k0 | (kBatch - 1)) : N)) {
    uint64_t* bar = &S.bars[pub_group(kl) % kNumBars];
    const uint32_t par = static_cast<uint32_t>((pub_group(kl) / kNumBars) & 1);
    const long long c_w = clock64();
    if (!mbar_test(bar, par)) {
      unsigned spins = 0;
      const unsigned long long w0 = global_ns();
      const bool spin = (P.debug & 4) != 0;  // dev: poll without the suspend hint
      while (!(spin ? mbar_test(bar, par) : mbar_wait_hint(bar, par, 100000u))) {
        if (ld_volatile_smem(&S.abort)) return;
        if (((++spins) & 255u) == 0) {
          if (*((volatile int*)&P.ctrl->abort)) return;
          if (global_ns() - w0 > P.timeout_ns) return;
        }
      }
    }
    const long long c_p = clock64();
    if (k0 == 0) {
      // f_0: enters the predictor sums only (the corrector interior starts at
      // k = 1; its k = 0 term is the first-node coefficient, added at handoff)
      const double* row = &S.ring[0][0];
#pragma unroll
      for (int c = 0; c < D; ++c) f0[c] = row[D + c];
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const int kh = (m[s] & ~(kChunk - 1)) - kChunk - 1;
        const double wb = (lo[s] == 0 && kh >= 0) ? S.wb[m[s]] : 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) accP[s][c] = fma(wb, f0[c], accP[s][c]);
      }
    } else {
      const bool skip = (P.debug & 2) != 0;  // dev: no far-window pushes (results invalid)
      bool in[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const int kh = (m[s] & ~(kChunk - 1)) - kChunk - 1;  // last far term: 32(c-1) - 1
        in[s] = (k0 >= lo[s]) & (kl <= kh) & !skip;
      }
      helper_batch<D>(S, k0, kl, m, in, accP, accC);
    }
    // handoffs: slots whose far window ends with this batch (chunks 0 and 1:
    // with f_0).  One branch per slot per batch.
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int kh = (m[s] & ~(kChunk - 1)) - kChunk - 1;
      const bool due = (k0 == 0) ? (kh <= 0) : (kl == kh);
      if (due && m[s] < N) {
        if (!helper_handoff<D>(P, S, m[s], f0, accP[s], accC[s])) return;
        m[s] += kSlots;
        lo[s] = static_cast<int>(lo_of(m[s]));
#pragma unroll
        for (int c = 0; c < D; ++c) { accP[s][c] = 0.0; accC[s][c] = 0.0; }
      }
    }
    __syncwarp();
    if (lane == 0) st_volatile_smem(&S.hprog[hwarp], kl);
    const long long c_e = clock64();
    c_wait += c_p - c_w;
    c_proc += c_e - c_p;
  }
  if (hwarp == 1 && lane == 0) {
    P.ctrl->prof[3] = static_cast<unsigned long long>(c_wait);
    P.ctrl->prof[7] = static_cast<unsigned long long>(c_proc);
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
    uint64_t* bar = &S.bars[pub_group(kend) % kNumBars];
    const uint32_t par = static_cast<uint32_t>((pub_group(kend) / kNumBars) & 1);
    unsigned spins = 0;
    const unsigned long long w0 = global_ns();
    while (!mbar_wait_hint(bar, par, 100000u)) {
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
    // rows k >= 1 carry step n = k - 1: its predictor rhs fP and corrector rhs
    // f_k; the first failing step, predictor before corrector (serial.py:157,167)
    int kind = KIND_NONE;
    if (k <= kend && k >= 1) {
      const double* row = &S.ring[static_cast<int>(k % kRing)][0];
      double fp[D], fk[D];
#pragma unroll
      for (int c = 0; c < D; ++c) { fp[c] = row[2 * D + c]; fk[c] = row[D + c]; }
      kind = any_nonfinite<D>(fp) ? KIND_PREDICTOR : (any_nonfinite<D>(fk) ? KIND_CORRECTOR : KIND_NONE);
    }
    const unsigned bad = __ballot_sync(0xffffffffu, kind != KIND_NONE);
    if (bad) {
      const int first = __ffs(bad) - 1;
      if (lane == first) {
        const long long n = k - 1;
        raise_abort(P, ERR_NONFINITE, kind, n, static_cast<double>(n + 1) * P.h);
        st_volatile_smem(&S.abort, 1);
      }
      return;
    }
    if (k <= kend) {
      FABM_CHECK(P, k >= 0 && k <= N && k < P.f_rows);
      const int ri = static_cast<int>(k % kRing);
      double yf[2 * D];
      ld_pairs<D>(&S.ring[ri][0], yf);
      double* yd = P.Y + k * D;
      double* fd = P.F + k * DS;
      double* fo = P.Fc + k * D;
#pragma unroll
      for (int c = 0; c < D; ++c) { yd[c] = yf[c]; fd[c] = yf[D + c]; fo[c] = yf[D + c]; }
      if (P.Yh) {  // trajectory streamed to mapped pinned host memory during the run (no D2H afterwards)
        double* yh = P.Yh + k * D;
        double* fh = P.Fch + k * D;
#pragma unroll
        for (int c = 0; c < D; ++c) { yh[c] = yf[c]; fh[c] = yf[D + c]; }
      }
      for (int sh = 1; sh < P.n_shards; ++sh) {  // peer copies of the f history
        double* fp = P.shard[sh].F + k * DS;
#pragma unroll
        for (int c = 0; c < D; ++c) fp[c] = yf[D + c];
      }
    }
    if (P.n_shards > 1 && ((kend + 1) % kB) == 0) __threadfence_system();
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
  int next_stage = 0;
  unsigned long long last_progress = global_ns();
  while (published < last_block || next_stage < nb) {
    bool progress = false;
    // (1) source blocks written by the writer warp -> GPU-scope publication
    int io_block = 0;
    if (lane == 0) io_block = ld_acquire_cta_smem(&S.io_block);
    io_block = __shfl_sync(0xffffffffu, io_block, 0);
    if (io_block > published) {
      if (lane == 0) {
        if (P.n_shards == 1) {
          __threadfence();  // cumulative over the writer's rows (acquired above)
          st_release_gpu(&P.ctrl->src_done, io_block);
        } else {
          __threadfence_system();
          for (int sh = 0; sh < P.n_shards; ++sh) st_release_sys(&P.shard[sh].ctrl->src_done, io_block);
        }
#ifdef FABM_PROFILE
        if (P.trace)
          for (int q = published; q < io_block; ++q) P.trace[4 * q + 0] = global_ns();
#endif
      }
      published = io_block;
      progress = true;
    }
    // (2) stage block J once the helpers are done with buffer J&1 (the leader
    // has published step (J-1)*B): first-node coefficients for every block,
    // plus, for J >= L, the bulk sums once the agents flagged them complete
    if (next_stage < nb && ld_volatile_smem(&S.io_done) - 1 >= static_cast<long long>(next_stage - 1) * kB) {
      int rdy = 1;
      if (next_stage >= kL) {
        if (lane == 0) rdy = P.n_shards == 1 ? ld_acquire_gpu(&P.ready[next_stage]) : ld_acquire_sys(&P.ready[next_stage]);
        rdy = __shfl_sync(0xffffffffu, rdy, 0);
      }
      if (rdy) {
        __syncwarp();
        const int J = next_stage;
        const long long m0 = static_cast<long long>(J) * kB;
        for (int r = lane; r < kB; r += 32) {
          const long long mm = m0 + r;
          double cf = 0.0;
          if (mm < P.N) cf = J >= kL ? P.wc[mm] - P.wa[mm] : P.wc[mm];
          S.cfirst[J & 1][r] = cf;
        }
        if (J >= kL) {
          const double* src = P.BK + m0 * 2 * DS;
          double* dst = &S.bulk[J & 1][0][0][0];
          for (int i = lane; i < kB * 2 * D; i += 32) {
            const int row = i / (2 * D), rem = i % (2 * D), half = rem / D, c = rem % D;
            dst[(row * 2 + half) * 4 + c] = __ldcg(src + (row * 2 + half) * DS + c);
          }
        }
        __syncwarp();
        if (lane == 0) st_release_cta_smem(&S.bulk_flag, J);
#ifdef FABM_PROFILE
        if (P.trace && lane == 0) P.trace[4 * J + 2] = global_ns();
#endif
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
  for (int i = tid; i < kSlots + 2 * kGFar; i += kThreads) {
    S.wb[i] = i < kSlots ? P.wb[i] : 0.0;
    S.wa[i] = i < kSlots ? P.wa[i] : 0.0;
  }
  for (int i = tid; i < 4 * kChunk; i += kThreads) {
    const int j = i - (2 * kChunk - 1);
    S.tb[i] = (j >= 1 && j < kSlots) ? P.wb[j] : 0.0;
    S.ta[i] = (j >= 1 && j < kSlots) ? P.wa[j] : 0.0;
  }
  for (int i = tid; i < kHR; i += kThreads) S.hflag[i] = -1;
  if (tid < kWarps) S.hprog[tid] = -1;
  if (tid == 0) {
    S.bulk_flag = -1;
    S.io_done = 0;
    S.io_block = 0;
    S.abort = 0;
    for (int i = 0; i < kNumBars; ++i) mbar_init(&S.bars[i], 1);
  }
  __syncthreads();
  if (warp == 0) { stepper_leader<SYS, D>(P, S, lane); return; }
  // SMSP 0 (warps 0, 4, 8, 12) belongs to the leader alone: the writer and
  // the publisher poll, and their issue slots would come out of the chain's
  if (warp == kWriterWarp) { stepper_writer<D>(P, S, lane); return; }
  if (warp == kPublisherWarp) { stepper_publisher<D>(P, S, lane); return; }
  if ((warp & 3) == 0) return;  // SMSP 0 stays with the leader warp
  const int hw = helper_index(warp);  // warps 1,2,3,5,6,7,9,10 -> 0..7
  if (hw >= kHelperWarps) return;
  stepper_helper<D>(P, S, hw * 32 + lane, warp);
}

// ======================================================================
// BULK AGENTS
// ======================================================================
}  // namespace fabm
#include "bulk_dmma.cuh"
namespace fabm {

// ---------------------------------------------------------------- units
// The bulk sums of target block J run over its n = J-L+1 chunks I = 0 .. J-L
// (Toeplitz tiles T_{J-I} F_I).  The chunks are cut at fixed points into
// SEGMENTS of S = 2^k chunks, k = max(0, floor(log2 n) - 4), so a target has
// 16..32 units (fewer below n = 16): unit (J, s) = chunks [sS, min((s+1)S, n)).
// A unit is one ascending DMMA chain from zero; a target's sum is its
// units' partial sums added in ascending s (one fixed-order reduction per
// target block).  The partition depends on J alone: results are bitwise
// independent of N (the first M steps of an N-step run equal the M-step
// run), of which agent or GPU computed which unit, and of the timing.
//
// Scheduling: agent a OWNS targets J = L + a + i*A
// (round-robin) and processes their units incrementally as source blocks
// are published, earliest target first.  A unit of a COMPLETE column (its
// segment's sources all published) that no owner has started is CLAIMED by
// any agent whose earliest owned work is later: targets with the same S
// form a class, each (class, segment) column has a cursor walking its
// targets in ascending J, and a per-unit claim word (CAS) arbitrates between
// owners and claimers.  Reduction in two stages so that the deadline path is
// short: the last non-final unit to finish sums the prefix p_0 + .. +
// p_{n-2} (usually long before the deadline), and whichever of {prefix,
// final unit} arrives second adds the final unit's partial.
constexpr int kMaxClasses = 32;
#ifndef FABM_DYN_BURST  // (dev overrides for A/B sweeps, tools/ab_engine.py)
#define FABM_DYN_BURST 4
#endif
#ifndef FABM_URGENT
#define FABM_URGENT 16
#endif
constexpr int kDynBurst = FABM_DYN_BURST;  // chunks of a claimed unit between selections (8: 200 vs 182 ms at N=1e6)
constexpr int kUrgent = FABM_URGENT;  // blocks before an owned target's deadline that end a claimed-unit burst
// segments of S = 2^k chunks, k = max(kSegMin, floor(log2 n) - 4): up to
// 16..32 units per target, none shorter than 2^kSegMin chunks -- with one-
// chunk units the first targets summed ~30 partials right at their deadline
// (kSegMin 0 -> 5: N=1e5 13.2 -> 12.66 ms, N=1e6 181.2 -> 180.3 ms)
#ifndef FABM_SEG_KMIN
#define FABM_SEG_KMIN 5
#endif
constexpr int kSegMin = FABM_SEG_KMIN;
__host__ __device__ __forceinline__ int seg_class_of_log(int lg) { return lg - 4 > kSegMin ? lg - 4 : kSegMin; }
__device__ __forceinline__ int seg_class(int n) { return seg_class_of_log(31 - __clz(n)); }
// class k covers n in [lo, hi): the lowest class starts at n = 1
__host__ __device__ __forceinline__ int class_lo(int k) { return k == kSegMin ? 1 : 1 << (k + 4); }
__host__ __device__ __forceinline__ int class_hi(int k) { return 1 << (k + 5); }
__host__ __device__ __forceinline__ long long seg_prefix(long long m, int k) {  // sum_{n'=1..m} ceil(n'/2^k)
  const long long q = m >> k, r = m & ((1LL << k) - 1);
  return ((q * (q + 1)) << k) / 2 + r * (q + 1);
}
// units of the classes below k: the lowest class (n = 1 .. 2^(kSegMin+5)-1)
// has seg_prefix(2^(kSegMin+5)-1, kSegMin); class j above it (n = 16S ..
// 32S-1, S = 2^j) has sum_{q=16..31} (qS + S - 1) = 392 S - 16
__host__ __device__ __forceinline__ long long class_base(int k) {
  if (k <= kSegMin) return 0;
  const long long t0 = seg_prefix((1LL << (kSegMin + 5)) - 1, kSegMin);
  return t0 + 392 * ((1LL << k) - (2LL << kSegMin)) - 16LL * (k - 1 - kSegMin);
}
// unit id of (J, 0): units of targets L .. J-1
__device__ __forceinline__ long long unit_base(const EngineParams&, int J) {
  const int n = J - kL + 1;
  const int k = seg_class(n);
  return class_base(k) + seg_prefix(n - 1, k) - seg_prefix(class_lo(k) - 1, k);
}

__device__ __forceinline__ int owned_target(int agent, int i, int nA) { return kL + agent + i * nA; }
__device__ __forceinline__ int owned_count(int agent, int nA, int n_targets) {
  return agent < n_targets ? (n_targets - 1 - agent) / nA + 1 : 0;
}

__device__ __forceinline__ int at_cas(int* p, int c, int v, bool sys) {
  return sys ? atomicCAS_system(p, c, v) : atomicCAS(p, c, v);
}
__device__ __forceinline__ int at_add(int* p, int v, bool sys) { return sys ? atomicAdd_system(p, v) : atomicAdd(p, v); }
__device__ __forceinline__ void at_max(int* p, int v, bool sys) {
  if (sys) atomicMax_system(p, v); else atomicMax(p, v);
}
__device__ __forceinline__ int ld_rlx(const int* p, bool sys) { return sys ? ld_relaxed_sys(p) : ld_relaxed_gpu(p); }
__device__ __forceinline__ void fence_scope(bool sys) {
  if (sys) __threadfence_system(); else __threadfence();
}

template <int D>
struct BulkSmem {
  DmmaSmem<D> t;
  int own_next[kMaxOwn];   // owned target i: (next chunk << 1) | (holds the unit of that chunk)
};

template <int D>
__device__ __forceinline__ double* unit_slot(const EngineParams& P, long long uid) {
  return P.PK + uid * (32 * 8 * D);
}

template <int D>
__device__ __forceinline__ void publish_target(const EngineParams& P, int J, int lane, const DmmaAcc<D>& acc, bool sys) {
  __syncwarp();
  dmma_store_rows<D>(P.BK, J, lane, acc);  // shard 0's BK (peer memory on other GPUs)
  fence_scope(sys);
  __syncwarp();
  if (lane == 0) {
    if (sys) st_release_sys(&P.ready[J], 1); else st_release_gpu(&P.ready[J], 1);
  }
#ifdef FABM_PROFILE
  if (P.trace && lane == 0) P.trace[4 * J + 1] = global_ns();
#endif
}

// second arrival at stage 2 of target J's reduction?
__device__ __forceinline__ bool stage2_second(const EngineParams& P, int J, int lane, bool sys) {
  int second = 0;
  if (lane == 0) {
    const int old = at_add(&P.tstage[J], 1, sys);
    FABM_CHECK(P, old == 0 || old == 1);
    second = old == 1;
  }
  second = __shfl_sync(0xffffffffu, second, 0);
  if (second) fence_scope(sys);
  return second != 0;
}

// A unit's chain is complete (acc = its partial sums).
template <int D>
__device__ void unit_finish(const EngineParams& P, int J, int s, long long uid, int lane, DmmaAcc<D>& acc, bool sys) {
  const int n = J - kL + 1;
  const int S = 1 << seg_class(n);
  const int nseg = (n + S - 1) / S;
  if (nseg == 1) {
    publish_target<D>(P, J, lane, acc, sys);
    return;
  }
  dmma_spill_slot<D>(unit_slot<D>(P, uid), lane, acc);
  fence_scope(sys);
  __syncwarp();
  const long long base = unit_base(P, J);
#ifdef FABM_CHECKED
  // each unit finishes exactly once: its claim word turns negative here
  if (lane == 0) {
    const int w = ld_rlx(&P.claim[uid], sys);
    FABM_CHECK(P, w > 0 && at_cas(&P.claim[uid], w, -w, sys) == w);
  }
#endif
  if (s == nseg - 1) {  // the final unit: P + p_final if the prefix is already there
    if (!stage2_second(P, J, lane, sys)) return;
    dmma_add_slot<D>(unit_slot<D>(P, base), lane, acc);  // p_final + P == P + p_final (IEEE add commutes)
    publish_target<D>(P, J, lane, acc, sys);
    return;
  }
  int last = 0;
  if (lane == 0) {
    const int old = at_add(&P.tdone[J], 1, sys);
    FABM_CHECK(P, old >= 0 && old <= nseg - 2);
    last = old == nseg - 2;
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
  fence_scope(sys);
  if (nseg > 2) {  // prefix p_0 + .. + p_{nseg-2} into unit 0's slot
    dmma_reload_slot<D>(unit_slot<D>(P, base), lane, acc);
    for (int q = 1; q < nseg - 1; ++q) dmma_add_slot<D>(unit_slot<D>(P, base + q), lane, acc);
    __syncwarp();
    dmma_spill_slot<D>(unit_slot<D>(P, base), lane, acc);
    fence_scope(sys);
    __syncwarp();
  } else {
    dmma_reload_slot<D>(unit_slot<D>(P, base), lane, acc);
  }
  if (!stage2_second(P, J, lane, sys)) return;
  dmma_add_slot<D>(unit_slot<D>(P, base + nseg - 1), lane, acc);
  publish_target<D>(P, J, lane, acc, sys);
}

// earliest claimable unit: the lowest class with a claimable column holds
// the smallest J (classes are ordered by J).  kc: lowest class not yet
// exhausted (only grows).  Returns J (or INT_MAX) and sets k/c.
__device__ __forceinline__ int scan_claimable(const EngineParams& P, int M, int lane, bool sys, int& kc, int& kk,
                                              int& cc) {
  const int nend_all = P.nb - kL + 1;  // n < nend_all
  // every target J <= M-1 is complete (the stepper passed it): a class whose
  // last target is below M has nothing left to claim
  while (kc <= P.k_max && class_hi(kc) + kL - 2 < M) ++kc;
  for (int k = kc; k <= P.k_max; ++k) {
    const int S = 1 << k;
    const int nend = min(class_hi(k), nend_all);
    const int ns = max(class_lo(k), (lane + 1) * S + 1);
    const bool col = lane < 31 && ns < nend;
    const int cur = col ? ns + ld_rlx(&P.col_next[k * 32 + lane], sys) : nend;
    const bool exhausted = cur >= nend;
    if (__all_sync(0xffffffffu, exhausted)) {
      if (k == kc) kc = k + 1;
      continue;
    }
    const int myJ = (!exhausted && M >= (lane + 1) * S) ? cur + kL - 1 : 0x7fffffff;
    const int mn = __reduce_min_sync(0xffffffffu, myJ);
    if (mn < 0x7fffffff) {
      kk = k;
      cc = __ffs(__ballot_sync(0xffffffffu, myJ == mn)) - 1;
      return mn;
    }
    if (M < 2 * S) break;  // no complete column in the classes above
  }
  return 0x7fffffff;
}

template <int D>
__device__ void bulk_agent(const EngineParams& P, BulkSmem<D>& A, int agent, int lane, const ShardView& sv) {
  const int nb = P.nb;
  const int n_targets = nb - kL;  // targets J = L .. nb-1
  if (n_targets <= 0) return;
  if (P.debug & 8) return;  // dev: no bulk agents (results invalid; the run reports FABM_ERR_CONFIG)
  FABM_CHECK(P, !(P.debug & 16));  // dev: positive control of the FABM_CHECKED reporting path
  const bool sys = P.n_shards > 1;
  const int nA = P.n_agents;
  const int nown = owned_count(agent, nA, n_targets);
  for (int i = lane; i < nown; i += 32) A.own_next[i] = 0;
  __syncwarp();
  DmmaAcc<D> acc;
  dmma_zero<D>(acc);
  long long cur_uid = -1;           // the unit whose chain is in acc
  int dJ = -1, ds = 0, dnext = 0;   // claimed (dynamic) unit, if any
  int kc = kSegMin;                 // lowest class with unclaimed columns
  int dyn_lb = 0, lb_M = -1;        // cached lower bound of the earliest claimable target (valid for lb_M)
  unsigned idle_polls = 0;
  unsigned long long tiles = 0, claims = 0;
  unsigned long long last_progress = global_ns();
  int last_M = -1;  // the watchdog counts the stepper's progress too (an agent may idle for long)

#ifdef FABM_PROFILE
  long long c_tile = 0, c_idle = 0, c_sw = 0, c_t = clock64();
  unsigned long long n_sel = 0, n_scan = 0, n_spill = 0, n_reload = 0, n_fin = 0, c_fin = 0, c_scan = 0, n_idle = 0;
  unsigned long long c_top = 0, c_spl = 0;
#define APROF(var) { const long long _t = clock64(); var += _t - c_t; c_t = _t; }
#define ACOUNT(var) ++var;
#else
#define APROF(var)
#define ACOUNT(var)
#endif
  while (true) {
    int M = 0, ab = 0;
#ifdef FABM_PROFILE
    const long long t_top = clock64();
#endif
    if (lane == 0) {
      M = sys ? ld_acquire_sys(&sv.ctrl->src_done) : ld_acquire_gpu(&sv.ctrl->src_done);
      ab = ld_rlx(&sv.ctrl->abort, sys);
    }
    M = __shfl_sync(0xffffffffu, M, 0);
    ab = __shfl_sync(0xffffffffu, ab, 0);
#ifdef FABM_PROFILE
    c_top += clock64() - t_top;
#endif
    if (ab) return;
    if (M != last_M) {
      last_M = M;
      last_progress = global_ns();
    }
    __syncwarp();
    // earliest owned target with a published chunk in its current unit
    int best = -1;
    for (int b0 = 0; b0 < nown; b0 += 32) {
      const int i = b0 + lane;
      bool pend = false;
      if (i < nown) {
        const int n = owned_target(agent, i, nA) - kL + 1;
        const int k = seg_class(n);
        const int nx = A.own_next[i] >> 1;
        const int uhi = min(((nx >> k) + 1) << k, n);
        pend = nx < min(uhi, M);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, pend);
      if (bal) { best = b0 + __ffs(bal) - 1; break; }
    }
    const int Jo = best >= 0 ? owned_target(agent, best, nA) : 0x7fffffff;
    // a claimed-unit burst yields once this owned target nears its deadline
    const int j_soon = Jo;
    // earliest claimable unit; the cursors only grow, so a bound read at
    // the same M stays a lower bound
    int Jd = 0x7fffffff, kd = 0, cd = -1;
    if (dJ >= 0) {
      Jd = dJ;
    } else if (Jo > dyn_lb || (M >> kc) != (lb_M >> kc) || lb_M < 0) {
      // a column of a class >= kc completes only when M crosses a multiple
      // of its segment length 2^k, k >= kc
#ifdef FABM_PROFILE
      const long long t_sc = clock64();
#endif
      Jd = scan_claimable(P, M, lane, sys, kc, kd, cd);
#ifdef FABM_PROFILE
      c_scan += clock64() - t_sc;
      ++n_scan;
#endif
      dyn_lb = Jd;
      lb_M = M;
    }
    const bool take_dyn = Jd < Jo;
    ACOUNT(n_sel)
    if (!take_dyn && best < 0) {
      // nothing to do: finished, or wait for the next source block
      bool fin = dJ < 0 && kc > P.k_max;
      for (int b0 = 0; b0 < nown && fin; b0 += 32) {
        const int i = b0 + lane;
        const bool od = i >= nown || (A.own_next[i] >> 1) >= owned_target(agent, i, nA) - kL + 1;
        fin = __all_sync(0xffffffffu, od);
      }
      if (fin) break;
      __nanosleep(256);
      ACOUNT(n_idle)
      if ((++idle_polls & 63) == 0) lb_M = -1;  // re-scan now and then (exit detection)
      APROF(c_idle)
      if (global_ns() - last_progress > P.timeout_ns) {
        if (lane == 0) raise_abort(P, ERR_TIMEOUT, KIND_NONE, -1, 0.0);
        return;
      }
      continue;
    }
    int J, s, nx, hi, lim;
    if (take_dyn) {
      if (dJ < 0) {
        // claim the first unclaimed unit of column (kd, cd) at or after Jd:
        // 32 candidates read at once, CAS on the first free one
        const int S = 1 << kd;
        const int ns = max(class_lo(kd), (cd + 1) * S + 1);
        const int nend = min(class_hi(kd), nb - kL + 1);
        const int j = Jd + lane;
        bool freeu = false;
        if (j - kL + 1 < nend) freeu = ld_rlx(&P.claim[unit_base(P, j) + cd], sys) == 0;
        const unsigned fb = __ballot_sync(0xffffffffu, freeu);
        int got = -1;
        if (lane == 0) {
          int* cursor = &P.col_next[kd * 32 + cd];
          if (fb) {
            const int jj = Jd + __ffs(fb) - 1;
            if (at_cas(&P.claim[unit_base(P, jj) + cd], 0, agent + 1, sys) == 0) got = jj;
            at_max(cursor, (jj - kL + 1) - ns + (got >= 0 ? 1 : 0), sys);
          } else {
            at_max(cursor, min(Jd - kL + 1 + 32, nend) - ns, sys);
          }
        }
        got = __shfl_sync(0xffffffffu, got, 0);
        lb_M = -1;  // re-scan next time
        if (got < 0) continue;
        dJ = got;
        ds = cd;
        dnext = cd * S;
        ++claims;
      }
      J = dJ;
      s = ds;
      nx = dnext;
      hi = min((s + 1) << seg_class(J - kL + 1), J - kL + 1);
      lim = hi;  // a complete column: every chunk is published
    } else {
      J = owned_target(agent, best, nA);
      const int n = J - kL + 1;
      const int k = seg_class(n);
      const int v = A.own_next[best];
      nx = v >> 1;
      s = nx >> k;
      hi = min((s + 1) << k, n);
      lim = min(hi, M);
      if (!(v & 1)) {  // first touch of this unit: claim it (a claimer may hold it)
        int ok = 0;
        if (lane == 0) ok = at_cas(&P.claim[unit_base(P, J) + s], 0, agent + 1, sys) == 0;
        ok = __shfl_sync(0xffffffffu, ok, 0);
        __syncwarp();
        if (lane == 0) A.own_next[best] = ok ? ((nx << 1) | 1) : (hi << 1);
        __syncwarp();
        if (!ok) continue;
      }
    }
    const long long uid = unit_base(P, J) + s;
    FABM_CHECK(P, J >= kL && J < nb && s >= 0 && s * (1 << seg_class(J - kL + 1)) <= nx && nx <= hi &&
                      hi <= J - kL + 1 && uid >= 0 && uid < P.n_units);
    FABM_CHECK(P, lane != 0 || ld_rlx(&P.claim[uid], sys) == agent + 1);  // only the unit's claimant computes it
    // the chunk's weight window [128(J-nx)-127, 128(J-nx)+128] and f rows < 128(J-L+1) are allocated
    FABM_CHECK(P, 128LL * (J - nx) - 127 >= 0 && 128LL * (J - nx) + 128 < P.wlen &&
                      128LL * (J - kL + 1) <= P.f_rows);
#ifdef FABM_PROFILE
    const long long t_spl = clock64();
#endif
    if (uid != cur_uid) {
      if (cur_uid >= 0) {
        dmma_spill_slot<D>(unit_slot<D>(P, cur_uid), lane, acc);
        ACOUNT(n_spill)
      }
      if (nx > (s << seg_class(J - kL + 1))) {
        __syncwarp();
        dmma_reload_slot<D>(unit_slot<D>(P, uid), lane, acc);
        ACOUNT(n_reload)
      } else {
        dmma_zero<D>(acc);
      }
      cur_uid = uid;
    }
#ifdef FABM_PROFILE
    c_spl += clock64() - t_spl;
#endif
    APROF(c_sw)
    // owned units: re-run the selection when a newer source block arrives;
    // claimed units: in bursts of kDynBurst chunks (fewer spill/reload
    // switches between a claimed unit and the owned frontier)
    const int burst_end = take_dyn ? min(lim, nx + kDynBurst) : lim;
    while (nx < burst_end) {
      int M2 = 0;
      if (lane == 0) M2 = ld_rlx(&sv.ctrl->src_done, sys);
      dmma_chunk<D>(P.wb, P.wa, sv.F, A.t, J * kB, nx * kB, (J - kL + 1) * kB, lane, acc);
      ++nx;
      ++tiles;
      M2 = __shfl_sync(0xffffffffu, M2, 0);
      // a newer source block: re-run the selection (owned units at once --
      // EDF may switch to an earlier target; claimed units only when an
      // owned target nears its deadline)
      if (M2 != M && (!take_dyn || j_soon - M2 <= kUrgent)) break;
    }
    APROF(c_tile)
    __syncwarp();
    if (take_dyn) {
      dnext = nx;
    } else if (lane == 0) {
      A.own_next[best] = nx == hi ? (nx << 1) : ((nx << 1) | 1);
    }
    __syncwarp();
    if (nx == hi) {
#ifdef FABM_PROFILE
      const long long t_f = clock64();
#endif
      unit_finish<D>(P, J, s, uid, lane, acc, sys);
#ifdef FABM_PROFILE
      c_fin += clock64() - t_f;
      ++n_fin;
#endif
      cur_uid = -1;
      if (take_dyn) dJ = -1;
    }
  }
  if (lane == 0) {
    atomicAdd(&sv.ctrl->bulk_tiles, tiles);
    atomicAdd(&sv.ctrl->bulk_claims, claims);
  }
#ifdef FABM_PROFILE
  if (lane == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&P.ctrl->prof[4]), (unsigned long long)c_tile);
    atomicAdd(reinterpret_cast<unsigned long long*>(&P.ctrl->prof[5]), (unsigned long long)c_idle);
    atomicAdd(reinterpret_cast<unsigned long long*>(&P.ctrl->prof[6]), (unsigned long long)c_sw);
    const unsigned long long ev[8] = {n_sel, n_scan, n_spill, c_top, n_fin, c_fin, c_scan, c_spl};
    for (int q = 0; q < 8; ++q) atomicAdd(&P.ctrl->prof2[q], ev[q]);
  }
#endif
}

// ======================================================================
template <int SYS, int D>
__global__ void __launch_bounds__(kThreads, 1) abm_engine_kernel(EngineParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  // the stepper is CTA 0 of the launch that hosts it (shard 0); the launches
  // of the other shards are agents only
  if (P.has_stepper && blockIdx.x == 0) {
    stepper_cta<SYS, D>(P, *reinterpret_cast<StepperSmem*>(smem_raw));
  } else {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    BulkSmem<D>* A = reinterpret_cast<BulkSmem<D>*>(smem_raw) + warp;
    const int lcta = blockIdx.x - (P.has_stepper ? 1 : 0);
    const int sh = P.my_shard >= 0 ? P.my_shard : lcta % P.n_shards;
    // agents are dealt warp-major across CTAs (of all shards) so every SM
    // hosts a mix of light and heavy owners
    const ShardView sv = P.shard[sh];
    bulk_agent<D>(P, *A, warp * P.n_agent_ctas + P.agent_cta_base + lcta, lane, sv);
  }
}

template <int D>
constexpr size_t engine_smem_bytes() {
  return sizeof(StepperSmem) > kWarps * sizeof(BulkSmem<D>) ? sizeof(StepperSmem) : kWarps * sizeof(BulkSmem<D>);
}

}  // namespace fabm
