// fabm_api.cu — the C ABI declared in include/fabm.h (libfabm.so).
//
// Host-side runtime: device buffers per plan (one stream, CUDA events for
// timing), weight generation, cooperative launch of the history engine,
// status translation.  No torch types cross this boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cerrno>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fabm.h"
#include "batch.cuh"
#include "csv_format.cuh"
#include "oracles.cuh"
#include "steps.cuh"
#include "engine.cuh"
#include "weights.cuh"

using namespace fabm;

namespace {

constexpr const char* kVersion = "fabm-b200 0.1.0 (sm_100a)";

void set_status(fabm_status* st, int code, const char* fmt, ...) {
  if (!st) return;
  st->code = code;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(st->message, sizeof(st->message), fmt, ap);
  va_end(ap);
}

void clear_status(fabm_status* st) {
  if (!st) return;
  std::memset(st, 0, sizeof(*st));
}

#define CUDA_TRY(expr)                                                              \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      set_status(status, FABM_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e));   \
      return FABM_ERR_CUDA;                                                         \
    }                                                                               \
  } while (0)

bool system_dim_ok(int sys, int dim) {
  switch (sys) {
    case FABM_SYS_CONSTANT:
    case FABM_SYS_LINEAR: return dim >= 1 && dim <= FABM_MAX_DIM;
    case FABM_SYS_POWER_LAW: return dim == 1;
    case FABM_SYS_HINDMARSH_ROSE:
    case FABM_SYS_LORENZ:
    case FABM_SYS_CHEN:
    case FABM_SYS_ROSSLER:
    case FABM_SYS_FINANCIAL: return dim == 3;
    default: return false;
  }
}

int validate(const fabm_problem* p, const fabm_grid* g, fabm_status* status) {
  if (!p || !g) { set_status(status, FABM_ERR_CONFIG, "null problem or grid"); return FABM_ERR_CONFIG; }
  if (!std::isfinite(p->alpha) || !(p->alpha > 0.0 && p->alpha <= 1.0)) {
    set_status(status, FABM_ERR_CONFIG, "alpha must lie in (0, 1], got %.17g", p->alpha);
    return FABM_ERR_CONFIG;
  }
  if (!system_dim_ok(p->system, p->dim)) {
    set_status(status, FABM_ERR_CONFIG, "system %d does not support dim %d (device engine: dim <= %d)",
               p->system, p->dim, FABM_MAX_DIM);
    return FABM_ERR_CONFIG;
  }
  for (int i = 0; i < p->dim; ++i)
    if (!std::isfinite(p->y0[i])) { set_status(status, FABM_ERR_CONFIG, "y0 must be finite"); return FABM_ERR_CONFIG; }
  if (g->n_steps < 1) { set_status(status, FABM_ERR_CONFIG, "n_steps must be >= 1"); return FABM_ERR_CONFIG; }
  if (!std::isfinite(g->h) || !(g->h > 0.0)) {
    set_status(status, FABM_ERR_CONFIG, "step size must be finite and positive, got %.17g", g->h);
    return FABM_ERR_CONFIG;
  }
  return FABM_OK;
}

// per-solve scalars, filled from libm when the caller left them zero
void fill_scalars(const fabm_problem* p, fabm_grid* g) {
  if (g->h_alpha == 0.0) g->h_alpha = std::pow(g->h, p->alpha);
  if (g->gamma1 == 0.0) g->gamma1 = std::tgamma(p->alpha + 1.0);
  if (g->gamma2 == 0.0) g->gamma2 = std::tgamma(p->alpha + 2.0);
  if (g->inv_gamma2 == 0.0) g->inv_gamma2 = 1.0 / g->gamma2;
}

// (system, dim) -> the LAUNCHER<SYS, D> instantiation compiled for it (every
// device rhs: constant/linear for d <= 4, the named systems at their dims)
#define FABM_PICK_SYSTEM(LAUNCHER)                                   \
  switch (sys) {                                                     \
    case FABM_SYS_CONSTANT:                                          \
      switch (dim) {                                                 \
        case 1: return LAUNCHER<SYS_CONSTANT, 1>;                    \
        case 2: return LAUNCHER<SYS_CONSTANT, 2>;                    \
        case 3: return LAUNCHER<SYS_CONSTANT, 3>;                    \
        case 4: return LAUNCHER<SYS_CONSTANT, 4>;                    \
      }                                                              \
      break;                                                         \
    case FABM_SYS_LINEAR:                                            \
      switch (dim) {                                                 \
        case 1: return LAUNCHER<SYS_LINEAR, 1>;                      \
        case 2: return LAUNCHER<SYS_LINEAR, 2>;                      \
        case 3: return LAUNCHER<SYS_LINEAR, 3>;                      \
        case 4: return LAUNCHER<SYS_LINEAR, 4>;                      \
      }                                                              \
      break;                                                         \
    case FABM_SYS_POWER_LAW: return LAUNCHER<SYS_POWER_LAW, 1>;      \
    case FABM_SYS_HINDMARSH_ROSE: return LAUNCHER<SYS_HINDMARSH_ROSE, 3>; \
    case FABM_SYS_LORENZ: return LAUNCHER<SYS_LORENZ, 3>;            \
    case FABM_SYS_CHEN: return LAUNCHER<SYS_CHEN, 3>;                \
    case FABM_SYS_ROSSLER: return LAUNCHER<SYS_ROSSLER, 3>;          \
    case FABM_SYS_FINANCIAL: return LAUNCHER<SYS_FINANCIAL, 3>;      \
  }                                                                  \
  return nullptr

using EngineLaunch = cudaError_t (*)(const EngineParams&, int grid, cudaStream_t);

template <int SYS, int D>
cudaError_t launch_engine(const EngineParams& P, int grid, cudaStream_t stream) {
  auto kern = abm_engine_kernel<SYS, D>;
  const size_t smem = engine_smem_bytes<D>();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  EngineParams Pc = P;
  void* args[] = {&Pc};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), dim3(grid), dim3(kThreads), args, smem, stream);
}

template <int SYS, int D>
cudaError_t engine_occupancy(int* blocks_per_sm) {
  auto kern = abm_engine_kernel<SYS, D>;
  const size_t smem = engine_smem_bytes<D>();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, kern, kThreads, smem);
}

EngineLaunch pick_engine(int sys, int dim) {
  FABM_PICK_SYSTEM(launch_engine);
}

int stride_of(int dim) { return dim == 1 ? 1 : (dim == 2 ? 2 : 4); }

// bulk-unit geometry, host side of engine.cuh's seg_class / unit_base
int host_seg_class(int n) {
  int lg = 0;
  while ((2 << lg) <= n) ++lg;  // floor(log2 n)
  return seg_class_of_log(lg);
}
long long host_unit_base(int J) {
  const int n = J - kL + 1;
  const int k = host_seg_class(n);
  return class_base(k) + seg_prefix(n - 1, k) - seg_prefix(class_lo(k) - 1, k);
}

}  // namespace

static unsigned long long g_last_prof[16];
extern "C" void fabm_debug_prof(unsigned long long* out) {
  for (int i = 0; i < 8; ++i) out[i] = g_last_prof[i];
}
extern "C" void fabm_debug_prof2(unsigned long long* out) {
  for (int i = 0; i < 8; ++i) out[i] = g_last_prof[8 + i];
}
#ifdef FABM_PROFILE
static unsigned long long* g_trace = nullptr;
static int g_trace_n = 0;
extern "C" int fabm_debug_trace(unsigned long long* out, int n) {
  if (!g_trace) return 0;
  const int m = n < g_trace_n ? n : g_trace_n;
  cudaMemcpy(out, g_trace, sizeof(unsigned long long) * m, cudaMemcpyDeviceToHost);
  return m;
}
#endif

struct fabm_plan {
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  fabm_problem prob{};
  fabm_grid grid{};
  long long N = 0;
  int nb = 0;
  int ds = 1;
  long long wlen = 0;
  double* wb = nullptr;
  double* wa = nullptr;
  double* wc = nullptr;
  double* y0 = nullptr;
  double* Y = nullptr;
  double* Fc = nullptr;
  double* Yh = nullptr;    // device aliases of the caller's mapped pinned output (fabm_plan_set_host_output)
  double* Fch = nullptr;
  // the shard arena: {ctrl, ready, F, BK} in one allocation so that one CUDA
  // IPC handle exposes it to the peer GPUs of a sharded run (config 5)
  char* arena = nullptr;
  size_t arena_bytes = 0;
  size_t shard_bytes = 0;      // the per-shard prefix {ctrl, ready, F, BK}; the rest is rank 0's unit state
  size_t off_ready = 0, off_F = 0, off_BK = 0;
  size_t off_claim = 0, off_tdone = 0, off_tstage = 0, off_col = 0, off_PK = 0;
  int k_max = 0;               // highest segment class (engine.cuh: units)
  long long n_units = 0;
  int bulk_default = 0;        // bulk CTAs chosen at creation (fabm_plan_set_bulk_ctas overrides)
  double* F = nullptr;
  double* BK = nullptr;
  int* ready = nullptr;
  DevCtrl* ctrl = nullptr;
  // sharding: n_shards = 1 (default), real (one process per GPU, peers opened
  // from IPC handles) or virtual (one-GPU emulation with local arenas)
  int n_shards = 1;
  int rank = 0;
  bool virt = false;
  bool emulate = false;        // attached peers, but one launch here serves every shard (fabm_plan_emulate_shards)
  bool armed = false;          // real sharded runs: flags reset and not yet run
  int agent_ctas_per_shard = 0;
  std::vector<char*> peer;     // arena base of every shard (peer[rank] = arena)
  std::vector<char*> opened;   // IPC mappings to close
  std::vector<char*> virt_arenas;
  ShardView* shard_tab = nullptr;  // device copy of the per-shard views
  bool weights_ready = false;
  int weights_mode = FABM_WEIGHTS_ACCURATE;
  int bulk_ctas = 0;
  EngineLaunch launch = nullptr;
  fabm_stats stats{};
};

static void plan_free(fabm_plan* p) {
  if (!p) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  for (char* m : p->opened) cudaIpcCloseMemHandle(m);
  for (char* m : p->virt_arenas) cudaFree(m);
  for (void* ptr : {(void*)p->wb, (void*)p->wa, (void*)p->wc, (void*)p->y0, (void*)p->Y, (void*)p->Fc,
                    (void*)p->arena, (void*)p->shard_tab})
    if (ptr) cudaFree(ptr);
  for (auto& e : p->ev)
    if (e) cudaEventDestroy(e);
  if (p->stream) cudaStreamDestroy(p->stream);
  cudaSetDevice(prev);
  delete p;
}

extern "C" {

const char* fabm_version(void) { return kVersion; }

int fabm_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

fabm_plan* fabm_plan_create(const fabm_problem* problem, const fabm_grid* grid_in, int device, fabm_status* status) {
  clear_status(status);
  if (validate(problem, grid_in, status) != FABM_OK) return nullptr;
  int ndev = fabm_device_count();
  if (ndev <= 0 || device < 0 || device >= ndev) {
    set_status(status, FABM_ERR_NODEVICE, "no CUDA device %d (found %d)", device, ndev);
    return nullptr;
  }
  auto* p = new fabm_plan();
  p->device = device;
  p->prob = *problem;
  p->grid = *grid_in;
  fill_scalars(problem, &p->grid);
  p->N = grid_in->n_steps;
  p->nb = static_cast<int>((p->N + kB - 1) / kB);
  p->ds = stride_of(problem->dim);
  p->wlen = static_cast<long long>(p->nb) * kB + 2 * kB;
  p->launch = pick_engine(problem->system, problem->dim);
  auto fail = [&](const char* what, cudaError_t e) -> fabm_plan* {
    set_status(status, FABM_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    plan_free(p);
    return nullptr;
  };
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail("cudaSetDevice", e);
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  if (prop.major < 10) {
    set_status(status, FABM_ERR_NODEVICE, "device %d is sm_%d%d; libfabm is built for sm_100a", device, prop.major,
               prop.minor);
    plan_free(p);
    return nullptr;
  }
  p->num_sms = prop.multiProcessorCount;
  // bulk agents: 16 per CTA, one CTA per SM besides the stepper
  const int n_targets = p->nb - kL;
  if (n_targets > 0) {
    int ctas = (n_targets + kWarps - 1) / kWarps;
    ctas = std::min(ctas, p->num_sms - 1);
    p->bulk_ctas = std::max(ctas, 1);
    p->bulk_default = p->bulk_ctas;
    const int n_agents = p->bulk_ctas * kWarps;
    if ((n_targets + n_agents - 1) / n_agents > kMaxOwn) {
      set_status(status, FABM_ERR_CONFIG, "n_steps=%lld exceeds the engine capacity", p->N);
      plan_free(p);
      return nullptr;
    }
  }
  if ((e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking)) != cudaSuccess) return fail("stream", e);
  for (auto& ev : p->ev)
    if ((e = cudaEventCreate(&ev)) != cudaSuccess) return fail("event", e);
  const size_t wbytes = sizeof(double) * p->wlen;
  const size_t fl = static_cast<size_t>(p->nb + 1) * kB * p->ds;
  if ((e = cudaMalloc(&p->wb, wbytes)) != cudaSuccess) return fail("malloc b", e);
  if ((e = cudaMalloc(&p->wa, wbytes)) != cudaSuccess) return fail("malloc a", e);
  if ((e = cudaMalloc(&p->wc, wbytes)) != cudaSuccess) return fail("malloc c", e);
  if ((e = cudaMalloc(&p->y0, sizeof(double) * FABM_MAX_DIM)) != cudaSuccess) return fail("malloc y0", e);
  if ((e = cudaMalloc(&p->Y, sizeof(double) * (p->N + 1) * problem->dim)) != cudaSuccess) return fail("malloc Y", e);
  if ((e = cudaMalloc(&p->Fc, sizeof(double) * (p->N + 1) * problem->dim)) != cudaSuccess) return fail("malloc Fc", e);
  {
    auto up = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
    p->off_ready = up(sizeof(DevCtrl));
    p->off_F = p->off_ready + up(sizeof(int) * (p->nb + 1));
    p->off_BK = p->off_F + up(sizeof(double) * fl);
    p->shard_bytes = p->off_BK + up(sizeof(double) * static_cast<size_t>(p->nb) * kB * 2 * p->ds);
    // bulk units (engine.cuh): segment classes, unit counts
    const int nt = std::max(p->nb - kL, 0);
    p->k_max = nt > 0 ? host_seg_class(nt) : 0;
    p->n_units = nt > 0 ? host_unit_base(p->nb) : 0;
    p->off_claim = p->shard_bytes;
    p->off_tdone = p->off_claim + up(sizeof(int) * static_cast<size_t>(p->n_units + 1));
    p->off_tstage = p->off_tdone + up(sizeof(int) * (p->nb + 1));
    p->off_col = p->off_tstage + up(sizeof(int) * (p->nb + 1));
    p->off_PK = p->off_col + up(sizeof(int) * kMaxClasses * 32);
    p->arena_bytes = p->off_PK + up(sizeof(double) * static_cast<size_t>(p->n_units) * 32 * 8 * problem->dim);
  }
  if ((e = cudaMalloc(&p->arena, p->arena_bytes)) != cudaSuccess) return fail("malloc arena", e);
  if ((e = cudaMalloc(&p->shard_tab, sizeof(ShardView) * kMaxShards)) != cudaSuccess) return fail("malloc shards", e);
  p->ctrl = reinterpret_cast<DevCtrl*>(p->arena);
  p->ready = reinterpret_cast<int*>(p->arena + p->off_ready);
  p->F = reinterpret_cast<double*>(p->arena + p->off_F);
  p->BK = reinterpret_cast<double*>(p->arena + p->off_BK);
  p->peer.assign(1, p->arena);
  p->agent_ctas_per_shard = p->bulk_ctas;
  cudaMemsetAsync(p->arena, 0, p->arena_bytes, p->stream);
  cudaMemsetAsync(p->wb, 0, wbytes, p->stream);
  cudaMemsetAsync(p->wa, 0, wbytes, p->stream);
  cudaMemsetAsync(p->wc, 0, wbytes, p->stream);
  cudaMemcpyAsync(p->y0, problem->y0, sizeof(double) * problem->dim, cudaMemcpyHostToDevice, p->stream);
  if ((e = cudaStreamSynchronize(p->stream)) != cudaSuccess) return fail("init", e);
  p->stats.block = kB;
  p->stats.window_blocks = kL;
  p->stats.bulk_ctas = p->bulk_ctas;
  return p;
}

int fabm_plan_set_weights(fabm_plan* p, int mode, const double* b, const double* a, const double* c,
                          fabm_status* status) {
  clear_status(status);
  if (!p) { set_status(status, FABM_ERR_CONFIG, "null plan"); return FABM_ERR_CONFIG; }
  CUDA_TRY(cudaSetDevice(p->device));
  const long long n1 = p->N + 1;
  if (mode == FABM_WEIGHTS_HOST) {
    if (!b || !a || !c) { set_status(status, FABM_ERR_CONFIG, "host weights need b, a and c"); return FABM_ERR_CONFIG; }
    // indices > N are never combined with a live history term; keep them 0
    CUDA_TRY(cudaMemsetAsync(p->wb, 0, sizeof(double) * p->wlen, p->stream));
    CUDA_TRY(cudaMemsetAsync(p->wa, 0, sizeof(double) * p->wlen, p->stream));
    CUDA_TRY(cudaMemsetAsync(p->wc, 0, sizeof(double) * p->wlen, p->stream));
    CUDA_TRY(cudaMemcpyAsync(p->wb, b, sizeof(double) * n1, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(p->wa, a, sizeof(double) * n1, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(p->wc, c, sizeof(double) * n1, cudaMemcpyHostToDevice, p->stream));
    p->stats.weights_ms = 0.0;
  } else if (mode == FABM_WEIGHTS_ACCURATE || mode == FABM_WEIGHTS_FORMULA) {
    CUDA_TRY(cudaEventRecord(p->ev[2], p->stream));
    const int threads = 256;
    const int blocks = static_cast<int>(std::min<long long>((p->wlen + threads - 1) / threads, 148LL * 16));
    weights_kernel<<<blocks, threads, 0, p->stream>>>(p->prob.alpha, p->grid.gamma1, p->grid.gamma2, p->wlen,
                                                      mode == FABM_WEIGHTS_FORMULA ? 1 : 0, p->wb, p->wa, p->wc);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(p->ev[3], p->stream));
    CUDA_TRY(cudaEventSynchronize(p->ev[3]));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p->ev[2], p->ev[3]);
    p->stats.weights_ms = ms;
  } else {
    set_status(status, FABM_ERR_CONFIG, "unknown weight mode %d", mode);
    return FABM_ERR_CONFIG;
  }
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  p->weights_ready = true;
  p->weights_mode = mode;
  return FABM_OK;
}

int fabm_plan_set_y0(fabm_plan* p, const double* y0, fabm_status* status) {
  clear_status(status);
  if (!p) { set_status(status, FABM_ERR_CONFIG, "null plan"); return FABM_ERR_CONFIG; }
  if (!y0) return FABM_OK;
  for (int i = 0; i < p->prob.dim; ++i) {
    if (!std::isfinite(y0[i])) { set_status(status, FABM_ERR_CONFIG, "y0 must be finite"); return FABM_ERR_CONFIG; }
    p->prob.y0[i] = y0[i];
  }
  CUDA_TRY(cudaSetDevice(p->device));
  CUDA_TRY(cudaMemcpyAsync(p->y0, p->prob.y0, sizeof(double) * p->prob.dim, cudaMemcpyHostToDevice, p->stream));
  return FABM_OK;
}

int fabm_plan_run(fabm_plan* p, double timeout_s, fabm_status* status) {
  clear_status(status);
  if (!p) { set_status(status, FABM_ERR_CONFIG, "null plan"); return FABM_ERR_CONFIG; }
  if (!p->launch) { set_status(status, FABM_ERR_CONFIG, "no engine for system/dim"); return FABM_ERR_CONFIG; }
  CUDA_TRY(cudaSetDevice(p->device));
  if (!p->weights_ready) {
    int rc = fabm_plan_set_weights(p, FABM_WEIGHTS_ACCURATE, nullptr, nullptr, nullptr, status);
    if (rc != FABM_OK) return rc;
  }
  const bool real_shards = p->n_shards > 1 && !p->virt && !p->emulate;
  if (real_shards) {
    if (!p->armed) {
      set_status(status, FABM_ERR_CONFIG, "sharded plan: call fabm_plan_reset on every rank, then barrier, then run");
      return FABM_ERR_CONFIG;
    }
    p->armed = false;
  } else {
    int rc = fabm_plan_reset(p, status);
    if (rc != FABM_OK) return rc;
  }
  EngineParams P{};
  P.N = p->N;
  P.h = p->grid.h;
  P.ha = p->grid.h_alpha;
  P.ig = p->grid.inv_gamma2;
  P.wb = p->wb;
  P.wa = p->wa;
  P.wc = p->wc;
  P.y0 = p->y0;
  P.Y = p->Y;
  P.F = p->F;
  P.Fc = p->Fc;
  P.Yh = p->Yh;
  P.Fch = p->Fch;
  P.BK = p->BK;
  P.ready = p->ready;
  P.ctrl = p->ctrl;
  std::memcpy(P.params, p->prob.params, sizeof(P.params));
  P.nb = p->nb;
  P.n_shards = p->n_shards;
  {
    ShardView tab[kMaxShards] = {};
    for (int sh = 0; sh < p->n_shards; ++sh) {
      char* base = p->peer[sh];
      tab[sh].ctrl = reinterpret_cast<DevCtrl*>(base);
      tab[sh].F = reinterpret_cast<double*>(base + p->off_F);
    }
    CUDA_TRY(cudaMemcpyAsync(p->shard_tab, tab, sizeof(tab), cudaMemcpyHostToDevice, p->stream));
    P.shard = p->shard_tab;
  }
  int grid = 1 + p->bulk_ctas;
  P.has_stepper = 1;
  {
    // the bulk units' shared state lives in shard 0's arena (peer memory on
    // the other GPUs of a sharded run)
    char* base0 = p->peer[0];
    P.k_max = p->k_max;
    P.n_units = p->n_units;
    P.wlen = p->wlen;
    P.f_rows = static_cast<long long>(p->nb + 1) * kB;
    P.claim = reinterpret_cast<int*>(base0 + p->off_claim);
    P.tdone = reinterpret_cast<int*>(base0 + p->off_tdone);
    P.tstage = reinterpret_cast<int*>(base0 + p->off_tstage);
    P.col_next = reinterpret_cast<int*>(base0 + p->off_col);
    P.PK = reinterpret_cast<double*>(base0 + p->off_PK);
  }
  if (real_shards) {
    // completed targets land in shard 0's accumulators; the stepper lives there
    P.BK = reinterpret_cast<double*>(p->peer[0] + p->off_BK);
    P.ready = reinterpret_cast<int*>(p->peer[0] + p->off_ready);
    P.my_shard = p->rank;
    P.agent_cta_base = p->rank * p->agent_ctas_per_shard;
    P.n_agent_ctas = p->n_shards * p->agent_ctas_per_shard;
    P.has_stepper = p->rank == 0;
    grid = (p->rank == 0 ? 1 : 0) + p->agent_ctas_per_shard;
  } else {
    P.my_shard = (p->virt || p->emulate) ? -1 : 0;
    P.agent_cta_base = 0;
    P.n_agent_ctas = p->bulk_ctas;
  }
  P.n_agents = P.n_agent_ctas * kWarps;
#ifdef FABM_PROFILE
  if (g_trace_n < 4 * (p->nb + 1)) {
    if (g_trace) cudaFree(g_trace);
    g_trace_n = 4 * (p->nb + 1);
    cudaMalloc(&g_trace, sizeof(unsigned long long) * g_trace_n);
  }
  cudaMemsetAsync(g_trace, 0, sizeof(unsigned long long) * g_trace_n, p->stream);
  P.trace = g_trace;
#endif
  const double tmo = timeout_s > 0 ? timeout_s : 60.0;
  P.timeout_ns = static_cast<unsigned long long>(tmo * 1e9);
  // dev switches (tools/solo_probe.py, the watchdog test): bits 1, 2 and 8
  // invalidate the trajectory, so a run that completes with one of them set
  // reports FABM_ERR_CONFIG instead of FABM_OK
  if (const char* dbg = getenv("FABM_DEBUG_MODE")) P.debug = atoi(dbg);
  CUDA_TRY(cudaEventRecord(p->ev[0], p->stream));
  CUDA_TRY(p->launch(P, grid, p->stream));
  CUDA_TRY(cudaEventRecord(p->ev[1], p->stream));
  CUDA_TRY(cudaEventSynchronize(p->ev[1]));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, p->ev[0], p->ev[1]);
  DevCtrl h{};
  CUDA_TRY(cudaMemcpy(&h, p->ctrl, sizeof(DevCtrl), cudaMemcpyDeviceToHost));
  if (p->virt || p->emulate) {  // emulated shards: their agents count tiles / raise errors in their own blocks
    for (int sh = 1; sh < p->n_shards; ++sh) {
      DevCtrl v{};
      CUDA_TRY(cudaMemcpy(&v, p->peer[sh], sizeof(DevCtrl), cudaMemcpyDeviceToHost));
      h.bulk_tiles += v.bulk_tiles;
      h.bulk_claims += v.bulk_claims;
      if (h.err_code == ERR_OK && v.err_code != ERR_OK) {
        h.err_code = v.err_code;
        h.err_kind = v.err_kind;
        h.err_step = v.err_step;
        h.err_t = v.err_t;
      }
    }
  }
  if (h.check_line) {  // FABM_CHECKED build: an invariant failed (engine.cuh line)
    set_status(status, FABM_ERR_CONFIG, "FABM_CHECKED: engine invariant violated at engine.cuh:%d", h.check_line);
    return FABM_ERR_CONFIG;
  }
  if (h.err_code == ERR_OK && h.abort) {  // stopped by a peer shard (its watchdog or its error)
    h.err_code = ERR_TIMEOUT;
    h.err_step = -3;
  }
  p->stats.kernel_ms = ms;
  p->stats.steps = p->N;
  p->stats.history_fma = static_cast<int64_t>(p->prob.dim) * p->N * p->N;
  p->stats.bulk_tiles = static_cast<int64_t>(h.bulk_tiles);
  p->stats.bulk_claims = static_cast<int64_t>(h.bulk_claims);
  p->stats.segment = 1 << p->k_max;
  p->stats.leader_wait_ns = static_cast<int64_t>(h.leader_wait_ns);
  p->stats.leader_throttle_ns = static_cast<int64_t>(h.leader_throttle_ns);
  for (int i = 0; i < 8; ++i) g_last_prof[i] = h.prof[i];
  for (int i = 0; i < 8; ++i) g_last_prof[8 + i] = h.prof2[i];
  if (h.err_code != ERR_OK) {
    if (status) {
      status->code = h.err_code == ERR_TIMEOUT ? FABM_ERR_TIMEOUT : FABM_ERR_NONFINITE;
      status->kind = h.err_kind;
      status->step = h.err_step;
      status->t = h.err_t;
      if (h.err_code == ERR_TIMEOUT && h.err_step == -3)
        snprintf(status->message, sizeof(status->message), "aborted by a peer shard");
      else if (h.err_code == ERR_TIMEOUT)
        snprintf(status->message, sizeof(status->message), "device watchdog expired (no progress for %.1f s)", tmo);
      else
        snprintf(status->message, sizeof(status->message), "rhs returned a non-finite value");
    }
    return h.err_code == ERR_TIMEOUT ? FABM_ERR_TIMEOUT : FABM_ERR_NONFINITE;
  }
  if (P.debug & (1 | 2 | 8)) {
    set_status(status, FABM_ERR_CONFIG, "FABM_DEBUG_MODE=%d: dev switches invalidate the trajectory", P.debug);
    return FABM_ERR_CONFIG;
  }
  return FABM_OK;
}

int fabm_plan_set_bulk_ctas(fabm_plan* p, int n_ctas, fabm_status* status) {
  clear_status(status);
  if (!p) { set_status(status, FABM_ERR_CONFIG, "null plan"); return FABM_ERR_CONFIG; }
  if (p->n_shards > 1) {
    set_status(status, FABM_ERR_CONFIG, "set the bulk CTA count before sharding the plan");
    return FABM_ERR_CONFIG;
  }
  const int n_targets = p->nb - kL;
  int want = n_ctas <= 0 ? p->bulk_default : n_ctas;
  if (want > p->num_sms - 1 || want < 1) {
    set_status(status, FABM_ERR_CONFIG, "bulk CTAs must lie in [1, %d], got %d", p->num_sms - 1, n_ctas);
    return FABM_ERR_CONFIG;
  }
  if (n_targets > 0 && (n_targets + want * kWarps - 1) / (want * kWarps) > kMaxOwn) {
    set_status(status, FABM_ERR_CONFIG, "%d bulk CTAs cannot own %d target blocks (at most %d per agent)", want,
               n_targets, kMaxOwn);
    return FABM_ERR_CONFIG;
  }
  p->bulk_ctas = want;
  p->agent_ctas_per_shard = want;
  p->stats.bulk_ctas = want;
  return FABM_OK;
}

int fabm_plan_reset(fabm_plan* p, fabm_status* status) {
  clear_status(status);
  if (!p) { set_status(status, FABM_ERR_CONFIG, "null plan"); return FABM_ERR_CONFIG; }
  CUDA_TRY(cudaSetDevice(p->device));
  CUDA_TRY(cudaMemsetAsync(p->ctrl, 0, sizeof(DevCtrl), p->stream));
  CUDA_TRY(cudaMemsetAsync(p->ready, 0, sizeof(int) * (p->nb + 1), p->stream));
  // claim words, finished-unit and stage-2 counts, cursors (contiguous)
  CUDA_TRY(cudaMemsetAsync(p->arena + p->off_claim, 0, p->off_PK - p->off_claim, p->stream));
  for (char* va : p->virt_arenas) CUDA_TRY(cudaMemsetAsync(va, 0, sizeof(DevCtrl), p->stream));
  if (p->emulate)  // the peers' control blocks (IPC mappings) belong to this launch too
    for (int sh = 1; sh < p->n_shards; ++sh) CUDA_TRY(cudaMemsetAsync(p->peer[sh], 0, sizeof(DevCtrl), p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  p->armed = true;
  return FABM_OK;
}

// agent CTAs per shard for a sharded run (every GPU hosts the same count)
static int shard_ctas(const fabm_plan* p, int n_shards) {
  const int n_targets = p->nb - kL;
  if (n_targets <= 0) return 1;
  const int want = (n_targets + kWarps - 1) / kWarps;
  return std::max(1, std::min(p->num_sms - 1, (want + n_shards - 1) / n_shards));
}

int fabm_plan_set_virtual_shards(fabm_plan* p, int n_shards, fabm_status* status) {
  clear_status(status);
  if (!p) { set_status(status, FABM_ERR_CONFIG, "null plan"); return FABM_ERR_CONFIG; }
  if (n_shards < 1 || n_shards > kMaxShards || (p->n_shards > 1 && !p->virt)) {
    set_status(status, FABM_ERR_CONFIG, "virtual shards: need 1..%d and a plan not attached to peers", kMaxShards);
    return FABM_ERR_CONFIG;
  }
  CUDA_TRY(cudaSetDevice(p->device));
  for (char* m : p->virt_arenas) cudaFree(m);
  p->virt_arenas.clear();
  p->peer.assign(1, p->arena);
  for (int sh = 1; sh < n_shards; ++sh) {
    char* m = nullptr;
    CUDA_TRY(cudaMalloc(&m, p->shard_bytes));
    CUDA_TRY(cudaMemsetAsync(m, 0, p->shard_bytes, p->stream));
    p->virt_arenas.push_back(m);
    p->peer.push_back(m);
  }
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  p->n_shards = n_shards;
  p->virt = n_shards > 1;
  return FABM_OK;
}

int fabm_plan_ipc_handle(fabm_plan* p, void* handle_out, fabm_status* status) {
  clear_status(status);
  if (!p || !handle_out) { set_status(status, FABM_ERR_CONFIG, "null plan/output"); return FABM_ERR_CONFIG; }
  static_assert(sizeof(cudaIpcMemHandle_t) == FABM_IPC_HANDLE_BYTES, "IPC handle size");
  CUDA_TRY(cudaSetDevice(p->device));
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, p->arena));
  std::memcpy(handle_out, &h, sizeof(h));
  return FABM_OK;
}

int fabm_plan_attach_shards(fabm_plan* p, int n_shards, int rank, const void* handles, fabm_status* status) {
  clear_status(status);
  if (!p || !handles) { set_status(status, FABM_ERR_CONFIG, "null plan/handles"); return FABM_ERR_CONFIG; }
  if (n_shards < 1 || n_shards > kMaxShards || rank < 0 || rank >= n_shards || p->virt) {
    set_status(status, FABM_ERR_CONFIG, "attach: need 1 <= n_shards <= %d, 0 <= rank < n_shards", kMaxShards);
    return FABM_ERR_CONFIG;
  }
  CUDA_TRY(cudaSetDevice(p->device));
  for (char* m : p->opened) cudaIpcCloseMemHandle(m);
  p->opened.clear();
  p->peer.assign(n_shards, nullptr);
  const auto* hb = static_cast<const unsigned char*>(handles);
  for (int sh = 0; sh < n_shards; ++sh) {
    if (sh == rank) { p->peer[sh] = p->arena; continue; }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hb + static_cast<size_t>(sh) * FABM_IPC_HANDLE_BYTES, sizeof(h));
    void* m = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&m, h, cudaIpcMemLazyEnablePeerAccess));
    p->opened.push_back(static_cast<char*>(m));
    p->peer[sh] = static_cast<char*>(m);
  }
  p->n_shards = n_shards;
  p->rank = rank;
  p->armed = false;
  p->agent_ctas_per_shard = shard_ctas(p, n_shards);
  const int n_agents = n_shards * p->agent_ctas_per_shard * kWarps;
  const int n_targets = p->nb - kL;
  if (n_targets > 0 && (n_targets + n_agents - 1) / n_agents > kMaxOwn) {
    set_status(status, FABM_ERR_CONFIG, "n_steps=%lld exceeds the engine capacity", p->N);
    return FABM_ERR_CONFIG;
  }
  p->stats.bulk_ctas = p->agent_ctas_per_shard;
  return FABM_OK;
}

int fabm_plan_emulate_shards(fabm_plan* p, int on, fabm_status* status) {
  clear_status(status);
  if (!p) { set_status(status, FABM_ERR_CONFIG, "null plan"); return FABM_ERR_CONFIG; }
  if (on && (p->n_shards < 2 || p->virt || p->rank != 0)) {
    set_status(status, FABM_ERR_CONFIG, "emulate: needs a plan attached to peer shards, on rank 0");
    return FABM_ERR_CONFIG;
  }
  p->emulate = on != 0;
  if (p->emulate) {
    p->agent_ctas_per_shard = p->bulk_ctas;
    p->stats.bulk_ctas = p->bulk_ctas;
  } else if (p->n_shards > 1) {
    p->agent_ctas_per_shard = shard_ctas(p, p->n_shards);
    p->stats.bulk_ctas = p->agent_ctas_per_shard;
  }
  return FABM_OK;
}

int fabm_plan_shard_counters(const fabm_plan* p, int64_t* src_done, int64_t* bulk_tiles, fabm_status* status) {
  clear_status(status);
  if (!p) { set_status(status, FABM_ERR_CONFIG, "null plan"); return FABM_ERR_CONFIG; }
  CUDA_TRY(cudaSetDevice(p->device));
  DevCtrl h{};
  CUDA_TRY(cudaMemcpy(&h, p->ctrl, sizeof(DevCtrl), cudaMemcpyDeviceToHost));
  if (src_done) *src_done = h.src_done;
  if (bulk_tiles) *bulk_tiles = static_cast<int64_t>(h.bulk_tiles);
  return FABM_OK;
}

int fabm_plan_detach_shards(fabm_plan* p, fabm_status* status) {
  clear_status(status);
  if (!p) { set_status(status, FABM_ERR_CONFIG, "null plan"); return FABM_ERR_CONFIG; }
  CUDA_TRY(cudaSetDevice(p->device));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  for (char* m : p->opened) CUDA_TRY(cudaIpcCloseMemHandle(m));
  p->opened.clear();
  for (char* m : p->virt_arenas) cudaFree(m);
  p->virt_arenas.clear();
  p->peer.assign(1, p->arena);
  p->n_shards = 1;
  p->rank = 0;
  p->virt = false;
  p->emulate = false;
  p->armed = false;
  p->agent_ctas_per_shard = p->bulk_ctas;
  p->stats.bulk_ctas = p->bulk_ctas;
  return FABM_OK;
}

int fabm_plan_download(fabm_plan* p, double* states, double* f_cache, fabm_status* status) {
  clear_status(status);
  if (!p) { set_status(status, FABM_ERR_CONFIG, "null plan"); return FABM_ERR_CONFIG; }
  CUDA_TRY(cudaSetDevice(p->device));
  const int d = p->prob.dim;
  if (states)
    CUDA_TRY(cudaMemcpyAsync(states, p->Y, sizeof(double) * (p->N + 1) * d, cudaMemcpyDeviceToHost, p->stream));
  if (f_cache)
    CUDA_TRY(cudaMemcpyAsync(f_cache, p->Fc, sizeof(double) * (p->N + 1) * d, cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  return FABM_OK;
}

int fabm_plan_download_last(fabm_plan* p, double* y_last, fabm_status* status) {
  clear_status(status);
  if (!p || !y_last) { set_status(status, FABM_ERR_CONFIG, "null plan/output"); return FABM_ERR_CONFIG; }
  CUDA_TRY(cudaSetDevice(p->device));
  const int d = p->prob.dim;
  CUDA_TRY(cudaMemcpyAsync(y_last, p->Y + p->N * d, sizeof(double) * d, cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  return FABM_OK;
}

int fabm_plan_stats(const fabm_plan* p, fabm_stats* s) {
  if (!p || !s) return FABM_ERR_CONFIG;
  *s = p->stats;
  return FABM_OK;
}

void fabm_plan_destroy(fabm_plan* p) { plan_free(p); }

int fabm_solve(const fabm_problem* problem, const fabm_grid* grid, int weight_mode, const double* b,
               const double* a, const double* c, double* states, double* f_cache, fabm_status* status) {
  fabm_plan* p = fabm_plan_create(problem, grid, 0, status);
  if (!p) return status ? status->code : FABM_ERR_CONFIG;
  int rc = fabm_plan_set_weights(p, weight_mode, b, a, c, status);
  if (rc == FABM_OK) rc = fabm_plan_run(p, 60.0, status);
  if (rc == FABM_OK) rc = fabm_plan_download(p, states, f_cache, status);
  plan_free(p);
  return rc;
}

int fabm_weights(double alpha, int64_t n_steps, int mode, double gamma1, double gamma2, double* b, double* a,
                 double* c, fabm_status* status) {
  clear_status(status);
  if (!std::isfinite(alpha) || !(alpha > 0.0 && alpha <= 1.0)) {
    set_status(status, FABM_ERR_CONFIG, "alpha must lie in (0, 1], got %.17g", alpha);
    return FABM_ERR_CONFIG;
  }
  if (n_steps < 1) { set_status(status, FABM_ERR_CONFIG, "n_steps must be >= 1"); return FABM_ERR_CONFIG; }
  if (mode != FABM_WEIGHTS_ACCURATE && mode != FABM_WEIGHTS_FORMULA) {
    set_status(status, FABM_ERR_CONFIG, "fabm_weights generates on device: mode must be ACCURATE or FORMULA");
    return FABM_ERR_CONFIG;
  }
  if (fabm_device_count() <= 0) { set_status(status, FABM_ERR_NODEVICE, "no CUDA device"); return FABM_ERR_NODEVICE; }
  if (gamma1 == 0.0) gamma1 = std::tgamma(alpha + 1.0);
  if (gamma2 == 0.0) gamma2 = std::tgamma(alpha + 2.0);
  const long long len = n_steps + 1;
  double *db = nullptr, *da = nullptr, *dc = nullptr;
  CUDA_TRY(cudaMalloc(&db, sizeof(double) * len));
  CUDA_TRY(cudaMalloc(&da, sizeof(double) * len));
  CUDA_TRY(cudaMalloc(&dc, sizeof(double) * len));
  const int threads = 256;
  const int blocks = static_cast<int>(std::min<long long>((len + threads - 1) / threads, 148LL * 16));
  weights_kernel<<<blocks, threads>>>(alpha, gamma1, gamma2, len, mode == FABM_WEIGHTS_FORMULA ? 1 : 0, db, da, dc);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(b, db, sizeof(double) * len, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(a, da, sizeof(double) * len, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(c, dc, sizeof(double) * len, cudaMemcpyDeviceToHost);
  cudaFree(db);
  cudaFree(da);
  cudaFree(dc);
  if (e != cudaSuccess) { set_status(status, FABM_ERR_CUDA, "weights: %s", cudaGetErrorString(e)); return FABM_ERR_CUDA; }
  return FABM_OK;
}

}  // extern "C"

namespace {
using BatchLaunch = cudaError_t (*)(const BatchParams&, int grid, cudaStream_t);

template <int SYS, int D>
cudaError_t launch_batch(const BatchParams& P, int grid, cudaStream_t stream) {
  auto kern = abm_batch_kernel<SYS, D>;
  const size_t smem = kWarps * sizeof(DmmaSmem<D>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, smem, stream>>>(P);
  return cudaGetLastError();
}

BatchLaunch pick_batch(int sys, int dim) {
  FABM_PICK_SYSTEM(launch_batch);
}

// device buffer; with a stream it is stream-ordered (cudaMallocAsync from the
// device's default pool, freed back to the pool without a device sync)
struct DevBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  ~DevBuf() {
    if (p) {
      if (s) cudaFreeAsync(p, s);
      else cudaFree(p);
    }
  }
  cudaError_t alloc(size_t bytes, cudaStream_t stream) {
    s = stream;
    return cudaMallocAsync(&p, bytes, stream);
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};
// the stream outlives the buffers declared after it (reverse destruction order)
struct StreamHolder {
  cudaStream_t s = nullptr;
  ~StreamHolder() {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
};
// keep freed pool memory cached on the device: repeated batch solves of the
// same size then allocate without cudaMalloc/cudaFree (~100 ms per GB-scale
// sweep otherwise)
void retain_pool_memory(int device) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
}
}  // namespace

extern "C" {

int fabm_solve_batch(const fabm_problem* problems, const fabm_grid* grids, int64_t count, int device, double* states,
                     double* f_cache, double* y_last, double* kernel_ms, fabm_status* status) {
  clear_status(status);
  if (status) status->index = -1;
  if (!problems || !grids || count < 1) {
    set_status(status, FABM_ERR_CONFIG, "batch needs count >= 1 problems and grids");
    return FABM_ERR_CONFIG;
  }
  if (count > (1LL << 30)) {
    set_status(status, FABM_ERR_CONFIG, "batch too large");
    return FABM_ERR_CONFIG;
  }
  const int T = static_cast<int>(count);
  const fabm_problem& p0 = problems[0];
  const long long N = grids[0].n_steps;
  for (int t = 0; t < T; ++t) {
    int rc = validate(&problems[t], &grids[t], status);
    if (rc != FABM_OK) {
      if (status) status->index = t;
      return rc;
    }
    if (problems[t].dim != p0.dim || problems[t].system != p0.system || grids[t].n_steps != N ||
        grids[t].h != grids[0].h) {
      set_status(status, FABM_ERR_CONFIG, "batch members must share dim, system, n_steps and h (member %d)", t);
      if (status) status->index = t;
      return FABM_ERR_CONFIG;
    }
  }
  const int D = p0.dim, DS = stride_of(D);
  BatchLaunch launch = pick_batch(p0.system, D);
  if (!launch) { set_status(status, FABM_ERR_CONFIG, "no batch engine for system/dim"); return FABM_ERR_CONFIG; }
  int ndev = fabm_device_count();
  if (ndev <= 0 || device < 0 || device >= ndev) {
    set_status(status, FABM_ERR_NODEVICE, "no CUDA device %d (found %d)", device, ndev);
    return FABM_ERR_NODEVICE;
  }
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop{};
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  const int nb = static_cast<int>((N + kB - 1) / kB);
  const long long WL = static_cast<long long>(nb) * kB + 2 * kB;
  // host-side per-trajectory scalars (the caller's CPython values when given)
  std::vector<double> hal(T), hg1(T), hg2(T), hha(T), hig(T), hy0(static_cast<size_t>(T) * kMaxDim, 0.0),
      hprm(static_cast<size_t>(T) * kMaxParams, 0.0);
  for (int t = 0; t < T; ++t) {
    fabm_grid g = grids[t];
    fill_scalars(&problems[t], &g);
    hal[t] = problems[t].alpha;
    hg1[t] = g.gamma1;
    hg2[t] = g.gamma2;
    hha[t] = g.h_alpha;
    hig[t] = g.inv_gamma2;
    for (int c = 0; c < D; ++c) hy0[static_cast<size_t>(t) * kMaxDim + c] = problems[t].y0[c];
    for (int i = 0; i < kMaxParams; ++i) hprm[static_cast<size_t>(t) * kMaxParams + i] = problems[t].params[i];
  }
  // pull segments: a body in pieces of G source blocks and a short tail
  // (batch.cuh pull_bounds); the ticket layout of round J is T * S_J pulls
  // then T steps
#ifndef FABM_BATCH_G
#define FABM_BATCH_G 32
#endif
  constexpr int kPullG = FABM_BATCH_G;
  int S_max = 1;
  std::vector<long long> hround(nb + 1, 0), hcum(nb, 0);
  for (int J = 0; J < nb; ++J) {
    const int SJ = pull_units(J, kPullG);
    S_max = std::max(S_max, SJ);
    hround[J + 1] = hround[J] + static_cast<long long>(T) * (SJ + 1);
    hcum[J] = (J >= 2 ? hcum[J - 2] : 0) + SJ;  // pulls of the rounds j <= J of J's parity
  }
  StreamHolder stream_holder;
  CUDA_TRY(cudaStreamCreateWithFlags(&stream_holder.s, cudaStreamNonBlocking));
  cudaStream_t stream = stream_holder.s;
  retain_pool_memory(device);
  DevBuf dal, dg1, dg2, dha, dig, dy0, dprm, dW, dF, dY, dFc, dyl, dnext, dek, des, dtk, dctrl, dround, dcum, dpart, dpdone;
  const size_t szF = sizeof(double) * static_cast<size_t>(T) * (nb + 1) * kB * DS;
  const size_t szY = sizeof(double) * static_cast<size_t>(T) * (N + 1) * D;
  CUDA_TRY(dal.alloc(sizeof(double) * T, stream));
  CUDA_TRY(dg1.alloc(sizeof(double) * T, stream));
  CUDA_TRY(dg2.alloc(sizeof(double) * T, stream));
  CUDA_TRY(dha.alloc(sizeof(double) * T, stream));
  CUDA_TRY(dig.alloc(sizeof(double) * T, stream));
  CUDA_TRY(dy0.alloc(sizeof(double) * hy0.size(), stream));
  CUDA_TRY(dprm.alloc(sizeof(double) * hprm.size(), stream));
  CUDA_TRY(dW.alloc(sizeof(double) * static_cast<size_t>(T) * 3 * WL, stream));
  CUDA_TRY(dF.alloc(szF, stream));
  if (states) CUDA_TRY(dY.alloc(szY, stream));
  if (f_cache) CUDA_TRY(dFc.alloc(szY, stream));
  CUDA_TRY(dyl.alloc(sizeof(double) * static_cast<size_t>(T) * D, stream));
  CUDA_TRY(dnext.alloc(sizeof(int) * T, stream));
  CUDA_TRY(dek.alloc(sizeof(int) * T, stream));
  CUDA_TRY(des.alloc(sizeof(long long) * T, stream));
  CUDA_TRY(dtk.alloc(sizeof(unsigned long long), stream));
  CUDA_TRY(dctrl.alloc(sizeof(DevCtrl), stream));
  CUDA_TRY(dround.alloc(sizeof(long long) * (nb + 1), stream));
  CUDA_TRY(dcum.alloc(sizeof(long long) * nb, stream));
  CUDA_TRY(dpart.alloc(sizeof(double) * static_cast<size_t>(T) * 2 * S_max * kB * 2 * DS, stream));
  CUDA_TRY(dpdone.alloc(sizeof(int) * 2 * T, stream));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto cleanup = [&]() {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  };
  cudaMemcpyAsync(dal.p, hal.data(), sizeof(double) * T, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(dg1.p, hg1.data(), sizeof(double) * T, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(dg2.p, hg2.data(), sizeof(double) * T, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(dha.p, hha.data(), sizeof(double) * T, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(dig.p, hig.data(), sizeof(double) * T, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(dy0.p, hy0.data(), sizeof(double) * hy0.size(), cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(dprm.p, hprm.data(), sizeof(double) * hprm.size(), cudaMemcpyHostToDevice, stream);
  cudaMemsetAsync(dF.p, 0, szF, stream);
  cudaMemsetAsync(dnext.p, 0, sizeof(int) * T, stream);
  cudaMemsetAsync(dek.p, 0, sizeof(int) * T, stream);
  cudaMemsetAsync(des.p, 0, sizeof(long long) * T, stream);
  cudaMemsetAsync(dtk.p, 0, sizeof(unsigned long long), stream);
  cudaMemsetAsync(dctrl.p, 0, sizeof(DevCtrl), stream);
  cudaMemsetAsync(dpdone.p, 0, sizeof(int) * 2 * T, stream);
  cudaMemcpyAsync(dround.p, hround.data(), sizeof(long long) * (nb + 1), cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(dcum.p, hcum.data(), sizeof(long long) * nb, cudaMemcpyHostToDevice, stream);
  {
    const long long total = static_cast<long long>(T) * WL;
    const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148LL * 64));
    weights_batch_kernel<<<blocks, 256, 0, stream>>>(dal.as<double>(), dg1.as<double>(), dg2.as<double>(), T, WL,
                                                     dW.as<double>());
  }
  BatchParams P{};
  P.T = T;
  P.nb = nb;
  P.N = N;
  P.WL = WL;
  P.h = grids[0].h;
  P.ha = dha.as<double>();
  P.ig = dig.as<double>();
  P.y0 = dy0.as<double>();
  P.params = dprm.as<double>();
  P.W = dW.as<double>();
  P.F = dF.as<double>();
  P.Y = dY.as<double>();
  P.Fc = dFc.as<double>();
  P.ylast = dyl.as<double>();
  P.next_block = dnext.as<int>();
  P.err_kind = dek.as<int>();
  P.err_step = des.as<long long>();
  P.ticket = dtk.as<unsigned long long>();
  P.timeout_ns = 600ull * 1000000000ull;
  P.ctrl = dctrl.as<DevCtrl>();
  P.G = kPullG;
  P.S_max = S_max;
  P.round_start = dround.as<long long>();
  P.pull_cum = dcum.as<long long>();
  P.part = dpart.as<double>();
  P.pulls_done = dpdone.as<int>();
  cudaEventRecord(e0, stream);
  cudaError_t le = launch(P, prop.multiProcessorCount, stream);
  cudaEventRecord(e1, stream);
  cudaError_t se = cudaStreamSynchronize(stream);
  if (le != cudaSuccess || se != cudaSuccess) {
    set_status(status, FABM_ERR_CUDA, "batch kernel: %s", cudaGetErrorString(le != cudaSuccess ? le : se));
    cleanup();
    return FABM_ERR_CUDA;
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  if (kernel_ms) *kernel_ms = ms;
  if (states) cudaMemcpy(states, dY.p, szY, cudaMemcpyDeviceToHost);
  if (f_cache) cudaMemcpy(f_cache, dFc.p, szY, cudaMemcpyDeviceToHost);
  if (y_last) cudaMemcpy(y_last, dyl.p, sizeof(double) * static_cast<size_t>(T) * D, cudaMemcpyDeviceToHost);
  std::vector<int> hek(T);
  std::vector<long long> hes(T);
  cudaMemcpy(hek.data(), dek.p, sizeof(int) * T, cudaMemcpyDeviceToHost);
  cudaMemcpy(hes.data(), des.p, sizeof(long long) * T, cudaMemcpyDeviceToHost);
  DevCtrl hc{};
  cudaMemcpy(&hc, dctrl.p, sizeof(DevCtrl), cudaMemcpyDeviceToHost);
  cleanup();
  if (hc.check_line) {
    set_status(status, FABM_ERR_CONFIG, "FABM_CHECKED: batch invariant violated at batch.cuh:%d", hc.check_line);
    return FABM_ERR_CONFIG;
  }
  if (hc.err_code == ERR_TIMEOUT) {
    set_status(status, FABM_ERR_TIMEOUT, "batch watchdog expired");
    return FABM_ERR_TIMEOUT;
  }
  for (int t = 0; t < T; ++t) {
    if (hek[t] != KIND_NONE) {
      if (status) {
        status->code = FABM_ERR_NONFINITE;
        status->kind = hek[t];
        status->step = hes[t];
        status->t = hek[t] == KIND_INITIAL ? 0.0 : static_cast<double>(hes[t] + 1) * grids[0].h;
        status->index = t;
        snprintf(status->message, sizeof(status->message), "trajectory %d: rhs returned a non-finite value", t);
      }
      return FABM_ERR_NONFINITE;
    }
  }
  return FABM_OK;
}

// ---------------------------------------------------------------- DFMA peak
static __global__ void dfma_peak_kernel(double* out, int iters, double x) {
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = x + i * threadIdx.x;
  const double m = 1.0 + 1e-12 * (threadIdx.x & 7);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], m, 1e-9);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 123.456) out[0] = s;
}

double fabm_measure_dfma_peak(int device) {
  if (cudaSetDevice(device) != cudaSuccess) return 0.0;
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  double* out = nullptr;
  cudaMalloc(&out, sizeof(double));
  const int threads = 512, blocks = prop.multiProcessorCount * 4, iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_peak_kernel<<<blocks, threads>>>(out, 200, 1.0);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    dfma_peak_kernel<<<blocks, threads>>>(out, iters, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  const double fmas = static_cast<double>(blocks) * threads * iters * 8.0;
  return fmas / (best * 1e-3);
}

}  // extern "C"

// ======================================================================
// Trajectory CSV (cli.py:97-105) — formatting kernels in csv_format.cuh
// ======================================================================
namespace {

std::string csv_header(int dim) {
  std::string h = "t";
  for (int i = 0; i < dim; ++i) h += ",y" + std::to_string(i);
  h += "\n";
  return h;
}

// The CSV of device states (and optional device times) into a fresh device
// buffer *d_out of *n_bytes (header included).  Synchronous on `stream`.
int csv_format_device(const double* d_states, const double* d_t, double h, long long n_rows, int dim,
                      cudaStream_t stream, char** d_out, long long* n_bytes, double* kernel_ms,
                      fabm_status* status) {
  *d_out = nullptr;
  *n_bytes = 0;
  const int rows = fabm_csv::tile_rows(dim);
  if (dim < 1 || rows < 32 || n_rows < 0) {
    set_status(status, FABM_ERR_CONFIG, "csv: need dim >= 1 (at most %d) and n_rows >= 0", 280);
    return FABM_ERR_CONFIG;
  }
  const std::string head = csv_header(dim);
  const long long n_tiles = (n_rows + rows - 1) / rows;
  int* row_len = nullptr;
  long long* tile_off = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  auto cleanup = [&]() {
    if (row_len) cudaFree(row_len);
    if (tile_off) cudaFree(tile_off);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  };
#define CSV_TRY(expr)                                                               \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      set_status(status, FABM_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e));   \
      cleanup();                                                                    \
      if (*d_out) { cudaFree(*d_out); *d_out = nullptr; }                           \
      return FABM_ERR_CUDA;                                                         \
    }                                                                               \
  } while (0)
  CSV_TRY(cudaEventCreate(&e0));
  CSV_TRY(cudaEventCreate(&e1));
  CSV_TRY(cudaMalloc(&row_len, sizeof(int) * (n_rows > 0 ? n_rows : 1)));
  CSV_TRY(cudaMalloc(&tile_off, sizeof(long long) * (n_tiles + 1)));
  CSV_TRY(cudaMemsetAsync(tile_off, 0, sizeof(long long) * (n_tiles + 1), stream));
  float ms_a = 0.f, ms_b = 0.f;
  long long body = 0;
  if (n_tiles > 0) {
    CSV_TRY(cudaEventRecord(e0, stream));
    fabm_csv::csv_len_kernel<<<static_cast<unsigned>(n_tiles), rows, 0, stream>>>(d_states, d_t, h, n_rows, dim,
                                                                                   row_len, tile_off);
    CSV_TRY(cudaGetLastError());
    fabm_csv::csv_scan_kernel<<<1, 1024, 0, stream>>>(tile_off, n_tiles);
    CSV_TRY(cudaGetLastError());
    CSV_TRY(cudaEventRecord(e1, stream));
    CSV_TRY(cudaMemcpyAsync(&body, tile_off + n_tiles, sizeof(long long), cudaMemcpyDeviceToHost, stream));
    CSV_TRY(cudaStreamSynchronize(stream));
    CSV_TRY(cudaEventElapsedTime(&ms_a, e0, e1));
  }
  const long long total = static_cast<long long>(head.size()) + body;
  CSV_TRY(cudaMalloc(d_out, total > 0 ? total : 1));
  CSV_TRY(cudaMemcpyAsync(*d_out, head.data(), head.size(), cudaMemcpyHostToDevice, stream));
  if (n_tiles > 0) {
    const size_t smem = fabm_csv::tile_smem_bytes(dim, rows);
    CSV_TRY(cudaFuncSetAttribute(fabm_csv::csv_write_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    CSV_TRY(cudaEventRecord(e0, stream));
    fabm_csv::csv_write_kernel<<<static_cast<unsigned>(n_tiles), rows, smem, stream>>>(
        d_states, d_t, h, n_rows, dim, row_len, tile_off, *d_out + head.size());
    CSV_TRY(cudaGetLastError());
    CSV_TRY(cudaEventRecord(e1, stream));
  }
  CSV_TRY(cudaStreamSynchronize(stream));
  if (n_tiles > 0) CSV_TRY(cudaEventElapsedTime(&ms_b, e0, e1));
#undef CSV_TRY
  cleanup();
  *n_bytes = total;
  if (kernel_ms) *kernel_ms = static_cast<double>(ms_a) + ms_b;
  return FABM_OK;
}

constexpr long long kCsvStageBytes = 32ll << 20;
std::mutex g_csv_stage_mu;
char* g_csv_stage[2] = {nullptr, nullptr};

// Device bytes -> file, through two pinned staging buffers so the D2H of
// chunk i+1 overlaps the write of chunk i.
int csv_write_file(const char* path, const char* d_bytes, long long n, cudaStream_t stream, fabm_status* status) {
  if (!path) { set_status(status, FABM_ERR_CONFIG, "csv: null path"); return FABM_ERR_CONFIG; }
  FILE* fh = std::fopen(path, "wb");
  if (!fh) {
    set_status(status, FABM_ERR_IO, "%s: %s", path, std::strerror(errno));
    return FABM_ERR_IO;
  }
  constexpr long long kChunk = kCsvStageBytes;
  // the pinned staging pair is allocated once per process (cudaMallocHost
  // costs milliseconds) and serialised by a mutex
  std::lock_guard<std::mutex> lock(g_csv_stage_mu);
  char** pin = g_csv_stage;
  cudaEvent_t done[2] = {nullptr, nullptr};
  int rc = FABM_OK;
  auto fail_cuda = [&](const char* what, cudaError_t e) {
    set_status(status, FABM_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    rc = FABM_ERR_CUDA;
  };
  cudaError_t e;
  for (int i = 0; i < 2 && rc == FABM_OK; ++i) {
    if (!pin[i] && (e = cudaMallocHost(&pin[i], kChunk)) != cudaSuccess) fail_cuda("cudaMallocHost", e);
    else if ((e = cudaEventCreate(&done[i])) != cudaSuccess) fail_cuda("cudaEventCreate", e);
  }
  const long long n_chunks = (n + kChunk - 1) / kChunk;
  auto issue = [&](long long c) {
    const long long off = c * kChunk, len = std::min(kChunk, n - off);
    cudaError_t ee = cudaMemcpyAsync(pin[c & 1], d_bytes + off, len, cudaMemcpyDeviceToHost, stream);
    if (ee == cudaSuccess) ee = cudaEventRecord(done[c & 1], stream);
    if (ee != cudaSuccess) fail_cuda("csv D2H", ee);
  };
  if (rc == FABM_OK && n_chunks > 0) issue(0);
  for (long long c = 0; c < n_chunks && rc == FABM_OK; ++c) {
    if ((e = cudaEventSynchronize(done[c & 1])) != cudaSuccess) { fail_cuda("csv D2H sync", e); break; }
    if (c + 1 < n_chunks) issue(c + 1);
    const long long len = std::min(kChunk, n - c * kChunk);
    if (std::fwrite(pin[c & 1], 1, static_cast<size_t>(len), fh) != static_cast<size_t>(len)) {
      set_status(status, FABM_ERR_IO, "%s: %s", path, std::strerror(errno));
      rc = FABM_ERR_IO;
    }
  }
  cudaStreamSynchronize(stream);
  if (std::fclose(fh) != 0 && rc == FABM_OK) {
    set_status(status, FABM_ERR_IO, "%s: %s", path, std::strerror(errno));
    rc = FABM_ERR_IO;
  }
  for (int i = 0; i < 2; ++i)
    if (done[i]) cudaEventDestroy(done[i]);
  return rc;
}

// host states/t -> device (one stream), for the host-pointer entry points
int csv_upload(const double* states, const double* t, long long n_rows, int dim, int device, cudaStream_t* stream,
               double** d_states, double** d_t, fabm_status* status) {
  *d_states = nullptr;
  *d_t = nullptr;
  if (n_rows < 0 || dim < 1 || (n_rows > 0 && !states)) {
    set_status(status, FABM_ERR_CONFIG, "csv: need states for n_rows >= 0 rows of dim >= 1");
    return FABM_ERR_CONFIG;
  }
  const int ndev = fabm_device_count();
  if (ndev <= 0 || device < 0 || device >= ndev) {
    set_status(status, FABM_ERR_NODEVICE, "no CUDA device %d (found %d)", device, ndev);
    return FABM_ERR_NODEVICE;
  }
  CUDA_TRY(cudaSetDevice(device));
  CUDA_TRY(cudaStreamCreateWithFlags(stream, cudaStreamNonBlocking));
  const size_t sb = sizeof(double) * static_cast<size_t>(n_rows > 0 ? n_rows : 1) * dim;
  CUDA_TRY(cudaMalloc(d_states, sb));
  if (n_rows > 0)
    CUDA_TRY(cudaMemcpyAsync(*d_states, states, sizeof(double) * n_rows * dim, cudaMemcpyHostToDevice, *stream));
  if (t && n_rows > 0) {
    CUDA_TRY(cudaMalloc(d_t, sizeof(double) * n_rows));
    CUDA_TRY(cudaMemcpyAsync(*d_t, t, sizeof(double) * n_rows, cudaMemcpyHostToDevice, *stream));
  }
  return FABM_OK;
}

void csv_release(cudaStream_t stream, double* d_states, double* d_t, char* d_out) {
  if (stream) cudaStreamSynchronize(stream);
  if (d_states) cudaFree(d_states);
  if (d_t) cudaFree(d_t);
  if (d_out) cudaFree(d_out);
  if (stream) cudaStreamDestroy(stream);
}

}  // namespace

extern "C" {

int fabm_format_csv(const double* states, const double* t, int64_t n_rows, int32_t dim, double h, int device,
                    char* out, int64_t out_cap, int64_t* n_bytes, double* kernel_ms, fabm_status* status) {
  clear_status(status);
  cudaStream_t stream = nullptr;
  double *d_states = nullptr, *d_t = nullptr;
  char* d_out = nullptr;
  int rc = csv_upload(states, t, n_rows, dim, device, &stream, &d_states, &d_t, status);
  long long total = 0;
  if (rc == FABM_OK) rc = csv_format_device(d_states, d_t, h, n_rows, dim, stream, &d_out, &total, kernel_ms, status);
  if (rc == FABM_OK) {
    if (n_bytes) *n_bytes = total;
    if (!out || out_cap < total) {
      set_status(status, FABM_ERR_CONFIG, "csv: output buffer of %lld bytes, %lld needed",
                 static_cast<long long>(out_cap), total);
      rc = FABM_ERR_CONFIG;
    } else {
      cudaError_t e = cudaMemcpyAsync(out, d_out, total, cudaMemcpyDeviceToHost, stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
      if (e != cudaSuccess) {
        set_status(status, FABM_ERR_CUDA, "csv D2H: %s", cudaGetErrorString(e));
        rc = FABM_ERR_CUDA;
      }
    }
  }
  csv_release(stream, d_states, d_t, d_out);
  return rc;
}

int fabm_write_csv(const char* path, const double* states, const double* t, int64_t n_rows, int32_t dim, double h,
                   int device, int64_t* n_bytes, double* kernel_ms, fabm_status* status) {
  clear_status(status);
  cudaStream_t stream = nullptr;
  double *d_states = nullptr, *d_t = nullptr;
  char* d_out = nullptr;
  int rc = csv_upload(states, t, n_rows, dim, device, &stream, &d_states, &d_t, status);
  long long total = 0;
  if (rc == FABM_OK) rc = csv_format_device(d_states, d_t, h, n_rows, dim, stream, &d_out, &total, kernel_ms, status);
  if (rc == FABM_OK) rc = csv_write_file(path, d_out, total, stream, status);
  if (rc == FABM_OK && n_bytes) *n_bytes = total;
  csv_release(stream, d_states, d_t, d_out);
  return rc;
}

int fabm_plan_write_csv(fabm_plan* p, const char* path, int64_t* n_bytes, double* kernel_ms, fabm_status* status) {
  clear_status(status);
  if (!p) { set_status(status, FABM_ERR_CONFIG, "null plan"); return FABM_ERR_CONFIG; }
  CUDA_TRY(cudaSetDevice(p->device));
  char* d_out = nullptr;
  long long total = 0;
  int rc = csv_format_device(p->Y, nullptr, p->grid.h, p->N + 1, p->prob.dim, p->stream, &d_out, &total, kernel_ms,
                             status);
  if (rc == FABM_OK) rc = csv_write_file(path, d_out, total, p->stream, status);
  if (rc == FABM_OK && n_bytes) *n_bytes = total;
  if (d_out) cudaFree(d_out);
  return rc;
}

}  // extern "C"

extern "C" int fabm_mittag_leffler(const double* alpha, const double* z, int64_t n, int device, double* out,
                                   int32_t* codes, fabm_status* status) {
  clear_status(status);
  if (n < 0 || (n > 0 && (!alpha || !z || !out))) {
    set_status(status, FABM_ERR_CONFIG, "mittag_leffler: need alpha, z and out for n >= 0 pairs");
    return FABM_ERR_CONFIG;
  }
  if (n == 0) return FABM_OK;
  const int ndev = fabm_device_count();
  if (ndev <= 0 || device < 0 || device >= ndev) {
    set_status(status, FABM_ERR_NODEVICE, "no CUDA device %d (found %d)", device, ndev);
    return FABM_ERR_NODEVICE;
  }
  CUDA_TRY(cudaSetDevice(device));
  double* d = nullptr;
  int* c = nullptr;
  const size_t nb = sizeof(double) * static_cast<size_t>(n);
  cudaError_t e = cudaMalloc(&d, 3 * nb);
  if (e == cudaSuccess) e = cudaMalloc(&c, sizeof(int) * static_cast<size_t>(n));
  if (e == cudaSuccess) e = cudaMemcpy(d, alpha, nb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d + n, z, nb, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    const int threads = 128;
    fabm_oracle::mittag_leffler_kernel<<<static_cast<unsigned>((n + threads - 1) / threads), threads>>>(
        d, d + n, n, d + 2 * n, c);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, d + 2 * n, nb, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && codes) e = cudaMemcpy(codes, c, sizeof(int) * static_cast<size_t>(n), cudaMemcpyDeviceToHost);
  if (d) cudaFree(d);
  if (c) cudaFree(c);
  if (e != cudaSuccess) {
    set_status(status, FABM_ERR_CUDA, "mittag_leffler: %s", cudaGetErrorString(e));
    return FABM_ERR_CUDA;
  }
  return FABM_OK;
}

// ======================================================================
// Single-step ops (serial.py:74-111) — steps.cuh
// ======================================================================
namespace {
using StepLaunch = cudaError_t (*)(const StepParams&, cudaStream_t);
template <int SYS, int D>
cudaError_t launch_steps(const StepParams& P, cudaStream_t stream) {
  const long long blocks = (P.count + 7) / 8;  // 8 warps (requests) per CTA
  step_pc_kernel<SYS, D><<<static_cast<unsigned>(blocks), 256, 0, stream>>>(P);
  return cudaGetLastError();
}
StepLaunch pick_steps(int sys, int dim) { FABM_PICK_SYSTEM(launch_steps); }
}  // namespace

extern "C" int fabm_step_pc(const fabm_problem* problem, const fabm_grid* grid, const double* b, const double* a,
                            const double* c, int64_t n_weights, const double* f_cache, int64_t n_rows,
                            const int64_t* ns, int64_t count, const double* y_pred, double* yp_out, double* y_out,
                            int32_t* err_out, int device, fabm_status* status) {
  clear_status(status);
  if (!problem || !grid || !b || !a || !c || !f_cache || (count > 0 && (!ns || !err_out)) || count < 0) {
    set_status(status, FABM_ERR_CONFIG, "step_pc: null argument");
    return FABM_ERR_CONFIG;
  }
  const int d = problem->dim;
  StepLaunch launch = pick_steps(problem->system, d);
  if (!launch) {
    set_status(status, FABM_ERR_CONFIG, "no device rhs for system %d with dim %d", problem->system, d);
    return FABM_ERR_CONFIG;
  }
  long long nmax = -1;
  for (int64_t i = 0; i < count; ++i) {
    const long long n = ns[i];
    // _history_transposed, serial.py:67-71
    if (n < 0 || n >= grid->n_steps) {
      set_status(status, FABM_ERR_CONFIG, "step index n=%lld outside [0, %lld)", n,
                 static_cast<long long>(grid->n_steps));
      return FABM_ERR_CONFIG;
    }
    if (n >= n_rows || n >= n_weights) {
      set_status(status, FABM_ERR_CONFIG, "step index n=%lld needs %lld f rows and weights (have %lld, %lld)", n,
                 n + 1, static_cast<long long>(n_rows), static_cast<long long>(n_weights));
      return FABM_ERR_CONFIG;
    }
    nmax = std::max(nmax, n);
  }
  if (count == 0) return FABM_OK;
  const int ndev = fabm_device_count();
  if (ndev <= 0 || device < 0 || device >= ndev) {
    set_status(status, FABM_ERR_NODEVICE, "no CUDA device %d (found %d)", device, ndev);
    return FABM_ERR_NODEVICE;
  }
  CUDA_TRY(cudaSetDevice(device));
  fabm_grid g = *grid;
  fill_scalars(problem, &g);
  const size_t nw = static_cast<size_t>(nmax + 1), nq = static_cast<size_t>(count);
  DevBuf buf;
  const size_t bytes = sizeof(double) * (3 * nw + nw * d + d + 3 * nq * d) + sizeof(long long) * nq + sizeof(int) * nq;
  CUDA_TRY(cudaMalloc(&buf.p, bytes));
  double* w = buf.as<double>();
  StepParams P{};
  P.count = count;
  P.wb = w;
  P.wa = w + nw;
  P.wc = w + 2 * nw;
  P.F = w + 3 * nw;
  double* y0 = w + 3 * nw + nw * d;
  double* yq = y0 + d;
  P.y0 = y0;
  P.yp_out = yq + nq * d;
  P.y_out = yq + 2 * nq * d;
  P.ypred = y_pred ? yq : nullptr;
  long long* dns = reinterpret_cast<long long*>(yq + 3 * nq * d);
  P.ns = dns;
  P.err = reinterpret_cast<int*>(dns + nq);
  P.h = g.h;
  P.ha = g.h_alpha;
  P.ig = g.inv_gamma2;
  std::memcpy(P.params, problem->params, sizeof(P.params));
  CUDA_TRY(cudaMemcpy(w, b, sizeof(double) * nw, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(w + nw, a, sizeof(double) * nw, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(w + 2 * nw, c, sizeof(double) * nw, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(w + 3 * nw, f_cache, sizeof(double) * nw * d, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(y0, problem->y0, sizeof(double) * d, cudaMemcpyHostToDevice));
  if (y_pred) CUDA_TRY(cudaMemcpy(yq, y_pred, sizeof(double) * nq * d, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dns, ns, sizeof(long long) * nq, cudaMemcpyHostToDevice));
  CUDA_TRY(launch(P, nullptr));
  CUDA_TRY(cudaDeviceSynchronize());
  if (yp_out) CUDA_TRY(cudaMemcpy(yp_out, P.yp_out, sizeof(double) * nq * d, cudaMemcpyDeviceToHost));
  if (y_out) CUDA_TRY(cudaMemcpy(y_out, P.y_out, sizeof(double) * nq * d, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(err_out, P.err, sizeof(int) * nq, cudaMemcpyDeviceToHost));
  return FABM_OK;
}

// ======================================================================
// Pinned host output (the trajectory streamed to the host during the run)
// ======================================================================
extern "C" {

void* fabm_host_alloc(int64_t bytes) {
  void* ptr = nullptr;
  if (bytes <= 0) return nullptr;
  if (cudaHostAlloc(&ptr, static_cast<size_t>(bytes), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
    return nullptr;
  return ptr;
}

void fabm_host_free(void* ptr) {
  if (ptr) cudaFreeHost(ptr);
}

int fabm_plan_set_host_output(fabm_plan* p, double* states, double* f_cache, fabm_status* status) {
  clear_status(status);
  if (!p) { set_status(status, FABM_ERR_CONFIG, "null plan"); return FABM_ERR_CONFIG; }
  if ((states == nullptr) != (f_cache == nullptr)) {
    set_status(status, FABM_ERR_CONFIG, "host output needs both states and f_cache (or neither)");
    return FABM_ERR_CONFIG;
  }
  if (p->n_shards > 1 && !p->virt && p->rank != 0) {
    set_status(status, FABM_ERR_CONFIG, "host output lives on the stepper's rank (0)");
    return FABM_ERR_CONFIG;
  }
  CUDA_TRY(cudaSetDevice(p->device));
  p->Yh = p->Fch = nullptr;
  if (!states) return FABM_OK;
  void *dy = nullptr, *df = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&dy, states, 0);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(&df, f_cache, 0);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_status(status, FABM_ERR_CONFIG, "host output must be mapped pinned memory (fabm_host_alloc): %s",
               cudaGetErrorString(e));
    return FABM_ERR_CONFIG;
  }
  p->Yh = static_cast<double*>(dy);
  p->Fch = static_cast<double*>(df);
  return FABM_OK;
}

}  // extern "C"

extern "C" int fabm_trim_memory(int device) {
  cudaMemPool_t pool;
  if (cudaSetDevice(device) != cudaSuccess) return FABM_ERR_NODEVICE;
  if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return FABM_ERR_CUDA;
  cudaDeviceSynchronize();
  return cudaMemPoolTrimTo(pool, 0) == cudaSuccess ? FABM_OK : FABM_ERR_CUDA;
}
