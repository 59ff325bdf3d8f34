// chunk_probe.cu — the engine's bulk chunk (bulk_dmma.cuh dmma_chunk) alone:
// 16 agent warps per SM, each sweeping `chunks` source chunks into one
// target block, as in the engine's steady state.  Reports FMA/s against the
// DMMA peak; profile with ncu --set full --import-source on.
// make -C tools chunk_probe
#include <cstdio>
#include <vector>

#include "engine.cuh"

using namespace fabm;

template <int D>
__global__ void __launch_bounds__(kThreads, 1) chunk_kernel(const double* wb, const double* wa, const double* F,
                                                            int chunks, double* out, int active = kWarps) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= active) return;
  auto* S = reinterpret_cast<DmmaSmem<D>*>(smem_raw) + warp;
  DmmaAcc<D> acc;
  dmma_zero<D>(acc);
  const int J = chunks + kL + (blockIdx.x * kWarps + warp) % 64;  // targets above the sources
  for (int I = 0; I < chunks; ++I) dmma_chunk<D>(wb, wa, F, *S, J * kB, I * kB, (J - kL + 1) * kB, lane, acc);
  double s = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int w = 0; w < 2; ++w) s += acc[h][c][w][0] + acc[h][c][w][1];
  out[blockIdx.x * kThreads + threadIdx.x] = s;
}

// prefetch variant: while chunk I is swept, the cache lines of chunk I+1's
// weight windows and f rows are prefetched into L1 (prefetch.global.L1), and
// the f rows are then loaded through L1 (__ldg)
template <int D>
__device__ __forceinline__ void chunk_prefetch_next(const double* wbp, const double* wap, const double* Fp, int T0,
                                                    int Xn, int xend, int lane) {
  constexpr int DS = Stride<D>::value;
  if (Xn >= xend) return;
  const long long wbase = static_cast<long long>(T0) - Xn - 127;
  // 256 doubles = 2 KB = 16 lines per weight array; 184 rows x 32 B = 46 lines of f
  if (lane < 16) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(wbp + wbase + 16 * lane));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(wap + wbase + 16 * lane));
  }
  for (int q = lane; q < 47; q += 32) {
    const int row = Xn - 56 + 4 * q;
    if (row >= 0 && row < xend) asm volatile("prefetch.global.L1 [%0];" ::"l"(Fp + static_cast<long long>(row) * DS));
  }
}

template <int D>
__device__ __forceinline__ void dmma_chunk_pf(const double* __restrict__ wbp, const double* __restrict__ wap,
                                              const double* Fp, DmmaSmem<D>& S, int T0, int X, int xend, int lane,
                                              DmmaAcc<D>& acc) {
  constexpr int DS = Stride<D>::value;
  __syncwarp();
  const long long wbase = static_cast<long long>(T0) - X - 127;
  for (int u = lane; u < 256; u += 32) {
    S.w[0][u] = __ldg(wbp + wbase + u);
    S.w[1][u] = __ldg(wap + wbase + u);
  }
  for (int rho = lane; rho < kDRows; rho += 32) {
    const int row = X - 56 + rho;
    const bool ok = row >= 0 && row < xend;
    const double* src = Fp + static_cast<long long>(ok ? row : 0) * DS;
#pragma unroll
    for (int c = 0; c < D; ++c) S.f[c][dmma_fidx(rho)] = ok ? __ldg(src + c) : 0.0;
  }
  __syncwarp();
  chunk_prefetch_next<D>(wbp, wap, Fp, T0, X + kB, xend, lane);
  const int i = lane >> 2, k = lane & 3;
  const int nsteps = (X + 128 >= xend) ? kDSweep + kDClose : kDSweep;
#pragma unroll 2
  for (int v = 0; v < nsteps; ++v) {
    const int sbr = 4 * v;
    double a[2][2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int u = 64 * h + i - k + 183 - sbr;
      a[h][0] = S.w[0][u];
      a[h][1] = S.w[1][u];
    }
    const int rho = sbr + k + 8 * i;
    double b[D];
#pragma unroll
    for (int c = 0; c < D; ++c) b[c] = rho < kDRows ? S.f[c][dmma_fidx(rho)] : 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int c = 0; c < D; ++c)
#pragma unroll
        for (int w = 0; w < 2; ++w) dmma_f64(acc[h][c][w][0], acc[h][c][w][1], a[h][w], b[c]);
  }
}

// batched staging: every load of the chunk issued before any shared store
template <int D>
__device__ __forceinline__ void dmma_chunk_batched(const double* __restrict__ wbp, const double* __restrict__ wap,
                                                   const double* __restrict__ Fp, DmmaSmem<D>& S, int T0, int X,
                                                   int xend, int lane, DmmaAcc<D>& acc) {
  constexpr int DS = Stride<D>::value;
  const long long wbase = static_cast<long long>(T0) - X - 127;
  double wv[2][8], fv[6][D];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    wv[0][q] = __ldg(wbp + wbase + lane + 32 * q);
    wv[1][q] = __ldg(wap + wbase + lane + 32 * q);
  }
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const int rho = lane + 32 * q;
    const int row = X - 56 + rho;
    const bool ok = rho < kDRows && row >= 0 && row < xend;
    const double* src = Fp + static_cast<long long>(ok ? row : 0) * DS;
#pragma unroll
    for (int c = 0; c < D; ++c) fv[q][c] = ok ? __ldcg(src + c) : 0.0;
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    S.w[0][lane + 32 * q] = wv[0][q];
    S.w[1][lane + 32 * q] = wv[1][q];
  }
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const int rho = lane + 32 * q;
    if (rho < kDRows) {
#pragma unroll
      for (int c = 0; c < D; ++c) S.f[c][dmma_fidx(rho)] = fv[q][c];
    }
  }
  __syncwarp();
  const int i = lane >> 2, k = lane & 3;
  const int nsteps = (X + 128 >= xend) ? kDSweep + kDClose : kDSweep;
#pragma unroll 2
  for (int v = 0; v < nsteps; ++v) {
    const int sbr = 4 * v;
    double a[2][2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int u = 64 * h + i - k + 183 - sbr;
      a[h][0] = S.w[0][u];
      a[h][1] = S.w[1][u];
    }
    const int rho = sbr + k + 8 * i;
    double b[D];
#pragma unroll
    for (int c = 0; c < D; ++c) b[c] = rho < kDRows ? S.f[c][dmma_fidx(rho)] : 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int c = 0; c < D; ++c)
#pragma unroll
        for (int w = 0; w < 2; ++w) dmma_f64(acc[h][c][w][0], acc[h][c][w][1], a[h][w], b[c]);
  }
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) batched_kernel(const double* wb, const double* wa, const double* F,
                                                              int chunks, double* out, int active) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= active) return;
  auto* S = reinterpret_cast<DmmaSmem<D>*>(smem_raw) + warp;
  DmmaAcc<D> acc;
  dmma_zero<D>(acc);
  const int J = chunks + kL + (blockIdx.x * kWarps + warp) % 64;
  for (int I = 0; I < chunks; ++I)
    dmma_chunk_batched<D>(wb, wa, F, *S, J * kB, I * kB, (J - kL + 1) * kB, lane, acc);
  double s = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int w = 0; w < 2; ++w) s += acc[h][c][w][0] + acc[h][c][w][1];
  out[blockIdx.x * kThreads + threadIdx.x] = s;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) pf_kernel(const double* wb, const double* wa, const double* F,
                                                         int chunks, double* out, int active) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= active) return;
  auto* S = reinterpret_cast<DmmaSmem<D>*>(smem_raw) + warp;
  DmmaAcc<D> acc;
  dmma_zero<D>(acc);
  const int J = chunks + kL + (blockIdx.x * kWarps + warp) % 64;
  for (int I = 0; I < chunks; ++I) dmma_chunk_pf<D>(wb, wa, F, *S, J * kB, I * kB, (J - kL + 1) * kB, lane, acc);
  double s = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int w = 0; w < 2; ++w) s += acc[h][c][w][0] + acc[h][c][w][1];
  out[blockIdx.x * kThreads + threadIdx.x] = s;
}

// sweep-only: stage one chunk, sweep it `chunks` times (no restaging) -- the
// DMMA sweep's own ceiling for k warps per SM
template <int D>
__global__ void __launch_bounds__(kThreads, 1) sweep_kernel(const double* wb, const double* wa, const double* F,
                                                            int chunks, double* out, int active) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= active) return;
  auto* S = reinterpret_cast<DmmaSmem<D>*>(smem_raw) + warp;
  DmmaAcc<D> acc;
  dmma_zero<D>(acc);
  const int J = chunks + kL + 8;
  DmmaAcc<D> tmp;
  dmma_zero<D>(tmp);
  dmma_chunk<D>(wb, wa, F, *S, J * kB, 0, (J - kL + 1) * kB, lane, tmp);  // stage chunk 0
  const int i = lane >> 2, k = lane & 3;
  for (int I = 0; I < chunks; ++I) {
#pragma unroll 2
    for (int v = 0; v < kDSweep; ++v) {
      const int sbr = 4 * v;
      double a[2][2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = 64 * h + i - k + 183 - sbr;
        a[h][0] = S->w[0][u];
        a[h][1] = S->w[1][u];
      }
      const int rho = sbr + k + 8 * i;
      double b[D];
#pragma unroll
      for (int c = 0; c < D; ++c) b[c] = S->f[c][dmma_fidx(rho)];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < D; ++c)
#pragma unroll
          for (int w = 0; w < 2; ++w) dmma_f64(acc[h][c][w][0], acc[h][c][w][1], a[h][w], b[c]);
    }
  }
  double s = tmp[0][0][0][0];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int w = 0; w < 2; ++w) s += acc[h][c][w][0] + acc[h][c][w][1];
  out[blockIdx.x * kThreads + threadIdx.x] = s;
}

// variant: the two weight windows staged by TMA bulk copies (one elected
// lane, mbarrier completion), the f rows by the lanes as in dmma_chunk
template <int D>
struct alignas(128) TmaSmem {
  double w[2][264];  // 258 used: the window starts one double early when misaligned
  double f[D][kDPad];
  uint64_t bar;
};

template <int D>
__global__ void __launch_bounds__(kThreads, 1) tma_kernel(const double* wb, const double* wa, const double* F,
                                                          int chunks, double* out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int DS = Stride<D>::value;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto& S = reinterpret_cast<TmaSmem<D>*>(smem_raw)[warp];
  if (lane == 0) mbar_init(&S.bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  DmmaAcc<D> acc;
  dmma_zero<D>(acc);
  const int J = chunks + kL + (blockIdx.x * kWarps + warp) % 64;
  const int T0 = J * kB, xend = (J - kL + 1) * kB;
  uint32_t phase = 0;
  for (int I = 0; I < chunks; ++I) {
    const int X = I * kB;
    __syncwarp();
    const long long wbase = static_cast<long long>(T0) - X - 127;
    const long long wal = wbase & ~1ll;
    const int off = static_cast<int>(wbase - wal);
    if (lane == 0) {
      const uint32_t bar = smem_u32(&S.bar);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2 * 2064) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(&S.w[0][0])), "l"(wb + wal), "r"(2064), "r"(bar) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(&S.w[1][0])), "l"(wa + wal), "r"(2064), "r"(bar) : "memory");
    }
    for (int rho = lane; rho < kDRows; rho += 32) {
      const int row = X - 56 + rho;
      const bool ok = row >= 0 && row < xend;
      const double* src = F + static_cast<long long>(ok ? row : 0) * DS;
#pragma unroll
      for (int c = 0; c < D; ++c) S.f[c][dmma_fidx(rho)] = ok ? __ldcg(src + c) : 0.0;
    }
    while (!mbar_try(&S.bar, phase)) {}
    phase ^= 1;
    __syncwarp();
    const int i = lane >> 2, k = lane & 3;
    const int nsteps = (X + 128 >= xend) ? kDSweep + kDClose : kDSweep;
#pragma unroll 2
    for (int v = 0; v < nsteps; ++v) {
      const int sbr = 4 * v;
      double a[2][2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = 64 * h + i - k + 183 - sbr + off;
        a[h][0] = S.w[0][u];
        a[h][1] = S.w[1][u];
      }
      const int rho = sbr + k + 8 * i;
      double b[D];
#pragma unroll
      for (int c = 0; c < D; ++c) b[c] = rho < kDRows ? S.f[c][dmma_fidx(rho)] : 0.0;
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < D; ++c)
#pragma unroll
          for (int w = 0; w < 2; ++w) dmma_f64(acc[h][c][w][0], acc[h][c][w][1], a[h][w], b[c]);
    }
  }
  double s = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int w = 0; w < 2; ++w) s += acc[h][c][w][0] + acc[h][c][w][1];
  out[blockIdx.x * kThreads + threadIdx.x] = s;
}

int main() {
  constexpr int D = 3;
  const int chunks = 256, nsm = 148;
  const long long nrows = (chunks + 64 + 2 * kL) * (long long)kB + 256;
  std::vector<double> hw(nrows), hf(nrows * 4);
  for (long long i = 0; i < nrows; ++i) hw[i] = 1.0 / (1.0 + i);
  for (long long i = 0; i < nrows * 4; ++i) hf[i] = 1e-3 * (i % 97);
  double *wb, *wa, *F, *out;
  cudaMalloc(&wb, nrows * 8);
  cudaMalloc(&wa, nrows * 8);
  cudaMalloc(&F, nrows * 32);
  cudaMalloc(&out, nsm * kThreads * 8);
  cudaMemcpy(wb, hw.data(), nrows * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(wa, hw.data(), nrows * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(F, hf.data(), nrows * 32, cudaMemcpyHostToDevice);
  const size_t smem = kWarps * sizeof(DmmaSmem<D>);
  cudaFuncSetAttribute(chunk_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  chunk_kernel<D><<<nsm, kThreads, smem>>>(wb, wa, F, 8, out);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    chunk_kernel<D><<<nsm, kThreads, smem>>>(wb, wa, F, chunks, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double fma = (double)nsm * kWarps * chunks * 2.0 * kB * kB * D;
  printf("engine chunk (bulk_dmma.cuh): %.3f ms  %.4e FMA/s  (%s)\n", best, fma / (best * 1e-3),
         cudaGetErrorString(cudaGetLastError()));
  for (int active : {1, 2, 4, 8}) {  // lone-warp chunk rate (the per-chain cap of the schedule)
    float tb = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      chunk_kernel<D><<<nsm, kThreads, smem>>>(wb, wa, F, chunks, out, active);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tb = ms < tb ? ms : tb;
    }
    const double f1 = (double)nsm * active * chunks * 2.0 * kB * kB * D;
    printf("  %2d warp(s)/SM: %.4e FMA/s = %.3f of the 16-warp rate per SM\n", active, f1 / (tb * 1e-3),
           (f1 / (tb * 1e-3)) / (fma / (best * 1e-3)));
  }
  cudaFuncSetAttribute(pf_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int active : {1, 2, 4, 8, 16}) {
    float tb = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      pf_kernel<D><<<nsm, kThreads, smem>>>(wb, wa, F, chunks, out, active);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tb = ms < tb ? ms : tb;
    }
    const double f1 = (double)nsm * active * chunks * 2.0 * kB * kB * D;
    printf("  L1 prefetch of the next chunk, %2d warp(s)/SM: %.4e FMA/s = %.3f of the 16-warp chunk rate\n", active,
           f1 / (tb * 1e-3), (f1 / (tb * 1e-3)) / (fma / (best * 1e-3)));
  }
  cudaFuncSetAttribute(batched_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int active : {1, 4, 8, 16}) {
    float tb = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      batched_kernel<D><<<nsm, kThreads, smem>>>(wb, wa, F, chunks, out, active);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tb = ms < tb ? ms : tb;
    }
    const double f1 = (double)nsm * active * chunks * 2.0 * kB * kB * D;
    printf("  batched staging loads, %2d warp(s)/SM: %.4e FMA/s = %.3f of the 16-warp chunk rate\n", active,
           f1 / (tb * 1e-3), (f1 / (tb * 1e-3)) / (fma / (best * 1e-3)));
  }
  {
    std::vector<double> r1(nsm * kThreads), r2(nsm * kThreads);
    chunk_kernel<D><<<nsm, kThreads, smem>>>(wb, wa, F, chunks, out);
    cudaMemcpy(r1.data(), out, 8 * r1.size(), cudaMemcpyDeviceToHost);
    batched_kernel<D><<<nsm, kThreads, smem>>>(wb, wa, F, chunks, out, kWarps);
    cudaMemcpy(r2.data(), out, 8 * r2.size(), cudaMemcpyDeviceToHost);
    bool same = true;
    for (size_t q = 0; q < r1.size(); ++q) same &= r1[q] == r2[q];
    printf("  batched staging bitwise %s\n", same ? "equal" : "DIFFERENT");
  }
  cudaFuncSetAttribute(sweep_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int active : {1, 4, 16}) {
    float tb = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      sweep_kernel<D><<<nsm, kThreads, smem>>>(wb, wa, F, chunks, out, active);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tb = ms < tb ? ms : tb;
    }
    const double f1 = (double)nsm * active * chunks * 2.0 * kB * kB * D;
    printf("  sweep only, %2d warp(s)/SM: %.4e FMA/s = %.3f of the 16-warp chunk rate\n", active, f1 / (tb * 1e-3),
           (f1 / (tb * 1e-3)) / (fma / (best * 1e-3)));
  }
  chunk_kernel<D><<<nsm, kThreads, smem>>>(wb, wa, F, chunks, out);
  cudaDeviceSynchronize();
  std::vector<double> ref(nsm * kThreads), got(nsm * kThreads);
  cudaMemcpy(ref.data(), out, 8 * ref.size(), cudaMemcpyDeviceToHost);
  {
    const size_t tsmem = kWarps * sizeof(TmaSmem<D>);
    cudaFuncSetAttribute(tma_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsmem);
    tma_kernel<D><<<nsm, kThreads, tsmem>>>(wb, wa, F, 8, out);
    float tb = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      tma_kernel<D><<<nsm, kThreads, tsmem>>>(wb, wa, F, chunks, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tb = ms < tb ? ms : tb;
    }
    cudaMemcpy(got.data(), out, 8 * got.size(), cudaMemcpyDeviceToHost);
    bool same = true;
    for (size_t q = 0; q < ref.size(); ++q) same &= ref[q] == got[q];
    printf("TMA weights + lane f staging: %.3f ms  %.4e FMA/s  bitwise %s (%s)\n", tb, fma / (tb * 1e-3),
           same ? "equal" : "DIFFERENT", cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
