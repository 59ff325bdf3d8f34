// pair_probe.cu — does a bulk agent holding TWO adjacent target blocks
// (J, J+1) per staged source chunk beat the engine's one-target chunk?
// The f rows of a chunk are staged once for both targets and the two weight
// windows overlap (target J+1's window is J's shifted by 128), so staging
// per DMMA drops by ~40 %; the accumulators double (48 doubles per lane), so
// the probe runs WPS warps per SM with up to 255 registers.
// Same products, same per-target order as dmma_chunk: results must match.
// make -C tools pair_probe; ./pair_probe
#include <cstdio>
#include <vector>

#include "engine.cuh"

using namespace fabm;

template <int D>
struct PairSmem {
  double w[2][384];    // b, a: w[u] = W[T0 - X - 127 + u] (target J: u < 256, J+1: u + 128)
  double f[D][kDPad];
};

template <int D>
using PairAcc = double[2][2][D][2][2];  // [target][half][c][w][e]

template <int D>
__device__ __forceinline__ void pair_chunk(const double* __restrict__ wbp, const double* __restrict__ wap,
                                           const double* Fp, PairSmem<D>& S, int T0, int X, int xend, int lane,
                                           PairAcc<D>& acc) {
  constexpr int DS = Stride<D>::value;
  __syncwarp();
  const long long wbase = static_cast<long long>(T0) - X - 127;
  for (int u = lane; u < 384; u += 32) {
    S.w[0][u] = __ldg(wbp + wbase + u);
    S.w[1][u] = __ldg(wap + wbase + u);
  }
#pragma unroll 3
  for (int rho = lane; rho < kDRows; rho += 32) {
    const int row = X - 56 + rho;
    const bool ok = row >= 0 && row < xend;
    const double* src = Fp + static_cast<long long>(ok ? row : 0) * DS;
#pragma unroll
    for (int c = 0; c < D; ++c) S.f[c][dmma_fidx(rho)] = ok ? __ldcg(src + c) : 0.0;
  }
  __syncwarp();
  const int i = lane >> 2, k = lane & 3;
#pragma unroll 2
  for (int v = 0; v < kDSweep; ++v) {
    const int sbr = 4 * v;
    double a[2][2][2];
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = 128 * t + 64 * h + i - k + 183 - sbr;
        a[t][h][0] = S.w[0][u];
        a[t][h][1] = S.w[1][u];
      }
    const int rho = sbr + k + 8 * i;
    double b[D];
#pragma unroll
    for (int c = 0; c < D; ++c) b[c] = S.f[c][dmma_fidx(rho)];
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < D; ++c)
#pragma unroll
          for (int w = 0; w < 2; ++w) dmma_f64(acc[t][h][c][w][0], acc[t][h][c][w][1], a[t][h][w], b[c]);
  }
}

template <int D, int WPS>
__global__ void __launch_bounds__(WPS * 32, 1) pair_kernel(const double* wb, const double* wa, const double* F,
                                                           int chunks, double* out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto* S = reinterpret_cast<PairSmem<D>*>(smem_raw) + warp;
  PairAcc<D> acc;
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int c = 0; c < D; ++c)
#pragma unroll
        for (int w = 0; w < 2; ++w) acc[t][h][c][w][0] = acc[t][h][c][w][1] = 0.0;
  const int J = chunks + kL + 2 * ((blockIdx.x * WPS + warp) % 32);
  for (int I = 0; I < chunks; ++I) pair_chunk<D>(wb, wa, F, *S, J * kB, I * kB, (J - kL + 2) * kB, lane, acc);
  double s = 0;
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int c = 0; c < D; ++c)
#pragma unroll
        for (int w = 0; w < 2; ++w) s += acc[t][h][c][w][0] + acc[t][h][c][w][1];
  out[blockIdx.x * 1024 + threadIdx.x] = s;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) single_kernel(const double* wb, const double* wa, const double* F,
                                                             int chunks, double* out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto* S = reinterpret_cast<DmmaSmem<D>*>(smem_raw) + warp;
  DmmaAcc<D> acc;
  dmma_zero<D>(acc);
  const int J = chunks + kL + (blockIdx.x * kWarps + warp) % 64;
  for (int I = 0; I < chunks; ++I) dmma_chunk<D>(wb, wa, F, *S, J * kB, I * kB, (J - kL + 1) * kB, lane, acc);
  double s = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int w = 0; w < 2; ++w) s += acc[h][c][w][0] + acc[h][c][w][1];
  out[blockIdx.x * 1024 + threadIdx.x] = s;
}

template <int WPS>
void run_pair(const double* wb, const double* wa, const double* F, double* out, int chunks, int nsm, double base) {
  constexpr int D = 3;
  const size_t smem = WPS * sizeof(PairSmem<D>);
  cudaFuncSetAttribute(pair_kernel<D, WPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  pair_kernel<D, WPS><<<nsm, WPS * 32, smem>>>(wb, wa, F, 8, out);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    pair_kernel<D, WPS><<<nsm, WPS * 32, smem>>>(wb, wa, F, chunks, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double fma = (double)nsm * WPS * 2 * chunks * 2.0 * kB * kB * D;
  printf("pair chunk, %2d warps/SM (2 targets each): %.3f ms  %.4e FMA/s = %.3f x the single chunk  (%s)\n", WPS, best,
         fma / (best * 1e-3), fma / (best * 1e-3) / base, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  constexpr int D = 3;
  const int chunks = 256, nsm = 148;
  const long long nrows = (chunks + 80 + 2 * kL) * (long long)kB + 512;
  std::vector<double> hw(nrows), hf(nrows * 4);
  for (long long i = 0; i < nrows; ++i) hw[i] = 1.0 / (1.0 + i);
  for (long long i = 0; i < nrows * 4; ++i) hf[i] = 1e-3 * (i % 97);
  double *wb, *wa, *F, *out;
  cudaMalloc(&wb, nrows * 8);
  cudaMalloc(&wa, nrows * 8);
  cudaMalloc(&F, nrows * 32);
  cudaMalloc(&out, nsm * 1024 * 8);
  cudaMemcpy(wb, hw.data(), nrows * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(wa, hw.data(), nrows * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(F, hf.data(), nrows * 32, cudaMemcpyHostToDevice);
  const size_t smem = kWarps * sizeof(DmmaSmem<D>);
  cudaFuncSetAttribute(single_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  single_kernel<D><<<nsm, kThreads, smem>>>(wb, wa, F, 8, out);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    single_kernel<D><<<nsm, kThreads, smem>>>(wb, wa, F, chunks, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double fma = (double)nsm * kWarps * chunks * 2.0 * kB * kB * D;
  const double base = fma / (best * 1e-3);
  printf("engine chunk (one target, 16 warps/SM): %.3f ms  %.4e FMA/s\n", best, base);
  run_pair<4>(wb, wa, F, out, chunks, nsm, base);
  run_pair<6>(wb, wa, F, out, chunks, nsm, base);
  run_pair<8>(wb, wa, F, out, chunks, nsm, base);
  run_pair<12>(wb, wa, F, out, chunks, nsm, base);
  return 0;
}
