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
                                                            int chunks, double* out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
  return 0;
}
