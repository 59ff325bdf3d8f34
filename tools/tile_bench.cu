// tile_bench.cu — throughput of the bulk Toeplitz tile (agent_tile) alone:
// every warp of 148 CTAs computes T tiles from L2-resident synthetic data.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1611_08678_b200/csrc -o tools/tile_bench tools/tile_bench.cu
#include <cstdio>
#include <vector>

#include "engine.cuh"
#include "dfma_tile.cuh"

using namespace fabm;

template <int D>
__global__ void __launch_bounds__(kThreads, 1) tile_kernel(EngineParams P, int tiles, double* out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  AgentSmem* A = reinterpret_cast<AgentSmem*>(smem_raw) + warp;
  double accP[kR][D], accC[kR][D];
  for (int r = 0; r < kR; ++r)
    for (int c = 0; c < D; ++c) { accP[r][c] = 0.0; accC[r][c] = 0.0; }
  const int agent = blockIdx.x * kWarps + warp;
  for (int t = 0; t < tiles; ++t) {
    const int J = 3 + (agent * 7 + t * 13) % (P.nb - 3);
    const int I = (agent + t) % (J - 2);
    agent_tile<D>(P.wb, P.wa, P.F, *A, I, J, lane, accP, accC);
  }
  double s = 0;
  for (int r = 0; r < kR; ++r)
    for (int c = 0; c < D; ++c) s += accP[r][c] + accC[r][c];
  if (s == 1.2345) out[0] = s;
}

int main(int argc, char** argv) {
  const int tiles = argc > 1 ? atoi(argv[1]) : 64;
  const int nb = 512;  // 64k steps of synthetic history
  const long long wl = (long long)nb * kB + 2 * kB;
  std::vector<double> h(wl);
  for (long long i = 0; i < wl; ++i) h[i] = 1.0 / (1.0 + i);
  double *wb, *wa, *F, *out;
  cudaMalloc(&wb, wl * 8);
  cudaMalloc(&wa, wl * 8);
  cudaMalloc(&F, (nb + 1) * kB * 4 * 8);
  cudaMalloc(&out, 8);
  cudaMemcpy(wb, h.data(), wl * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(wa, h.data(), wl * 8, cudaMemcpyHostToDevice);
  cudaMemset(F, 0, (nb + 1) * kB * 4 * 8);
  EngineParams P{};
  P.wb = wb; P.wa = wa; P.F = F; P.nb = nb;
  const size_t smem = kWarps * sizeof(AgentSmem);
  cudaFuncSetAttribute(tile_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tile_kernel<3><<<148, kThreads, smem>>>(P, 2, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  tile_kernel<3><<<148, kThreads, smem>>>(P, tiles, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fma = 148.0 * kWarps * tiles * 2.0 * kB * kB * 3;
  printf("tiles/warp=%d  %.3f ms  %.3e FMA/s  (%s)\n", tiles, ms, fma / (ms * 1e-3),
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
