// tile_variants.cu — DFMA operand-order variants of the bulk Toeplitz tile
// (agent_tile in csrc/engine.cuh) measured alone: every warp of 148 CTAs
// computes T tiles of L2-resident synthetic data; checks all variants agree.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1611_08678_b200/csrc -o tools/tile_variants tools/tile_variants.cu
#include <cstdio>
#include <vector>

#include "engine.cuh"
#include "dfma_tile.cuh"

using namespace fabm;

__device__ __forceinline__ double fma_ab(double a, double b, double c) {
  double d;
  asm("fma.rn.f64 %0, %1, %2, %3;" : "=d"(d) : "d"(a), "d"(b), "d"(c));
  return d;
}

// V: 0 = engine agent_tile; 1 = f-major order, asm fma(f, w, acc);
// 2 = w-major order, asm fma(w, f, acc)
template <int D, int V>
__device__ __forceinline__ void tile_v(const double* __restrict__ wbp, const double* __restrict__ wap,
                                       const double* Fp, AgentSmem& A, int I, int J, int lane,
                                       double (&accP)[kR][D], double (&accC)[kR][D]) {
  if (V == 0) {
    agent_tile<D>(wbp, wap, Fp, A, I, J, lane, accP, accC);
    return;
  }
  constexpr int DS = Stride<D>::value;
  __syncwarp();
  const long long base = static_cast<long long>(J - I) * kB - (kB - 1);
  for (int jl = lane; jl < 2 * kB - 1; jl += 32) {
    const double vb = __ldg(wbp + base + jl);
    const double va = __ldg(wap + base + jl);
    A.w[0][jl & 3][jl >> 2] = vb;
    A.w[1][jl & 3][jl >> 2] = va;
  }
  {
    const double* src = Fp + static_cast<long long>(I) * kB * DS;
    for (int i = lane; i < kB * DS / 2; i += 32) {
      const double2 v = __ldcg(reinterpret_cast<const double2*>(src) + i);
      const int row = (2 * i) / DS, c = (2 * i) % DS;
      A.f[row][c] = v.x;
      A.f[row][c + 1] = v.y;
    }
  }
  __syncwarp();
  double wb[7], wa[7];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
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
      if (V == 1) {
#pragma unroll
        for (int c = 0; c < D; ++c)
#pragma unroll
          for (int r = 0; r < kR; ++r) {
            accP[r][c] = fma_ab(fk[c], wb[3 + r - t], accP[r][c]);
            accC[r][c] = fma_ab(fk[c], wa[3 + r - t], accC[r][c]);
          }
      } else {
#pragma unroll
        for (int r = 0; r < kR; ++r) {
#pragma unroll
          for (int c = 0; c < D; ++c) accP[r][c] = fma_ab(wb[3 + r - t], fk[c], accP[r][c]);
#pragma unroll
          for (int c = 0; c < D; ++c) accC[r][c] = fma_ab(wa[3 + r - t], fk[c], accC[r][c]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) { wb[4 + i] = wb[i]; wa[4 + i] = wa[i]; }
  }
}

template <int D, int V>
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
    tile_v<D, V>(P.wb, P.wa, P.F, *A, I, J, lane, accP, accC);
  }
  double s = 0;
  for (int r = 0; r < kR; ++r)
    for (int c = 0; c < D; ++c) s += accP[r][c] * (1 + r) + accC[r][c] * (3 + c);
  out[blockIdx.x * kThreads + threadIdx.x] = s;
}

template <int V>
double run(EngineParams P, int tiles, double* out, std::vector<double>& res) {
  const size_t smem = kWarps * sizeof(AgentSmem);
  cudaFuncSetAttribute(tile_kernel<3, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  tile_kernel<3, V><<<148, kThreads, smem>>>(P, 2, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    tile_kernel<3, V><<<148, kThreads, smem>>>(P, tiles, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  res.resize(148 * kThreads);
  cudaMemcpy(res.data(), out, res.size() * 8, cudaMemcpyDeviceToHost);
  const double fma = 148.0 * kWarps * tiles * 2.0 * kB * kB * 3;
  printf("variant %d: %.3f ms  %.3e FMA/s  (%s)\n", V, best, fma / (best * 1e-3), cudaGetErrorString(cudaGetLastError()));
  return fma / (best * 1e-3);
}

int main(int argc, char** argv) {
  const int tiles = argc > 1 ? atoi(argv[1]) : 64;
  const int nb = 512;
  const long long wl = (long long)nb * kB + 2 * kB;
  std::vector<double> h(wl), hf((nb + 1) * kB * 4);
  for (long long i = 0; i < wl; ++i) h[i] = 1.0 / (1.0 + i);
  for (size_t i = 0; i < hf.size(); ++i) hf[i] = 1e-3 * ((i * 7919) % 1000);
  double *wb, *wa, *F, *out;
  cudaMalloc(&wb, wl * 8);
  cudaMalloc(&wa, wl * 8);
  cudaMalloc(&F, hf.size() * 8);
  cudaMalloc(&out, 148 * kThreads * 8);
  cudaMemcpy(wb, h.data(), wl * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(wa, h.data(), wl * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(F, hf.data(), hf.size() * 8, cudaMemcpyHostToDevice);
  EngineParams P{};
  P.wb = wb; P.wa = wa; P.F = F; P.nb = nb;
  std::vector<double> r0, r1, r2;
  run<0>(P, tiles, out, r0);
  run<1>(P, tiles, out, r1);
  run<2>(P, tiles, out, r2);
  double d1 = 0, d2 = 0;
  for (size_t i = 0; i < r0.size(); ++i) {
    d1 = fmax(d1, fabs(r1[i] - r0[i]) / fmax(1e-300, fabs(r0[i])));
    d2 = fmax(d2, fabs(r2[i] - r0[i]) / fmax(1e-300, fabs(r0[i])));
  }
  printf("max rel diff vs engine: v1 %.3e  v2 %.3e\n", d1, d2);
  return 0;
}
