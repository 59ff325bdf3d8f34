// tile_dmma.cu — the bulk Toeplitz product on the FP64 tensor cores
// (mma.sync m8n8k4 f64) vs the DFMA tile (agent_tile), standalone.
//
// One DMMA: D[i][j] += sum_k W[tb + i - sb - k] * f[sb + k + 8j][c]
//   = contribution to target tb + i + 8j from sources sb + 8j + k
// (Toeplitz: the weight only depends on target - source), so the 8 columns
// are 8 diagonal shifts and every column is useful for any d.  A target half
// block (64 targets) times one source chunk X..X+127 is swept with
// sb in [X-56, X+72) (32 DMMAs per component and weight); column j then covers
// sources [X-56+8j, X+72+8j), contiguous across chunks; the last chunk adds a
// closing sweep sb in [X+72, X+128) over zero-padded rows.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1611_08678_b200/csrc -o tools/tile_dmma tools/tile_dmma.cu
#include <cstdio>
#include <vector>

#include "engine.cuh"
#include "dfma_tile.cuh"

using namespace fabm;

constexpr int kFRows = 240;                    // rows X-56 .. X+183 (zeros past the chunk)
constexpr int kFPad = kFRows + 4 * (kFRows / 8);  // padded: conflict-free 8-strided reads
struct DSmem {
  double w[2][256];   // b, a: w[u] = W[T0 - X - 127 + u]
  double f[3][kFPad];  // f[c][rho + 4*(rho>>3)], rho = row - (X - 56)
};

__device__ __forceinline__ int fidx(int rho) { return rho + 4 * (rho >> 3); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// acc[h][c][w][2]: targets T0 + 64h + (lane>>2) + 8*(2*(lane&3) + e)
template <int D>
__device__ __forceinline__ void dmma_chunk(const double* __restrict__ wbp, const double* __restrict__ wap,
                                           const double* Fp, DSmem& S, int T0, int X, int Xend, bool closing,
                                           int lane, double (&acc)[2][D][2][2]) {
  constexpr int DS = Stride<D>::value;
  __syncwarp();
  const long long wbase = static_cast<long long>(T0) - X - 127;
  for (int u = lane; u < 256; u += 32) {
    const long long j = wbase + u;
    S.w[0][u] = __ldg(wbp + j);
    S.w[1][u] = __ldg(wap + j);
  }
  for (int rho = lane; rho < kFRows; rho += 32) {
    const int row = X - 56 + rho;
    const bool ok = row >= 0 && row < Xend;
#pragma unroll
    for (int c = 0; c < D; ++c) S.f[c][fidx(rho)] = ok ? __ldcg(Fp + static_cast<long long>(row) * DS + c) : 0.0;
  }
  __syncwarp();
  const int i = lane >> 2, k = lane & 3;
  const int nsteps = closing ? 46 : 32;  // sb = X - 56 + 4v
#pragma unroll 2
  for (int v = 0; v < nsteps; ++v) {
    const int sbr = 4 * v;  // sb - (X - 56)
    // A: W[tb + i - sb - k], tb = T0 + 64h  ->  u = tb + i - sb - k - wbase
    //   = 64h + i - k + 127 - (sb - X) = 64h + i - k + 183 - sbr
    double a[2][2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int u = 64 * h + i - k + 183 - sbr;
      a[h][0] = S.w[0][u];
      a[h][1] = S.w[1][u];
    }
    double b[D];
#pragma unroll
    for (int c = 0; c < D; ++c) b[c] = S.f[c][fidx(sbr + k + 8 * i)];  // B: row k, col j = lane>>2
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int c = 0; c < D; ++c)
#pragma unroll
        for (int w = 0; w < 2; ++w) dmma(acc[h][c][w][0], acc[h][c][w][1], a[h][w], b[c]);
  }
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1) dmma_kernel(const double* wb, const double* wa, const double* F,
                                                           int chunks, double* out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  DSmem* S = reinterpret_cast<DSmem*>(smem_raw) + warp;
  double acc[2][D][2][2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int w = 0; w < 2; ++w) acc[h][c][w][0] = acc[h][c][w][1] = 0.0;
  const int J = chunks + 3 + (blockIdx.x % 5);  // target block; sources 0 .. 128*chunks
  const int T0 = 128 * J;
  for (int I = 0; I < chunks; ++I)
    dmma_chunk<D>(wb, wa, F, *S, T0, 128 * I, 128 * chunks, I == chunks - 1, lane, acc);
  // out[gwarp][target 0..127][c][w]
  double* o = out + (static_cast<long long>(blockIdx.x) * kWarps + warp) * 128 * D * 2;
  const int i = lane >> 2, q = lane & 3;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int w = 0; w < 2; ++w)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int t = 64 * h + i + 8 * (2 * q + e);
          o[(t * D + c) * 2 + w] = acc[h][c][w][e];
        }
}

// DFMA reference: the engine's agent_tile over the same chunks
template <int D>
__global__ void __launch_bounds__(kThreads, 1) dfma_kernel(const double* wb, const double* wa, const double* F,
                                                           int chunks, double* out) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  AgentSmem* A = reinterpret_cast<AgentSmem*>(smem_raw) + warp;
  double accP[kR][D], accC[kR][D];
  for (int r = 0; r < kR; ++r)
    for (int c = 0; c < D; ++c) accP[r][c] = accC[r][c] = 0.0;
  const int J = chunks + 3 + (blockIdx.x % 5);
  for (int I = 0; I < chunks; ++I) agent_tile<D>(wb, wa, F, *A, I, J, lane, accP, accC);
  double* o = out + (static_cast<long long>(blockIdx.x) * kWarps + warp) * 128 * D * 2;
  for (int r = 0; r < kR; ++r)
    for (int c = 0; c < D; ++c) {
      const int t = kR * lane + r;
      o[(t * D + c) * 2 + 0] = accP[r][c];
      o[(t * D + c) * 2 + 1] = accC[r][c];
    }
}

int main(int argc, char** argv) {
  const int chunks = argc > 1 ? atoi(argv[1]) : 64;
  constexpr int D = 3;
  const int nb = chunks + 16;
  const long long wl = (long long)nb * kB + 2 * kB;
  std::vector<double> hw(wl), hwa(wl), hf((long long)(nb + 1) * kB * 4);
  for (long long j = 0; j < wl; ++j) { hw[j] = 1.0 / (1.0 + j); hwa[j] = 1.0 / (2.0 + 0.5 * j); }
  for (size_t i = 0; i < hf.size(); ++i) hf[i] = 1e-3 * (double)((i * 7919) % 1000) - 0.5;
  double *wb, *wa, *F, *o1, *o2;
  const size_t outn = 148ull * kWarps * 128 * D * 2;
  cudaMalloc(&wb, wl * 8);
  cudaMalloc(&wa, wl * 8);
  cudaMalloc(&F, hf.size() * 8);
  cudaMalloc(&o1, outn * 8);
  cudaMalloc(&o2, outn * 8);
  cudaMemcpy(wb, hw.data(), wl * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(wa, hwa.data(), wl * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(F, hf.data(), hf.size() * 8, cudaMemcpyHostToDevice);
  const size_t s1 = kWarps * sizeof(DSmem), s2 = kWarps * sizeof(AgentSmem);
  printf("smem/CTA: dmma %zu B, dfma %zu B\n", s1, s2);
  cudaFuncSetAttribute(dmma_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1);
  cudaFuncSetAttribute(dfma_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best1 = 1e30f, best2 = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    cudaEventRecord(e0);
    dmma_kernel<D><<<148, kThreads, s1>>>(wb, wa, F, chunks, o1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best1 = ms < best1 ? ms : best1;
    cudaEventRecord(e0);
    dfma_kernel<D><<<148, kThreads, s2>>>(wb, wa, F, chunks, o2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best2 = ms < best2 ? ms : best2;
  }
  const double fma = 148.0 * kWarps * chunks * 2.0 * kB * kB * D;
  printf("DMMA tile: %.3f ms  %.3e FMA/s\nDFMA tile: %.3f ms  %.3e FMA/s   (%s)\n", best1, fma / (best1 * 1e-3), best2,
         fma / (best2 * 1e-3), cudaGetErrorString(cudaGetLastError()));
  std::vector<double> r1(outn), r2(outn);
  cudaMemcpy(r1.data(), o1, outn * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(r2.data(), o2, outn * 8, cudaMemcpyDeviceToHost);
  double md = 0, mx = 0;
  for (size_t i = 0; i < outn; ++i) {
    md = fmax(md, fabs(r1[i] - r2[i]));
    mx = fmax(mx, fabs(r2[i]));
  }
  printf("max |dmma - dfma| = %.3e (max |value| %.3e, rel %.3e)\n", md, mx, md / mx);
  return 0;
}
