// dfma_tile.cuh — the bulk tile on the CUDA-core FP64 FMA pipe (the design
// before bulk_dmma.cuh), kept for the A/B probes in tools/ (tile_dmma.cu,
// tile_bench.cu, tile_variants.cu): register-blocked 4 targets x d components
// x {b, a} per lane, weights staged in a mod-4 transposed smem layout.  The
// shipped engine uses the FP64 tensor-core tile; both give bitwise equal sums.
#pragma once
#include "engine.cuh"

namespace fabm {

constexpr int kWCols = 2 * kB / 4 + 2;  // transposed weight row length (+2 pad)

struct AgentSmem {
  double w[2][4][kWCols];  // b, a in mod-4 transposed layout
  double f[kB][4];         // f tile of the source block (row stride 4)
  int own_next[kMaxOwn];   // next source block per owned target
};

template <int D>
__device__ __forceinline__ void agent_store_acc(double* BK, int J, int lane,
                                                const double (&accP)[kR][D], const double (&accC)[kR][D]) {
  constexpr int DS = Stride<D>::value;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    double* dst = BK + (static_cast<long long>(J) * kB + kR * lane + r) * 2 * DS;
#pragma unroll
    for (int c = 0; c < D; ++c) { dst[c] = accP[r][c]; dst[DS + c] = accC[r][c]; }
  }
}

template <int D>
__device__ __forceinline__ void agent_load_acc(const double* BK, int J, int lane,
                                               double (&accP)[kR][D], double (&accC)[kR][D]) {
  constexpr int DS = Stride<D>::value;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const double* src = BK + (static_cast<long long>(J) * kB + kR * lane + r) * 2 * DS;
#pragma unroll
    for (int c = 0; c < D; ++c) { accP[r][c] = __ldcg(src + c); accC[r][c] = __ldcg(src + DS + c); }
  }
}

// acc[n] += sum_{k in block I} w[n - k] f_k for the lane's 4 targets of block J,
// ascending k.  Weight window u = 127 - s + r (jl = 4*lane + u), mod-4 transposed.
template <int D>
__device__ __forceinline__ void agent_tile(const double* __restrict__ wbp, const double* __restrict__ wap,
                                           const double* Fp, AgentSmem& A, int I, int J, int lane,
                                           double (&accP)[kR][D], double (&accC)[kR][D]) {
  constexpr int DS = Stride<D>::value;
  __syncwarp();
  // ---- stage weights j in [Delta-127, Delta+127] (transposed) and the f tile
  const long long base = static_cast<long long>(J - I) * kB - (kB - 1);
  for (int jl = lane; jl < 2 * kB - 1; jl += 32) {
    const double vb = __ldg(wbp + base + jl);
    const double va = __ldg(wap + base + jl);
    A.w[0][jl & 3][jl >> 2] = vb;
    A.w[1][jl & 3][jl >> 2] = va;
  }
  {
    const double* src = Fp + static_cast<long long>(I) * kB * DS;
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

}  // namespace fabm
