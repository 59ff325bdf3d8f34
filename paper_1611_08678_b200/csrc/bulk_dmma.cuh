// bulk_dmma.cuh — the bulk Toeplitz products on the FP64 tensor cores.
//
// One m8n8k4 DMMA computes
//     D[i][j] += sum_k W[tb + i - sb - k] * f[sb + k + 8j][c]
// i.e. the contribution to target tb + i + 8j of sources sb + 8j + k.  The
// weight depends only on target - source (Toeplitz), so the 8 columns are 8
// diagonal shifts of one weight fragment: all 8 columns are useful for any
// state dimension d (a (target x component) mapping would fill only d of 8).
//
// A bulk agent computes one target block J at a time (128 targets = two
// halves of 64, 24 accumulator doubles per lane for d = 3, the same register
// budget as the DFMA tile) -- a whole block, or one unit of it (a fixed
// segment of its sources; engine.cuh "units") -- and sweeps source chunks
// X = 128 I in ascending order: chunk I runs sb over [X-56, X+72) in steps of 4, so column
// j covers sources [X-56+8j, X+72+8j) -- contiguous from chunk to chunk --
// and the last chunk adds a closing sweep sb in [X+72, X+128) whose rows past
// the bulk end read as zero.  Every (target, source) product is taken once,
// in ascending source order per target, with the DMMA's sequential-FMA
// accumulation: the sums are bitwise equal to the DFMA tile's (agent_tile;
// tools/tile_dmma.cu checks this and measures 1.69e13 vs 1.38e13 FMA/s).
#pragma once

namespace fabm {

constexpr int kDRows = 184;                           // staged rows X-56 .. X+127
constexpr int kDPad = kDRows + 4 * (kDRows / 8);      // +4 per 8 rows: conflict-free 8-strided B reads
constexpr int kDSweep = 32, kDClose = 14;             // sb steps per chunk / closing sweep

template <int D>
struct DmmaSmem {
  double w[2][256];    // b, a: w[u] = W[T0 - X - 127 + u]
  double f[D][kDPad];  // f[c][rho + 4 (rho >> 3)], rho = row - (X - 56)
};

__device__ __forceinline__ int dmma_fidx(int rho) { return rho + 4 * (rho >> 3); }

__device__ __forceinline__ void dmma_f64(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// accumulators: acc[h][c][w][e] <-> target 64h + (lane>>2) + 8 (2 (lane&3) + e)
// of the block, component c, weight w (0 = predictor b, 1 = corrector a)
template <int D>
using DmmaAcc = double[2][D][2][2];

__device__ __forceinline__ int dmma_target(int lane, int h, int e) {
  return 64 * h + (lane >> 2) + 8 * (2 * (lane & 3) + e);
}

// sources of chunk I (X = 128 I) into the sums of target block J (T0 = 128 J);
// xend = bulk end of the block (128 (J - L + 1)); closing on its last chunk
template <int D, bool BATCHED = false>
__device__ __forceinline__ void dmma_chunk(const double* __restrict__ wbp, const double* __restrict__ wap,
                                           const double* Fp, DmmaSmem<D>& S, int T0, int X, int xend,
                                           int lane, DmmaAcc<D>& acc) {
  constexpr int DS = Stride<D>::value;
  if constexpr (BATCHED) {
    const long long wbase = static_cast<long long>(T0) - X - 127;
    // every global load of the chunk issued before its shared stores, so the
    // loads overlap instead of serialising one round trip per loop iteration:
    // the batch kernel stages from HBM (sweep working sets exceed L2);
    // 4096 x 1e5 sweep 7.43 -> 7.11 s.  (In the engine, whose staging hits
    // L2, the extra registers cost more than they gain.)
    constexpr int kFQ = (kDRows + 31) / 32;  // 6 rows per lane
    {
      double wv[2][8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        wv[0][q] = __ldg(wbp + wbase + lane + 32 * q);
        wv[1][q] = __ldg(wap + wbase + lane + 32 * q);
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        S.w[0][lane + 32 * q] = wv[0][q];
        S.w[1][lane + 32 * q] = wv[1][q];
      }
    }
    double fv[kFQ][D];
#pragma unroll
    for (int q = 0; q < kFQ; ++q) {
      const int rho = lane + 32 * q;
      const int row = X - 56 + rho;
      const bool ok = rho < kDRows && row >= 0 && row < xend;
      const double* src = Fp + static_cast<long long>(ok ? row : 0) * DS;
#pragma unroll
      for (int c = 0; c < D; ++c) fv[q][c] = ok ? __ldcg(src + c) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kFQ; ++q) {
      const int rho = lane + 32 * q;
      if (rho < kDRows) {
#pragma unroll
        for (int c = 0; c < D; ++c) S.f[c][dmma_fidx(rho)] = fv[q][c];
      }
    }
    __syncwarp();
  } else {
    __syncwarp();
    const long long wbase = static_cast<long long>(T0) - X - 127;
    for (int u = lane; u < 256; u += 32) {
      S.w[0][u] = __ldg(wbp + wbase + u);
      S.w[1][u] = __ldg(wap + wbase + u);
    }
#pragma unroll 3  // 3 rows' loads in flight: N=1e6 193.7 -> 190.9 ms (2 or 6: worse)
    for (int rho = lane; rho < kDRows; rho += 32) {
      const int row = X - 56 + rho;
      const bool ok = row >= 0 && row < xend;
      const double* src = Fp + static_cast<long long>(ok ? row : 0) * DS;
#pragma unroll
      for (int c = 0; c < D; ++c) S.f[c][dmma_fidx(rho)] = ok ? __ldcg(src + c) : 0.0;
    }
    __syncwarp();
  }
  const int i = lane >> 2, k = lane & 3;
  // the 32 regular sweep steps read staged rows only (rho <= 183); the
  // closing steps of a target's last chunk run past them and read zeros
  auto step = [&](int v, bool guard) {
    const int sbr = 4 * v;  // sb - (X - 56)
    // A = W[tb + i - sb - k], tb = T0 + 64 h  ->  u = 64 h + i - k + 183 - sbr
    double a[2][2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int u = 64 * h + i - k + 183 - sbr;
      a[h][0] = S.w[0][u];
      a[h][1] = S.w[1][u];
    }
    // B = f[sb + k + 8j], column j = lane >> 2
    const int rho = sbr + k + 8 * i;
    double b[D];
#pragma unroll
    for (int c = 0; c < D; ++c) b[c] = (!guard || rho < kDRows) ? S.f[c][dmma_fidx(rho)] : 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int c = 0; c < D; ++c)
#pragma unroll
        for (int w = 0; w < 2; ++w) dmma_f64(acc[h][c][w][0], acc[h][c][w][1], a[h][w], b[c]);
  };
#pragma unroll 2
  for (int v = 0; v < kDSweep; ++v) step(v, false);
  if (X + 128 >= xend) {
#pragma unroll 1
    for (int v = kDSweep; v < kDSweep + kDClose; ++v) step(v, true);
  }
}

template <int D>
__device__ __forceinline__ void dmma_zero(DmmaAcc<D>& acc) {
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int w = 0; w < 2; ++w) acc[h][c][w][0] = acc[h][c][w][1] = 0.0;
}

// spill / reload of an unfinished target (lane-major, inside the target's BK rows)
template <int D>
__device__ __forceinline__ void dmma_spill(double* BK, int J, int lane, const DmmaAcc<D>& acc) {
  constexpr int DS = Stride<D>::value;
  double* dst = BK + static_cast<long long>(J) * kB * 2 * DS + lane * (8 * D);
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int w = 0; w < 2; ++w)
        reinterpret_cast<double2*>(dst)[(h * D + c) * 2 + w] = make_double2(acc[h][c][w][0], acc[h][c][w][1]);
}
template <int D>
__device__ __forceinline__ void dmma_reload(const double* BK, int J, int lane, DmmaAcc<D>& acc) {
  constexpr int DS = Stride<D>::value;
  const double* src = BK + static_cast<long long>(J) * kB * 2 * DS + lane * (8 * D);
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const double2 v = __ldcg(reinterpret_cast<const double2*>(src) + (h * D + c) * 2 + w);
        acc[h][c][w][0] = v.x;
        acc[h][c][w][1] = v.y;
      }
}
// a unit's partial-sum slot (lane-major, 8D doubles per lane)
template <int D>
__device__ __forceinline__ void dmma_spill_slot(double* slot, int lane, const DmmaAcc<D>& acc) {
  dmma_spill<D>(slot, 0, lane, acc);
}
template <int D>
__device__ __forceinline__ void dmma_reload_slot(const double* slot, int lane, DmmaAcc<D>& acc) {
  dmma_reload<D>(slot, 0, lane, acc);
}
// acc += slot, element by element (the fixed-order reduction of partials)
template <int D>
__device__ __forceinline__ void dmma_add_slot(const double* slot, int lane, DmmaAcc<D>& acc) {
  const double* src = slot + lane * (8 * D);
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int w = 0; w < 2; ++w) {
        const double2 v = __ldcg(reinterpret_cast<const double2*>(src) + (h * D + c) * 2 + w);
        acc[h][c][w][0] = __dadd_rn(acc[h][c][w][0], v.x);
        acc[h][c][w][1] = __dadd_rn(acc[h][c][w][1], v.y);
      }
}
// final sums in the row layout the stepper stages: BK[(J B + t) 2 DS + w DS + c]
template <int D>
__device__ __forceinline__ void dmma_store_rows(double* BK, int J, int lane, const DmmaAcc<D>& acc) {
  constexpr int DS = Stride<D>::value;
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double* dst = BK + (static_cast<long long>(J) * kB + dmma_target(lane, h, e)) * 2 * DS;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        dst[c] = acc[h][c][0][e];
        dst[DS + c] = acc[h][c][1][e];
      }
    }
}

}  // namespace fabm
