// fp64_mix_bench.cu — do the FP64 tensor-core path (DMMA m8n8k4) and the
// DFMA path share one pipe on B200?  Runs DMMA alone, DFMA alone, and both
// at once (split warps, and interleaved in one warp); if the mixed rate is
// above either alone, the bulk tile can issue both.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_mix_bench tools/fp64_mix_bench.cu
#include <cstdio>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

// mode 0: DMMA only; 1: DFMA only; 2: even warps DMMA, odd warps DFMA;
// 3: every warp interleaves NM DMMA and NF DFMA-groups per iteration
template <int MODE, int NM, int NF>
__global__ void __launch_bounds__(512, 1) mix(int iters, double* out) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2], f[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = i * 1e-3;
  const int warp = threadIdx.x >> 5;
  const bool do_m = MODE == 0 || MODE == 3 || (MODE == 2 && (warp & 1) == 0);
  const bool do_f = MODE == 1 || MODE == 3 || (MODE == 2 && (warp & 1) == 1);
  for (int it = 0; it < iters; ++it) {
    if (do_m) {
#pragma unroll
      for (int i = 0; i < NM; ++i) dmma(c[i & 7], a, b);
    }
    if (do_f) {
#pragma unroll
      for (int r = 0; r < NF; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] = fma(a, f[i], b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < 16; ++i) s += f[i];
  if (s == 1.2345) out[0] = s;
}

template <int MODE, int NM, int NF>
void run(const char* name, int warps, int iters) {
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mix<MODE, NM, NF><<<148, 32 * warps>>>(10, out);
  cudaEventRecord(e0);
  mix<MODE, NM, NF><<<148, 32 * warps>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  double mw = 0, fw = 0;  // warps doing each
  if (MODE == 0) mw = warps;
  if (MODE == 1) fw = warps;
  if (MODE == 2) { mw = (warps + 1) / 2; fw = warps / 2; }
  if (MODE == 3) { mw = warps; fw = warps; }
  const double fm = 148.0 * mw * iters * NM * 256.0;
  const double ff = 148.0 * fw * iters * NF * 16 * 32.0;
  const double s = ms * 1e-3;
  printf("%-28s warps=%2d  DMMA %.3e  DFMA %.3e  total %.3e FMA/s (%s)\n", name, warps, fm / s, ff / s,
         (fm + ff) / s, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  const int it = 20000;
  for (int w : {8, 16}) {
    run<0, 8, 1>("dmma only", w, it);
    run<1, 8, 1>("dfma only (16 chains)", w, it / 2);
    run<2, 8, 1>("split warps dmma|dfma", w, it / 2);
    run<3, 8, 1>("interleave 8 dmma + 16 dfma", w, it / 2);
    run<3, 8, 2>("interleave 8 dmma + 32 dfma", w, it / 2);
    run<3, 4, 2>("interleave 4 dmma + 32 dfma", w, it / 2);
  }
  return 0;
}
