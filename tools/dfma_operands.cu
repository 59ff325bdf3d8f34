// DFMA throughput vs operand pattern (register-bank / reuse effects). dev tool
#include <cstdio>
template <int MODE>
__global__ void k(double* out, int iters, double x) {
  double acc[12], w[4], f[3];
  for (int i = 0; i < 12; ++i) acc[i] = x + i;
  for (int i = 0; i < 4; ++i) w[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  for (int i = 0; i < 3; ++i) f[i] = 1.0 - 1e-9 * (threadIdx.x + 2 * i);
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {  // r-outer: w[r] reused across c
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[r * 3 + c] = fma(w[r], f[c], acc[r * 3 + c]);
    } else if (MODE == 1) {  // c-outer: f[c] reused across r
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[r * 3 + c] = fma(w[r], f[c], acc[r * 3 + c]);
    } else {  // 2-operand: acc = fma(acc, w, const)
#pragma unroll
      for (int i = 0; i < 12; ++i) acc[i] = fma(acc[i], w[i & 3], 1e-9);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = __shfl_xor_sync(0xffffffff, w[i], 1) ;  // keep w live/variant
  }
  double s = 0;
  for (int i = 0; i < 12; ++i) s += acc[i];
  if (s == 1.2345) out[0] = s;
}
template <int M> void run(const char* name) {
  double* out; cudaMalloc(&out, 8);
  const int blocks = 148 * 4, threads = 256, iters = 4000;
  k<M><<<blocks, threads>>>(out, 10, 1.0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<M><<<blocks, threads>>>(out, iters, 1.0); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%s: %.3e FMA/s\n", name, double(blocks) * threads * iters * 12 / (ms * 1e-3));
}
int main() { run<0>("w-reuse (r outer)"); run<1>("f-reuse (c outer)"); run<2>("2-operand"); return 0; }
