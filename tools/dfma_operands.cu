// DFMA throughput vs operand pattern (register-bank / reuse effects). dev tool
#include <cstdio>
template <int MODE>
__global__ void k(double* out, int iters, double x) {
  double acc[24], w[8], f[3];
  for (int i = 0; i < 24; ++i) acc[i] = x + i;
  for (int i = 0; i < 8; ++i) w[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  for (int i = 0; i < 3; ++i) f[i] = 1.0 - 1e-9 * (threadIdx.x + 2 * i);
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {  // tile-like: acc[r][c] += w[r] * f[c], r-outer
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[r * 3 + c] = fma(w[r], f[c], acc[r * 3 + c]);
    } else if (MODE == 1) {  // c-outer
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int r = 0; r < 8; ++r) acc[r * 3 + c] = fma(w[r], f[c], acc[r * 3 + c]);
    } else {  // 2 register operands + immediate
#pragma unroll
      for (int i = 0; i < 24; ++i) acc[i] = fma(acc[i], w[i & 7], 1e-9);
    }
  }
  double s = 0;
  for (int i = 0; i < 24; ++i) s += acc[i];
  if (s == 1.2345) out[0] = s;
}
template <int M> void run(const char* name, int threads) {
  double* out; cudaMalloc(&out, 8);
  const int blocks = 148 * (1024 / threads), iters = 2000;
  k<M><<<blocks, threads>>>(out, 10, 1.0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); k<M><<<blocks, threads>>>(out, iters, 1.0); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%-28s threads/SM=1024: %.3e FMA/s\n", name, double(blocks) * threads * iters * 24 / (ms * 1e-3));
}
int main() {
  run<0>("3-reg w-reuse (r outer)", 256);
  run<1>("3-reg f-reuse (c outer)", 256);
  run<2>("2-reg + imm", 256);
  return 0;
}
