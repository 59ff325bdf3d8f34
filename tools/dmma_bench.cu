// dmma_bench.cu — FP64 tensor-core (mma.sync m8n8k4 f64) throughput vs the
// DFMA path on this GPU: decides whether the bulk tile belongs on DMMA
// (BASELINE north star: "tensor cores only if ncu shows DMMA beating FMA").
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_bench tools/dmma_bench.cu
#include <cstdio>

template <int NACC>
__global__ void __launch_bounds__(512, 1) dmma_loop(int iters, double* out) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 1.2345) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    dmma_loop<8><<<148, 32 * warps>>>(10, out);
    cudaEventRecord(e0);
    dmma_loop<8><<<148, 32 * warps>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fma = 148.0 * warps * iters * 8 * 256.0;  // 8x8x4 = 256 FMA per mma
    printf("DMMA m8n8k4: %2d warps/SM  %.3e FMA/s = %.2f TFLOP/s (%s)\n", warps, fma / (ms * 1e-3),
           2 * fma / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
