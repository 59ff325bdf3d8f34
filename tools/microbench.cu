// microbench.cu — latency probes that shape the stepper design (dev tool).
//   dependent DFMA / DADD / DMUL latency, LDS latency,
//   smem flag ping-pong between two warps (volatile poll),
//   mbarrier arrive -> try_wait wake-up latency.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ long long clk() { return clock64(); }

__global__ void fp64_latency(double* out, long long* cyc, double x, double y) {
  double a = x;
  long long t0 = clk();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) {
    a = fma(a, y, 1e-9);
    a = fma(a, y, 1e-9);
    a = fma(a, y, 1e-9);
    a = fma(a, y, 1e-9);
  }
  long long t1 = clk();
  double b = x;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) {
    b = __dadd_rn(b, y);
    b = __dadd_rn(b, y);
    b = __dadd_rn(b, y);
    b = __dadd_rn(b, y);
  }
  long long t2 = clk();
  double c = x;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) {
    c = __dmul_rn(c, y);
    c = __dmul_rn(c, y);
    c = __dmul_rn(c, y);
    c = __dmul_rn(c, y);
  }
  long long t3 = clk();
  out[0] = a + b + c;
  cyc[0] = (t1 - t0);
  cyc[1] = (t2 - t1);
  cyc[2] = (t3 - t2);
}

__global__ void lds_latency(long long* cyc, int* dummy) {
  __shared__ int buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i + 1) & 1023;
  __syncthreads();
  if (threadIdx.x != 0) return;
  int p = 0;
  long long t0 = clk();
#pragma unroll 1
  for (int i = 0; i < 4000; ++i) p = ((volatile int*)buf)[p];
  long long t1 = clk();
  dummy[0] = p;
  cyc[3] = t1 - t0;
}

// two warps ping-pong a counter through smem (volatile polling)
__global__ void pingpong(long long* cyc) {
  __shared__ int flag;
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0) return;
  volatile int* f = &flag;
  long long t0 = clk();
  for (int i = 0; i < 2000; ++i) {
    if (w == 0) {
      while (*f != 2 * i) {}
      *f = 2 * i + 1;
    } else {
      while (*f != 2 * i + 1) {}
      *f = 2 * i + 2;
    }
  }
  long long t1 = clk();
  if (w == 0) cyc[4] = t1 - t0;
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ bool trywait(uint64_t* b, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
               : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
  return ok;
}
__device__ __forceinline__ bool testwait(uint64_t* b, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
               : "=r"(ok) : "r"(sa(b)), "r"(par) : "memory");
  return ok;
}

// mbarrier ping-pong: warp 0 arrives on bar[0], warp 1 waits then arrives on bar[1]
template <bool TRY>
__global__ void mbar_pingpong(long long* cyc, int slot) {
  __shared__ uint64_t bar[2];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[1])));
  }
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0) return;
  long long t0 = clk();
  for (int i = 0; i < 2000; ++i) {
    const uint32_t par = i & 1;
    if (w == 0) {
      arrive(&bar[0]);
      if (TRY) { while (!trywait(&bar[1], par)) {} } else { while (!testwait(&bar[1], par)) {} }
    } else {
      if (TRY) { while (!trywait(&bar[0], par)) {} } else { while (!testwait(&bar[0], par)) {} }
      arrive(&bar[1]);
    }
  }
  long long t1 = clk();
  if (w == 0) cyc[slot] = t1 - t0;
}

int main() {
  double* out; long long* cyc; int* dummy;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 16 * 8); cudaMalloc(&dummy, 4);
  fp64_latency<<<1, 1>>>(out, cyc, 1.0, 1.0000001);
  lds_latency<<<1, 32>>>(cyc, dummy);
  pingpong<<<1, 64>>>(cyc);
  mbar_pingpong<true><<<1, 64>>>(cyc, 5);
  mbar_pingpong<false><<<1, 64>>>(cyc, 6);
  // warps on different SMSPs (0 and 1) vs same SMSP (0 and 4)
  long long h[16];
  cudaMemcpy(h, cyc, 16 * 8, cudaMemcpyDeviceToHost);
  printf("DFMA dep latency   %.2f cyc\n", h[0] / 4000.0);
  printf("DADD dep latency   %.2f cyc\n", h[1] / 4000.0);
  printf("DMUL dep latency   %.2f cyc\n", h[2] / 4000.0);
  printf("LDS  dep latency   %.2f cyc\n", h[3] / 4000.0);
  printf("smem flag pingpong %.2f cyc per one-way handoff\n", h[4] / 4000.0);
  printf("mbar try_wait pp   %.2f cyc per one-way handoff\n", h[5] / 4000.0);
  printf("mbar test_wait pp  %.2f cyc per one-way handoff\n", h[6] / 4000.0);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("clock attr %d kHz\n", clk_khz);
  return 0;
}
