// leader_bench.cu — cycles per step of the stepper's sequential chain in
// isolation (one thread), adding one ingredient per variant (dev tool).
#include <cstdint>
#include <cstdio>

struct Prm { double ha, ig, b0, a0, sigma, rho, beta, h; double y0[3]; };

__device__ __forceinline__ void lorenz(const double* s, double* f, const Prm& p) {
  const double x = s[0], y = s[1], z = s[2];
  f[0] = __dmul_rn(p.sigma, __dsub_rn(y, x));
  f[1] = __dsub_rn(__dmul_rn(x, __dsub_rn(p.rho, z)), y);
  f[2] = __dsub_rn(__dmul_rn(x, y), __dmul_rn(p.beta, z));
}

template <int V>
__global__ void chain(Prm p, long long steps, double* out, long long* cyc) {
  __shared__ double ring[64][8];
  __shared__ double hbuf[8][8];
  __shared__ uint64_t bar[64];
  if (threadIdx.x == 0)
    for (int i = 0; i < 64; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[i])));
  for (int i = threadIdx.x; i < 64; i += blockDim.x) hbuf[i / 8][i % 8] = 1e-3 * i;
  __syncthreads();
  if (threadIdx.x != 0) return;
  bool bad = false;
  __shared__ int flagw;
  double fc[3] = {1.0, 2.0, 3.0}, preP[3] = {0.1, 0.2, 0.3}, preC[3] = {0.1, 0.2, 0.3};
  long long t0 = clock64();
  for (long long n = 0; n < steps; ++n) {
    double hp[3] = {0, 0, 0};
    if (V >= 4) {
      const int s = n & 7;
      for (int c = 0; c < 3; ++c) hp[c] = hbuf[s][c];
    }
    const double t1 = (double)(n + 1) * p.h;
    double yP[3], fP[3], y1[3], f1[3];
    for (int c = 0; c < 3; ++c) yP[c] = __dadd_rn(__dmul_rn(fma(p.b0, fc[c], preP[c]), p.ha), p.y0[c]);
    lorenz(yP, fP, p);
    if (V >= 2 && V <= 4) {
      if (!(isfinite(fP[0]) && isfinite(fP[1]) && isfinite(fP[2]))) { out[1] = t1; break; }
    }
    if (V >= 5) bad |= !(isfinite(fP[0]) && isfinite(fP[1]) && isfinite(fP[2]));
    for (int c = 0; c < 3; ++c)
      y1[c] = __dadd_rn(__dmul_rn(__dadd_rn(fma(p.a0, fc[c], preC[c]), __dmul_rn(p.ig, fP[c])), p.ha), p.y0[c]);
    lorenz(y1, f1, p);
    if (V >= 2 && V <= 4) {
      if (!(isfinite(f1[0]) && isfinite(f1[1]) && isfinite(f1[2]))) { out[1] = t1; break; }
    }
    if (V >= 5) {
      bad |= !(isfinite(f1[0]) && isfinite(f1[1]) && isfinite(f1[2]));
      if ((n & 7) == 7 && bad) { out[1] = t1; break; }
    }
    if (V == 6 || V == 7 || V == 8) {
      const int ri = (n + 1) & 63;
      for (int c = 0; c < 3; ++c) { ring[ri][c] = y1[c]; ring[ri][4 + c] = f1[c]; }
    }
    if (V == 6 || V == 9)
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&bar[(n + 1) & 63])) : "memory");
    if (V == 8)
      asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&bar[(n + 1) & 63])) : "memory");
    if (V == 7) *(volatile int*)&flagw = (int)(n + 1);
    if (V == 10 || V == 11) {  // ring store every step; 11: release arrive once per 8 steps
      const int ri = (n + 1) & 63;
      for (int c = 0; c < 3; ++c) { ring[ri][c] = y1[c]; ring[ri][4 + c] = f1[c]; }
      if (V == 11 && ((n + 1) & 7) == 7)
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                         (unsigned)__cvta_generic_to_shared(&bar[((n + 1) >> 3) & 63])) : "memory");
    }
    if (V >= 3 && V <= 4) {
      const int ri = (n + 1) & 63;
      for (int c = 0; c < 3; ++c) { ring[ri][c] = y1[c]; ring[ri][4 + c] = f1[c]; }
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&bar[(n + 1) & 63]))
                   : "memory");
    }
    for (int c = 0; c < 3; ++c) {
      preP[c] = fma(1e-3, fc[c], hp[c] + 1e-3 * y1[c]);
      preC[c] = fma(1e-3, fc[c], hp[c] + 2e-3 * y1[c]);
      fc[c] = f1[c] * 1e-6 + 1e-3 * y1[c];
    }
  }
  long long t1c = clock64();
  out[0] = fc[0] + fc[1] + fc[2] + preP[0] + preC[1] + ((V >= 3 && V <= 11 && V != 5 && V != 9) ? ring[5][1] : 0.0) + flagw;
  cyc[V] = t1c - t0;
}

int main() {
  Prm p{0.01, 0.5, 0.99, 0.5, 10.0, 28.0, 8.0 / 3.0, 1e-4, {1.0, 1.0, 1.0}};
  double* out; long long* cyc;
  cudaMalloc(&out, 16); cudaMalloc(&cyc, 16 * 8);
  const long long steps = 100000;
  chain<1><<<1, 32>>>(p, steps, out, cyc);
  chain<2><<<1, 32>>>(p, steps, out, cyc);
  chain<3><<<1, 32>>>(p, steps, out, cyc);
  chain<4><<<1, 32>>>(p, steps, out, cyc);
  chain<5><<<1, 32>>>(p, steps, out, cyc);
  chain<6><<<1, 32>>>(p, steps, out, cyc);
  chain<7><<<1, 32>>>(p, steps, out, cyc);
  chain<8><<<1, 32>>>(p, steps, out, cyc);
  chain<9><<<1, 32>>>(p, steps, out, cyc);
  chain<10><<<1, 32>>>(p, steps, out, cyc);
  chain<11><<<1, 32>>>(p, steps, out, cyc);
  long long h[16];
  cudaMemcpy(h, cyc, 16 * 8, cudaMemcpyDeviceToHost);
  for (int v = 1; v <= 11; ++v) printf("variant %d: %.1f cycles/step\n", v, h[v] / (double)steps);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
