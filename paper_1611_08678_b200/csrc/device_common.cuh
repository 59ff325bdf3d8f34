// device_common.cuh — sm_100a primitives shared by the fabm kernels:
// memory-ordering helpers (acquire/release at CTA and GPU scope), mbarrier
// wrappers, the device watchdog clock and the rhs library.
//
// The rhs expressions reproduce the Python evaluation order of the
// reference factories (systems.py:26-123) and of the BASELINE systems in
// paper_1611_08678_b200/systems.py with explicit round-to-nearest
// intrinsics, so nvcc never contracts them into FMAs (NumPy does none).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fabm {

enum System : int {
  SYS_CONSTANT = 0,
  SYS_POWER_LAW = 1,
  SYS_LINEAR = 2,
  SYS_HINDMARSH_ROSE = 3,
  SYS_LORENZ = 4,
  SYS_CHEN = 5,
  SYS_ROSSLER = 6,
  SYS_FINANCIAL = 7,
};

constexpr int kMaxDim = 4;
constexpr int kMaxParams = 16;

// padded row stride of the f history in HBM / smem
template <int D> struct Stride { static constexpr int value = D == 1 ? 1 : (D == 2 ? 2 : 4); };

// ---------------------------------------------------------------- rounding
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// ---------------------------------------------------------------- addresses
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- ordering
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// system scope: flags shared with peer GPUs over NVLink (sharded engine)
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed_sys(const int* p) {
  int v;
  asm volatile("ld.relaxed.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire_cta_smem(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_smem(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_volatile_smem(const int* p) {
  return *reinterpret_cast<const volatile int*>(p);
}
__device__ __forceinline__ void st_volatile_smem(int* p, int v) {
  *reinterpret_cast<volatile int*>(p) = v;
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// arrive with release semantics at CTA scope; the state token is discarded
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// arrive only where `pred` holds, without a branch (keeps a warp converged)
__device__ __forceinline__ void mbar_arrive_if(uint64_t* bar, bool pred) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "@p mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n\t}" ::"r"(smem_u32(bar)),
      "r"(static_cast<uint32_t>(pred))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_if_u32(uint32_t bar, bool pred) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "@p mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n\t}" ::"r"(bar),
      "r"(static_cast<uint32_t>(pred))
      : "memory");
}
// non-blocking probe of phase completion, acquire semantics on success
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// potentially-blocking probe (hardware suspend up to an implementation limit)
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// blocking probe with a suspend-time hint: the thread sleeps in hardware until
// the phase completes or ~hint_ns elapse (no spinning on the SYNCS unit)
__device__ __forceinline__ bool mbar_wait_hint(uint64_t* bar, uint32_t parity, uint32_t hint_ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(hint_ns)
      : "memory");
  return ok != 0;
}

// ---------------------------------------------------------------- clock
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------- finiteness
// core.py:50-59: a finite sum proves the vector finite; the elementwise check
// settles the rare non-finite sum.  Both branches agree with isfinite(all).
template <int D>
__device__ __forceinline__ bool all_finite(const double* v) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < D; ++i) ok = ok && isfinite(v[i]);
  return ok;
}

// ---------------------------------------------------------------- rhs
// Each specialisation evaluates f(t, y) in the Python operator order of its
// host factory (left-to-right, ** before *, no FMA contraction).
template <int SYS, int D> struct Rhs;

// systems.py:26-36 — f = value
template <int D> struct Rhs<SYS_CONSTANT, D> {
  __device__ __forceinline__ static void eval(double, const double*, double* f, const double* p) {
#pragma unroll
    for (int i = 0; i < D; ++i) f[i] = p[i];
  }
};

// systems.py:39-61 — (coef * t ** expo if t > 0.0 else 0.0,)
template <> struct Rhs<SYS_POWER_LAW, 1> {
  __device__ __forceinline__ static void eval(double t, const double*, double* f, const double* p) {
    f[0] = t > 0.0 ? mul_rn(p[0], pow(t, p[1])) : 0.0;
  }
};

// systems.py:64-73 — lam * y
template <int D> struct Rhs<SYS_LINEAR, D> {
  __device__ __forceinline__ static void eval(double, const double* y, double* f, const double* p) {
#pragma unroll
    for (int i = 0; i < D; ++i) f[i] = mul_rn(p[0], y[i]);
  }
};

// systems.py:101-123 — Hindmarsh–Rose; params {a,b,c,d,r,s,x_rest,i_ext}
template <> struct Rhs<SYS_HINDMARSH_ROSE, 3> {
  __device__ __forceinline__ static void eval(double, const double* s, double* f, const double* p) {
    const double x = s[0], y = s[1], z = s[2];
    const double x2 = mul_rn(x, x);
    // y - a * x2 * x + b * x2 - z + i_ext
    double f0 = sub_rn(y, mul_rn(mul_rn(p[0], x2), x));
    f0 = add_rn(f0, mul_rn(p[1], x2));
    f0 = sub_rn(f0, z);
    f0 = add_rn(f0, p[7]);
    // c - d * x2 - y
    const double f1 = sub_rn(sub_rn(p[2], mul_rn(p[3], x2)), y);
    // r * (s * (x - x_rest) - z)
    const double f2 = mul_rn(p[4], sub_rn(mul_rn(p[5], sub_rn(x, p[6])), z));
    f[0] = f0; f[1] = f1; f[2] = f2;
  }
};

// Lorenz: (sigma * (y - x), x * (rho - z) - y, x * y - beta * z)
template <> struct Rhs<SYS_LORENZ, 3> {
  __device__ __forceinline__ static void eval(double, const double* s, double* f, const double* p) {
    const double x = s[0], y = s[1], z = s[2];
    f[0] = mul_rn(p[0], sub_rn(y, x));
    f[1] = sub_rn(mul_rn(x, sub_rn(p[1], z)), y);
    f[2] = sub_rn(mul_rn(x, y), mul_rn(p[2], z));
  }
};

// Chen: (a * (y - x), (c - a) * x - x * z + c * y, x * y - b * z)
template <> struct Rhs<SYS_CHEN, 3> {
  __device__ __forceinline__ static void eval(double, const double* s, double* f, const double* p) {
    const double x = s[0], y = s[1], z = s[2];
    const double a = p[0], b = p[1], c = p[2];
    f[0] = mul_rn(a, sub_rn(y, x));
    f[1] = add_rn(sub_rn(mul_rn(sub_rn(c, a), x), mul_rn(x, z)), mul_rn(c, y));
    f[2] = sub_rn(mul_rn(x, y), mul_rn(b, z));
  }
};

// Rossler: (-y - z, x + a * y, b + z * (x - c))
template <> struct Rhs<SYS_ROSSLER, 3> {
  __device__ __forceinline__ static void eval(double, const double* s, double* f, const double* p) {
    const double x = s[0], y = s[1], z = s[2];
    f[0] = sub_rn(-y, z);
    f[1] = add_rn(x, mul_rn(p[0], y));
    f[2] = add_rn(p[1], mul_rn(z, sub_rn(x, p[2])));
  }
};

// financial: (z + (y - a) * x, 1.0 - b * y - x * x, -x - c * z)
template <> struct Rhs<SYS_FINANCIAL, 3> {
  __device__ __forceinline__ static void eval(double, const double* s, double* f, const double* p) {
    const double x = s[0], y = s[1], z = s[2];
    f[0] = add_rn(z, mul_rn(sub_rn(y, p[0]), x));
    f[1] = sub_rn(sub_rn(1.0, mul_rn(p[1], y)), mul_rn(x, x));
    f[2] = sub_rn(-x, mul_rn(p[2], z));
  }
};

}  // namespace fabm
