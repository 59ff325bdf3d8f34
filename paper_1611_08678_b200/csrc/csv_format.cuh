// csv_format.cuh — the trajectory CSV writer on the GPU.
//
// Replaces write_trajectory_csv (reference cli.py:97-105):
//     header  "t,y0,..,y{d-1}\n"
//     row n   f"{t[n]:.17g}," + ",".join(f"{v:.17g}" for v in states[n]) + "\n"
// CPython's ".17g" is correctly rounded (dtoa mode 2, 17 digits, ties to
// even), with trailing zeros removed and Python's 'g' layout rules:
// fixed notation when -4 <= X < 17 (X = decimal exponent after rounding),
// else d.ddde+XX with at least two exponent digits; "inf", "-inf", "nan",
// "-0".  The device conversion below is exact integer arithmetic, so the
// bytes are identical to CPython's for every double (tests/test_gpu_csv.py
// checks random bit patterns over the whole exponent range, the ties and
// the trajectories).
//
// Work layout: one thread per row, a tile of rows per CTA.
//   pass 1 (csv_len_kernel)   row lengths and the tile's total
//   pass 2 (csv_scan_kernel)  exclusive scan of the tile totals (one CTA)
//   pass 3 (csv_write_kernel) rows formatted into shared memory at their
//                             in-tile offsets, then the tile's bytes are
//                             stored contiguously (word stores) at its offset
// The output is byte work: 1 conversion per value in each of passes 1 and 3
// and ~22 output bytes per value; states are read twice (8 B per value).
#pragma once
#include <cstdint>

namespace fabm_csv {

constexpr int kFieldMax = 24;    // "-1.2345678901234567e-308"
constexpr int kMaxTileRows = 256;  // rows per CTA (one thread each; blockDim.x, a multiple of 32)

__device__ const unsigned long long kPow5[28] = {
    1ull, 5ull, 25ull, 125ull, 625ull, 3125ull, 15625ull, 78125ull, 390625ull, 1953125ull, 9765625ull,
    48828125ull, 244140625ull, 1220703125ull, 6103515625ull, 30517578125ull, 152587890625ull,
    762939453125ull, 3814697265625ull, 19073486328125ull, 95367431640625ull, 476837158203125ull,
    2384185791015625ull, 11920928955078125ull, 59604644775390625ull, 298023223876953125ull,
    1490116119384765625ull, 7450580596923828125ull};

constexpr unsigned long long kE16 = 10000000000000000ull;   // 10^16
constexpr unsigned long long kE17 = 100000000000000000ull;  // 10^17

// ---------------------------------------------------------------- bigint
// Rare path only (|v| < 1e-11 or |v| >= 1e17): little-endian 32-bit limbs.
constexpr int kLimbs = 36;  // 1152 bits: m * 5^340 (843 bits), m << 971 (1024 bits)
struct Big {
  uint32_t w[kLimbs];
  int n;  // limbs in use (w[n..] == 0)
};

__device__ __forceinline__ void big_set(Big& a, unsigned long long x) {
  for (int i = 0; i < kLimbs; ++i) a.w[i] = 0;
  a.w[0] = static_cast<uint32_t>(x);
  a.w[1] = static_cast<uint32_t>(x >> 32);
  a.n = a.w[1] ? 2 : 1;
}
__device__ __forceinline__ void big_mul32(Big& a, uint32_t m) {
  unsigned long long carry = 0;
  for (int i = 0; i < a.n; ++i) {
    const unsigned long long p = static_cast<unsigned long long>(a.w[i]) * m + carry;
    a.w[i] = static_cast<uint32_t>(p);
    carry = p >> 32;
  }
  if (carry) a.w[a.n++] = static_cast<uint32_t>(carry);
}
__device__ __forceinline__ void big_pow5(Big& a, int k) {  // a *= 5^k
  while (k >= 13) { big_mul32(a, 1220703125u); k -= 13; }
  if (k > 0) big_mul32(a, static_cast<uint32_t>(kPow5[k]));
}
__device__ __forceinline__ void big_shl(Big& a, int s) {
  const int ws = s >> 5, bs = s & 31;
  const int n = a.n + ws + 1;
  for (int i = n - 1; i >= 0; --i) {
    const int j = i - ws;
    const uint32_t hi = (j >= 0 && j < kLimbs) ? a.w[j] : 0u;
    const uint32_t lo = (j - 1 >= 0 && j - 1 < kLimbs) ? a.w[j - 1] : 0u;
    a.w[i] = bs ? (hi << bs) | (lo >> (32 - bs)) : hi;
  }
  a.n = n;
  while (a.n > 1 && a.w[a.n - 1] == 0) --a.n;
}
__device__ __forceinline__ uint32_t big_bit(const Big& a, int b) {
  return (b >> 5) < a.n ? (a.w[b >> 5] >> (b & 31)) & 1u : 0u;
}
__device__ __forceinline__ int big_cmp(const Big& a, const Big& b) {
  const int n = a.n > b.n ? a.n : b.n;
  for (int i = n - 1; i >= 0; --i) {
    const uint32_t x = i < a.n ? a.w[i] : 0u, y = i < b.n ? b.w[i] : 0u;
    if (x != y) return x < y ? -1 : 1;
  }
  return 0;
}
__device__ __forceinline__ void big_sub(Big& a, const Big& b) {  // a -= b, a >= b
  long long borrow = 0;
  for (int i = 0; i < a.n; ++i) {
    const long long d = static_cast<long long>(a.w[i]) - (i < b.n ? b.w[i] : 0u) - borrow;
    a.w[i] = static_cast<uint32_t>(d);
    borrow = d < 0;
  }
  while (a.n > 1 && a.w[a.n - 1] == 0) --a.n;
}
// r = a >> s
__device__ __forceinline__ void big_shr_into(const Big& a, int s, Big& r) {
  const int ws = s >> 5, bs = s & 31;
  for (int i = 0; i < kLimbs; ++i) {
    const int j = i + ws;
    const uint32_t lo = j < a.n ? a.w[j] : 0u;
    const uint32_t hi = j + 1 < a.n ? a.w[j + 1] : 0u;
    r.w[i] = bs ? (lo >> bs) | (hi << (32 - bs)) : lo;
  }
  r.n = a.n - ws > 1 ? a.n - ws : 1;
  while (r.n > 1 && r.w[r.n - 1] == 0) --r.n;
}
// bits [s, s+64) of a
__device__ __forceinline__ unsigned long long big_bits64(const Big& a, int s) {
  unsigned long long r = 0;
  for (int b = 63; b >= 0; --b) r = (r << 1) | big_bit(a, s + b);
  return r;
}
// any bit below position s set?
__device__ __forceinline__ bool big_sticky(const Big& a, int s) {
  const int ws = s >> 5, bs = s & 31;
  for (int i = 0; i < ws && i < a.n; ++i)
    if (a.w[i]) return true;
  return bs && ws < a.n && (a.w[ws] & ((1u << bs) - 1u));
}

// ------------------------------------------------------ exact scaling
// q = m * 2^e * 10^k rounded to an integer, ties to even; sets *fl to
// floor(q) (for the range check).  m < 2^53.
__device__ __forceinline__ unsigned long long round_half_even(unsigned long long q, bool half, bool sticky) {
  return q + ((half && (sticky || (q & 1ull))) ? 1ull : 0ull);
}

__device__ __noinline__ unsigned long long scale_big(unsigned long long m, int e, int k, unsigned long long* fl) {
  Big a;
  big_set(a, m);
  if (k >= 0) {
    big_pow5(a, k);
    const int s = e + k;
    if (s >= 0) {  // q is an integer (< 2^60): no rounding
      const unsigned long long q = big_bits64(a, 0) << s;
      *fl = q;
      return q;
    }
    const int sh = -s;
    const unsigned long long q = big_bits64(a, sh);
    *fl = q;
    return round_half_even(q, big_bit(a, sh - 1) != 0, big_sticky(a, sh - 1));
  }
  // k < 0: q = (m << (e + k)) / 5^(-k), long division (q < 2^60)
  Big d;
  big_set(d, 1);
  big_pow5(d, -k);
  const int s = e + k;
  big_shl(a, s > 0 ? s : 0);
  Big r;  // r = a >> 60, then the low 60 bits are shifted in one at a time
  big_shr_into(a, 60, r);
  unsigned long long q = 0;
  for (int b = 59; b >= 0; --b) {
    big_shl(r, 1);
    r.w[0] |= big_bit(a, b);
    q <<= 1;
    if (big_cmp(r, d) >= 0) {
      big_sub(r, d);
      q |= 1ull;
    }
  }
  *fl = q;
  big_shl(r, 1);  // compare 2r with the divisor
  const int c = big_cmp(r, d);
  return q + ((c > 0 || (c == 0 && (q & 1ull))) ? 1ull : 0ull);
}

__device__ __forceinline__ unsigned long long scale(unsigned long long m, int e, int k, unsigned long long* fl) {
  if (k >= 0 && k <= 27) {
    // M = m * 5^k < 2^116 as (hi, lo)
    const unsigned long long p5 = kPow5[k];
    const unsigned long long lo = m * p5, hi = __umul64hi(m, p5);
    const int s = e + k;
    if (s >= 0) {
      if (s < 64 && hi == 0 && (lo >> (63 - s)) == 0) {
        *fl = lo << s;
        return lo << s;
      }
      return scale_big(m, e, k, fl);
    }
    const int sh = -s;
    if (sh >= 64 + 52) return scale_big(m, e, k, fl);
    unsigned long long q;
    bool half, sticky;
    if (sh < 64) {
      q = (lo >> sh) | (sh ? (hi << (64 - sh)) : 0ull);
      if ((hi >> sh) != 0 && sh < 64) return scale_big(m, e, k, fl);  // q >= 2^64: estimate far off
      half = sh ? ((lo >> (sh - 1)) & 1ull) : false;
      sticky = sh > 1 ? (lo & ((1ull << (sh - 1)) - 1ull)) != 0 : false;
    } else {
      const int t = sh - 64;
      q = hi >> t;
      half = t ? ((hi >> (t - 1)) & 1ull) : (lo >> 63);
      sticky = t ? (((hi & ((1ull << (t - 1)) - 1ull)) != 0) || lo != 0) : ((lo << 1) != 0);
    }
    *fl = q;
    return round_half_even(q, half, sticky);
  }
  return scale_big(m, e, k, fl);
}

// 17 correctly rounded significant digits of v = m * 2^e > 0:
// v ~= D * 10^(X - 16), 10^16 <= D < 10^17
__device__ __forceinline__ void decimal17(unsigned long long m, int e, unsigned long long* D, int* X) {
  const int p = e + 63 - __clzll(static_cast<long long>(m));  // 2^p <= v < 2^(p+1)
  // floor(p * log10(2)) for |p| < 1700 (X is this or one more)
  int x = (p >= 0) ? (p * 78913) >> 18 : -((-p * 78913 + (1 << 18) - 1) >> 18);
  unsigned long long fl = 0;
  unsigned long long q = scale(m, e, 16 - x, &fl);
  if (fl >= kE17) {  // the estimate was one low
    x += 1;
    q = scale(m, e, 16 - x, &fl);
  }
  if (q >= kE17) {  // 99999999999999999.5.. rounded up to 10^17
    q = kE16;
    x += 1;
  }
  *D = q;
  *X = x;
}

// the field f"{v:.17g}" into out (no terminator); returns its length
__device__ __forceinline__ int format_g17(double v, char* out) {
  const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
  const bool neg = (bits >> 63) != 0;
  const int ef = static_cast<int>((bits >> 52) & 0x7ff);
  const unsigned long long frac = bits & ((1ull << 52) - 1ull);
  int n = 0;
  if (ef == 0x7ff) {
    if (frac) { out[0] = 'n'; out[1] = 'a'; out[2] = 'n'; return 3; }
    if (neg) out[n++] = '-';
    out[n++] = 'i'; out[n++] = 'n'; out[n++] = 'f';
    return n;
  }
  if (neg) out[n++] = '-';
  if (ef == 0 && frac == 0) { out[n++] = '0'; return n; }
  const unsigned long long m = ef ? (frac | (1ull << 52)) : frac;
  const int e = ef ? ef - 1075 : -1074;
  unsigned long long D;
  int X;
  decimal17(m, e, &D, &X);
  // 17 digits as 1 + 8 + 8: one 64-bit split, then 32-bit arithmetic
  char dg[17];
  const unsigned long long top = D / 100000000ull;  // < 10^9
  uint32_t lo = static_cast<uint32_t>(D - top * 100000000ull);
  uint32_t mid = static_cast<uint32_t>(top % 100000000ull);
  dg[0] = static_cast<char>('0' + static_cast<uint32_t>(top / 100000000ull));
#pragma unroll
  for (int i = 8; i >= 1; --i) {
    const uint32_t q = mid / 10u;
    dg[i] = static_cast<char>('0' + (mid - 10u * q));
    mid = q;
  }
#pragma unroll
  for (int i = 16; i >= 9; --i) {
    const uint32_t q = lo / 10u;
    dg[i] = static_cast<char>('0' + (lo - 10u * q));
    lo = q;
  }
  int nd = 17;
  while (nd > 1 && dg[nd - 1] == '0') --nd;
  if (X >= -4 && X < 17) {
    if (X >= 0) {
      for (int i = 0; i <= X; ++i) out[n++] = i < nd ? dg[i] : '0';
      if (nd > X + 1) {
        out[n++] = '.';
        for (int i = X + 1; i < nd; ++i) out[n++] = dg[i];
      }
    } else {
      out[n++] = '0';
      out[n++] = '.';
      for (int i = 0; i < -X - 1; ++i) out[n++] = '0';
      for (int i = 0; i < nd; ++i) out[n++] = dg[i];
    }
    return n;
  }
  out[n++] = dg[0];
  if (nd > 1) {
    out[n++] = '.';
    for (int i = 1; i < nd; ++i) out[n++] = dg[i];
  }
  out[n++] = 'e';
  out[n++] = X < 0 ? '-' : '+';
  const int ax = X < 0 ? -X : X;
  if (ax >= 100) out[n++] = static_cast<char>('0' + ax / 100);
  out[n++] = static_cast<char>('0' + (ax / 10) % 10);
  out[n++] = static_cast<char>('0' + ax % 10);
  return n;
}

__device__ __forceinline__ double row_time(const double* t, double h, long long row) {
  return t ? t[row] : static_cast<double>(row) * h;  // GridSpec.times(): arange(N+1) * h, core.py:179-181
}

// ------------------------------------------------------------- kernels
// pass 1: row lengths (bytes incl. commas and newline) and tile totals
__global__ void __launch_bounds__(kMaxTileRows) csv_len_kernel(const double* __restrict__ states,
                                                            const double* __restrict__ t, double h,
                                                            long long n_rows, int dim, int* __restrict__ row_len,
                                                            long long* __restrict__ tile_len) {
  __shared__ long long red[kMaxTileRows / 32];
  const long long row = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  int len = 0;
  if (row < n_rows) {
    char buf[kFieldMax];
    len = format_g17(row_time(t, h, row), buf) + dim + 1;
    const double* s = states + row * dim;
    for (int c = 0; c < dim; ++c) len += format_g17(s[c], buf);
    row_len[row] = len;
  }
  long long v = len;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long s = 0;
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) s += red[i];
    tile_len[blockIdx.x] = s;
  }
}

// pass 2: exclusive scan of the tile totals in place (one CTA of 1024);
// tile_len[n_tiles] receives the grand total
__global__ void __launch_bounds__(1024) csv_scan_kernel(long long* tile_len, long long n_tiles) {
  __shared__ long long part[1024];
  const int tid = threadIdx.x;
  const long long per = (n_tiles + 1023) / 1024;
  const long long b0 = tid * per, b1 = (b0 + per < n_tiles) ? b0 + per : n_tiles;
  long long s = 0;
  for (long long i = b0; i < b1; ++i) s += tile_len[i];
  part[tid] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // Hillis-Steele inclusive scan
    const long long x = tid >= off ? part[tid - off] : 0;
    __syncthreads();
    part[tid] += x;
    __syncthreads();
  }
  long long run = part[tid] - s;  // exclusive prefix of this thread's range
  for (long long i = b0; i < b1; ++i) {
    const long long x = tile_len[i];
    tile_len[i] = run;
    run += x;
  }
  if (tid == 1023) tile_len[n_tiles] = part[1023];
}

// pass 3: format the tile into shared memory and store it at its offset.
// Dynamic smem: the tile's bytes (<= blockDim.x * (dim + 1) * (kFieldMax + 1)).
__global__ void __launch_bounds__(kMaxTileRows) csv_write_kernel(const double* __restrict__ states,
                                                              const double* __restrict__ t, double h,
                                                              long long n_rows, int dim,
                                                              const int* __restrict__ row_len,
                                                              const long long* __restrict__ tile_off,
                                                              char* __restrict__ out) {
  extern __shared__ __align__(16) char tile[];
  __shared__ int wsum[kMaxTileRows / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const long long row = static_cast<long long>(blockIdx.x) * blockDim.x + tid;
  const int len = row < n_rows ? row_len[row] : 0;
  // block exclusive scan of the row lengths
  int incl = len;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < warp; ++w) base += wsum[w];
  int total = 0;
  for (int w = 0; w < nwarps; ++w) total += wsum[w];
  const int off = base + incl - len;
  if (row < n_rows) {
    char* p = tile + off;
    int n = format_g17(row_time(t, h, row), p);
    const double* s = states + row * dim;
    for (int c = 0; c < dim; ++c) {
      p[n++] = ',';
      n += format_g17(s[c], p + n);
    }
    p[n++] = '\n';
  }
  __syncthreads();
  // contiguous store of [0, total) at out + tile_off[b]: head bytes up to a
  // 4-byte boundary of the destination, then words, then the tail
  char* dst = out + tile_off[blockIdx.x];
  int head = static_cast<int>((4 - (reinterpret_cast<uintptr_t>(dst) & 3)) & 3);
  head = head < total ? head : total;
  if (tid < head) dst[tid] = tile[tid];
  const int nw = (total - head) >> 2;
  uint32_t* dw = reinterpret_cast<uint32_t*>(dst + head);
  for (int i = tid; i < nw; i += blockDim.x) {
    const int b = head + 4 * i;
    const uint32_t w = static_cast<uint32_t>(static_cast<unsigned char>(tile[b])) |
                       (static_cast<uint32_t>(static_cast<unsigned char>(tile[b + 1])) << 8) |
                       (static_cast<uint32_t>(static_cast<unsigned char>(tile[b + 2])) << 16) |
                       (static_cast<uint32_t>(static_cast<unsigned char>(tile[b + 3])) << 24);
    dw[i] = w;
  }
  const int tail0 = head + 4 * nw;
  if (tid < total - tail0) dst[tail0 + tid] = tile[tail0 + tid];
}

constexpr size_t kMaxTileBytes = 200 * 1024;  // dynamic smem budget of the write pass

// rows per tile for this dim (0: dim too large for one row per thread)
inline int tile_rows(int dim) {
  const size_t row_max = static_cast<size_t>(dim + 1) * (kFieldMax + 1);
  size_t r = kMaxTileBytes / row_max;
  r = r > kMaxTileRows ? kMaxTileRows : (r & ~static_cast<size_t>(31));
  return static_cast<int>(r);
}
inline size_t tile_smem_bytes(int dim, int rows) {
  return static_cast<size_t>(rows) * static_cast<size_t>(dim + 1) * (kFieldMax + 1);
}

}  // namespace fabm_csv
