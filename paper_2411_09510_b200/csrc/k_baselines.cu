// Comparison codecs of the reference (mx/baselines.py) on sm_100a:
//
//   channel-wise INT  (mx/baselines.py:138-178)
//     K_ci_amax   per-channel max |x| (column reduction, atomicMax on the
//                 order-preserving f32 bit pattern), non-finite flag
//     K_ci_scale  scale = f16_RNE(amax / qmax) from the exact float64 quotient
//     K_ci_quant  level = round-half-even(x / scale) clamped to +-qmax,
//                 sign-magnitude code, 8 codes per thread -> `bits` bytes
//                 (LSB-first, mx/bitpack.py:22-34)
//     K_ci_dequant  level * scale in float64 -> f64 / f32 / bf16
//   TopK  (mx/baselines.py:95-135)
//     radix select of the K-th largest |x| key, 8 bits per pass, digit
//     choice on the device (no host round trip), then a stable compaction:
//     element i is kept iff key > T, or key == T and fewer than `take`
//     equal keys precede it (ties toward the lower index); kept entries are
//     written in index order as (u32 index, f16 value).
//
// Exactness: for bf16/f16/f32 inputs x / scale is rounded with an exact
// integer test against (k + 1/2) * scale (scale is an f16, k < 2^9: every
// product is an exact f32), which equals numpy's rint(float64(x / scale))
// because a float64 quotient of such operands can only be a .5 tie when the
// true quotient is one.  float64 inputs use float64 division + rint.
// These are HBM-bound byte/integer kernels; no tensor cores.
#include <cuda_fp16.h>
#include <string.h>

#include "mx_kernels.cuh"

namespace mxb {
namespace bl {

constexpr int kT = 256;

// value i of a typed array as f64 (exact) / f32 (exact for <= f32)
template <typename T>
__device__ __forceinline__ double ld64(const T* x, int64_t i) {
  if constexpr (std::is_same<T, double>::value) return x[i];
  else return (double)InTraits<T>::to_f32(x[i]);
}

// |x| as an order-preserving key (f32 bits for <= f32 inputs, f64 bits else);
// NaN/Inf are flagged by the caller.
template <typename T>
struct Key {
  using U = uint32_t;
  __device__ static U of_val(T v) { return __float_as_uint(fabsf(InTraits<T>::to_f32(v))); }
  __device__ static U of(const T* x, int64_t i) { return of_val(x[i]); }
  __device__ static bool bad(U k) { return k >= 0x7f800000u; }
};
template <>
struct Key<double> {
  using U = unsigned long long;
  __device__ static U of_val(double v) { return (U)__double_as_longlong(fabs(v)); }
  __device__ static U of(const double* x, int64_t i) { return of_val(x[i]); }
  __device__ static bool bad(U k) { return k >= 0x7ff0000000000000ull; }
};

// V consecutive values at p (16-byte aligned, V*sizeof(T) a multiple of 16)
template <typename T, int V>
__device__ __forceinline__ void ldv(const T* p, T (&out)[V]) {
  static_assert((V * sizeof(T)) % 16 == 0, "vector width");
#pragma unroll
  for (int i = 0; i < (int)(V * sizeof(T) / 16); ++i) {
    const uint4 w = __ldg(reinterpret_cast<const uint4*>(p) + i);
    memcpy(reinterpret_cast<char*>(out) + 16 * i, &w, 16);
  }
}

// float64 -> IEEE binary16 bits, round to nearest even, overflow -> inf
// (numpy's astype(float16), mx/baselines.py:124,153).
__device__ __forceinline__ uint16_t f64_to_f16_bits(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const uint16_t sign = (uint16_t)((b >> 48) & 0x8000u);
  const int e = (int)((b >> 52) & 0x7ff);
  unsigned long long m = b & 0xfffffffffffffull;
  if (e == 0x7ff) return sign | 0x7c00u | (m ? 0x200u : 0u);
  if (e == 0 && m == 0) return sign;
  const int E = e - 1023;  // v = 1.m * 2^E (f64 subnormals underflow to 0 below)
  if (E > 15) return sign | 0x7c00u;
  unsigned long long sig = m | (1ull << 52);  // 53-bit significand
  int shift;  // bits to drop from the 53-bit significand
  uint32_t ebits;
  if (E >= -14) {
    shift = 52 - 10;
    ebits = (uint32_t)(E + 15);
  } else {
    shift = 52 - 10 + (-14 - E);
    ebits = 0;
    if (shift > 63) return sign;
  }
  unsigned long long q = sig >> shift;
  const unsigned long long rem = sig & ((1ull << shift) - 1ull);
  const unsigned long long half = 1ull << (shift - 1);
  if (rem > half || (rem == half && (q & 1ull))) ++q;
  uint32_t r;
  if (ebits == 0) {
    r = (uint32_t)q;  // may carry into the smallest normal: still right
  } else {
    r = (ebits << 10) + ((uint32_t)q - 1024u);  // q in [1024, 2048]
    if (r >= 0x7c00u) r = 0x7c00u;
  }
  return sign | (uint16_t)r;
}

__device__ __forceinline__ double f16_bits_to_f64(uint16_t h) {
  return (double)__half2float(__ushort_as_half(h));  // exact
}

// ---------------------------------------------------------------------------
// channel-wise INT
// ---------------------------------------------------------------------------

// one thread: channel c, rows [r0, r0 + RB)
template <typename T, int RB>
__global__ void __launch_bounds__(kT) k_ci_amax(const T* __restrict__ x, int64_t rows, int64_t C,
                                               typename Key<T>::U* __restrict__ amax,
                                               unsigned long long* nonfinite) {
  using U = typename Key<T>::U;
  const int64_t c = blockIdx.x * (int64_t)kT + threadIdx.x;
  if (c >= C) return;
  const int64_t r0 = (int64_t)blockIdx.y * RB;
  const int64_t r1 = min(rows, r0 + RB);
  U m = 0;
  int64_t bad = -1;
  for (int64_t r = r0; r < r1; ++r) {
    const U k = Key<T>::of(x, r * C + c);
    if (Key<T>::bad(k)) {
      if (bad < 0) bad = r * C + c;
    } else {
      m = k > m ? k : m;
    }
  }
  if (m) atomicMax(amax + c, m);
  if (bad >= 0 && nonfinite) atomicMin(nonfinite, (unsigned long long)bad);
}

// C % 8 == 0, 16-B aligned rows: thread (tx, ty) owns channels
// 8*(32*bx + tx) .. +8 and rows by*RB + ty, +8, ...; column maxima reduced
// over ty in shared memory, one atomicMax per channel per block
template <typename T, int RB>
__global__ void __launch_bounds__(256) k_ci_amax_v(const T* __restrict__ x, int64_t rows,
                                                  int64_t C, typename Key<T>::U* __restrict__ amax,
                                                  unsigned long long* nonfinite) {
  using U = typename Key<T>::U;
  __shared__ U red[8][256];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t c0 = ((int64_t)blockIdx.x * 32 + tx) * 8;
  const bool live = c0 < C;
  U m[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) m[j] = 0;
  unsigned long long bad = ~0ull;
  if (live) {
    // the thread's RB/8 rows: every load in flight before the reduction
    constexpr int NR = RB / 8;
    const int64_t rb = (int64_t)blockIdx.y * RB + ty;
    T v[NR][8];
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const int64_t r = rb + 8 * i;
      if (r < rows) ldv<T, 8>(x + r * C + c0, v[i]);
    }
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const int64_t r = rb + 8 * i;
      if (r >= rows) break;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const U k = Key<T>::of_val(v[i][j]);
        if (Key<T>::bad(k)) bad = min(bad, (unsigned long long)(r * C + c0 + j));
        else m[j] = k > m[j] ? k : m[j];
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) red[ty][tx * 8 + j] = m[j];
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (c < C) {
    U r = red[0][threadIdx.x];
#pragma unroll
    for (int y = 1; y < 8; ++y) r = red[y][threadIdx.x] > r ? red[y][threadIdx.x] : r;
    if (r) atomicMax(amax + c, r);
  }
  if (bad != ~0ull && nonfinite) atomicMin(nonfinite, bad);
}

template <typename U>
__device__ __forceinline__ double key_value(U k);
template <>
__device__ __forceinline__ double key_value<uint32_t>(uint32_t k) {
  return (double)__uint_as_float(k);
}
template <>
__device__ __forceinline__ double key_value<unsigned long long>(unsigned long long k) {
  return __longlong_as_double((long long)k);
}

template <typename U>
__global__ void k_ci_scale(const U* __restrict__ amax, int64_t C, int qmax,
                           uint16_t* __restrict__ scales) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c < C) scales[c] = f64_to_f16_bits(__ddiv_rn(key_value<U>(amax[c]), (double)qmax));
}

// round-half-even(|x| / s) for an exact f32 |x| and an f16 scale s > 0;
// `rs` ~ 1/s (approximate: floor(mag*rs) is then off by at most one, and
// the exact products below fix it)
__device__ __forceinline__ int level_f32(float mag, float s, float rs, int qmax) {
  float k = floorf(mag * rs);
  k = fminf(k, (float)(2 * qmax + 2));
  if (k * s > mag) k -= 1.f;           // exact products (s: 11 bits, k < 2^9)
  if ((k + 1.f) * s <= mag) k += 1.f;
  const float half = (k + 0.5f) * s;
  int l = (int)k;
  l += (mag > half) | ((mag == half) & (l & 1));
  return min(l, qmax);
}

// Fast form: floor/fraction of the approximate quotient decide directly
// unless the fraction is within 1e-3 of one half (the approximation error is
// < 1e-4 for quotients up to 2^8), where the exact test above decides.
__device__ __forceinline__ int level_f32_fast(float mag, float s, float rs, int qmax) {
  const float r = mag * rs;
  const float fl = floorf(r);
  const float t = r - fl;
  int l;
  if (fabsf(t - 0.5f) > 1e-3f) l = (int)fl + (t > 0.5f ? 1 : 0);
  else l = level_f32(mag, s, rs, qmax);
  return min(l, qmax);
}

__device__ __forceinline__ float rcp_approx(float s) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(s));
  return r;
}

template <typename T>
__device__ __forceinline__ uint32_t ci_code(const T* x, int64_t i, uint16_t sb, int bits,
                                            int qmax) {
  if ((sb & 0x7fffu) == 0 || (sb & 0x7c00u) == 0x7c00u) return 0u;  // scale 0 or inf: level 0
  int l;
  bool neg;
  if constexpr (std::is_same<T, double>::value) {
    const double r = rint(__ddiv_rn(x[i], f16_bits_to_f64(sb)));
    const double c = fmin(fmax(r, (double)-qmax), (double)qmax);
    l = (int)fabs(c);
    neg = c < 0.0;
  } else {
    const float v = InTraits<T>::to_f32(x[i]);
    const float sf = __half2float(__ushort_as_half(sb));
    l = level_f32_fast(fabsf(v), sf, rcp_approx(sf), qmax);
    neg = v < 0.f && l > 0;
  }
  return (uint32_t)l | (neg ? (1u << (bits - 1)) : 0u);
}

// 8 flat-consecutive values per thread -> `bits` bytes of the code stream
template <typename T>
__global__ void __launch_bounds__(kT) k_ci_quant(const T* __restrict__ x, int64_t n, int64_t C,
                                                const uint16_t* __restrict__ scales, int bits,
                                                uint8_t* __restrict__ out) {
  const int64_t g = blockIdx.x * (int64_t)kT + threadIdx.x;
  const int64_t i0 = g * 8;
  if (i0 >= n) return;
  const int qmax = (1 << (bits - 1)) - 1;
  const int cnt = (int)min((int64_t)8, n - i0);
  unsigned long long w = 0;
  int64_t c = i0 % C;
  for (int j = 0; j < cnt; ++j) {
    w |= (unsigned long long)ci_code<T>(x, i0 + j, scales[c], bits, qmax) << (j * bits);
    if (++c == C) c = 0;
  }
  const int nb = (cnt * bits + 7) / 8;
  uint8_t* p = out + g * bits;
  for (int b = 0; b < nb; ++b) p[b] = (uint8_t)(w >> (8 * b));
}

// C % 8 == 0: a thread's 8 values share a row; values and their 8 scales
// arrive in vector loads; BITS is compile-time (constant shifts, one store)
template <typename T, int BITS>
__global__ void __launch_bounds__(kT) k_ci_quant_v(const T* __restrict__ x, int64_t n, int64_t C,
                                                  const uint16_t* __restrict__ scales,
                                                  uint8_t* __restrict__ out) {
  const int64_t g = blockIdx.x * (int64_t)kT + threadIdx.x;
  const int64_t i0 = g * 8;
  if (i0 >= n) return;
  constexpr int qmax = (1 << (BITS - 1)) - 1;
  T v[8];
  ldv<T, 8>(x + i0, v);
  const int64_t c0 = (n < 0x100000000ll) ? (int64_t)((uint32_t)i0 % (uint32_t)C) : i0 % C;
  const uint4 sw = __ldg(reinterpret_cast<const uint4*>(scales + c0));
  const uint32_t sv[4] = {sw.x, sw.y, sw.z, sw.w};
  unsigned long long w = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint16_t sb = (uint16_t)(sv[j >> 1] >> (16 * (j & 1)));
    w |= (unsigned long long)ci_code<T>(v + j, 0, sb, BITS, qmax) << (j * BITS);
  }
  uint8_t* p = out + g * BITS;
  if constexpr (BITS == 4) {
    *reinterpret_cast<uint32_t*>(p) = (uint32_t)w;
  } else if constexpr (BITS == 8) {
    *reinterpret_cast<unsigned long long*>(p) = w;
  } else if constexpr (BITS == 2) {
    *reinterpret_cast<uint16_t*>(p) = (uint16_t)w;
  } else {
#pragma unroll
    for (int b = 0; b < BITS; ++b) p[b] = (uint8_t)(w >> (8 * b));
  }
}

// C % 8 == 0, f32 / bf16 output: level * scale is exact in f32 (a 7-bit
// level times an f16 scale), so the float64 product of the reference rounds
// to the same f32 / bf16; vector loads of codes and scales, one 16/32-byte
// store per 8 values.
template <typename OutT, int BITS>
__global__ void __launch_bounds__(kT) k_ci_dequant_v(const uint8_t* __restrict__ codes,
                                                    const uint16_t* __restrict__ scales,
                                                    int64_t n, int64_t C, OutT* __restrict__ out) {
  const int64_t g = blockIdx.x * (int64_t)kT + threadIdx.x;
  const int64_t i0 = g * 8;
  if (i0 >= n) return;
  const uint8_t* p = codes + g * BITS;
  unsigned long long w = 0;
  if constexpr (BITS == 4) w = *reinterpret_cast<const uint32_t*>(p);
  else if constexpr (BITS == 8) w = *reinterpret_cast<const unsigned long long*>(p);
  else if constexpr (BITS == 2) w = *reinterpret_cast<const uint16_t*>(p);
  else {
#pragma unroll
    for (int b = 0; b < BITS; ++b) w |= (unsigned long long)p[b] << (8 * b);
  }
  const int64_t c0 = (n < 0x100000000ll) ? (int64_t)((uint32_t)i0 % (uint32_t)C) : i0 % C;
  const uint4 sw = __ldg(reinterpret_cast<const uint4*>(scales + c0));
  const uint32_t sv[4] = {sw.x, sw.y, sw.z, sw.w};
  constexpr uint32_t MM = (1u << (BITS - 1)) - 1u;
  float v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t code = (uint32_t)(w >> (j * BITS)) & ((1u << BITS) - 1u);
    const float sc = __half2float(__ushort_as_half((uint16_t)(sv[j >> 1] >> (16 * (j & 1)))));
    const float lev = (float)(code & MM);
    v[j] = ((code >> (BITS - 1)) ? -lev : lev) * sc;  // exact (or inf/nan, like numpy)
  }
  if constexpr (std::is_same<OutT, float>::value) {
    reinterpret_cast<float4*>(out + i0)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(out + i0)[1] = make_float4(v[4], v[5], v[6], v[7]);
  } else {
    uint4 o;
    o.x = pack2<__nv_bfloat16>(v[0], v[1]);
    o.y = pack2<__nv_bfloat16>(v[2], v[3]);
    o.z = pack2<__nv_bfloat16>(v[4], v[5]);
    o.w = pack2<__nv_bfloat16>(v[6], v[7]);
    *reinterpret_cast<uint4*>(out + i0) = o;
  }
}

template <typename OutT>
__global__ void __launch_bounds__(kT) k_ci_dequant(const uint8_t* __restrict__ codes,
                                                  const uint16_t* __restrict__ scales, int64_t n,
                                                  int64_t C, int bits, OutT* __restrict__ out) {
  const int64_t g = blockIdx.x * (int64_t)kT + threadIdx.x;
  const int64_t i0 = g * 8;
  if (i0 >= n) return;
  const int cnt = (int)min((int64_t)8, n - i0);
  const int nb = (cnt * bits + 7) / 8;
  unsigned long long w = 0;
  const uint8_t* p = codes + g * bits;
  for (int b = 0; b < nb; ++b) w |= (unsigned long long)p[b] << (8 * b);
  const uint32_t mmask = (1u << (bits - 1)) - 1u;
  int64_t c = i0 % C;
  for (int j = 0; j < cnt; ++j) {
    const uint32_t code = (uint32_t)(w >> (j * bits)) & ((1u << bits) - 1u);
    const double lev = (double)(code & mmask) * ((code >> (bits - 1)) ? -1.0 : 1.0);
    const double v = lev * f16_bits_to_f64(scales[c]);  // exact, or inf/nan like numpy
    if (++c == C) c = 0;
    if constexpr (std::is_same<OutT, double>::value) out[i0 + j] = v;
    else if constexpr (std::is_same<OutT, float>::value) out[i0 + j] = (float)v;
    else out[i0 + j] = __float2bfloat16_rn((float)v);
  }
}

// ---------------------------------------------------------------------------
// TopK
// ---------------------------------------------------------------------------

// select state in device memory: prefix, mask (key words), take, pass
template <typename U>
struct Sel {
  U prefix, mask;
  unsigned long long take;  // equal-to-threshold entries still to keep
  unsigned long long hist[256];
};

template <typename U>
__global__ void k_tk_init(Sel<U>* sel, unsigned long long k) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sel->hist[i] = 0;
  if (threadIdx.x == 0) {
    sel->prefix = 0;
    sel->mask = 0;
    sel->take = k;
  }
}

template <typename T>
__global__ void __launch_bounds__(kT) k_tk_hist(const T* __restrict__ x, int64_t n,
                                               Sel<typename Key<T>::U>* sel, int shift,
                                               unsigned long long* nonfinite, int vec, int agg) {
  using U = typename Key<T>::U;
  __shared__ unsigned int h[256];
  __shared__ unsigned int hw[kT / 32][256];  // per-warp bins (passes after the top one)
  for (int i = threadIdx.x; i < 256; i += kT) h[i] = 0;
  for (int i = threadIdx.x; i < 256 * (kT / 32); i += kT) (&hw[0][0])[i] = 0;
  __syncthreads();
  unsigned int* mine = hw[threadIdx.x >> 5];
  const U prefix = sel->prefix, mask = sel->mask;
  const int lane = threadIdx.x & 31;
  // warp tiles of 256 values, 8 consecutive per lane; every lane runs the
  // same trip count so __match_any_sync sees the full warp
  const int64_t ntiles = (n + 255) / 256;
  const int64_t nw = (int64_t)gridDim.x * (kT / 32);
  for (int64_t t = blockIdx.x * (int64_t)(kT / 32) + (threadIdx.x >> 5); t < ntiles; t += nw) {
    const int64_t i0 = t * 256 + lane * 8;
    T v[8];
    if (vec && i0 + 8 <= n) {
      ldv<T, 8>(x + i0, v);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = i0 + j < n ? x[i0 + j] : T(0);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const bool in = i0 + j < n;
      const U k = Key<T>::of_val(v[j]);
      if (nonfinite && in && Key<T>::bad(k)) atomicMin(nonfinite, (unsigned long long)(i0 + j));
      const uint32_t d = (in && (k & mask) == prefix) ? ((uint32_t)(k >> shift) & 255u) : 256u;
      if (agg) {  // top digit: few distinct values, heavy collisions
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        if (d < 256u && lane == __ffs(peers) - 1) atomicAdd(&h[d], (unsigned)__popc(peers));
      } else if (d < 256u) {
        atomicAdd(&mine[d], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += kT) {
    unsigned int t = h[i];
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) t += hw[w][i];
    if (t) atomicAdd(&sel->hist[i], (unsigned long long)t);
  }
}

// one warp: choose the digit where the descending cumulative count reaches
// `take`, fold it into the prefix, clear the histogram for the next pass
template <typename U>
__global__ void k_tk_select(Sel<U>* sel, int shift) {
  // one warp: lane l holds bins 255-8l .. 248-8l (descending); a warp scan of
  // the lane sums finds the lane, then the bin, where the count reaches take
  const int lane = threadIdx.x;
  unsigned long long c[8], tot = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    c[i] = sel->hist[255 - 8 * lane - i];
    tot += c[i];
  }
  unsigned long long incl = tot;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const unsigned long long take = sel->take, excl = incl - tot;
  const unsigned int hit = __ballot_sync(0xffffffffu, incl >= take);
  const int L = hit ? __ffs(hit) - 1 : 31;
  if (lane == L) {
    unsigned long long above = excl;
    int d = 255 - 8 * L;
    for (int i = 0; i < 8; ++i, --d) {
      if (above + c[i] >= take || d == 0) break;
      above += c[i];
    }
    sel->take = take - above;
    sel->prefix |= (U)d << shift;
    sel->mask |= (U)255 << shift;
  }
  __syncwarp();
  for (int i = lane; i < 256; i += 32) sel->hist[i] = 0;
}

constexpr int kPer = 16;               // elements per thread in the compaction
constexpr int kTile = kT * kPer;       // elements per block

// per-block counts of key > T and key == T
// the thread's kPer values (vector loads when whole and aligned)
template <typename T>
__device__ __forceinline__ int load_per(const T* x, int64_t i0, int64_t n, int vec, T (&v)[kPer]) {
  if (vec && i0 + kPer <= n) {
    ldv<T, kPer>(x + i0, v);
    return kPer;
  }
  const int cnt = (int)max((int64_t)0, min((int64_t)kPer, n - i0));
#pragma unroll
  for (int j = 0; j < kPer; ++j) v[j] = j < cnt ? x[i0 + j] : T(0);
  return cnt;
}

template <typename T>
__global__ void __launch_bounds__(kT) k_tk_count(const T* __restrict__ x, int64_t n,
                                                const Sel<typename Key<T>::U>* sel,
                                                unsigned long long* __restrict__ cnt, int vec) {
  using U = typename Key<T>::U;
  const U t = sel->prefix;
  const int64_t i0 = blockIdx.x * (int64_t)kTile + threadIdx.x * kPer;
  T v[kPer];
  const int m = load_per<T>(x, i0, n, vec, v);
  uint32_t gt = 0, eq = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const U k = Key<T>::of_val(v[j]);
    gt += (j < m) & (k > t);
    eq += (j < m) & (k == t);
  }
  __shared__ uint32_t sg[kT / 32], se[kT / 32];
  for (int o = 16; o; o >>= 1) {
    gt += __shfl_xor_sync(0xffffffffu, gt, o);
    eq += __shfl_xor_sync(0xffffffffu, eq, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sg[threadIdx.x >> 5] = gt;
    se[threadIdx.x >> 5] = eq;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t a = 0, b = 0;
    for (int w = 0; w < kT / 32; ++w) { a += sg[w]; b += se[w]; }
    cnt[2 * blockIdx.x] = a;
    cnt[2 * blockIdx.x + 1] = b;
  }
}

// exclusive scan of the (gt, eq) block counts in place, one block
__global__ void __launch_bounds__(1024) k_tk_scan(unsigned long long* cnt, int64_t nblocks) {
  __shared__ unsigned long long carry_g, carry_e;
  __shared__ unsigned long long wg[32], we[32];
  if (threadIdx.x == 0) carry_g = carry_e = 0;
  __syncthreads();
  for (int64_t base = 0; base < nblocks; base += 1024) {
    const int64_t i = base + threadIdx.x;
    unsigned long long g = i < nblocks ? cnt[2 * i] : 0, e = i < nblocks ? cnt[2 * i + 1] : 0;
    unsigned long long ig = g, ie = e;  // inclusive scan inside the warp
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long a = __shfl_up_sync(0xffffffffu, ig, o), b = __shfl_up_sync(0xffffffffu, ie, o);
      if ((threadIdx.x & 31) >= o) { ig += a; ie += b; }
    }
    if ((threadIdx.x & 31) == 31) { wg[threadIdx.x >> 5] = ig; we[threadIdx.x >> 5] = ie; }
    __syncthreads();
    if (threadIdx.x < 32) {
      unsigned long long a = wg[threadIdx.x], b = we[threadIdx.x];
      for (int o = 1; o < 32; o <<= 1) {
        unsigned long long c = __shfl_up_sync(0xffffffffu, a, o), d = __shfl_up_sync(0xffffffffu, b, o);
        if (threadIdx.x >= o) { a += c; b += d; }
      }
      wg[threadIdx.x] = a;
      we[threadIdx.x] = b;
    }
    __syncthreads();
    const int w = threadIdx.x >> 5;
    const unsigned long long pg = carry_g + (w ? wg[w - 1] : 0) + ig - g;
    const unsigned long long pe = carry_e + (w ? we[w - 1] : 0) + ie - e;
    if (i < nblocks) { cnt[2 * i] = pg; cnt[2 * i + 1] = pe; }
    __syncthreads();
    if (threadIdx.x == 0) { carry_g += wg[31]; carry_e += we[31]; }
    __syncthreads();
  }
}

template <typename T>
__device__ __forceinline__ uint16_t to_f16_bits(T v) {
  if constexpr (std::is_same<T, double>::value) return f64_to_f16_bits(v);
  else return __half_as_ushort(__float2half_rn(InTraits<T>::to_f32(v)));
}

template <typename T>
__global__ void __launch_bounds__(kT) k_tk_write(const T* __restrict__ x, int64_t n,
                                                const Sel<typename Key<T>::U>* sel,
                                                const unsigned long long* __restrict__ cnt,
                                                uint32_t* __restrict__ idx,
                                                uint16_t* __restrict__ val, int vec) {
  using U = typename Key<T>::U;
  const U t = sel->prefix;
  const unsigned long long take = sel->take;
  const int64_t i0 = blockIdx.x * (int64_t)kTile + threadIdx.x * kPer;
  T v[kPer];
  const int m = load_per<T>(x, i0, n, vec, v);
  uint32_t gt = 0, eq = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const U k = Key<T>::of_val(v[j]);
    gt += (j < m) & (k > t);
    eq += (j < m) & (k == t);
  }
  // block-exclusive prefix of (gt, eq) over threads
  __shared__ uint32_t sg[kT / 32], se[kT / 32];
  uint32_t ig = gt, ie = eq;
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t a = __shfl_up_sync(0xffffffffu, ig, o), b = __shfl_up_sync(0xffffffffu, ie, o);
    if ((threadIdx.x & 31) >= o) { ig += a; ie += b; }
  }
  if ((threadIdx.x & 31) == 31) { sg[threadIdx.x >> 5] = ig; se[threadIdx.x >> 5] = ie; }
  __syncthreads();
  uint32_t wg = 0, we = 0;
  for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) { wg += sg[w]; we += se[w]; }
  // block-local (32-bit) positions: the block's kept entries form one
  // contiguous output range starting at base; equal keys are kept while
  // fewer than `rem` equal keys of earlier blocks and threads precede them
  const unsigned long long e0 = cnt[2 * blockIdx.x + 1];
  const unsigned long long base = cnt[2 * blockIdx.x] + (e0 < take ? e0 : take);
  const uint32_t rem = e0 < take ? (uint32_t)min(take - e0, 0x7fffffffull) : 0u;
  uint32_t lg = wg + ig - gt, le = we + ie - eq;
  __shared__ uint32_t s_idx[kTile];
  __shared__ uint16_t s_val[kTile];
  __shared__ uint32_t s_cnt;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    if (j >= m) break;
    const U k = Key<T>::of_val(v[j]);
    const bool g1 = k > t, e1 = k == t;
    if (g1 || (e1 && le < rem)) {
      const uint32_t pos = lg + min(le, rem);
      s_idx[pos] = (uint32_t)(i0 + j);
      s_val[pos] = to_f16_bits<T>(v[j]);
    }
    lg += g1;
    le += e1;
  }
  if (threadIdx.x == kT - 1) s_cnt = lg + min(le, rem);  // the block's kept count
  __syncthreads();
  const uint32_t cntb = s_cnt;
  for (uint32_t q = threadIdx.x; q < cntb; q += kT) {
    idx[base + q] = s_idx[q];
    val[base + q] = s_val[q];
  }
}

template <typename OutT>
__global__ void k_tk_scatter(const uint32_t* __restrict__ idx, const uint16_t* __restrict__ val,
                             int64_t k, OutT* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= k) return;
  const float v = __half2float(__ushort_as_half(val[i]));
  if constexpr (std::is_same<OutT, __nv_bfloat16>::value) out[idx[i]] = __float2bfloat16_rn(v);
  else out[idx[i]] = (OutT)v;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

template <typename T>
void ci_compress(const T* x, int64_t rows, int64_t C, int bits, uint16_t* scales, uint8_t* codes,
                 void* ws, unsigned long long* nf, cudaStream_t st) {
  using U = typename Key<T>::U;
  U* amax = reinterpret_cast<U*>(ws);
  cudaMemsetAsync(amax, 0, C * sizeof(U), st);
  const bool vec = C % 8 == 0 && ((uintptr_t)x % 16) == 0;
  if (vec) {
    constexpr int RB = 64;
    dim3 g((unsigned)((C / 8 + 31) / 32), (unsigned)((rows + RB - 1) / RB));
    k_ci_amax_v<T, RB><<<g, 256, 0, st>>>(x, rows, C, amax, nf);
  } else {
    constexpr int RB = 32;
    dim3 g((unsigned)((C + kT - 1) / kT), (unsigned)((rows + RB - 1) / RB));
    k_ci_amax<T, RB><<<g, kT, 0, st>>>(x, rows, C, amax, nf);
  }
  k_ci_scale<U><<<(unsigned)((C + kT - 1) / kT), kT, 0, st>>>(amax, C, (1 << (bits - 1)) - 1,
                                                              scales);
  const int64_t n = rows * C, groups = (n + 7) / 8;
  const unsigned qg = (unsigned)((groups + kT - 1) / kT);
  if (vec && ((uintptr_t)scales % 16) == 0) {
    switch (bits) {
      case 2: k_ci_quant_v<T, 2><<<qg, kT, 0, st>>>(x, n, C, scales, codes); break;
      case 3: k_ci_quant_v<T, 3><<<qg, kT, 0, st>>>(x, n, C, scales, codes); break;
      case 4: k_ci_quant_v<T, 4><<<qg, kT, 0, st>>>(x, n, C, scales, codes); break;
      case 5: k_ci_quant_v<T, 5><<<qg, kT, 0, st>>>(x, n, C, scales, codes); break;
      case 6: k_ci_quant_v<T, 6><<<qg, kT, 0, st>>>(x, n, C, scales, codes); break;
      case 7: k_ci_quant_v<T, 7><<<qg, kT, 0, st>>>(x, n, C, scales, codes); break;
      default: k_ci_quant_v<T, 8><<<qg, kT, 0, st>>>(x, n, C, scales, codes); break;
    }
  } else
    k_ci_quant<T><<<(unsigned)((groups + kT - 1) / kT), kT, 0, st>>>(x, n, C, scales, bits, codes);
}

template <typename OutT>
void ci_decompress(const uint16_t* scales, const uint8_t* codes, int64_t n, int64_t C, int bits,
                   void* out, cudaStream_t st) {
  const int64_t groups = (n + 7) / 8;
  const unsigned gg = (unsigned)((groups + kT - 1) / kT);
  if constexpr (!std::is_same<OutT, double>::value) {
    if (C % 8 == 0 && ((uintptr_t)scales % 16) == 0 && ((uintptr_t)out % 32) == 0 &&
        ((uintptr_t)codes % 8) == 0) {
      OutT* o = reinterpret_cast<OutT*>(out);
      switch (bits) {
        case 2: k_ci_dequant_v<OutT, 2><<<gg, kT, 0, st>>>(codes, scales, n, C, o); return;
        case 3: k_ci_dequant_v<OutT, 3><<<gg, kT, 0, st>>>(codes, scales, n, C, o); return;
        case 4: k_ci_dequant_v<OutT, 4><<<gg, kT, 0, st>>>(codes, scales, n, C, o); return;
        case 5: k_ci_dequant_v<OutT, 5><<<gg, kT, 0, st>>>(codes, scales, n, C, o); return;
        case 6: k_ci_dequant_v<OutT, 6><<<gg, kT, 0, st>>>(codes, scales, n, C, o); return;
        case 7: k_ci_dequant_v<OutT, 7><<<gg, kT, 0, st>>>(codes, scales, n, C, o); return;
        default: k_ci_dequant_v<OutT, 8><<<gg, kT, 0, st>>>(codes, scales, n, C, o); return;
      }
    }
  }
  k_ci_dequant<OutT><<<gg, kT, 0, st>>>(codes, scales, n, C, bits, reinterpret_cast<OutT*>(out));
}

inline int64_t tk_blocks(int64_t n) { return (n + kTile - 1) / kTile; }

// 16-bit inputs (bf16 / f16): the 15-bit magnitude IS an order-preserving
// key, so one pass builds the full 32768-bin histogram (per-block bins in
// shared memory, non-zero bins flushed to global) and one block picks the
// threshold -- instead of two 8-bit radix passes over the data.
constexpr int kBins16 = 32768;

template <typename T>
__global__ void __launch_bounds__(1024) k_tk_hist16(const T* __restrict__ x, int64_t n, int vec,
                                                   unsigned int* __restrict__ ghist,
                                                   unsigned long long* nonfinite) {
  extern __shared__ unsigned int h16[];
  for (int i = threadIdx.x; i < kBins16; i += 1024) h16[i] = 0;
  __syncthreads();
  const uint32_t bad_key = std::is_same<T, __half>::value ? 0x7c00u : 0x7f80u;
  const int64_t stride = (int64_t)gridDim.x * 1024 * 8;
  for (int64_t i0 = ((int64_t)blockIdx.x * 1024 + threadIdx.x) * 8; i0 < n; i0 += stride) {
    T v[8];
    if (vec && i0 + 8 <= n) {
      ldv<T, 8>(x + i0, v);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = i0 + j < n ? x[i0 + j] : T(0);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (i0 + j >= n) break;
      const uint32_t k = (uint32_t)(*reinterpret_cast<const uint16_t*>(&v[j])) & 0x7fffu;
      if (k >= bad_key && nonfinite) atomicMin(nonfinite, (unsigned long long)(i0 + j));
      atomicAdd(&h16[k], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kBins16; i += 1024)
    if (h16[i]) atomicAdd(&ghist[i], h16[i]);
}

// one block: thread t owns bins 32767-32t .. 32736-32t (descending); a block
// scan of the thread sums finds the threshold bin; writes the f32-domain
// key of that bin and the number of equal keys to keep into *sel
template <typename T>
__global__ void __launch_bounds__(1024) k_tk_select16(const unsigned int* __restrict__ ghist,
                                                     Sel<uint32_t>* sel) {
  extern __shared__ unsigned int hs[];  // the histogram, loaded coalesced
  __shared__ unsigned long long wsum[32];
  __shared__ unsigned long long s_take;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  for (int i = t; i < kBins16 / 4; i += 1024)
    reinterpret_cast<uint4*>(hs)[i] = reinterpret_cast<const uint4*>(ghist)[i];
  __syncthreads();
  unsigned long long tot = 0;
#pragma unroll 8
  for (int i = 0; i < 32; ++i) tot += hs[kBins16 - 1 - 32 * t - ((i + lane) & 31)];
  unsigned long long incl = tot;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  if (t == 0) s_take = sel->take;
  __syncthreads();
  unsigned long long before = 0;
  for (int j = 0; j < w; ++j) before += wsum[j];
  const unsigned long long take = s_take;
  const unsigned long long excl = before + incl - tot;
  if (excl < take && excl + tot >= take) {  // exactly one thread
    unsigned long long above = excl;
    int b = kBins16 - 1 - 32 * t;
    for (int i = 0; i < 32; ++i, --b) {
      const unsigned int c = hs[b];
      if (above + c >= take || b == 0) break;
      above += c;
    }
    uint32_t key32;
    if constexpr (std::is_same<T, __half>::value)
      key32 = __float_as_uint(__half2float(__ushort_as_half((unsigned short)b)));
    else
      key32 = (uint32_t)b << 16;
    sel->prefix = key32;
    sel->mask = 0xffffffffu;
    sel->take = take - above;
  }
}



template <typename T>
void tk_compress(const T* x, int64_t n, int64_t k, uint32_t* idx, uint16_t* val, void* ws,
                 unsigned long long* nf, int low_shift, cudaStream_t st) {
  using U = typename Key<T>::U;
  Sel<U>* sel = reinterpret_cast<Sel<U>*>(ws);
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(
      reinterpret_cast<uint8_t*>(ws) + ((sizeof(Sel<U>) + 255) / 256) * 256);
  k_tk_init<U><<<1, 256, 0, st>>>(sel, (unsigned long long)k);  // graph-capturable
  const int vec = ((uintptr_t)x % 16) == 0 && (8 * sizeof(T)) % 16 == 0;
  static thread_local int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const unsigned hg = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((int64_t)sms * 8, (n + kT * 8 - 1) / (kT * 8)));
  if constexpr (sizeof(T) == 2) {
    unsigned int* gh = reinterpret_cast<unsigned int*>(
        reinterpret_cast<uint8_t*>(cnt) + ((16 * tk_blocks(n) + 255) / 256) * 256);
    cudaMemsetAsync(gh, 0, kBins16 * sizeof(unsigned int), st);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_tk_hist16<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kBins16 * 4);
      attr = true;
    }
    const unsigned g16 = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>((int64_t)sms, (n + 8191) / 8192));
    k_tk_hist16<T><<<g16, 1024, kBins16 * 4, st>>>(x, n, vec, gh, nf);
    static bool attr2 = false;
    if (!attr2) {
      cudaFuncSetAttribute(k_tk_select16<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kBins16 * 4);
      attr2 = true;
    }
    k_tk_select16<T><<<1, 1024, kBins16 * 4, st>>>(gh, reinterpret_cast<Sel<uint32_t>*>(sel));
  } else
  for (int shift = (int)(8 * sizeof(U)) - 8; shift >= low_shift; shift -= 8) {
    const bool top = shift == (int)(8 * sizeof(U)) - 8;
    k_tk_hist<T><<<hg, kT, 0, st>>>(x, n, sel, shift, top ? nf : nullptr, vec, top ? 1 : 0);
    k_tk_select<U><<<1, 32, 0, st>>>(sel, shift);
  }
  const int64_t nb = tk_blocks(n);
  k_tk_count<T><<<(unsigned)nb, kT, 0, st>>>(x, n, sel, cnt, vec);
  k_tk_scan<<<1, 1024, 0, st>>>(cnt, nb);
  k_tk_write<T><<<(unsigned)nb, kT, 0, st>>>(x, n, sel, cnt, idx, val, vec);
}

}  // namespace bl

// dtype codes as in mxb200.h
int64_t topk_workspace_bytes(int64_t n) {
  return ((int64_t)sizeof(bl::Sel<unsigned long long>) + 255) / 256 * 256 +
         (16 * bl::tk_blocks(n) + 255) / 256 * 256 + 4 * bl::kBins16 + 256;
}

void launch_chanint_compress(const void* x, int dtype, int64_t rows, int64_t C, int bits,
                             uint16_t* scales, uint8_t* codes, void* ws,
                             unsigned long long* nf, cudaStream_t st) {
  switch (dtype) {
    case 0: bl::ci_compress(static_cast<const float*>(x), rows, C, bits, scales, codes, ws, nf, st); break;
    case 1: bl::ci_compress(static_cast<const __half*>(x), rows, C, bits, scales, codes, ws, nf, st); break;
    case 2: bl::ci_compress(static_cast<const __nv_bfloat16*>(x), rows, C, bits, scales, codes, ws, nf, st); break;
    default: bl::ci_compress(static_cast<const double*>(x), rows, C, bits, scales, codes, ws, nf, st); break;
  }
}

void launch_chanint_decompress(const uint16_t* scales, const uint8_t* codes, int64_t n, int64_t C,
                               int bits, void* out, int out_dtype, cudaStream_t st) {
  switch (out_dtype) {
    case 0: bl::ci_decompress<float>(scales, codes, n, C, bits, out, st); break;
    case 2: bl::ci_decompress<__nv_bfloat16>(scales, codes, n, C, bits, out, st); break;
    default: bl::ci_decompress<double>(scales, codes, n, C, bits, out, st); break;
  }
}

void launch_topk_compress(const void* x, int dtype, int64_t n, int64_t k, uint32_t* idx,
                          uint16_t* val, void* ws, unsigned long long* nf, cudaStream_t st) {
  switch (dtype) {
    case 0: bl::tk_compress(static_cast<const float*>(x), n, k, idx, val, ws, nf, 0, st); break;
    case 1: bl::tk_compress(static_cast<const __half*>(x), n, k, idx, val, ws, nf, 8, st); break;
    case 2: bl::tk_compress(static_cast<const __nv_bfloat16*>(x), n, k, idx, val, ws, nf, 16, st); break;
    default: bl::tk_compress(static_cast<const double*>(x), n, k, idx, val, ws, nf, 0, st); break;
  }
}

void launch_topk_decompress(const uint32_t* idx, const uint16_t* val, int64_t k, int64_t n,
                            void* out, int out_dtype, cudaStream_t st) {
  const int es = out_dtype == 0 ? 4 : (out_dtype == 2 ? 2 : 8);
  cudaMemsetAsync(out, 0, n * es, st);
  if (k <= 0) return;
  const unsigned g = (unsigned)((k + 255) / 256);
  switch (out_dtype) {
    case 0: bl::k_tk_scatter<float><<<g, 256, 0, st>>>(idx, val, k, static_cast<float*>(out)); break;
    case 2: bl::k_tk_scatter<__nv_bfloat16><<<g, 256, 0, st>>>(idx, val, k, static_cast<__nv_bfloat16*>(out)); break;
    default: bl::k_tk_scatter<double><<<g, 256, 0, st>>>(idx, val, k, static_cast<double*>(out)); break;
  }
}

}  // namespace mxb
