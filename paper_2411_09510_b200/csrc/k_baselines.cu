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
  __device__ static U of(const T* x, int64_t i) {
    return __float_as_uint(fabsf(InTraits<T>::to_f32(x[i])));
  }
  __device__ static bool bad(U k) { return k >= 0x7f800000u; }
};
template <>
struct Key<double> {
  using U = unsigned long long;
  __device__ static U of(const double* x, int64_t i) {
    return (U)__double_as_longlong(fabs(x[i]));
  }
  __device__ static bool bad(U k) { return k >= 0x7ff0000000000000ull; }
};

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

// round-half-even(|x| / s) for an exact f32 |x| and an f16 scale s > 0
__device__ __forceinline__ int level_f32(float mag, float s, int qmax) {
  float k = floorf(mag * __frcp_rn(s));
  k = fminf(fmaxf(k, 0.f), (float)(2 * qmax + 2));
  if (k * s > mag) k -= 1.f;           // exact products (s: 11 bits, k < 2^9)
  if ((k + 1.f) * s <= mag) k += 1.f;
  const float half = (k + 0.5f) * s;
  int l = (int)k;
  if (mag > half || (mag == half && (l & 1))) ++l;
  return min(l, qmax);
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
    l = level_f32(fabsf(v), __half2float(__ushort_as_half(sb)), qmax);
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
                                               unsigned long long* nonfinite) {
  using U = typename Key<T>::U;
  __shared__ unsigned int h[256];
  for (int i = threadIdx.x; i < 256; i += kT) h[i] = 0;
  __syncthreads();
  const U prefix = sel->prefix, mask = sel->mask;
  const int64_t stride = (int64_t)gridDim.x * kT;
  for (int64_t i = blockIdx.x * (int64_t)kT + threadIdx.x; i < n; i += stride) {
    const U k = Key<T>::of(x, i);
    if (nonfinite && Key<T>::bad(k)) atomicMin(nonfinite, (unsigned long long)i);
    if ((k & mask) == prefix) atomicAdd(&h[(uint32_t)(k >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += kT)
    if (h[i]) atomicAdd(&sel->hist[i], (unsigned long long)h[i]);
}

// one warp: choose the digit where the descending cumulative count reaches
// `take`, fold it into the prefix, clear the histogram for the next pass
template <typename U>
__global__ void k_tk_select(Sel<U>* sel, int shift) {
  if (threadIdx.x == 0) {
    unsigned long long take = sel->take, above = 0;
    int d = 255;
    for (; d > 0; --d) {
      if (above + sel->hist[d] >= take) break;
      above += sel->hist[d];
    }
    sel->take = take - above;
    sel->prefix |= (U)d << shift;
    sel->mask |= (U)255 << shift;
  }
  __syncwarp();
  for (int i = threadIdx.x; i < 256; i += 32) sel->hist[i] = 0;
}

constexpr int kPer = 16;               // elements per thread in the compaction
constexpr int kTile = kT * kPer;       // elements per block

// per-block counts of key > T and key == T
template <typename T>
__global__ void __launch_bounds__(kT) k_tk_count(const T* __restrict__ x, int64_t n,
                                                const Sel<typename Key<T>::U>* sel,
                                                unsigned long long* __restrict__ cnt) {
  using U = typename Key<T>::U;
  const U t = sel->prefix;
  const int64_t i0 = blockIdx.x * (int64_t)kTile + threadIdx.x * kPer;
  uint32_t gt = 0, eq = 0;
  for (int j = 0; j < kPer; ++j) {
    if (i0 + j >= n) break;
    const U k = Key<T>::of(x, i0 + j);
    gt += k > t;
    eq += k == t;
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
__device__ __forceinline__ uint16_t to_f16_bits(const T* x, int64_t i) {
  if constexpr (std::is_same<T, double>::value) return f64_to_f16_bits(x[i]);
  else return __half_as_ushort(__float2half_rn(InTraits<T>::to_f32(x[i])));
}

template <typename T>
__global__ void __launch_bounds__(kT) k_tk_write(const T* __restrict__ x, int64_t n,
                                                const Sel<typename Key<T>::U>* sel,
                                                const unsigned long long* __restrict__ cnt,
                                                uint32_t* __restrict__ idx,
                                                uint16_t* __restrict__ val) {
  using U = typename Key<T>::U;
  const U t = sel->prefix;
  const unsigned long long take = sel->take;
  const int64_t i0 = blockIdx.x * (int64_t)kTile + threadIdx.x * kPer;
  uint32_t gt = 0, eq = 0;
  for (int j = 0; j < kPer; ++j) {
    if (i0 + j >= n) break;
    const U k = Key<T>::of(x, i0 + j);
    gt += k > t;
    eq += k == t;
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
  unsigned long long pg = cnt[2 * blockIdx.x] + wg + ig - gt;
  unsigned long long pe = cnt[2 * blockIdx.x + 1] + we + ie - eq;
  for (int j = 0; j < kPer; ++j) {
    const int64_t i = i0 + j;
    if (i >= n) break;
    const U k = Key<T>::of(x, i);
    bool keep = false;
    if (k > t) {
      keep = true;
    } else if (k == t) {
      keep = pe < take;
    }
    if (keep) {
      const unsigned long long pos = pg + (pe < take ? pe : take);
      idx[pos] = (uint32_t)i;
      val[pos] = to_f16_bits<T>(x, i);
    }
    pg += k > t;
    pe += k == t;
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
  constexpr int RB = 32;
  dim3 g((unsigned)((C + kT - 1) / kT), (unsigned)((rows + RB - 1) / RB));
  k_ci_amax<T, RB><<<g, kT, 0, st>>>(x, rows, C, amax, nf);
  k_ci_scale<U><<<(unsigned)((C + kT - 1) / kT), kT, 0, st>>>(amax, C, (1 << (bits - 1)) - 1,
                                                              scales);
  const int64_t n = rows * C, groups = (n + 7) / 8;
  k_ci_quant<T><<<(unsigned)((groups + kT - 1) / kT), kT, 0, st>>>(x, n, C, scales, bits, codes);
}

template <typename OutT>
void ci_decompress(const uint16_t* scales, const uint8_t* codes, int64_t n, int64_t C, int bits,
                   void* out, cudaStream_t st) {
  const int64_t groups = (n + 7) / 8;
  k_ci_dequant<OutT><<<(unsigned)((groups + kT - 1) / kT), kT, 0, st>>>(
      codes, scales, n, C, bits, reinterpret_cast<OutT*>(out));
}

inline int64_t tk_blocks(int64_t n) { return (n + kTile - 1) / kTile; }

template <typename T>
void tk_compress(const T* x, int64_t n, int64_t k, uint32_t* idx, uint16_t* val, void* ws,
                 unsigned long long* nf, int low_shift, cudaStream_t st) {
  using U = typename Key<T>::U;
  Sel<U>* sel = reinterpret_cast<Sel<U>*>(ws);
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(
      reinterpret_cast<uint8_t*>(ws) + ((sizeof(Sel<U>) + 255) / 256) * 256);
  k_tk_init<U><<<1, 256, 0, st>>>(sel, (unsigned long long)k);  // graph-capturable
  static thread_local int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const unsigned hg = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((int64_t)sms * 8, (n + kT * 8 - 1) / (kT * 8)));
  for (int shift = (int)(8 * sizeof(U)) - 8; shift >= low_shift; shift -= 8) {
    k_tk_hist<T><<<hg, kT, 0, st>>>(x, n, sel, shift, shift == (int)(8 * sizeof(U)) - 8 ? nf : nullptr);
    k_tk_select<U><<<1, 32, 0, st>>>(sel, shift);
  }
  const int64_t nb = tk_blocks(n);
  k_tk_count<T><<<(unsigned)nb, kT, 0, st>>>(x, n, sel, cnt);
  k_tk_scan<<<1, 1024, 0, st>>>(cnt, nb);
  k_tk_write<T><<<(unsigned)nb, kT, 0, st>>>(x, n, sel, cnt, idx, val);
}

}  // namespace bl

// dtype codes as in mxb200.h
int64_t topk_workspace_bytes(int64_t n) {
  return ((int64_t)sizeof(bl::Sel<unsigned long long>) + 255) / 256 * 256 +
         16 * bl::tk_blocks(n) + 256;
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
