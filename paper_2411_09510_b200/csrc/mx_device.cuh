// Device-side MX arithmetic shared by the quantise / dequant-sum / requant
// kernels.  Every routine here is exact (bit-identical to the float64
// reference mx/codec.py:127-188): no fast-math, no FTZ, no FMA contraction on
// the rounding adds.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace mxb {

// Element + scale parameters of one SchemeDescriptor, precomputed on the host.
struct Fmt {
  int bits;     // b = 1 + exponent_bits + mantissa_bits
  int y;        // mantissa bits (INTn: n-1 magnitude bits)
  int lo;       // lowest normal exponent 1-bias (float); y for INT (all "subnormal")
  int emax;     // floor(log2(grid max))             mx/formats.py:208-212
  int kbits;    // scale exponent bits k
  int sbias;    // 2^(k-1)-1                          mx/formats.py:116-118
  int s_min;    // 1-sbias                            mx/formats.py:120-123
  int s_max;    // 2^k-1-sbias                        mx/formats.py:125-128
  int block;    // B
  int s_fast_lo;   // block exponents for which grid*2^s is exactly an f32
  int s_fast_hi;   // (decode = one FFMA into the fp32 accumulator)
  uint32_t ovf32;  // fraction threshold of the overshoot bump (mx/codec.py:159)
  uint64_t ovf64;
  float gmax;
  double gmax64;
};

__device__ __forceinline__ float pow2f(int e) {  // exact, e in [-149, 127]
  return e >= -126 ? __uint_as_float((uint32_t)(e + 127) << 23)
                   : __uint_as_float(1u << (e + 149));
}
__device__ __forceinline__ double pow2d(int e) {  // exact, e in [-1022, 1023]
  return __longlong_as_double((long long)(e + 1023) << 52);
}

// ---------------------------------------------------------------------------
// Shared exponent (mx/codec.py:152-161): floor(log2 amax) - emax, +1 when the
// scaled max still exceeds grid max, clamped.  `ab` = |amax| bits, finite >0.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int shared_exp32(uint32_t ab, const Fmt& f) {
  int E = (int)(ab >> 23);
  uint32_t frac = ab & 0x7fffffu;
  int flog;
  if (E == 0) {  // subnormal amax: normalise
    int lz = __clz(frac);
    flog = (31 - lz) - 149;
    frac = (frac << (lz - 8)) & 0x7fffffu;
  } else {
    flog = E - 127;
  }
  int s = flog - f.emax + (frac > f.ovf32 ? 1 : 0);
  return min(max(s, f.s_min), f.s_max);
}

__device__ __forceinline__ int shared_exp64(uint64_t ab, const Fmt& f) {
  int E = (int)(ab >> 52);
  uint64_t frac = ab & 0xfffffffffffffull;
  int flog;
  if (E == 0) {
    int lz = __clzll(frac);
    flog = (63 - lz) - 1074;
    frac = (frac << (lz - 11)) & 0xfffffffffffffull;
  } else {
    flog = E - 1023;
  }
  int s = flog - f.emax + (frac > f.ovf64 ? 1 : 0);
  return min(max(s, f.s_min), f.s_max);
}

// ---------------------------------------------------------------------------
// Element encoders: x is the block-scaled value v * 2^-s (exact except for
// f32 underflow below 2^-126, which is far below every grid midpoint).
// Result: sign << (b-1) | grid index, ties to the even index, saturating
// (mx/codec.py:127-137,163-168).
// ---------------------------------------------------------------------------

// Generic closed form: q = max(floor(log2 a), lo); quantum 2^(q-y);
// r = RNE(a / quantum) via the magic-add; index = r + ((q-lo) << y).
__device__ __forceinline__ uint32_t encode_gen(float x, const Fmt& f) {
  uint32_t sign = __float_as_uint(x) >> 31;
  float a = fminf(fabsf(x), f.gmax);
  int E = (int)(__float_as_uint(a) >> 23);
  int q = max(E - 127, f.lo);
  int qe = q - f.y;
  float C = __uint_as_float(((uint32_t)(qe + 150) << 23) | 0x400000u);  // 1.5*2^(qe+23)
  float sum = __fadd_rn(a, C);
  uint32_t idx = (__float_as_uint(sum) - __float_as_uint(C)) + ((uint32_t)(q - f.lo) << f.y);
  if (f.y == 0) {
    // zero-mantissa formats: the offset (q-lo) can be odd, so RNE on r is not
    // "ties to the even grid index"; redo ties explicitly.
    float d = __fsub_rn(a, __fsub_rn(sum, C));
    if (fabsf(d) == pow2f(qe - 1)) {
      uint32_t lo_idx = d > 0.f ? idx : idx - 1u;
      idx = lo_idx + (lo_idx & 1u);
    }
  }
  return (sign << (f.bits - 1)) | idx;
}

__device__ __forceinline__ uint32_t encode_gen(double x, const Fmt& f) {
  uint32_t sign = (uint32_t)((unsigned long long)__double_as_longlong(x) >> 63);
  double a = fmin(fabs(x), f.gmax64);
  int E = (int)((unsigned long long)__double_as_longlong(a) >> 52);
  int q = max(E - 1023, f.lo);
  int qe = q - f.y;
  double C = __longlong_as_double(((long long)(qe + 1075) << 52) | (1ll << 51));
  double sum = __dadd_rn(a, C);
  uint32_t idx = (uint32_t)(__double_as_longlong(sum) - __double_as_longlong(C)) +
                 ((uint32_t)(q - f.lo) << f.y);
  if (f.y == 0) {
    double d = __dsub_rn(a, __dsub_rn(sum, C));
    if (fabs(d) == pow2d(qe - 1)) {
      uint32_t lo_idx = d > 0. ? idx : idx - 1u;
      idx = lo_idx + (lo_idx & 1u);
    }
  }
  return (sign << (f.bits - 1)) | idx;
}

// Hardware OCP conversions (RNE + satfinite).  For E2M1/E2M3/E3M2 the OCP
// code point layout equals the reference's sign|e|m grid index
// (mx/formats.py:199-204) and none of them has Inf/NaN codes.
__device__ __forceinline__ uint32_t cvt_e2m1x2(float lo, float hi) {
  uint32_t r;
  asm("{.reg .b8 t; cvt.rn.satfinite.e2m1x2.f32 t, %1, %2; cvt.u32.u8 %0, t;}"
      : "=r"(r) : "f"(hi), "f"(lo));
  return r & 0xffu;  // lo value in bits 0-3, hi value in bits 4-7
}
__device__ __forceinline__ uint32_t cvt_e2m3x2(float lo, float hi) {
  uint16_t r;
  asm("cvt.rn.satfinite.e2m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;  // lo code in byte 0, hi code in byte 1 (6 bits each)
}
__device__ __forceinline__ uint32_t cvt_e3m2x2(float lo, float hi) {
  uint16_t r;
  asm("cvt.rn.satfinite.e3m2x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

// ---------------------------------------------------------------------------
// Decoders (mx/codec.py:175-188): value = (-1)^sign * grid[idx] * 2^s.
// ---------------------------------------------------------------------------

// M * 2^E rounded once to f32 (RNE, subnormals kept, overflow -> inf).
__device__ __forceinline__ float ldexp_exact(uint32_t M, int E) {
  float m = (float)M;  // exact, M < 2^8
  if (E >= -126) {
    if (E <= 127) return m * pow2f(E);
    return (m * pow2f(127)) * pow2f(min(E - 127, 127));
  }
  return (m * pow2f(max(E + 100, -126))) * pow2f(-100);
}

__device__ __forceinline__ void split_code(uint32_t code, const Fmt& f, uint32_t& M, int& E,
                                           uint32_t& sign) {
  sign = code >> (f.bits - 1);
  uint32_t idx = code & ((1u << (f.bits - 1)) - 1u);
  int ef = (int)(idx >> f.y);
  uint32_t mant = idx & ((1u << f.y) - 1u);
  M = ef ? (mant | (1u << f.y)) : mant;
  E = max(ef, 1) + f.lo - 1 - f.y;
}

// Generic decode to f32; `s` is the unbiased block exponent; zero-scale
// blocks (stored code 0) decode to +-0 like grid*0.0 in the reference.
__device__ __forceinline__ float decode_gen(uint32_t code, int s, bool zero_block,
                                            const Fmt& f) {
  uint32_t M, sign;
  int E;
  split_code(code, f, M, E, sign);
  float v = zero_block ? 0.f : ldexp_exact(M, E + s);
  return __uint_as_float(__float_as_uint(v) | (sign << 31));
}

__device__ __forceinline__ double decode_gen64(uint32_t code, int s, bool zero_block,
                                               const Fmt& f) {
  uint32_t M, sign;
  int E;
  split_code(code, f, M, E, sign);
  double v = zero_block ? 0. : (double)M * pow2d(E + s);
  return __longlong_as_double(__double_as_longlong(v) | ((long long)sign << 63));
}

// FP4 E2M1 fast decode.  (mag << 22) as f32 bits is grid*2^-126 for every
// magnitude code (the e=0 code lands in the f32 subnormal range exactly like
// the E2M1 subnormal), so value = (raw * P) * F with P*F = 2^(126+s) split so
// that the first product is exact and the second rounds once.
struct E2M1Scale {
  float P, F;
};
__device__ __forceinline__ E2M1Scale e2m1_scale(int stored, int sbias) {
  E2M1Scale r;
  if (stored == 0) {
    r.P = pow2f(126);
    r.F = 0.f;
  } else {
    int s = stored - sbias;
    if (s <= 127) {
      r.P = pow2f(126);
      r.F = pow2f(s);
    } else {
      r.P = pow2f(127);
      r.F = pow2f(s - 1);
    }
  }
  return r;
}
__device__ __forceinline__ float e2m1_raw(uint32_t word, int nib) {
  // nibble `nib` of `word` -> sign bit 31, magnitude bits 22..24
  uint32_t t = word >> (4 * nib);
  return __uint_as_float(((t & 7u) << 22) | ((t & 8u) << 28));
}

// ---------------------------------------------------------------------------
// Loads of 8 consecutive values -> f32 (and f64 for the generic path)
// ---------------------------------------------------------------------------
template <typename T>
struct InTraits;
template <>
struct InTraits<float> {
  static constexpr int kBytes = 4;
  __device__ static float to_f32(float v) { return v; }
};
template <>
struct InTraits<__half> {
  static constexpr int kBytes = 2;
  __device__ static float to_f32(__half v) { return __half2float(v); }
};
template <>
struct InTraits<__nv_bfloat16> {
  static constexpr int kBytes = 2;
  __device__ static float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
};

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// 8 values starting at x[g]; `valid` = how many of them exist (0..8).
template <typename T>
__device__ __forceinline__ void load8(const T* __restrict__ x, int64_t g, int valid, float v[8]) {
  if (valid == 8) {
    if constexpr (sizeof(T) == 2) {
      uint4 w = ldg_stream(x + g);
      uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if constexpr (std::is_same<T, __nv_bfloat16>::value) {
          v[2 * i] = __uint_as_float(u[i] << 16);
          v[2 * i + 1] = __uint_as_float(u[i] & 0xffff0000u);
        } else {
          __half2 h = *reinterpret_cast<__half2*>(&u[i]);
          float2 ff = __half22float2(h);
          v[2 * i] = ff.x;
          v[2 * i + 1] = ff.y;
        }
      }
    } else {
      uint4 a = ldg_stream(x + g);
      uint4 b = ldg_stream(x + g + 4);
      v[0] = __uint_as_float(a.x); v[1] = __uint_as_float(a.y);
      v[2] = __uint_as_float(a.z); v[3] = __uint_as_float(a.w);
      v[4] = __uint_as_float(b.x); v[5] = __uint_as_float(b.y);
      v[6] = __uint_as_float(b.z); v[7] = __uint_as_float(b.w);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = i < valid ? InTraits<T>::to_f32(x[g + i]) : 0.f;
  }
}

// Output conversion of the fp32 accumulator (one RNE rounding).
template <typename T>
__device__ __forceinline__ T from_f32(float v);
template <>
__device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half from_f32<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

template <typename T>
__device__ __forceinline__ uint32_t pack2(float lo, float hi);
template <>
__device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float lo, float hi) {
  __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);  // F2FP.BF16.F32.PACK_AB, RNE
  return *reinterpret_cast<uint32_t*>(&p);
}
template <>
__device__ __forceinline__ uint32_t pack2<__half>(float lo, float hi) {
  __half2 p = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&p);
}

template <typename T>
__device__ __forceinline__ void store8(T* __restrict__ out, int64_t g, int valid, const float v[8]) {
  if (valid == 8) {
    if constexpr (sizeof(T) == 2) {
      uint4 u = make_uint4(pack2<T>(v[0], v[1]), pack2<T>(v[2], v[3]), pack2<T>(v[4], v[5]),
                           pack2<T>(v[6], v[7]));
      *reinterpret_cast<uint4*>(out + g) = u;
    } else {
      *reinterpret_cast<float4*>(out + g) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(out + g + 4) = make_float4(v[4], v[5], v[6], v[7]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < valid) out[g + i] = from_f32<T>(v[i]);
  }
}

// k-bit scale code `blk` of a packed scale stream (LSB-first).
template <bool CG = false>
__device__ __forceinline__ uint8_t ld_byte(const uint8_t* p) {
  if constexpr (CG) return __ldcg(p);
  else return *p;
}

// k-bit scale code of block blk (CG: the stream was written in this kernel)
template <bool CG = false>
__device__ __forceinline__ int read_scale(const uint8_t* sc, int64_t blk, int k) {
  if (k == 8) return ld_byte<CG>(sc + blk);
  int64_t bit = blk * k;
  int64_t byte = bit >> 3;
  int sh = (int)(bit & 7);
  uint32_t w = ld_byte<CG>(sc + byte);
  if (sh + k > 8) w |= (uint32_t)ld_byte<CG>(sc + byte + 1) << 8;
  return (int)((w >> sh) & ((1u << k) - 1u));
}

}  // namespace mxb
