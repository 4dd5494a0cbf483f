// sm_100a fast-path kernels of the compressed TP all-reduce (arXiv 2411.09510).
//
//   K1 k_quant      MX block quantise + bit-pack        (mx/codec.py:140-172, 238-263;
//                                                        mx/bitpack.py:22-34)
//   K2 k_dqsum      unpack + dequantise + fp32 rank-order sum -> bf16/f16/f32
//                                                       (mx/codec.py:175-188, 266-284;
//                                                        mx/netbench.py:329-334)
//   K3 k_requant    K2's sum re-quantised in registers (two-shot middle step)
//
// Work layout.  A warp owns a UNIT of 1024 consecutive values of one chunk;
// lane L holds values [32L, 32L+32): two 256-bit loads for bf16/f16
// (LDG.E.ENL2.256 -- every request is one full 32-byte sector, so the warp
// streams whole sectors with no re-reads).  A block of B values is
//   B <= 32 : owned by one lane (32/B blocks per lane, no cross-lane work),
//   B  = 64 : spread over 2 adjacent lanes, amax reduced with __shfl_xor_sync.
// The lane's 32 codes are 4b contiguous bytes of the element stream (FP4: one
// 16-byte store, the warp writes 512 contiguous bytes; INT8: one 32-byte
// store).  E8M0 scale codes (k = 8) leave as 1-4 bytes per lane; k < 8 is
// packed through a per-warp smem stage.  Each warp takes its units in pairs
// and issues both units' loads before any arithmetic (register double
// buffering), over a grid sized to the work (at most one resident wave).
// HBM-bound; no tensor cores (not a contraction).  The element width b is a
// compile-time constant on this path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>

#include "mx_device.cuh"

namespace mxb {

enum Enc { ENC_GEN = 0, ENC_E2M1 = 1, ENC_E2M3 = 2, ENC_E3M2 = 3 };

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kVPL = 32;          // values per lane
constexpr int kUnit = 32 * kVPL;  // values per warp unit
constexpr int kUPW = 2;           // units per warp per step (loads issued together)

struct QArgs {
  const void* x;
  int64_t n;             // total values
  int64_t cv;            // values per chunk
  int64_t units_per_chunk;
  int64_t total_units;
  uint8_t* scale_base;   // chunk j's scale stream at scale_base + j*chunk_stride
  uint8_t* elem_base;
  int64_t chunk_stride;
  unsigned long long* nonfinite;
  Fmt f;
};

struct DArgs {
  const uint8_t* in;
  int64_t rank_stride;
  int nranks;
  int64_t chunk_stride;
  int64_t scale_off, elem_off;
  int64_t n, cv;
  int64_t units_per_chunk;
  int64_t total_units;
  void* out;
  int plain;  // 1: plain decode (no +0 accumulation semantics)
  Fmt f;
};

struct RArgs {  // two-shot middle step: one chunk, nranks shards -> one shard
  const uint8_t* in;
  int64_t rank_stride;
  int nranks;
  int64_t scale_off, elem_off;  // input and output shards share the layout
  int64_t n;
  int64_t total_units;
  uint8_t* out_scale;
  uint8_t* out_elem;
  unsigned long long* nonfinite;
  Fmt f;
};

template <int B>
struct Geo {
  static constexpr int NSB = B >= kVPL ? 1 : kVPL / B;  // scale blocks per lane
  static constexpr int LPB = B > kVPL ? B / kVPL : 1;   // lanes per block
  static constexpr int SBV = kVPL / NSB;                // values per owned block
};

// ---------------------------------------------------------------------------
// 256-bit global accesses (sm_100)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ldg256(const void* p, uint32_t* r) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}
__device__ __forceinline__ void stg256(void* p, const uint32_t* r) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

// ---------------------------------------------------------------------------
// 32 raw input values per lane
// ---------------------------------------------------------------------------
template <typename T>
struct Raw {
  static constexpr int NW = kVPL * (int)sizeof(T) / 4;  // 16 (bf16/f16) or 32 (f32)
  uint32_t w[NW];
};

template <typename T>
__device__ __forceinline__ void load_raw(const T* __restrict__ p, Raw<T>& r) {
#pragma unroll
  for (int i = 0; i < Raw<T>::NW / 8; ++i)
    ldg256(reinterpret_cast<const uint32_t*>(p) + 8 * i, r.w + 8 * i);
}

template <typename T>
__device__ __forceinline__ void load_raw_partial(const T* __restrict__ p, int valid, Raw<T>& r) {
  if constexpr (sizeof(T) == 4) {
    const uint32_t* q = reinterpret_cast<const uint32_t*>(p);
#pragma unroll
    for (int i = 0; i < 32; ++i) r.w[i] = i < valid ? q[i] : 0u;
  } else {
    const uint16_t* q = reinterpret_cast<const uint16_t*>(p);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      uint32_t lo = 2 * i < valid ? q[2 * i] : 0u;
      uint32_t hi = 2 * i + 1 < valid ? q[2 * i + 1] : 0u;
      r.w[i] = lo | (hi << 16);
    }
  }
}

// |amax| of raw words [W0, W0+NWS) as f32 bits; NaN/Inf map to >= 0x7f800000.
template <typename T, int W0, int NWS>
__device__ __forceinline__ uint32_t absmax_bits(const Raw<T>& r) {
  if constexpr (sizeof(T) == 4) {
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < NWS; ++i) m = max(m, r.w[W0 + i] & 0x7fffffffu);
    return m;
  } else {
    const uint32_t M = 0x7fff7fffu;
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < NWS; ++i) m = __vmaxu2(m, r.w[W0 + i] & M);
    uint32_t h = max(m & 0xffffu, m >> 16);
    if constexpr (std::is_same<T, __nv_bfloat16>::value) {
      return h << 16;
    } else {  // f16: exact widening; Inf/NaN (>= 0x7c00) flagged explicitly
      return h >= 0x7c00u ? (0x7f800000u | h)
                          : __float_as_uint(__half2float(__ushort_as_half((unsigned short)h)));
    }
  }
}

// value i of the lane as f32 (exact)
template <typename T>
__device__ __forceinline__ float raw_f32(const Raw<T>& r, int i) {
  if constexpr (sizeof(T) == 4) {
    return __uint_as_float(r.w[i]);
  } else if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    return (i & 1) ? __uint_as_float(r.w[i >> 1] & 0xffff0000u)
                   : __uint_as_float(r.w[i >> 1] << 16);
  } else {
    uint32_t u = r.w[i >> 1];
    return __half2float(__ushort_as_half((unsigned short)((i & 1) ? (u >> 16) : (u & 0xffffu))));
  }
}

// Shared exponent from |amax| bits without branches (subnormals rescaled
// by 2^64 first); mx/codec.py:152-161.
__device__ __forceinline__ int shared_exp_fast(uint32_t ab, const Fmt& f) {
  bool sub = ab < 0x00800000u;
  uint32_t nb = sub ? __float_as_uint(__uint_as_float(ab) * 0x1p64f) : ab;
  int flog = (int)(nb >> 23) - (sub ? 191 : 127);
  int s = flog - f.emax + ((nb & 0x7fffffu) > f.ovf32 ? 1 : 0);
  return min(max(s, f.s_min), f.s_max);
}

// Encode 8 block-scaled values -> packed word (8*b bits, value i at bit i*b).
template <int ENC, int BITS>
__device__ __forceinline__ uint64_t encode8(const float* x, const Fmt& f) {
  uint64_t w = 0;
  if constexpr (ENC == ENC_E2M1) {
    uint32_t u = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) u |= cvt_e2m1x2(x[2 * i], x[2 * i + 1]) << (8 * i);
    w = u;
  } else if constexpr (ENC == ENC_E2M3 || ENC == ENC_E3M2) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t p = ENC == ENC_E2M3 ? cvt_e2m3x2(x[2 * i], x[2 * i + 1])
                                   : cvt_e3m2x2(x[2 * i], x[2 * i + 1]);
      w |= (uint64_t)(p & 0x3fu) << (12 * i);
      w |= (uint64_t)((p >> 8) & 0x3fu) << (12 * i + 6);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) w |= (uint64_t)encode_gen(x[i], f) << (i * BITS);
  }
  return w;
}

// The lane's 32 codes as 4b contiguous bytes = BITS 32-bit words.
template <int BITS>
struct LaneCodes {
  uint32_t w[BITS];
};

// Put group g (values 8g..8g+7; 8b bits = b bytes) into the lane words.
template <int BITS>
__device__ __forceinline__ void put_group(LaneCodes<BITS>& c, int g, uint64_t v) {
  if constexpr (BITS == 4) {
    c.w[g] = (uint32_t)v;
  } else if constexpr (BITS == 8) {
    c.w[2 * g] = (uint32_t)v;
    c.w[2 * g + 1] = (uint32_t)(v >> 32);
  } else {
#pragma unroll
    for (int t = 0; t < BITS; ++t) {
      const int byte = g * BITS + t;  // compile-time after unrolling
      c.w[byte >> 2] |= (uint32_t)((v >> (8 * t)) & 0xffu) << (8 * (byte & 3));
    }
  }
}

template <int BITS>
__device__ __forceinline__ uint64_t get_group(const LaneCodes<BITS>& c, int g) {
  if constexpr (BITS == 4) {
    return c.w[g];
  } else if constexpr (BITS == 8) {
    return (uint64_t)c.w[2 * g] | ((uint64_t)c.w[2 * g + 1] << 32);
  } else {
    uint64_t v = 0;
#pragma unroll
    for (int t = 0; t < BITS; ++t) {
      const int byte = g * BITS + t;
      v |= (uint64_t)((c.w[byte >> 2] >> (8 * (byte & 3))) & 0xffu) << (8 * t);
    }
    return v;
  }
}

// Store / load the lane's 4b code bytes at p (= unit base + 4b*lane).
template <int BITS>
__device__ __forceinline__ void store_lane_codes(uint8_t* __restrict__ p, const LaneCodes<BITS>& c,
                                                 int valid) {
  if (valid == kVPL) {
    if constexpr (BITS == 8) {
      stg256(p, c.w);
    } else if constexpr (BITS == 4) {
      *reinterpret_cast<uint4*>(p) = make_uint4(c.w[0], c.w[1], c.w[2], c.w[3]);
    } else if constexpr (BITS % 2 == 0) {
#pragma unroll
      for (int i = 0; i < BITS / 2; ++i)
        reinterpret_cast<uint2*>(p)[i] = make_uint2(c.w[2 * i], c.w[2 * i + 1]);
    } else {
#pragma unroll
      for (int i = 0; i < BITS; ++i) reinterpret_cast<uint32_t*>(p)[i] = c.w[i];
    }
  } else if (valid > 0) {
    const int nb = (valid * BITS + 7) / 8;
#pragma unroll
    for (int i = 0; i < 4 * BITS; ++i)
      if (i < nb) p[i] = (uint8_t)(c.w[i >> 2] >> (8 * (i & 3)));
  }
}

template <int BITS>
__device__ __forceinline__ LaneCodes<BITS> load_lane_codes(const uint8_t* __restrict__ p,
                                                           int valid) {
  LaneCodes<BITS> c;
#pragma unroll
  for (int i = 0; i < BITS; ++i) c.w[i] = 0u;
  if (valid == kVPL) {
    if constexpr (BITS == 8) {
      uint4 a = __ldg(reinterpret_cast<const uint4*>(p));
      uint4 b = __ldg(reinterpret_cast<const uint4*>(p) + 1);
      c.w[0] = a.x; c.w[1] = a.y; c.w[2] = a.z; c.w[3] = a.w;
      c.w[4] = b.x; c.w[5] = b.y; c.w[6] = b.z; c.w[7] = b.w;
    } else if constexpr (BITS == 4) {
      uint4 a = __ldg(reinterpret_cast<const uint4*>(p));
      c.w[0] = a.x; c.w[1] = a.y; c.w[2] = a.z; c.w[3] = a.w;
    } else if constexpr (BITS % 2 == 0) {
#pragma unroll
      for (int i = 0; i < BITS / 2; ++i) {
        uint2 a = __ldg(reinterpret_cast<const uint2*>(p) + i);
        c.w[2 * i] = a.x;
        c.w[2 * i + 1] = a.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < BITS; ++i) c.w[i] = __ldg(reinterpret_cast<const uint32_t*>(p) + i);
    }
  } else if (valid > 0) {
    const int nb = (valid * BITS + 7) / 8;
#pragma unroll
    for (int i = 0; i < 4 * BITS; ++i)
      if (i < nb) c.w[i >> 2] |= (uint32_t)p[i] << (8 * (i & 3));
  }
  return c;
}

// Quantise the lane's 32 values.  stored[sb] = scale code of owned block sb
// (B = 64: both lanes of the block hold it).  Zero and non-finite blocks get
// scale code 0 and zero codes (mx/codec.py:170-171).
template <typename T, int B, int ENC, int BITS>
__device__ __forceinline__ LaneCodes<BITS> quant_lane(const Raw<T>& raw, const Fmt& f,
                                                      int stored[Geo<B>::NSB], bool& bad_any) {
  constexpr int NSB = Geo<B>::NSB;
  constexpr int LPB = Geo<B>::LPB;
  constexpr int SBV = Geo<B>::SBV;
  constexpr int WPB = Raw<T>::NW / NSB;  // raw words per owned block
  LaneCodes<BITS> c;
#pragma unroll
  for (int i = 0; i < BITS; ++i) c.w[i] = 0u;
  bad_any = false;
  uint32_t abs_[NSB];
  if constexpr (NSB == 1) {
    abs_[0] = absmax_bits<T, 0, WPB>(raw);
  } else if constexpr (NSB == 2) {
    abs_[0] = absmax_bits<T, 0, WPB>(raw);
    abs_[1] = absmax_bits<T, WPB, WPB>(raw);
  } else {
    abs_[0] = absmax_bits<T, 0, WPB>(raw);
    abs_[1] = absmax_bits<T, WPB, WPB>(raw);
    abs_[2] = absmax_bits<T, 2 * WPB, WPB>(raw);
    abs_[3] = absmax_bits<T, 3 * WPB, WPB>(raw);
  }
#pragma unroll
  for (int sb = 0; sb < NSB; ++sb) {
    uint32_t ab = abs_[sb];
    if constexpr (LPB > 1) ab = max(ab, __shfl_xor_sync(0xffffffffu, ab, 1));
    const bool bad = ab >= 0x7f800000u;
    bad_any |= bad;
    const int s = shared_exp_fast(bad ? 0u : ab, f);
    const float inv = pow2f(-s);
    const bool zero = (ab == 0u) | bad;
    stored[sb] = zero ? 0 : s + f.sbias;
#pragma unroll
    for (int g = 0; g < SBV / 8; ++g) {
      float x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = raw_f32<T>(raw, sb * SBV + 8 * g + i) * inv;  // exact
      uint64_t w = encode8<ENC, BITS>(x, f);
      put_group<BITS>(c, sb * (SBV / 8) + g, zero ? 0ull : w);
    }
  }
  return c;
}

// First non-finite value among the lane's `valid` values -> atomicMin.
template <typename T>
__device__ __forceinline__ void report_nonfinite_raw(const Raw<T>& raw, int valid, int64_t flat0,
                                                     unsigned long long* nonfinite) {
  if (!nonfinite) return;
  int first = kVPL;
#pragma unroll
  for (int i = kVPL - 1; i >= 0; --i)  // unrolled: no dynamic register indexing
    if (i < valid && (__float_as_uint(raw_f32<T>(raw, i)) & 0x7fffffffu) >= 0x7f800000u)
      first = i;
  if (first < kVPL) atomicMin(nonfinite, (unsigned long long)(flat0 + first));
}

// Scale codes of a unit: k = 8 -> direct stores (1-4 bytes per lane);
// k < 8 -> pack through the warp's smem stage (1024/B codes = k bytes per 8).
template <int B>
__device__ __forceinline__ void store_unit_scales(uint8_t* __restrict__ sc, int64_t blk0,
                                                  const int stored[Geo<B>::NSB], int uvalid,
                                                  int lane, int k, uint8_t* stage) {
  constexpr int NSB = Geo<B>::NSB;
  constexpr int LPB = Geo<B>::LPB;
  const int nblk = (uvalid + B - 1) / B;  // blocks of this unit that exist
  if (k == 8) {
    if (uvalid == kUnit) {
      uint8_t* p = sc + blk0 + (lane / LPB) * NSB;
      if constexpr (NSB == 4) {
        *reinterpret_cast<uint32_t*>(p) = (uint32_t)stored[0] | ((uint32_t)stored[1] << 8) |
                                          ((uint32_t)stored[2] << 16) | ((uint32_t)stored[3] << 24);
      } else if constexpr (NSB == 2) {
        *reinterpret_cast<uint16_t*>(p) = (uint16_t)(stored[0] | (stored[1] << 8));
      } else {
        if (lane % LPB == 0) *p = (uint8_t)stored[0];
      }
    } else if (lane % LPB == 0) {
#pragma unroll
      for (int sb = 0; sb < NSB; ++sb) {
        int bi = (lane / LPB) * NSB + sb;
        if (bi < nblk) sc[blk0 + bi] = (uint8_t)stored[sb];
      }
    }
    return;
  }
  __syncwarp();
  if (lane % LPB == 0) {
#pragma unroll
    for (int sb = 0; sb < NSB; ++sb) stage[(lane / LPB) * NSB + sb] = (uint8_t)stored[sb];
  }
  __syncwarp();
  const int ngrp = (nblk + 7) / 8;
  if (lane < ngrp) {
    int cnt = min(8, nblk - 8 * lane);
    uint64_t w = 0;
    for (int i = 0; i < cnt; ++i) w |= (uint64_t)stage[8 * lane + i] << (i * k);
    uint8_t* p = sc + (blk0 / 8 + lane) * k;
    int nb = (cnt * k + 7) / 8;
    for (int i = 0; i < nb; ++i) p[i] = (uint8_t)(w >> (8 * i));
  }
  __syncwarp();
}

// Position of warp unit u: chunk, first value (chunk-local) and how many of
// its values exist.  32-bit arithmetic; no division for one chunk.
struct UnitPos {
  int64_t cbase;  // first value of the chunk (flat index)
  int64_t uoff;   // unit offset inside the chunk
  int chunk;
  int uvalid;
};

__device__ __forceinline__ UnitPos unit_pos(uint32_t u, uint32_t upc, bool one_chunk, int64_t cv,
                                            int64_t n) {
  UnitPos p;
  uint32_t chunk = one_chunk ? 0u : u / upc;
  p.chunk = (int)chunk;
  p.cbase = (int64_t)chunk * cv;
  p.uoff = (int64_t)(u - chunk * upc) * kUnit;
  int64_t len = one_chunk ? n : min(cv, n - p.cbase);
  p.uvalid = (int)min((int64_t)kUnit, len - p.uoff);
  return p;
}

// ---------------------------------------------------------------------------
// K1: quantise + pack
// ---------------------------------------------------------------------------
template <typename InT>
__device__ __forceinline__ void load_unit(const InT* __restrict__ x, const UnitPos& p, int lane,
                                          Raw<InT>& r) {
  const InT* q = x + p.cbase + p.uoff + lane * kVPL;
  if (p.uvalid == kUnit) {
    load_raw<InT>(q, r);
  } else {
    int valid = max(0, min(kVPL, p.uvalid - lane * kVPL));
    load_raw_partial<InT>(q, valid, r);
  }
}

template <typename InT, int B, int ENC, int BITS>
__device__ __forceinline__ void quant_unit(const QArgs& A, const Fmt& f, const UnitPos& p,
                                           const Raw<InT>& raw, int lane, uint8_t* stage) {
  constexpr int NSB = Geo<B>::NSB;
  const int valid = max(0, min(kVPL, p.uvalid - lane * kVPL));
  int stored[NSB];
  bool bad;
  LaneCodes<BITS> c = quant_lane<InT, B, ENC, BITS>(raw, f, stored, bad);
  if (bad) report_nonfinite_raw<InT>(raw, valid, p.cbase + p.uoff + lane * kVPL, A.nonfinite);
  const int64_t cofs = (int64_t)p.chunk * A.chunk_stride;
  store_lane_codes<BITS>(A.elem_base + cofs + (p.uoff / 8) * BITS + lane * 4 * BITS, c, valid);
  store_unit_scales<B>(A.scale_base + cofs, p.uoff / B, stored, p.uvalid, lane, f.kbits, stage);
}

template <typename InT, int B, int ENC, int BITS>
__global__ void __launch_bounds__(kThreads) k_quant(const QArgs A) {
  __shared__ __align__(16) uint8_t s_stage[kWarps][kUnit / 8];  // one byte per block (B >= 8)
  const Fmt f = A.f;
  const int lane = threadIdx.x & 31;
  uint8_t* stage = s_stage[threadIdx.x >> 5];
  const InT* x = reinterpret_cast<const InT*>(A.x);
  const uint32_t total = (uint32_t)A.total_units, upc = (uint32_t)A.units_per_chunk;
  const bool one = total == upc;
  const uint32_t nw = (uint32_t)(gridDim.x * kWarps);
  // units u0, u0+nw (a pair per step, both loads in flight before any math)
  for (uint32_t u0 = blockIdx.x * kWarps + (threadIdx.x >> 5); u0 < total; u0 += kUPW * nw) {
    const uint32_t u1 = u0 + nw;
    const bool has1 = u1 < total;
    UnitPos p0 = unit_pos(u0, upc, one, A.cv, A.n), p1;
    Raw<InT> r0, r1;
    load_unit<InT>(x, p0, lane, r0);
    if (has1) {
      p1 = unit_pos(u1, upc, one, A.cv, A.n);
      load_unit<InT>(x, p1, lane, r1);
    }
    quant_unit<InT, B, ENC, BITS>(A, f, p0, r0, lane, stage);
    if (has1) quant_unit<InT, B, ENC, BITS>(A, f, p1, r1, lane, stage);
  }
}

// ---------------------------------------------------------------------------
// K2: unpack + dequantise + rank-order fp32 sum
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 e2m1x2_to_f32x2(uint32_t byte) {
  uint32_t h;
  asm("{.reg .b8 t; cvt.u8.u32 t, %1; cvt.rn.f16x2.e2m1x2 %0, t;}" : "=r"(h) : "r"(byte));
  return __half22float2(*reinterpret_cast<const __half2*>(&h));
}

// Decode 8 codes (a group) of one block and add them to acc.
// `lut` = signed grid values (generic formats), smem.
template <int DEC, int BITS>
__device__ __forceinline__ void decode8_acc(uint64_t w, int stored, const Fmt& f, float* acc,
                                            bool plain, const float* lut) {
  const int s = stored - f.sbias;
  // g*2^s exactly representable -> one FFMA is exactly acc + value
  const bool fast = !plain && stored != 0 && s >= f.s_fast_lo && s <= f.s_fast_hi;
  if constexpr (DEC == ENC_E2M1) {
    uint32_t w32 = (uint32_t)w;
    if (fast) {
      const float F = pow2f(s);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float2 g = e2m1x2_to_f32x2((w32 >> (8 * j)) & 0xffu);
        acc[2 * j] = fmaf(g.x, F, acc[2 * j]);
        acc[2 * j + 1] = fmaf(g.y, F, acc[2 * j + 1]);
      }
    } else {
      E2M1Scale sp = e2m1_scale(stored, f.sbias);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float val = (e2m1_raw(w32, i) * sp.P) * sp.F;
        acc[i] = plain ? val : __fadd_rn(acc[i], val);
      }
    }
  } else {
    const uint32_t mask = (1u << BITS) - 1u;
    if (fast) {
      const float F = pow2f(s);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        acc[i] = fmaf(lut[(uint32_t)(w >> (i * BITS)) & mask], F, acc[i]);
    } else {
      const bool zero = stored == 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float val = decode_gen((uint32_t)(w >> (i * BITS)) & mask, s, zero, f);
        acc[i] = plain ? val : __fadd_rn(acc[i], val);
      }
    }
  }
}

// Signed grid values of a generic format into smem (code -> value).
__device__ __forceinline__ void fill_lut(float* lut, const Fmt& f) {
  const int ncodes = 1 << f.bits;
  for (int c = threadIdx.x; c < ncodes; c += blockDim.x) {
    uint32_t M, sign;
    int E;
    split_code((uint32_t)c, f, M, E, sign);
    float v = ldexp_exact(M, E);
    lut[c] = __uint_as_float(__float_as_uint(v) | (sign << 31));
  }
}

// One rank's shard, loaded: the lane's codes and the scale codes of its blocks.
template <int B, int BITS>
struct RankLoad {
  LaneCodes<BITS> c;
  int st[Geo<B>::NSB];
};

template <int B, int BITS>
__device__ __forceinline__ void load_rank(RankLoad<B, BITS>& r, const uint8_t* __restrict__ base,
                                          int64_t scale_off, int64_t elem_off, int64_t uoff,
                                          int lane, int valid, int kbits) {
  constexpr int NSB = Geo<B>::NSB;
  constexpr int LPB = Geo<B>::LPB;
  r.c = load_lane_codes<BITS>(base + elem_off + (uoff / 8) * BITS + lane * 4 * BITS, valid);
  const uint8_t* sc = base + scale_off;
  const int64_t blk0 = uoff / B + (lane / LPB) * NSB;
#pragma unroll
  for (int sb = 0; sb < NSB; ++sb) r.st[sb] = 0;
  if (valid == kVPL && kbits == 8) {
    if constexpr (NSB == 4) {
      uint32_t v = __ldg(reinterpret_cast<const unsigned int*>(sc + blk0));
#pragma unroll
      for (int sb = 0; sb < 4; ++sb) r.st[sb] = (v >> (8 * sb)) & 0xff;
    } else if constexpr (NSB == 2) {
      uint32_t v = __ldg(reinterpret_cast<const unsigned short*>(sc + blk0));
      r.st[0] = v & 0xff;
      r.st[1] = v >> 8;
    } else {
      r.st[0] = __ldg(sc + blk0);
    }
  } else if (valid > 0) {
#pragma unroll
    for (int sb = 0; sb < NSB; ++sb)
      if (sb * Geo<B>::SBV < valid) r.st[sb] = read_scale(sc, blk0 + sb, kbits);
  }
}

template <int B, int DEC, int BITS>
__device__ __forceinline__ void decode_rank(const RankLoad<B, BITS>& r, const Fmt& f,
                                            float acc[kVPL], bool plain, const float* lut) {
  constexpr int SBV = Geo<B>::SBV;
#pragma unroll
  for (int g = 0; g < kVPL / 8; ++g)
    decode8_acc<DEC, BITS>(get_group<BITS>(r.c, g), r.st[(8 * g) / SBV], f, acc + 8 * g, plain,
                           lut);
}

template <typename OutT>
__device__ __forceinline__ void store_lane_out(OutT* __restrict__ out, int valid,
                                               const float acc[kVPL]) {
  if (valid == kVPL) {
    uint32_t o[8];
    if constexpr (sizeof(OutT) == 2) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          o[i] = pack2<OutT>(acc[16 * h + 2 * i], acc[16 * h + 2 * i + 1]);
        stg256(out + 16 * h, o);
      }
    } else {
#pragma unroll
      for (int h = 0; h < 4; ++h) {
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = __float_as_uint(acc[8 * h + i]);
        stg256(out + 8 * h, o);
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < kVPL; ++i)
      if (i < valid) out[i] = from_f32<OutT>(acc[i]);
  }
}

template <typename OutT, int B, int DEC, int BITS>
__global__ void __launch_bounds__(kThreads) k_dqsum(const DArgs A) {
  __shared__ float s_lut[DEC == ENC_E2M1 ? 1 : 256];
  const Fmt f = A.f;
  if constexpr (DEC != ENC_E2M1) {
    fill_lut(s_lut, f);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const bool plain = A.plain != 0;
  const uint32_t total = (uint32_t)A.total_units, upc = (uint32_t)A.units_per_chunk;
  const bool one = total == upc;
  const uint32_t nw = (uint32_t)(gridDim.x * kWarps);
  for (uint32_t u = blockIdx.x * kWarps + (threadIdx.x >> 5); u < total; u += nw) {
    const UnitPos p = unit_pos(u, upc, one, A.cv, A.n);
    const int valid = max(0, min(kVPL, p.uvalid - lane * kVPL));
    float acc[kVPL];
#pragma unroll
    for (int i = 0; i < kVPL; ++i) acc[i] = 0.f;  // +0.0 (mx/netbench.py:332)
    const uint8_t* base = A.in + (int64_t)p.chunk * A.chunk_stride;
    int rk = 0;
    // two ranks per iteration: both ranks' loads are in flight together
    for (; rk + 1 < A.nranks; rk += 2, base += 2 * A.rank_stride) {
      RankLoad<B, BITS> r0, r1;
      load_rank<B, BITS>(r0, base, A.scale_off, A.elem_off, p.uoff, lane, valid, f.kbits);
      load_rank<B, BITS>(r1, base + A.rank_stride, A.scale_off, A.elem_off, p.uoff, lane, valid,
                         f.kbits);
      decode_rank<B, DEC, BITS>(r0, f, acc, plain, s_lut);
      decode_rank<B, DEC, BITS>(r1, f, acc, plain, s_lut);
    }
    if (rk < A.nranks) {
      RankLoad<B, BITS> r0;
      load_rank<B, BITS>(r0, base, A.scale_off, A.elem_off, p.uoff, lane, valid, f.kbits);
      decode_rank<B, DEC, BITS>(r0, f, acc, plain, s_lut);
    }
    if (valid > 0)
      store_lane_out<OutT>(reinterpret_cast<OutT*>(A.out) + p.cbase + p.uoff + lane * kVPL,
                           valid, acc);
  }
}

// ---------------------------------------------------------------------------
// K3: two-shot middle step -- sum N shards of one chunk, re-quantise
// ---------------------------------------------------------------------------
template <int B, int ENC, int BITS>
__global__ void __launch_bounds__(kThreads) k_requant(const RArgs A) {
  constexpr int DEC = ENC == ENC_E2M1 ? ENC_E2M1 : ENC_GEN;
  __shared__ __align__(16) uint8_t s_stage[kWarps][kUnit / 8];  // one byte per block (B >= 8)
  __shared__ float s_lut[DEC == ENC_E2M1 ? 1 : 256];
  const Fmt f = A.f;
  if constexpr (DEC != ENC_E2M1) {
    fill_lut(s_lut, f);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  uint8_t* stage = s_stage[threadIdx.x >> 5];
  const uint32_t nw = (uint32_t)(gridDim.x * kWarps);
  for (uint32_t u = blockIdx.x * kWarps + (threadIdx.x >> 5); u < (uint32_t)A.total_units;
       u += nw) {
    const int64_t uoff = (int64_t)u * kUnit;
    const int uvalid = (int)min((int64_t)kUnit, A.n - uoff);
    const int valid = max(0, min(kVPL, uvalid - lane * kVPL));
    float acc[kVPL];
#pragma unroll
    for (int i = 0; i < kVPL; ++i) acc[i] = 0.f;
    const uint8_t* base = A.in;
    for (int rk = 0; rk < A.nranks; ++rk, base += A.rank_stride) {
      RankLoad<B, BITS> r0;
      load_rank<B, BITS>(r0, base, A.scale_off, A.elem_off, uoff, lane, valid, f.kbits);
      decode_rank<B, DEC, BITS>(r0, f, acc, false, s_lut);
    }
    // values past the end hold +0 sums, exactly like zero padding
    Raw<float> raw;
#pragma unroll
    for (int i = 0; i < kVPL; ++i) raw.w[i] = __float_as_uint(acc[i]);
    int stored[Geo<B>::NSB];
    bool bad;
    LaneCodes<BITS> c = quant_lane<float, B, ENC, BITS>(raw, f, stored, bad);
    if (bad) report_nonfinite_raw<float>(raw, valid, uoff + lane * kVPL, A.nonfinite);
    store_lane_codes<BITS>(A.out_elem + (uoff / 8) * BITS + lane * 4 * BITS, c, valid);
    store_unit_scales<B>(A.out_scale, uoff / B, stored, uvalid, lane, f.kbits, stage);
  }
}

// launchers (one translation unit per dtype, compiled in parallel)
void launch_quant_bf16(const QArgs& a, int block, int enc, int bits, cudaStream_t st);
void launch_quant_f16(const QArgs& a, int block, int enc, int bits, cudaStream_t st);
void launch_quant_f32(const QArgs& a, int block, int enc, int bits, cudaStream_t st);
void launch_dqsum_bf16(const DArgs& a, int block, int enc, int bits, cudaStream_t st);
void launch_dqsum_f16(const DArgs& a, int block, int enc, int bits, cudaStream_t st);
void launch_dqsum_f32(const DArgs& a, int block, int enc, int bits, cudaStream_t st);
void launch_requant(const RArgs& a, int block, int enc, int bits, cudaStream_t st);

// Grid: enough CTAs that every warp gets `per_warp` units, never more than
// one resident wave (#SMs x occupancy).
template <typename K>
inline unsigned work_grid(K kernel, int64_t total_units, int per_warp) {
  static thread_local int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, 0);
  if (occ <= 0) occ = 1;
  int64_t need = (total_units + (int64_t)kWarps * per_warp - 1) / ((int64_t)kWarps * per_warp);
  int64_t g = std::min<int64_t>((int64_t)sms * occ, need);
  return (unsigned)std::max<int64_t>(g, 1);
}

}  // namespace mxb
