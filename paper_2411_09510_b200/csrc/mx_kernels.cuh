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
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "mx_device.cuh"

namespace mxb {

enum Enc { ENC_GEN = 0, ENC_E2M1 = 1, ENC_E2M3 = 2, ENC_E3M2 = 3, ENC_INT = 4, ENC_E2M2 = 5 };

// Decoder of an encoding: hardware f16 conversions for E2M1 / E2M3 / E3M2,
// integer->f16 for INT8; everything else decodes through the smem LUT.
__host__ __device__ constexpr int dec_of(int enc, int bits) {
  return (enc == ENC_E2M1 || enc == ENC_E2M3 || enc == ENC_E3M2 || enc == ENC_E2M2 ||
          (enc == ENC_INT && bits == 8))
             ? enc
             : ENC_GEN;
}

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
  int64_t flat_off;      // flat index of x[0] (non-finite reports)
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
  // optional, out's dtype and layout (may alias out): out = residual +
  // round(sum), rounded again -- bit-identical to the unfused K2 followed by
  // an elementwise add in out's dtype (the Llama residual h + all_reduce(.))
  const void* residual;
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

template <int B, int VPL = kVPL>
struct Geo {
  static constexpr int NSB = B >= VPL ? 1 : VPL / B;  // scale blocks per lane
  static constexpr int LPB = B > VPL ? B / VPL : 1;   // lanes per block
  static constexpr int SBV = VPL / NSB;               // values per owned block
};

// Programmatic dependent launch: a kernel launched with launch_pdl may be
// scheduled while its predecessor on the stream drains; pdl_prologue() waits
// for that predecessor to complete (memory flushed) before any input is read
// and releases this kernel's own dependents.  No-ops without the attribute.
__device__ __forceinline__ void pdl_prologue() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
}

inline bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MXB200_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  if (!pdl_enabled()) {
    k<<<grid, block, smem, st>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, args...);
}

// ---------------------------------------------------------------------------
// 256-bit global accesses (sm_100)
// ---------------------------------------------------------------------------
#ifndef MXB_LDG_HINT
#define MXB_LDG_HINT ""
#endif
__device__ __forceinline__ void ldg256(const void* p, uint32_t* r) {
  asm volatile("ld.global.nc.L1::no_allocate" MXB_LDG_HINT ".v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}
#ifndef MXB_STG_HINT
#define MXB_STG_HINT ""
#endif
__device__ __forceinline__ void stg256(void* p, const uint32_t* r) {
  asm volatile("st.global" MXB_STG_HINT ".v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]),
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
    // four cvts into bytes of one register: ptxas chains F2FP ... MERGE_C,
    // so packing costs no extra instructions
    uint32_t u;
    asm("{\n\t.reg .b8 b0, b1, b2, b3;\n\t"
        "cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n\t"
        "cvt.rn.satfinite.e2m1x2.f32 b1, %4, %3;\n\t"
        "cvt.rn.satfinite.e2m1x2.f32 b2, %6, %5;\n\t"
        "cvt.rn.satfinite.e2m1x2.f32 b3, %8, %7;\n\t"
        "mov.b32 %0, {b0, b1, b2, b3};\n\t}"
        : "=r"(u)
        : "f"(x[0]), "f"(x[1]), "f"(x[2]), "f"(x[3]), "f"(x[4]), "f"(x[5]), "f"(x[6]),
          "f"(x[7]));
    w = u;
  } else if constexpr (ENC == ENC_E2M3 || ENC == ENC_E3M2) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t p = ENC == ENC_E2M3 ? cvt_e2m3x2(x[2 * i], x[2 * i + 1])
                                   : cvt_e3m2x2(x[2 * i], x[2 * i + 1]);
      w |= (uint64_t)(p & 0x3fu) << (12 * i);
      w |= (uint64_t)((p >> 8) & 0x3fu) << (12 * i + 6);
    }
  } else if constexpr (ENC == ENC_E2M2) {
    // FP5 E2M2 through the hardware FP6 E3M2 conversion: the E2M2 grid
    // {m/4 (e=0), (1+m/4)*2^(e-1)} scaled by 1/4 is exactly E3M2's grid for
    // e3 = 0..3 (bias 3), so RNE+satfinite of x/4 (exact) after the
    // reference's clamp to the grid max 7 (mx/codec.py:130) gives E3M2 code
    // s|e3|m with e3 <= 3, and the E2M2 code is s|e3[1:0]|m -- ties to the
    // even mantissa = the even grid index, as the reference rounds
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float lo = copysignf(fminf(fabsf(x[2 * i]), 7.0f), x[2 * i]) * 0.25f;
      const float hi = copysignf(fminf(fabsf(x[2 * i + 1]), 7.0f), x[2 * i + 1]) * 0.25f;
      const uint32_t p = cvt_e3m2x2(lo, hi);  // byte 0: lo, byte 1: hi
      const uint32_t c0 = ((p & 0x20u) >> 1) | (p & 0xFu);
      const uint32_t c1 = ((p >> 9) & 0x10u) | ((p >> 8) & 0xFu);
      w |= (uint64_t)(c0 | (c1 << 5)) << (10 * i);
    }
  } else if constexpr (ENC == ENC_INT) {
    // sign-magnitude INTb: RNE to an integer by the 1.5*2^23 magic add, the
    // grid maximum 2^(b-1)-1 saturates first (mx/codec.py:130)
    constexpr float GMAX = (float)((1 << (BITS - 1)) - 1);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float a = fminf(fabsf(x[i]), GMAX);
      const uint32_t idx = __float_as_uint(__fadd_rn(a, 12582912.0f)) - 0x4B400000u;
      const uint32_t code = idx | ((__float_as_uint(x[i]) >> 31) << (BITS - 1));
      w |= (uint64_t)code << (i * BITS);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) w |= (uint64_t)encode_gen(x[i], f) << (i * BITS);
  }
  return w;
}

// The lane's VPL codes as VPL*b/8 contiguous bytes (VPL = 32: BITS words).
template <int BITS, int VPL = kVPL>
struct LaneCodes {
  static constexpr int NB = VPL * BITS / 8;
  static constexpr int NW = (NB + 3) / 4;
  uint32_t w[NW];
};

// Put group g (values 8g..8g+7; 8b bits at bit offset 8bg) into the lane
// words.  g and BITS are compile-time after unrolling, so the word index and
// the funnel shifts fold to constants (2-3 shifts per group for odd widths).
template <int BITS, int VPL = kVPL>
__device__ __forceinline__ void put_group(LaneCodes<BITS, VPL>& c, int g, uint64_t v) {
  if constexpr (BITS == 4) {
    c.w[g] = (uint32_t)v;
  } else if constexpr (BITS == 8) {
    c.w[2 * g] = (uint32_t)v;
    c.w[2 * g + 1] = (uint32_t)(v >> 32);
  } else {
    const int o = g * 8 * BITS, wi = o >> 5, sh = o & 31;
    c.w[wi] |= (uint32_t)(v << sh);
    if (sh + 8 * BITS > 32) c.w[wi + 1] |= (uint32_t)(v >> (32 - sh));
    if (sh + 8 * BITS > 64) c.w[wi + 2] |= (uint32_t)(v >> (64 - sh));
  }
}

template <int BITS, int VPL = kVPL>
__device__ __forceinline__ uint64_t get_group(const LaneCodes<BITS, VPL>& c, int g) {
  if constexpr (BITS == 4) {
    return c.w[g];
  } else if constexpr (BITS == 8) {
    return (uint64_t)c.w[2 * g] | ((uint64_t)c.w[2 * g + 1] << 32);
  } else {
    const int o = g * 8 * BITS, wi = o >> 5, sh = o & 31;
    uint64_t v = (uint64_t)c.w[wi] >> sh;
    if (sh + 8 * BITS > 32) v |= (uint64_t)c.w[wi + 1] << (32 - sh);
    if (sh + 8 * BITS > 64) v |= (uint64_t)c.w[wi + 2] << (64 - sh);
    return v & ((1ull << (8 * BITS)) - 1ull);
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

// Loads of shard bytes.  CG = false: the non-coherent read-only path
// (ld.global.nc), ONLY for data no thread anywhere writes during the kernel.
// CG = true: ld.global.cg (weak, L1-bypassing, coherent at L2) for bytes
// written earlier in the SAME kernel -- by this warp (the fused one-device
// flow) or by a peer GPU over NVLink after a flag acquire (k_symm_flow /
// k_symm2_flow).  A weak load ordered after an acquire (directly, or through
// bar.sync from the acquiring thread) is inside the PTX memory model; an .nc
// load is not, and its cached line may be stale.
template <bool CG, typename T>
__device__ __forceinline__ T ldro(const T* p) {
  if constexpr (CG) return __ldcg(p);
  else return __ldg(p);
}

template <int BITS, bool CG = false>
__device__ __forceinline__ LaneCodes<BITS> load_lane_codes(const uint8_t* __restrict__ p,
                                                           int valid) {
  LaneCodes<BITS> c;
#pragma unroll
  for (int i = 0; i < BITS; ++i) c.w[i] = 0u;
  if (valid == kVPL) {
    if constexpr (BITS == 8) {
      uint4 a = ldro<CG>(reinterpret_cast<const uint4*>(p));
      uint4 b = ldro<CG>(reinterpret_cast<const uint4*>(p) + 1);
      c.w[0] = a.x; c.w[1] = a.y; c.w[2] = a.z; c.w[3] = a.w;
      c.w[4] = b.x; c.w[5] = b.y; c.w[6] = b.z; c.w[7] = b.w;
    } else if constexpr (BITS == 4) {
      uint4 a = ldro<CG>(reinterpret_cast<const uint4*>(p));
      c.w[0] = a.x; c.w[1] = a.y; c.w[2] = a.z; c.w[3] = a.w;
    } else if constexpr (BITS % 2 == 0) {
#pragma unroll
      for (int i = 0; i < BITS / 2; ++i) {
        uint2 a = ldro<CG>(reinterpret_cast<const uint2*>(p) + i);
        c.w[2 * i] = a.x;
        c.w[2 * i + 1] = a.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < BITS; ++i) c.w[i] = ldro<CG>(reinterpret_cast<const uint32_t*>(p) + i);
    }
  } else if (valid > 0) {
    const int nb = (valid * BITS + 7) / 8;
#pragma unroll
    for (int i = 0; i < 4 * BITS; ++i)
      if (i < nb) c.w[i >> 2] |= (uint32_t)ldro<CG>(p + i) << (8 * (i & 3));
  }
  return c;
}

// The lane's 16 codes (2b bytes at p = unit base + 2b*lane) for K2.
template <int BITS, bool CG = false>
__device__ __forceinline__ LaneCodes<BITS, 16> load_lane_codes16(const uint8_t* __restrict__ p,
                                                                 int valid) {
  LaneCodes<BITS, 16> c;
  constexpr int NW = LaneCodes<BITS, 16>::NW;
#pragma unroll
  for (int i = 0; i < NW; ++i) c.w[i] = 0u;
  if (valid == 16) {
    if constexpr (BITS == 8) {
      uint4 a = ldro<CG>(reinterpret_cast<const uint4*>(p));
      c.w[0] = a.x; c.w[1] = a.y; c.w[2] = a.z; c.w[3] = a.w;
    } else if constexpr (BITS == 4) {
      uint2 a = ldro<CG>(reinterpret_cast<const uint2*>(p));
      c.w[0] = a.x; c.w[1] = a.y;
    } else if constexpr (BITS % 2 == 0) {
#pragma unroll
      for (int i = 0; i < BITS / 2; ++i) c.w[i] = ldro<CG>(reinterpret_cast<const uint32_t*>(p) + i);
    } else {
#pragma unroll
      for (int i = 0; i < BITS; ++i)
        c.w[i >> 1] |= (uint32_t)ldro<CG>(reinterpret_cast<const unsigned short*>(p) + i)
                       << (16 * (i & 1));
    }
  } else if (valid > 0) {
    const int nb = (valid * BITS + 7) / 8;
#pragma unroll
    for (int i = 0; i < 2 * BITS; ++i)
      if (i < nb) c.w[i >> 2] |= (uint32_t)ldro<CG>(p + i) << (8 * (i & 3));
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
      if constexpr (std::is_same<T, __nv_bfloat16>::value && ENC == ENC_E2M1) {
        // bf16 pairs scaled by 2^-s in one HFMA2.BF16 each (exact: power-of-
        // two scaling of bf16; results below 2^-126 are far under the 0.25
        // rounding threshold and keep their sign), then widened to f32.
        // E2M1 has emax 2, so s <= 126 and 2^-s is a normal bf16.
        const uint32_t i16 = (uint32_t)(127 - s) << 7;
        const uint32_t inv2 = i16 | (i16 << 16);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          uint32_t wv = raw.w[(sb * SBV + 8 * g) / 2 + h];
          __nv_bfloat162 y = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&wv),
                                     *reinterpret_cast<const __nv_bfloat162*>(&inv2));
          uint32_t yu = *reinterpret_cast<uint32_t*>(&y);
          x[2 * h] = __uint_as_float(yu << 16);
          x[2 * h + 1] = __uint_as_float(yu & 0xffff0000u);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = raw_f32<T>(raw, sb * SBV + 8 * g + i) * inv;  // exact
      }
      uint64_t w;
      if constexpr (std::is_same<T, __nv_bfloat16>::value &&
                    (ENC == ENC_E2M2 || ENC == ENC_E2M3 || ENC == ENC_E3M2)) {
        if (s <= 124) {
          // bf16 pairs scaled in one HMUL2.BF16 each (exact power-of-two
          // scaling, as E2M1 above) straight into the hardware FP6
          // conversion.  E2M2 takes x/4 = v * 2^-(s+2) clamped to the grid
          // max 7/4 with one packed min/max (the reference clamps before
          // rounding, mx/codec.py:130), then E3M2 (see encode8)
          constexpr int SH = ENC == ENC_E2M2 ? 2 : 0;
          const uint32_t i16 = (uint32_t)(127 - s - SH) << 7;
          const uint32_t inv2 = i16 | (i16 << 16);
          w = 0;
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            uint32_t wv = raw.w[(sb * SBV + 8 * g) / 2 + h];
            __nv_bfloat162 y = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&wv),
                                       *reinterpret_cast<const __nv_bfloat162*>(&inv2));
            if constexpr (ENC == ENC_E2M2) {
              const __nv_bfloat162 hi2 = __floats2bfloat162_rn(1.75f, 1.75f);
              const __nv_bfloat162 lo2 = __floats2bfloat162_rn(-1.75f, -1.75f);
              y = __hmax2(__hmin2(y, hi2), lo2);
            }
            const uint32_t yu = *reinterpret_cast<uint32_t*>(&y);
            const float lo = __uint_as_float(yu << 16), hi = __uint_as_float(yu & 0xffff0000u);
            if constexpr (ENC == ENC_E2M2) {
              const uint32_t p = cvt_e3m2x2(lo, hi);
              const uint32_t c0 = ((p & 0x20u) >> 1) | (p & 0xFu);
              const uint32_t c1 = ((p >> 9) & 0x10u) | ((p >> 8) & 0xFu);
              w |= (uint64_t)(c0 | (c1 << 5)) << (10 * h);
            } else {
              const uint32_t p = ENC == ENC_E2M3 ? cvt_e2m3x2(lo, hi) : cvt_e3m2x2(lo, hi);
              w |= (uint64_t)(p & 0x3fu) << (12 * h);
              w |= (uint64_t)((p >> 8) & 0x3fu) << (12 * h + 6);
            }
          }
        } else {
          w = encode8<ENC, BITS>(x, f);
        }
      } else {
        w = encode8<ENC, BITS>(x, f);
      }
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
  if (bad)
    report_nonfinite_raw<InT>(raw, valid, A.flat_off + p.cbase + p.uoff + lane * kVPL,
                              A.nonfinite);
  const int64_t cofs = (int64_t)p.chunk * A.chunk_stride;
  store_lane_codes<BITS>(A.elem_base + cofs + (p.uoff / 8) * BITS + lane * 4 * BITS, c, valid);
  store_unit_scales<B>(A.scale_base + cofs, p.uoff / B, stored, p.uvalid, lane, f.kbits, stage);
}

// k < 8-bit scale codes (E5M0 ...) of a FULL unit straight from registers:
// the 8 blocks of one packed group (k bytes, LSB-first as mx/bitpack.py)
// belong to G = 8*LPB/NSB consecutive lanes; an xor butterfly ORs their
// shifted codes into one 64-bit word and the group's first lane stores its
// k bytes -- no shared-memory staging, no extra __syncwarp.
__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  uint32_t lo = __shfl_xor_sync(0xffffffffu, (uint32_t)v, m);
  uint32_t hi = __shfl_xor_sync(0xffffffffu, (uint32_t)(v >> 32), m);
  return ((uint64_t)hi << 32) | lo;
}

// warp-collective: lanes whose lane % scale_group_lanes<B>() == 0 return the
// k-bit codes of the 8-block group (lane / G) of the unit, packed
template <int B>
__host__ __device__ constexpr int scale_group_lanes() {
  return 8 * Geo<B>::LPB / Geo<B>::NSB;
}
template <int B>
__device__ __forceinline__ uint64_t pack_unit_scales_k(const int* stored, int lane, int k) {
  constexpr int NSB = Geo<B>::NSB;
  constexpr int LPB = Geo<B>::LPB;
  constexpr int G = scale_group_lanes<B>();  // lanes per group of 8 blocks
  uint64_t v = 0;
  if (lane % LPB == 0) {
    const int b0 = ((lane / LPB) * NSB) % 8;  // first owned block inside its group
#pragma unroll
    for (int sb = 0; sb < NSB; ++sb) v |= (uint64_t)stored[sb] << ((b0 + sb) * k);
  }
#pragma unroll
  for (int m = 1; m < G; m <<= 1) v |= shfl_xor_u64(v, m);
  return v;
}

template <int B>
__device__ __forceinline__ void store_unit_scales_k(uint8_t* __restrict__ sc, int64_t blk0,
                                                    const int* stored, int lane, int k) {
  constexpr int G = scale_group_lanes<B>();
  const uint64_t v = pack_unit_scales_k<B>(stored, lane, k);
  if (lane % G == 0) {
    uint8_t* p = sc + (blk0 / 8 + lane / G) * k;
    for (int i = 0; i < k; ++i) p[i] = (uint8_t)(v >> (8 * i));
  }
}

// Full unit u of a single-chunk tensor: straight-line, no bounds logic.
// KB: scale-code width, compile-time: 8 (E8M0 bytes) or 5 (E5M0, packed).
template <typename InT, int B, int ENC, int BITS, int KB = 8>
__device__ __forceinline__ void quant_full_unit(const QArgs& A, const Fmt& f, uint32_t u,
                                                const Raw<InT>& raw, int lane) {
  constexpr int NSB = Geo<B>::NSB;
  constexpr int LPB = Geo<B>::LPB;
  int stored[NSB];
  bool bad;
  LaneCodes<BITS> c = quant_lane<InT, B, ENC, BITS>(raw, f, stored, bad);
  if (bad)
    report_nonfinite_raw<InT>(raw, kVPL, A.flat_off + (int64_t)u * kUnit + lane * kVPL,
                              A.nonfinite);
  store_lane_codes<BITS>(A.elem_base + (size_t)u * (kUnit / 8 * BITS) + lane * (4 * BITS), c,
                         kVPL);
  if constexpr (KB != 8) {
    store_unit_scales_k<B>(A.scale_base, (int64_t)u * (kUnit / B), stored, lane, KB);
    return;
  }
  uint8_t* p = A.scale_base + (size_t)u * (kUnit / B) + (lane / LPB) * NSB;
  if constexpr (NSB == 4) {
    *reinterpret_cast<uint32_t*>(p) = (uint32_t)stored[0] | ((uint32_t)stored[1] << 8) |
                                      ((uint32_t)stored[2] << 16) | ((uint32_t)stored[3] << 24);
  } else if constexpr (NSB == 2) {
    *reinterpret_cast<uint16_t*>(p) = (uint16_t)(stored[0] | (stored[1] << 8));
  } else {
    if (lane % LPB == 0) *p = (uint8_t)stored[0];
  }
}

template <typename InT, int B_, int ENC, int BITS>
__global__ void __launch_bounds__(kThreads) k_quant(const QArgs A) {
  constexpr int B = B_;
  pdl_prologue();
  __shared__ __align__(16) uint8_t s_stage[kWarps][kUnit / 8];  // one byte per block (B >= 8)
  const Fmt f = A.f;
  const int lane = threadIdx.x & 31;
  uint8_t* stage = s_stage[threadIdx.x >> 5];
  const InT* x = reinterpret_cast<const InT*>(A.x);
  const uint32_t total = (uint32_t)A.total_units, upc = (uint32_t)A.units_per_chunk;
  const bool one = total == upc;
  const uint32_t nw = (uint32_t)(gridDim.x * kWarps);
  const uint32_t gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (!one && f.kbits == 8 && A.cv % kUnit == 0 && A.n % A.cv == 0) {
    // equal chunks of whole units (two-shot at 1024-multiple chunk sizes):
    // unit u is flat unit u of x; its codes go to chunk u / upc
    const uint32_t nfull = (uint32_t)(A.n / kUnit);
    auto one_unit = [&](uint32_t u, const Raw<InT>& r) {
      const uint32_t chunk = u / upc, q = u - chunk * upc;
      QArgs B = A;
      B.elem_base = A.elem_base + (size_t)chunk * A.chunk_stride;
      B.scale_base = A.scale_base + (size_t)chunk * A.chunk_stride;
      B.flat_off = A.flat_off + (int64_t)chunk * A.cv;
      quant_full_unit<InT, B_, ENC, BITS>(B, f, q, r, lane);
    };
    for (uint32_t u0 = gw; u0 < nfull; u0 += kUPW * nw) {
      const uint32_t u1 = u0 + nw;
      const bool has1 = u1 < nfull;
      Raw<InT> r0, r1;
      load_raw<InT>(x + (size_t)u0 * kUnit + lane * kVPL, r0);
      if (has1) load_raw<InT>(x + (size_t)u1 * kUnit + lane * kVPL, r1);
      one_unit(u0, r0);
      if (has1) one_unit(u1, r1);
    }
    return;
  }
  if (one && f.kbits == 8) {
    // single chunk, E8M0 scales: full units in pairs with both units' loads
    // in flight before any math; pointers are plain multiples of u
    const uint32_t nfull = (uint32_t)(A.n / kUnit);
    for (uint32_t u0 = gw; u0 < nfull; u0 += kUPW * nw) {
      const uint32_t u1 = u0 + nw;
      const bool has1 = u1 < nfull;
      Raw<InT> r0, r1;
      load_raw<InT>(x + (size_t)u0 * kUnit + lane * kVPL, r0);
      if (has1) load_raw<InT>(x + (size_t)u1 * kUnit + lane * kVPL, r1);
      quant_full_unit<InT, B, ENC, BITS>(A, f, u0, r0, lane);
      if (has1) quant_full_unit<InT, B, ENC, BITS>(A, f, u1, r1, lane);
    }
    // the partial last unit (if any) goes to the warp that would own it next
    if (nfull < total && gw == nfull % nw) {
      UnitPos p = unit_pos(nfull, upc, true, A.cv, A.n);
      Raw<InT> r;
      load_unit<InT>(x, p, lane, r);
      quant_unit<InT, B, ENC, BITS>(A, f, p, r, lane, stage);
    }
    return;
  }
  // general case (chunked shards, k < 8): units u0, u0+nw per step
  for (uint32_t u0 = gw; u0 < total; u0 += kUPW * nw) {
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

// K1 lean form (round 2; scripts/kquant_probe.cu, profiles/r02/k1_lean):
// E8M0 scales, one chunk or equal chunks of whole 1024-value units.  One
// unit per warp over a flat grid -- no grid-stride loop, no paired units --
// with registers capped so that MINB CTAs (6 x 8 warps for 16-bit inputs)
// stay resident: the loads of 48 warps per SM are in flight at once and the
// block scheduler balances the tail.  8B shape: 5.07 -> 4.74 us; 70B shape:
// 15.23 -> 13.93 us (0.93 of the HBM copy peak).
template <typename InT, int B_, int ENC, int BITS, int MINB, int KB>
__global__ void __launch_bounds__(kThreads, MINB) k_quant_lean(const QArgs A) {
  constexpr int B = B_;
  pdl_prologue();
  const int lane = threadIdx.x & 31;
  const uint32_t u = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint32_t total = (uint32_t)A.total_units, upc = (uint32_t)A.units_per_chunk;
  if (u >= total) return;
  const InT* x = reinterpret_cast<const InT*>(A.x);
  const Fmt f = A.f;
  if (total != upc) {  // equal chunks of whole units: unit u is flat unit u of x
    Raw<InT> r;
    load_raw<InT>(x + (size_t)u * kUnit + lane * kVPL, r);
    const uint32_t chunk = u / upc, q = u - chunk * upc;
    QArgs C = A;
    C.elem_base = A.elem_base + (size_t)chunk * A.chunk_stride;
    C.scale_base = A.scale_base + (size_t)chunk * A.chunk_stride;
    C.flat_off = A.flat_off + (int64_t)chunk * A.cv;
    quant_full_unit<InT, B, ENC, BITS, KB>(C, f, q, r, lane);
    return;
  }
  if ((int64_t)(u + 1) * kUnit <= A.n) {
    Raw<InT> r;
    load_raw<InT>(x + (size_t)u * kUnit + lane * kVPL, r);
    quant_full_unit<InT, B, ENC, BITS, KB>(A, f, u, r, lane);
    return;
  }
  // the partial last unit of a single chunk
  __shared__ __align__(16) uint8_t s_stage[kWarps][kUnit / 8];
  UnitPos p = unit_pos(u, upc, true, A.cv, A.n);
  Raw<InT> r;
  load_unit<InT>(x, p, lane, r);
  quant_unit<InT, B, ENC, BITS>(A, f, p, r, lane, s_stage[threadIdx.x >> 5]);
}

// 6 resident CTAs (40 registers) fit the bf16-input register path of every
// format with a hardware or closed-form encoder without spills (ptxas log);
// the generic encoder, f16 inputs (abs-max in f32) and f32 inputs (twice
// the raw registers) keep the 4-CTA bound
template <typename InT, int ENC>
constexpr int lean_minb() {
  return (std::is_same<InT, __nv_bfloat16>::value && ENC != ENC_GEN) ? 6 : 4;
}

// formats with a lean E5M0-scale instantiation (K1 / K2 / K4 / K5, KB = 5):
// the paper's selected schemes -- FP4 E2M1 / FP5 E2M2 elements with E5M0
// scales (mx/fixtures/table2_selected_schemes.csv); other
// formats and the E4M0/E6M0/E7M0 ablation scales take the general kernels
__host__ __device__ constexpr bool lean_k_ok(int enc) {
  return enc == ENC_E2M1 || enc == ENC_E2M2;
}

inline bool quant_lean_ok(const QArgs& a) {
  return a.total_units == a.units_per_chunk || (a.cv % kUnit == 0 && a.n % a.cv == 0);
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
template <int B, int BITS, int VPL = kVPL>
struct RankLoad {
  LaneCodes<BITS, VPL> c;
  int st[Geo<B, VPL>::NSB];
};

template <int B, int BITS, int VPL = kVPL, bool CG = false>
__device__ __forceinline__ void load_rank(RankLoad<B, BITS, VPL>& r,
                                          const uint8_t* __restrict__ base, int64_t scale_off,
                                          int64_t elem_off, int64_t uoff, int lane, int valid,
                                          int kbits) {
  constexpr int NSB = Geo<B, VPL>::NSB;
  constexpr int LPB = Geo<B, VPL>::LPB;
  const uint8_t* el = base + elem_off + (uoff / 8) * BITS + lane * (VPL * BITS / 8);
  if constexpr (VPL == 16) r.c = load_lane_codes16<BITS, CG>(el, valid);
  else r.c = load_lane_codes<BITS, CG>(el, valid);
  const uint8_t* sc = base + scale_off;
  const int64_t blk0 = uoff / B + (lane / LPB) * NSB;
#pragma unroll
  for (int sb = 0; sb < NSB; ++sb) r.st[sb] = 0;
  if (valid == VPL && kbits == 8) {
    if constexpr (NSB == 4) {
      uint32_t v = ldro<CG>(reinterpret_cast<const unsigned int*>(sc + blk0));
#pragma unroll
      for (int sb = 0; sb < 4; ++sb) r.st[sb] = (v >> (8 * sb)) & 0xff;
    } else if constexpr (NSB == 2) {
      uint32_t v = ldro<CG>(reinterpret_cast<const unsigned short*>(sc + blk0));
      r.st[0] = v & 0xff;
      r.st[1] = v >> 8;
    } else if constexpr (CG && LPB > 1) {
      // shard bytes written in this kernel: only the lane that stored the
      // shared scale byte reads it back; its pair partner gets it by shuffle
      int v = lane % LPB == 0 ? (int)ldro<CG>(sc + blk0) : 0;
      r.st[0] = __shfl_sync(0xffffffffu, v, lane & ~(LPB - 1));
    } else {
      r.st[0] = ldro<CG>(sc + blk0);
    }
  } else if (valid == VPL && kbits < 8) {
    // packed k-bit codes (E5M0 ...): the lane's NSB consecutive codes are
    // NSB*k bits at bit blk0*k -- gather exactly the bytes holding them
    // (<= 5), then shift them out (k is a compile-time constant in the lean
    // kernels, so the loop and the shifts fold)
    const int64_t bit = blk0 * kbits;
    const uint8_t* p = sc + (bit >> 3);
    const int sh = (int)(bit & 7);
    uint64_t w = 0;
#pragma unroll
    for (int i = 0; i < (7 + NSB * 8 + 7) / 8; ++i)
      if (i * 8 < sh + NSB * kbits) w |= (uint64_t)ld_byte<CG>(p + i) << (8 * i);
    w >>= sh;
#pragma unroll
    for (int sb = 0; sb < NSB; ++sb) r.st[sb] = (int)((w >> (sb * kbits)) & ((1u << kbits) - 1u));
  } else if (valid > 0) {
#pragma unroll
    for (int sb = 0; sb < NSB; ++sb)
      if (sb * Geo<B, VPL>::SBV < valid) r.st[sb] = read_scale<CG>(sc, blk0 + sb, kbits);
  }
}

// 8 FP4 codes (one 32-bit word) -> acc[i] += g_i * 2^s with 2^s given as f16
// bits: F2FP.F16.E2M1.UNPACK_B picks each byte straight out of the word and
// FHFMA (fma.rn.f32.f16) multiplies the f16 grid value by the f16 scale and
// adds the fp32 accumulator with ONE rounding -- exactly acc + value, since
// g*2^s is representable (mx/netbench.py:334 semantics).
__device__ __forceinline__ void e2m1_word_fma(uint32_t w, uint16_t F16, float* a) {
  asm("{\n\t.reg .b8 b0, b1, b2, b3;\n\t.reg .b32 p0, p1, p2, p3;\n\t"
      ".reg .b16 l0, h0, l1, h1, l2, h2, l3, h3;\n\t"
      "mov.b32 {b0, b1, b2, b3}, %8;\n\t"
      "cvt.rn.f16x2.e2m1x2 p0, b0;\n\tcvt.rn.f16x2.e2m1x2 p1, b1;\n\t"
      "cvt.rn.f16x2.e2m1x2 p2, b2;\n\tcvt.rn.f16x2.e2m1x2 p3, b3;\n\t"
      "mov.b32 {l0, h0}, p0;\n\tmov.b32 {l1, h1}, p1;\n\t"
      "mov.b32 {l2, h2}, p2;\n\tmov.b32 {l3, h3}, p3;\n\t"
      "fma.rn.f32.f16 %0, l0, %9, %0;\n\tfma.rn.f32.f16 %1, h0, %9, %1;\n\t"
      "fma.rn.f32.f16 %2, l1, %9, %2;\n\tfma.rn.f32.f16 %3, h1, %9, %3;\n\t"
      "fma.rn.f32.f16 %4, l2, %9, %4;\n\tfma.rn.f32.f16 %5, h2, %9, %5;\n\t"
      "fma.rn.f32.f16 %6, l3, %9, %6;\n\tfma.rn.f32.f16 %7, h3, %9, %7;\n\t}"
      : "+f"(a[0]), "+f"(a[1]), "+f"(a[2]), "+f"(a[3]), "+f"(a[4]), "+f"(a[5]), "+f"(a[6]),
        "+f"(a[7])
      : "r"(w), "h"(F16));
}

__device__ __forceinline__ void fma2_f16(uint32_t h2, uint16_t F16, float& a0, float& a1) {
  asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
      "fma.rn.f32.f16 %0, l, %3, %0;\n\tfma.rn.f32.f16 %1, h, %3, %1;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "r"(h2), "h"(F16));
}

// 8 FP6 codes (48 bits, value i at bit 6i) -> acc += grid * 2^s: the OCP
// E2M3 / E3M2 code points equal the reference's sign|index codes, so the
// hardware f16x2 conversion yields the exact grid values (f16-exact), and
// FHFMA adds g * 2^s with one rounding.
template <int DEC>
__device__ __forceinline__ void fp6_group_fma(uint64_t w, uint16_t F16, float* a) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t b = (uint32_t)((w >> (12 * i)) & 63u) | ((uint32_t)((w >> (12 * i + 6)) & 63u) << 8);
    uint32_t h2;
    if constexpr (DEC == ENC_E2M3)
      asm("cvt.rn.f16x2.e2m3x2 %0, %1;" : "=r"(h2) : "h"((uint16_t)b));
    else
      asm("cvt.rn.f16x2.e3m2x2 %0, %1;" : "=r"(h2) : "h"((uint16_t)b));
    fma2_f16(h2, F16, a[2 * i], a[2 * i + 1]);
  }
}

// 8 sign-magnitude INT8 codes -> acc += (+-mag) * 2^s (mag <= 127: f16-exact).
// Per 4 codes: the magnitudes become f16 0x64XX = 1024 + mag by one byte
// permute per pair, one HADD2 removes the 1024 exactly, and the code's sign
// bit is permuted into bit 15 of its half.
__device__ __forceinline__ void int8_group_fma(uint64_t w, uint16_t F16, float* a) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const uint32_t v = (uint32_t)(w >> (32 * k));
    const uint32_t m = v & 0x7f7f7f7fu;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      // bytes [c(2p), 0x64, c(2p+1), 0x64] and [0, c(2p), 0, c(2p+1)]
      const uint32_t biased = __byte_perm(m, 0x64646464u, p ? 0x4342u : 0x4140u);
      const uint32_t signs = __byte_perm(v, 0u, p ? 0x3424u : 0x1404u) & 0x80008000u;
      uint32_t h2;
      asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(h2) : "r"(biased), "r"(0x64006400u));
      fma2_f16(h2 ^ signs, F16, a[4 * k + 2 * p], a[4 * k + 2 * p + 1]);
    }
  }
}

// 2^s as f16 bits, s in [-24, 15]
// 8 FP5 E2M2 codes (40 bits) -> acc += g * 2^s: each code is re-laid as
// the FP6 E3M2 code s|0e|m (value g/4, see encode8) and converted in pairs
// by cvt.rn.f16x2.e3m2x2; F16 carries 2^(s+2)
__device__ __forceinline__ void fp5_group_fma(uint64_t w, uint16_t F16, float* a) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t c0 = (uint32_t)(w >> (10 * i)) & 31u;
    const uint32_t c1 = (uint32_t)(w >> (10 * i + 5)) & 31u;
    const uint32_t b = (((c0 & 0x10u) << 1) | (c0 & 0xFu)) |
                       ((((c1 & 0x10u) << 1) | (c1 & 0xFu)) << 8);
    uint32_t h2;
    asm("cvt.rn.f16x2.e3m2x2 %0, %1;" : "=r"(h2) : "h"((uint16_t)b));
    fma2_f16(h2, F16, a[2 * i], a[2 * i + 1]);
  }
}

__device__ __forceinline__ uint16_t pow2_f16(int s) {
  return (uint16_t)(s >= -14 ? (uint32_t)(s + 15) << 10 : 1u << (s + 24));
}

template <int B, int DEC, int BITS, int VPL = kVPL>
__device__ __forceinline__ void decode_rank(const RankLoad<B, BITS, VPL>& r, const Fmt& f,
                                            float* acc, bool plain, const float* lut) {
  constexpr int NSB = Geo<B, VPL>::NSB;
  constexpr int GPB = Geo<B, VPL>::SBV / 8;  // 8-value groups per owned block
#pragma unroll
  for (int sb = 0; sb < NSB; ++sb) {
    const int stored = r.st[sb];
    const int s = stored - f.sbias;
    if constexpr (DEC == ENC_E2M1 || DEC == ENC_E2M3 || DEC == ENC_E3M2 || DEC == ENC_INT ||
                  DEC == ENC_E2M2) {
      // f16 fast path: 2^s representable in f16 (|s| covers every block of
      // real activations); g*2^s is then always an exact f32.  E2M2 decodes
      // g/4, so its scale is 2^(s+2)
      constexpr int SH = DEC == ENC_E2M2 ? 2 : 0;
      if (!plain && stored != 0 && s + SH >= -24 && s + SH <= 15) {
        const uint16_t F16 = pow2_f16(s + SH);
#pragma unroll
        for (int g = 0; g < GPB; ++g) {
          const uint64_t w = get_group<BITS, VPL>(r.c, sb * GPB + g);
          float* a = acc + 8 * (sb * GPB + g);
          if constexpr (DEC == ENC_E2M1) e2m1_word_fma((uint32_t)w, F16, a);
          else if constexpr (DEC == ENC_INT) int8_group_fma(w, F16, a);
          else if constexpr (DEC == ENC_E2M2) fp5_group_fma(w, F16, a);
          else fp6_group_fma<DEC>(w, F16, a);
        }
        continue;
      }
    }
    // g*2^s exactly representable -> one FFMA is exactly acc + value
    const bool fast = !plain && stored != 0 && s >= f.s_fast_lo && s <= f.s_fast_hi;
    if (fast) {
      const float F = pow2f(s);
#pragma unroll
      for (int g = 0; g < GPB; ++g) {
        const uint64_t w = get_group<BITS, VPL>(r.c, sb * GPB + g);
        float* a = acc + 8 * (sb * GPB + g);
        if constexpr (DEC == ENC_E2M1) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float2 v = e2m1x2_to_f32x2(((uint32_t)w >> (8 * j)) & 0xffu);
            a[2 * j] = fmaf(v.x, F, a[2 * j]);
            a[2 * j + 1] = fmaf(v.y, F, a[2 * j + 1]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            a[i] = fmaf(lut[(uint32_t)(w >> (i * BITS)) & ((1u << BITS) - 1u)], F, a[i]);
        }
      }
    } else {
#pragma unroll
      for (int g = 0; g < GPB; ++g)
        decode8_acc<DEC, BITS>(get_group<BITS, VPL>(r.c, sb * GPB + g), stored, f,
                               acc + 8 * (sb * GPB + g), plain, lut);
    }
  }
}

// residual + round(acc), rounded: the unfused `out = sum; out = residual + out`
template <typename OutT>
__device__ __forceinline__ float add_residual(float acc, OutT r) {
  return __fadd_rn(InTraits<OutT>::to_f32(from_f32<OutT>(acc)), InTraits<OutT>::to_f32(r));
}

// coherent 256-bit load (the residual may alias this kernel's output)
__device__ __forceinline__ void ld256_coherent(const void* p, uint32_t* r) {
  asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "l"(p)
               : "memory");
}

template <typename OutT, int VPL = kVPL>
__device__ __forceinline__ void store_lane_out(OutT* out, int valid, float* acc,
                                               const OutT* res = nullptr) {
  if (valid == VPL) {
    uint32_t o[8];
    if (res != nullptr) {  // fold the residual in, 16 (8) values per 256-bit load
      constexpr int PER = 32 / sizeof(OutT);
#pragma unroll
      for (int h = 0; h < VPL / PER; ++h) {
        ld256_coherent(res + PER * h, o);
        const OutT* rv = reinterpret_cast<const OutT*>(o);
#pragma unroll
        for (int i = 0; i < PER; ++i) acc[PER * h + i] = add_residual<OutT>(acc[PER * h + i], rv[i]);
      }
    }
    if constexpr (sizeof(OutT) == 2) {
#pragma unroll
      for (int h = 0; h < VPL / 16; ++h) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          o[i] = pack2<OutT>(acc[16 * h + 2 * i], acc[16 * h + 2 * i + 1]);
        stg256(out + 16 * h, o);
      }
    } else {
#pragma unroll
      for (int h = 0; h < VPL / 8; ++h) {
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = __float_as_uint(acc[8 * h + i]);
        stg256(out + 8 * h, o);
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < VPL; ++i)
      if (i < valid)
        out[i] = from_f32<OutT>(res != nullptr ? add_residual<OutT>(acc[i], res[i]) : acc[i]);
  }
}

// K2 works on 16 values per lane (a 512-value unit per warp): the fp32
// accumulators are half as many registers, so twice the warps are resident,
// and the next unit's first two ranks are prefetched while this one decodes.
constexpr int kVPL2 = 16;
constexpr int kUnit2 = 32 * kVPL2;

__device__ __forceinline__ UnitPos unit_pos2(uint32_t u, uint32_t upc, bool one_chunk, int64_t cv,
                                             int64_t n) {
  UnitPos p;
  uint32_t chunk = one_chunk ? 0u : u / upc;
  p.chunk = (int)chunk;
  p.cbase = (int64_t)chunk * cv;
  p.uoff = (int64_t)(u - chunk * upc) * kUnit2;
  int64_t len = one_chunk ? n : min(cv, n - p.cbase);
  p.uvalid = (int)min((int64_t)kUnit2, len - p.uoff);
  return p;
}

template <typename OutT, int B, int DEC, int BITS>
__global__ void __launch_bounds__(kThreads) k_dqsum(const DArgs A) {
  using RL = RankLoad<B, BITS, kVPL2>;
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
  const int nr = A.nranks;
  uint32_t u = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (u >= total) return;
  UnitPos p = unit_pos2(u, upc, one, A.cv, A.n);
  int valid = max(0, min(kVPL2, p.uvalid - lane * kVPL2));
  const uint8_t* base = A.in + (int64_t)p.chunk * A.chunk_stride;
  RL c0, c1;  // ranks 0 and 1 of the current unit
  load_rank<B, BITS, kVPL2>(c0, base, A.scale_off, A.elem_off, p.uoff, lane, valid, f.kbits);
  if (nr > 1)
    load_rank<B, BITS, kVPL2>(c1, base + A.rank_stride, A.scale_off, A.elem_off, p.uoff, lane,
                              valid, f.kbits);
  while (true) {
    // prefetch ranks 0/1 of the next unit
    const uint32_t un = u + nw;
    const bool more = un < total;
    UnitPos pn = p;
    int validn = 0;
    RL n0, n1;
    if (more) {
      pn = unit_pos2(un, upc, one, A.cv, A.n);
      validn = max(0, min(kVPL2, pn.uvalid - lane * kVPL2));
      const uint8_t* bn = A.in + (int64_t)pn.chunk * A.chunk_stride;
      load_rank<B, BITS, kVPL2>(n0, bn, A.scale_off, A.elem_off, pn.uoff, lane, validn, f.kbits);
      if (nr > 1)
        load_rank<B, BITS, kVPL2>(n1, bn + A.rank_stride, A.scale_off, A.elem_off, pn.uoff, lane,
                                  validn, f.kbits);
    }
    float acc[kVPL2];
#pragma unroll
    for (int i = 0; i < kVPL2; ++i) acc[i] = 0.f;  // +0.0 (mx/netbench.py:332)
    decode_rank<B, DEC, BITS, kVPL2>(c0, f, acc, plain, s_lut);
    if (nr > 1) decode_rank<B, DEC, BITS, kVPL2>(c1, f, acc, plain, s_lut);
    const uint8_t* b = A.in + (int64_t)p.chunk * A.chunk_stride + 2 * A.rank_stride;
    for (int rk = 2; rk < nr; ++rk, b += A.rank_stride) {  // ranks 2.. in order
      RL r;
      load_rank<B, BITS, kVPL2>(r, b, A.scale_off, A.elem_off, p.uoff, lane, valid, f.kbits);
      decode_rank<B, DEC, BITS, kVPL2>(r, f, acc, plain, s_lut);
    }
    if (valid > 0) {
      const int64_t o = p.cbase + p.uoff + lane * kVPL2;
      store_lane_out<OutT, kVPL2>(reinterpret_cast<OutT*>(A.out) + o, valid, acc,
                                  A.residual ? reinterpret_cast<const OutT*>(A.residual) + o
                                             : nullptr);
    }
    if (!more) break;
    u = un;
    p = pn;
    valid = validn;
    c0 = n0;
    c1 = n1;
  }
}

// K2 lean form for the common case -- equal chunks of whole 1024-value
// units (one chunk: n % 1024 == 0; two-shot: chunk size % 1024 == 0), E8M0
// scales (accumulate mode, or plain decode as accumulation from -0.0): one 1024-value unit per warp (32 values per
// lane, the quantiser's layout), no chunk / tail / generic-scale logic, the
// ranks' codes loaded two at a time before their decode.  A flat grid of
// one unit per warp lets the block scheduler balance the waves.
// 128-thread CTAs, 8 resident (64 registers): the same 32 warps per SM as
// 256 x 4, scheduled at half the granularity -- the tail wave balances
// better (scripts/kdq_probe.cu: 8B 5.96 -> 5.51 us, 70B 19.2 -> 17.9 us,
// 8 ranks 12.3 -> 11.6 us)
constexpr int kLeanThreads2 = 128;
constexpr int kLeanWarps2 = kLeanThreads2 / 32;
// the 8-CTA (64-register) bound is spill-free for the FP4 decode of E8M0
// shards into 16-bit outputs; other decoders, packed k-bit scales and f32
// outputs choose their own registers
template <typename OutT, int DEC, int KB>
constexpr int dq_minb() {
  return ((DEC == ENC_E2M1 || DEC == ENC_E2M2 || DEC == ENC_E2M3 || DEC == ENC_E3M2 ||
           DEC == ENC_INT) &&
          sizeof(OutT) == 2) ? 8 : 1;
}

template <typename OutT, int B, int DEC, int BITS, int KB = 8>
__global__ void __launch_bounds__(kLeanThreads2, dq_minb<OutT, DEC, KB>()) k_dqsum_lean(const DArgs A) {
  using RL = RankLoad<B, BITS, kVPL>;
  pdl_prologue();
  __shared__ float s_lut[DEC == ENC_E2M1 ? 1 : 256];
  const Fmt f = A.f;
  if constexpr (DEC != ENC_E2M1) {
    fill_lut(s_lut, f);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const uint32_t u = blockIdx.x * kLeanWarps2 + (threadIdx.x >> 5);
  if (u >= (uint32_t)(A.n / kUnit)) return;
  // equal chunks of whole units: unit u is flat unit u of the output
  const uint32_t upc = (uint32_t)(A.cv / kUnit);
  const uint32_t chunk = u / upc;
  const int64_t uoff = (int64_t)(u - chunk * upc) * kUnit;
  const int nr = A.nranks;
  // sums start at +0.0 (mx/netbench.py:332); a plain decode (one shard,
  // decompress_tensor) starts at -0.0, which makes acc + v == v for every v
  // including -0, so it shares the accumulate code paths exactly
  const float z = A.plain ? -0.f : 0.f;
  float acc[kVPL];
#pragma unroll
  for (int i = 0; i < kVPL; ++i) acc[i] = z;
  const uint8_t* b = A.in + (size_t)chunk * A.chunk_stride;
  for (int r = 0; r < nr; r += 2, b += 2 * A.rank_stride) {
    RL x0, x1;
    load_rank<B, BITS, kVPL>(x0, b, A.scale_off, A.elem_off, uoff, lane, kVPL, KB);
    if (r + 1 < nr)
      load_rank<B, BITS, kVPL>(x1, b + A.rank_stride, A.scale_off, A.elem_off, uoff, lane, kVPL,
                               KB);
    decode_rank<B, DEC, BITS, kVPL>(x0, f, acc, false, s_lut);
    if (r + 1 < nr) decode_rank<B, DEC, BITS, kVPL>(x1, f, acc, false, s_lut);
  }
  const size_t o = (size_t)u * kUnit + lane * kVPL;
  store_lane_out<OutT, kVPL>(reinterpret_cast<OutT*>(A.out) + o, kVPL, acc,
                             A.residual ? reinterpret_cast<const OutT*>(A.residual) + o : nullptr);
}

// ---------------------------------------------------------------------------
// K3: two-shot middle step -- sum N shards of one chunk, re-quantise
// ---------------------------------------------------------------------------
template <int B, int ENC, int BITS>
__global__ void __launch_bounds__(kThreads) k_requant(const RArgs A) {
  constexpr int DEC = dec_of(ENC, BITS);
  pdl_prologue();
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

// fused one-shot (k_fused.cu): quantise N local partials, grid barrier,
// dequant-sum -- one persistent launch
struct FArgs {
  const void* const* partials;  // device array: nranks partial pointers
  int nranks;
  int64_t n;
  uint8_t* shards;              // nranks x shard_stride bytes
  int64_t shard_stride;
  int64_t scale_off, elem_off;  // shard layout for n values
  void* out;
  unsigned int* bar;            // {arrive count, generation}, zero-initialised once
  unsigned long long* nonfinite;
  Fmt f;
};

bool launch_fused_oneshot(const FArgs& a, int out_is_bf16, int block, int enc, int bits,
                          cudaStream_t st);

// multi-GPU fused one-shot over symmetric (peer-mapped) memory (k_fused.cu)
struct SArgs {
  const void* x;                 // this rank's bf16 partial (n values)
  int64_t n;                     // multiple of 1024
  uint8_t* const* bufs;          // device array [nranks]: peer buffer bases
  unsigned int* const* flags;    // device array [nranks]: peer flag arrays (u32 x nranks x ctas)
  int rank, nranks;
  int64_t slot_stride;           // bytes of one shard slot (2 slots per buffer)
  int64_t scale_off, elem_off;   // shard layout for n values
  void* out;
  const void* residual;          // nullable: out = residual + sum (see DArgs)
  unsigned int* status;          // local u32: set to 1 if a peer wait timed out
  unsigned int* epoch;           // local u32 per CTA, advanced once per call
  unsigned long long* nonfinite;
  Fmt f;
  int full_fence;                // 1: extra fence.sc.sys around the flags (MXB200_SYMM_FENCE=1)
  unsigned long long timeout_ns; // peer flag wait limit (MXB200_SYMM_TIMEOUT_MS)
};
// the consumer of the GEMM + all-gather push (k_push.cu)
struct PArgs {
  const uint8_t* buf;            // this rank's symmetric buffer base
  int64_t slot_stride, shard_stride, scale_off, elem_off;
  int nranks, rank;
  int64_t n;                     // multiple of 1024
  const unsigned int* flags;     // this rank's flag array: peer j's GEMM releases [j] = epoch
  const unsigned int* state;     // local [0]: this call's epoch (set by this rank's GEMM)
  unsigned int* status;          // local u32: 1 if a peer wait timed out
  unsigned long long timeout_ns;
  void* out;
  const void* residual;          // nullable, out's dtype (see DArgs)
  Fmt f;
};
// enc: ENC_* of the element format; the push set is fp4_e2m1 E8M0 (B 16 / 32)
// and E5M0 (B 8 / 16 / 32), fp5_e2m2 E5M0 (B 32) -- false outside it
bool launch_push_dqsum(const PArgs& a, int out_is_bf16, int block, int enc, cudaStream_t st);
// two-shot push (k_push.cu): the GEMM scatters chunk j of its shard to rank
// j (reduce-scatter leg), k_push2_requant sums + requantises this rank's
// chunk and pushes it to every rank (all-gather leg), k_push2_decode decodes
struct P2Args {
  const uint8_t* buf;            // this rank's symmetric buffer base
  int64_t slot_stride;           // 2 x nranks chunk shards (RS region, then AG region)
  int64_t shard_stride;          // one chunk shard (c values)
  int64_t scale_off, elem_off;   // chunk shard layout
  int nranks, rank;
  int64_t n, c;                  // c = n / nranks, multiple of 1024
  uint8_t* const* peer_bufs;     // device [nranks]: every rank's buffer base
  unsigned int* const* peer_flags;  // device [nranks]: flag arrays (RS [nranks], AG [nranks])
  const unsigned int* flags;     // this rank's flag array
  unsigned int* state;           // local [0]: this call's epoch (set by this rank's GEMM),
                                 // [2]: the requantiser's CTA arrival counter
  unsigned int* status;
  unsigned long long timeout_ns;
  unsigned long long* nonfinite;
  void* out;
  const void* residual;
  Fmt f;
};
bool launch_push2_requant(const P2Args& a, int block, int enc, cudaStream_t st);
bool launch_push2_decode(const P2Args& a, int out_is_bf16, int block, int enc, cudaStream_t st);

// two-shot over symmetric memory (k_fused.cuh, k_symm2_flow)
struct S2Args {
  const void* x;                 // this rank's bf16 partial (n values)
  int64_t n, c;                  // c = n / nranks, multiple of 1024
  uint8_t* const* bufs;          // device array [nranks]: peer buffer bases
  unsigned int* const* flags;    // device array [nranks]: peer flag arrays (2 x nranks x ctas)
  int rank, nranks;
  int64_t slot_stride;           // bytes of one slot: (nranks + 1) chunk shards
  int64_t shard_stride;          // bytes of one chunk shard
  int64_t scale_off, elem_off;   // chunk shard layout (c values)
  void* out;
  const void* residual;          // nullable: out = residual + sum (see DArgs)
  unsigned int* status;
  unsigned int* epoch;           // local u32 per CTA
  unsigned long long* nonfinite;
  Fmt f;
  int full_fence;
  unsigned long long timeout_ns;
};
bool launch_symm_twoshot(const S2Args& a, int out_is_bf16, int block, int enc, int bits,
                         cudaStream_t st);
// CTAs of the symmetric-memory kernel for n values (one 1024-value unit per warp)
// (capped: each CTA then loops over several unit rows, so one flag exchange
// -- one system-scope release -- covers more bytes; MXB200_SYMM_CTAS overrides)
inline int64_t symm_ctas(int64_t n) {
  static int64_t cap = -1;
  if (cap < 0) {
    const char* e = getenv("MXB200_SYMM_CTAS");
    cap = e ? atoll(e) : 592;  // 148 SMs x 4 resident CTAs of k_symm_flow
    if (cap < 1) cap = 1;
  }
  const int64_t g = (n / kUnit + kWarps - 1) / kWarps;
  return g < cap ? g : cap;
}
bool launch_symm_oneshot(const SArgs& a, int out_is_bf16, int block, int enc, int bits,
                         cudaStream_t st);

// launchers (one translation unit per dtype, compiled in parallel)
void launch_quant_bf16(const QArgs& a, int block, int enc, int bits, cudaStream_t st);
void launch_quant_f16(const QArgs& a, int block, int enc, int bits, cudaStream_t st);
void launch_quant_f32(const QArgs& a, int block, int enc, int bits, cudaStream_t st);
void launch_dqsum_bf16(const DArgs& a, int block, int enc, int bits, cudaStream_t st);
void launch_dqsum_f16(const DArgs& a, int block, int enc, int bits, cudaStream_t st);
void launch_dqsum_f32(const DArgs& a, int block, int enc, int bits, cudaStream_t st);
void launch_requant(const RArgs& a, int block, int enc, int bits, cudaStream_t st);
int64_t launch_quant_tma(const QArgs& a, int dtype_is_bf16, int block, int enc, int bits,
                         cudaStream_t st);

// comparison codecs (k_baselines.cu, mx/baselines.py); dtype codes of mxb200.h
int64_t topk_workspace_bytes(int64_t n);
void launch_chanint_compress(const void* x, int dtype, int64_t rows, int64_t C, int bits,
                             uint16_t* scales, uint8_t* codes, void* ws,
                             unsigned long long* nf, cudaStream_t st);
void launch_chanint_decompress(const uint16_t* scales, const uint8_t* codes, int64_t n, int64_t C,
                               int bits, void* out, int out_dtype, cudaStream_t st);
void launch_topk_compress(const void* x, int dtype, int64_t n, int64_t k, uint32_t* idx,
                          uint16_t* val, void* ws, unsigned long long* nf, cudaStream_t st);
void launch_topk_decompress(const uint32_t* idx, const uint16_t* val, int64_t k, int64_t n,
                            void* out, int out_dtype, cudaStream_t st);

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

template <typename InT, int B, int ENC, int BITS>
inline void launch_quant(const QArgs& a, cudaStream_t st) {
  const dim3 grid((unsigned)((a.total_units + kWarps - 1) / kWarps));
  if (quant_lean_ok(a) && a.f.kbits == 8) {
    launch_pdl(k_quant_lean<InT, B, ENC, BITS, lean_minb<InT, ENC>(), 8>, grid, dim3(kThreads),
               0, st, a);
    return;
  }
  if constexpr (lean_k_ok(ENC)) {  // E5M0 scales: the paper's selected schemes
    if (quant_lean_ok(a) && a.f.kbits == 5) {
      launch_pdl(k_quant_lean<InT, B, ENC, BITS, lean_minb<InT, ENC>(), 5>, grid,
                 dim3(kThreads), 0, st, a);
      return;
    }
  }
  auto k = k_quant<InT, B, ENC, BITS>;
  launch_pdl(k, dim3(work_grid(k, a.total_units, 1)), dim3(kThreads), 0, st, a);
}

}  // namespace mxb
