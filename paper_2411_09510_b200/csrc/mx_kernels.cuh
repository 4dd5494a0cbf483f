// sm_100a kernels of the compressed TP all-reduce (arXiv 2411.09510) and
// the C ABI declared in include/mxb200.h.
//
//   K1 k_quant      MX block quantise + bit-pack        (mx/codec.py:140-172, 238-263;
//                                                        mx/bitpack.py:22-34)
//   K2 k_dqsum      unpack + dequantise + fp32 rank-order sum -> bf16/f16/f32
//                                                       (mx/codec.py:175-188, 266-284;
//                                                        mx/netbench.py:329-334)
//   K3 k_requant    K2's sum re-quantised in registers (two-shot middle step)
//   G*              generic kernels for any block size / input alignment
//
// Layout: every CTA owns a TILE of 256 threads x 8 values x U rows of one
// chunk.  A lane holds 8 consecutive values (one 16-byte bf16 load), so a
// warp row covers 256 values = 32*b bytes of element stream, and a block of B
// values is spread over B/8 adjacent lanes whose amax is reduced with
// __shfl_xor_sync.  Scale codes are staged per tile in shared memory and
// packed (k bits each) at the end of the tile.  Everything is HBM-bound: no
// tensor cores (not a contraction).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "mx_device.cuh"

namespace mxb {

enum Enc { ENC_GEN = 0, ENC_E2M1 = 1, ENC_E2M3 = 2, ENC_E3M2 = 3 };

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

struct QArgs {
  const void* x;
  int64_t n;            // total values
  int64_t cv;           // values per chunk
  int tiles_per_chunk;
  uint8_t* scale_base;  // chunk j's scale stream at scale_base + j*chunk_stride
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
  int tiles_per_chunk;
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
  uint8_t* out_scale;
  uint8_t* out_elem;
  unsigned long long* nonfinite;
  Fmt f;
};

// ---------------------------------------------------------------------------
// Row helpers
// ---------------------------------------------------------------------------

// Quantise the 8 values a lane holds (block = LPB adjacent lanes).
// Returns the packed code word (8*b bits) and the block's stored scale code.
template <int LPB, int ENC, int BITS>
__device__ __forceinline__ uint64_t quant8(const float v[8], int valid, int64_t flat0,
                                           const Fmt& f, unsigned long long* nonfinite,
                                           int& stored_out) {
  uint32_t ab = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) ab = max(ab, __float_as_uint(v[i]) & 0x7fffffffu);
#pragma unroll
  for (int o = LPB / 2; o > 0; o >>= 1) ab = max(ab, __shfl_xor_sync(0xffffffffu, ab, o));
  int stored = 0;
  if (ab >= 0x7f800000u) {  // NaN / Inf somewhere in the block (mx/codec.py:191-199)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < valid && (__float_as_uint(v[i]) & 0x7fffffffu) >= 0x7f800000u) {
        if (nonfinite) atomicMin(nonfinite, (unsigned long long)(flat0 + i));
        break;
      }
    ab = 0;
  }
  stored_out = 0;
  if (ab == 0) return 0;  // all-zero block: scale code 0, codes 0 (mx/codec.py:170-171)
  int s = shared_exp32(ab, f);
  stored = s + f.sbias;
  stored_out = stored;
  float inv = pow2f(-s);
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = v[i] * inv;  // exact power-of-two scaling
  uint64_t w = 0;
  if constexpr (ENC == ENC_E2M1) {
#pragma unroll
    for (int i = 0; i < 4; ++i) w |= (uint64_t)cvt_e2m1x2(x[2 * i], x[2 * i + 1]) << (8 * i);
  } else if constexpr (ENC == ENC_E2M3 || ENC == ENC_E3M2) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t p = ENC == ENC_E2M3 ? cvt_e2m3x2(x[2 * i], x[2 * i + 1])
                                   : cvt_e3m2x2(x[2 * i], x[2 * i + 1]);
      w |= (uint64_t)(p & 0x3fu) << (12 * i);
      w |= (uint64_t)((p >> 8) & 0x3fu) << (12 * i + 6);
    }
  } else {
    const int b = BITS ? BITS : f.bits;
#pragma unroll
    for (int i = 0; i < 8; ++i) w |= (uint64_t)encode_gen(x[i], f) << (i * b);
  }
  return w;
}

// Store one lane's packed word (b bytes) of the element stream.
// `row_el` = element-stream pointer of this warp row (4-byte aligned);
// `valid` values of the lane's 8 exist.  Runtime-width rows go through the
// warp's shared staging buffer so the global stores are whole 32-bit words.
template <int BITS>
__device__ __forceinline__ void store_codes(uint8_t* __restrict__ row_el, int lane, uint64_t w,
                                            int valid, int row_valid, int b, uint8_t* stage) {
  if constexpr (BITS == 4) {
    uint8_t* p = row_el + lane * 4;
    if (valid == 8) *reinterpret_cast<uint32_t*>(p) = (uint32_t)w;
    else for (int i = 0; i < (valid * 4 + 7) / 8; ++i) p[i] = (uint8_t)(w >> (8 * i));
  } else if constexpr (BITS == 8) {
    uint8_t* p = row_el + lane * 8;
    if (valid == 8) *reinterpret_cast<uint64_t*>(p) = w;
    else for (int i = 0; i < valid; ++i) p[i] = (uint8_t)(w >> (8 * i));
  } else {
    for (int i = 0; i < b; ++i) stage[lane * b + i] = (uint8_t)(w >> (8 * i));
    __syncwarp();
    int nbytes = (row_valid * b + 7) / 8;
    int nw = nbytes >> 2;
    for (int k = lane; k < nw; k += 32)
      reinterpret_cast<uint32_t*>(row_el)[k] = reinterpret_cast<const uint32_t*>(stage)[k];
    if (lane < (nbytes & 3)) row_el[nw * 4 + lane] = stage[nw * 4 + lane];
    __syncwarp();
  }
}

// Load one lane's b bytes of codes.
template <int BITS>
__device__ __forceinline__ uint64_t load_codes(const uint8_t* __restrict__ row_el, int lane,
                                               int valid, int row_valid, int b, uint8_t* stage) {
  if constexpr (BITS == 4) {
    const uint8_t* p = row_el + lane * 4;
    if (valid == 8) return __ldg(reinterpret_cast<const uint32_t*>(p));
    uint64_t w = 0;
    for (int i = 0; i < (valid * 4 + 7) / 8; ++i) w |= (uint64_t)p[i] << (8 * i);
    return w;
  } else if constexpr (BITS == 8) {
    const uint8_t* p = row_el + lane * 8;
    if (valid == 8) return __ldg(reinterpret_cast<const unsigned long long*>(p));
    uint64_t w = 0;
    for (int i = 0; i < valid; ++i) w |= (uint64_t)p[i] << (8 * i);
    return w;
  } else {
    int nbytes = (row_valid * b + 7) / 8;
    int nw = nbytes >> 2;
    __syncwarp();
    for (int k = lane; k < nw; k += 32)
      reinterpret_cast<uint32_t*>(stage)[k] = __ldg(reinterpret_cast<const uint32_t*>(row_el) + k);
    if (lane < (nbytes & 3)) stage[nw * 4 + lane] = row_el[nw * 4 + lane];
    __syncwarp();
    uint64_t w = 0;
    if (valid > 0) {
      int nb = (valid * b + 7) / 8;
      for (int i = 0; i < nb; ++i) w |= (uint64_t)stage[lane * b + i] << (8 * i);
    }
    return w;
  }
}

// Pack the tile's staged scale codes (one byte each in smem) into k-bit
// groups of 8 blocks = k bytes each.
__device__ __forceinline__ void pack_tile_scales(const uint8_t* s_scale, int nbt, uint8_t* dst,
                                                 int k) {
  int ng = (nbt + 7) / 8;
  for (int g = threadIdx.x; g < ng; g += blockDim.x) {
    uint64_t w = 0;
    int cnt = min(8, nbt - 8 * g);
    for (int i = 0; i < cnt; ++i) w |= (uint64_t)s_scale[8 * g + i] << (i * k);
    uint8_t* p = dst + (int64_t)g * k;
    if (k == 8 && cnt == 8 && ((uintptr_t)p & 7) == 0) {
      *reinterpret_cast<uint64_t*>(p) = w;
    } else {
      int nb = (cnt * k + 7) / 8;
      for (int i = 0; i < nb; ++i) p[i] = (uint8_t)(w >> (8 * i));
    }
  }
}

// ---------------------------------------------------------------------------
// K1: quantise + pack
// ---------------------------------------------------------------------------
template <typename InT, int LPB, int ENC, int BITS, int U>
__global__ void __launch_bounds__(kThreads) k_quant(const QArgs A) {
  constexpr int B = 8 * LPB;
  constexpr int TILE = kThreads * 8 * U;
  __shared__ uint8_t s_scale[TILE / B];
  __shared__ __align__(16) uint8_t s_stage[kWarps][256];
  const int tile = blockIdx.x, chunk = blockIdx.y;
  const int64_t cbase = (int64_t)chunk * A.cv;
  const int64_t len = min(A.cv, A.n - cbase);
  const int64_t t0 = (int64_t)tile * TILE;
  if (t0 >= len) return;
  const InT* __restrict__ x = reinterpret_cast<const InT*>(A.x) + cbase;
  uint8_t* sc = A.scale_base + chunk * A.chunk_stride;
  uint8_t* el = A.elem_base + chunk * A.chunk_stride;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = BITS ? BITS : A.f.bits;

  float v[U][8];
#pragma unroll
  for (int r = 0; r < U; ++r) {
    int64_t g = t0 + (int64_t)(warp * U + r) * 256 + lane * 8;
    int valid = (int)max((int64_t)0, min((int64_t)8, len - g));
    if (valid > 0) load8<InT>(x, g, valid, v[r]);
    else
#pragma unroll
      for (int i = 0; i < 8; ++i) v[r][i] = 0.f;
  }
#pragma unroll
  for (int r = 0; r < U; ++r) {
    int64_t row0 = t0 + (int64_t)(warp * U + r) * 256;
    int64_t g = row0 + lane * 8;
    int valid = (int)max((int64_t)0, min((int64_t)8, len - g));
    int row_valid = (int)max((int64_t)0, min((int64_t)256, len - row0));
    int stored;
    uint64_t w = quant8<LPB, ENC, BITS>(v[r], valid, cbase + g, A.f, A.nonfinite, stored);
    if (row_valid > 0) {
      if ((lane % LPB) == 0 && valid > 0) s_scale[(int)((g - t0) / B)] = (uint8_t)stored;
      uint8_t* row_el = el + (row0 / 8) * b;
      store_codes<BITS>(row_el, lane, w, valid, row_valid, b, s_stage[warp]);
    }
  }
  __syncthreads();
  int nbt = (int)((min((int64_t)TILE, len - t0) + B - 1) / B);
  pack_tile_scales(s_scale, nbt, sc + (t0 / B / 8) * A.f.kbits, A.f.kbits);
}

// ---------------------------------------------------------------------------
// K2: unpack + dequantise + rank-order fp32 sum
// ---------------------------------------------------------------------------
template <int LPB, int DEC, int BITS>
__device__ __forceinline__ void decode_acc(uint64_t w, int stored, const Fmt& f, float acc[8],
                                           bool plain) {
  constexpr int B = 8 * LPB;
  (void)B;
  if constexpr (DEC == ENC_E2M1) {
    E2M1Scale sp = e2m1_scale(stored, f.sbias);
    uint32_t w32 = (uint32_t)w;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float val = (e2m1_raw(w32, i) * sp.P) * sp.F;
      acc[i] = plain ? val : __fadd_rn(acc[i], val);
    }
  } else {
    const int b = BITS ? BITS : f.bits;
    const uint32_t mask = (1u << b) - 1u;
    const bool zero = stored == 0;
    const int s = stored - f.sbias;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float val = decode_gen((uint32_t)(w >> (i * b)) & mask, s, zero, f);
      acc[i] = plain ? val : __fadd_rn(acc[i], val);
    }
  }
}

template <typename OutT, int LPB, int DEC, int BITS, int U>
__global__ void __launch_bounds__(kThreads) k_dqsum(const DArgs A) {
  constexpr int B = 8 * LPB;
  constexpr int TILE = kThreads * 8 * U;
  __shared__ __align__(16) uint8_t s_stage[kWarps][256];
  const int tile = blockIdx.x, chunk = blockIdx.y;
  const int64_t cbase = (int64_t)chunk * A.cv;
  const int64_t len = min(A.cv, A.n - cbase);
  const int64_t t0 = (int64_t)tile * TILE;
  if (t0 >= len) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = BITS ? BITS : A.f.bits;
  const bool plain = A.plain != 0;

  float acc[U][8];
#pragma unroll
  for (int r = 0; r < U; ++r)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[r][i] = 0.f;  // +0.0 (mx/netbench.py:332)

  for (int rk = 0; rk < A.nranks; ++rk) {
    const uint8_t* base = A.in + rk * A.rank_stride + chunk * A.chunk_stride;
    const uint8_t* sc = base + A.scale_off;
    const uint8_t* el = base + A.elem_off;
    uint64_t w[U];
    int st[U];
#pragma unroll
    for (int r = 0; r < U; ++r) {
      int64_t row0 = t0 + (int64_t)(warp * U + r) * 256;
      int64_t g = row0 + lane * 8;
      int valid = (int)max((int64_t)0, min((int64_t)8, len - g));
      int row_valid = (int)max((int64_t)0, min((int64_t)256, len - row0));
      w[r] = 0;
      st[r] = 0;
      if (row_valid > 0) {
        w[r] = load_codes<BITS>(el + (row0 / 8) * b, lane, valid, row_valid, b, s_stage[warp]);
        if (valid > 0) st[r] = read_scale(sc, g / B, A.f.kbits);
      }
    }
#pragma unroll
    for (int r = 0; r < U; ++r) decode_acc<LPB, DEC, BITS>(w[r], st[r], A.f, acc[r], plain);
  }
  OutT* out = reinterpret_cast<OutT*>(A.out) + cbase;
#pragma unroll
  for (int r = 0; r < U; ++r) {
    int64_t g = t0 + (int64_t)(warp * U + r) * 256 + lane * 8;
    int valid = (int)max((int64_t)0, min((int64_t)8, len - g));
    if (valid > 0) store8<OutT>(out, g, valid, acc[r]);
  }
}

// ---------------------------------------------------------------------------
// K3: two-shot middle step -- sum N shards of one chunk, re-quantise
// ---------------------------------------------------------------------------
template <int LPB, int ENC, int BITS, int U>
__global__ void __launch_bounds__(kThreads) k_requant(const RArgs A) {
  constexpr int B = 8 * LPB;
  constexpr int TILE = kThreads * 8 * U;
  __shared__ uint8_t s_scale[TILE / B];
  __shared__ __align__(16) uint8_t s_stage[kWarps][256];
  const int64_t len = A.n;
  const int64_t t0 = (int64_t)blockIdx.x * TILE;
  if (t0 >= len) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = BITS ? BITS : A.f.bits;
  constexpr int DEC = ENC == ENC_E2M1 ? ENC_E2M1 : ENC_GEN;

  float acc[U][8];
#pragma unroll
  for (int r = 0; r < U; ++r)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[r][i] = 0.f;
  for (int rk = 0; rk < A.nranks; ++rk) {
    const uint8_t* base = A.in + rk * A.rank_stride;
    const uint8_t* sc = base + A.scale_off;
    const uint8_t* el = base + A.elem_off;
    uint64_t w[U];
    int st[U];
#pragma unroll
    for (int r = 0; r < U; ++r) {
      int64_t row0 = t0 + (int64_t)(warp * U + r) * 256;
      int64_t g = row0 + lane * 8;
      int valid = (int)max((int64_t)0, min((int64_t)8, len - g));
      int row_valid = (int)max((int64_t)0, min((int64_t)256, len - row0));
      w[r] = 0;
      st[r] = 0;
      if (row_valid > 0) {
        w[r] = load_codes<BITS>(el + (row0 / 8) * b, lane, valid, row_valid, b, s_stage[warp]);
        if (valid > 0) st[r] = read_scale(sc, g / B, A.f.kbits);
      }
    }
#pragma unroll
    for (int r = 0; r < U; ++r) decode_acc<LPB, DEC, BITS>(w[r], st[r], A.f, acc[r], false);
  }
#pragma unroll
  for (int r = 0; r < U; ++r) {
    int64_t row0 = t0 + (int64_t)(warp * U + r) * 256;
    int64_t g = row0 + lane * 8;
    int valid = (int)max((int64_t)0, min((int64_t)8, len - g));
    int row_valid = (int)max((int64_t)0, min((int64_t)256, len - row0));
    // lanes past the end hold +0 sums, exactly like zero padding
    int stored;
    uint64_t w = quant8<LPB, ENC, BITS>(acc[r], valid, g, A.f, A.nonfinite, stored);
    if (row_valid > 0) {
      if ((lane % LPB) == 0 && valid > 0) s_scale[(int)((g - t0) / B)] = (uint8_t)stored;
      store_codes<BITS>(A.out_elem + (row0 / 8) * b, lane, w, valid, row_valid, b, s_stage[warp]);
    }
  }
  __syncthreads();
  int nbt = (int)((min((int64_t)TILE, len - t0) + B - 1) / B);
  pack_tile_scales(s_scale, nbt, A.out_scale + (t0 / B / 8) * A.f.kbits, A.f.kbits);
}


// launchers (one translation unit per dtype, compiled in parallel)
constexpr int kU = 4;  // rows per thread
constexpr int kTile = kThreads * 8 * kU;

void launch_quant_bf16(const QArgs& a, int64_t nchunks, int lpb, int enc, int bits, cudaStream_t st);
void launch_quant_f16(const QArgs& a, int64_t nchunks, int lpb, int enc, int bits, cudaStream_t st);
void launch_quant_f32(const QArgs& a, int64_t nchunks, int lpb, int enc, int bits, cudaStream_t st);
void launch_dqsum_bf16(const DArgs& a, int64_t nchunks, int lpb, int enc, int bits, cudaStream_t st);
void launch_dqsum_f16(const DArgs& a, int64_t nchunks, int lpb, int enc, int bits, cudaStream_t st);
void launch_dqsum_f32(const DArgs& a, int64_t nchunks, int lpb, int enc, int bits, cudaStream_t st);
void launch_requant(const RArgs& a, int lpb, int enc, int bits, cudaStream_t st);

}  // namespace mxb
