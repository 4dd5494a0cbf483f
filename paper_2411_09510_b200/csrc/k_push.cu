// The consumer half of the GEMM + all-gather push (k_gemm.cu, PUSH = true):
// every rank's GEMM epilogue has written its MX shard into slot (epoch & 1)
// of THIS rank's symmetric buffer over NVLink, and its last CTA has
// published the epoch into flag [rank] of every rank (one system fence).
// This launch waits for the N flags (acquire, system scope; a wait past the
// timeout sets a status word instead of hanging),
// then decodes the N local shards in rank order, fp32 from +0.0
// (mx/netbench.py:332-334), into bf16 / f32, with the optional residual
// add fused into the store -- K2's arithmetic, so the result is
// bit-identical to the NCCL one-shot.  The shard bytes arrived during this
// kernel's lifetime: coherent (ld.global.cg) loads only.
#include "mx_kernels.cuh"

namespace mxb {
namespace {

__device__ __forceinline__ unsigned int ld_acquire_sys_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// wait (threads < nr) until flags[j] >= epoch for every j, then bar.sync:
// the acquiring threads' view covers the whole CTA
__device__ __forceinline__ void wait_flags(const unsigned int* flags, int nr, unsigned int e,
                                           unsigned int* status, unsigned long long timeout_ns) {
  if ((int)threadIdx.x < nr) {
    const unsigned int* fl = flags + threadIdx.x;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while ((int)(ld_acquire_sys_u32(fl) - e) < 0) {
      __nanosleep(64);
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        atomicExch(status, 1u);
        break;
      }
    }
  }
  __syncthreads();
}

template <typename OutT, int B, int ENC, int BITS, int KB>
__global__ void __launch_bounds__(kLeanThreads2, 8) k_push_dqsum(const PArgs P) {
  constexpr int DEC = dec_of(ENC, BITS);
  using RL = RankLoad<B, BITS, kVPL>;
  __shared__ float s_lut[DEC == ENC_E2M1 ? 1 : 256];
  if constexpr (DEC != ENC_E2M1) fill_lut(s_lut, P.f);  // visible after the wait's barrier
  pdl_prologue();  // this rank's GEMM (same stream) is complete: state[0] = epoch
  __shared__ unsigned int s_e;
  if (threadIdx.x == 0) s_e = *reinterpret_cast<const volatile unsigned int*>(P.state);
  __syncthreads();
  const unsigned int e = s_e;
  wait_flags(P.flags, P.nranks, e, P.status, P.timeout_ns);
  const int lane = threadIdx.x & 31;
  const uint32_t u = blockIdx.x * kLeanWarps2 + (threadIdx.x >> 5);
  if (u >= (uint32_t)(P.n / kUnit)) return;
  const uint8_t* base = P.buf + (int64_t)(e & 1u) * P.slot_stride;
  const Fmt f = P.f;
  float acc[kVPL];
#pragma unroll
  for (int i = 0; i < kVPL; ++i) acc[i] = 0.f;  // +0.0 (mx/netbench.py:332)
  const int nr = P.nranks;
  for (int r = 0; r < nr; r += 2) {
    RL x0, x1;
    load_rank<B, BITS, kVPL, true>(x0, base + (int64_t)r * P.shard_stride, P.scale_off,
                                   P.elem_off, (int64_t)u * kUnit, lane, kVPL, KB);
    if (r + 1 < nr)
      load_rank<B, BITS, kVPL, true>(x1, base + (int64_t)(r + 1) * P.shard_stride, P.scale_off,
                                     P.elem_off, (int64_t)u * kUnit, lane, kVPL, KB);
    decode_rank<B, DEC, BITS, kVPL>(x0, f, acc, false, s_lut);
    if (r + 1 < nr) decode_rank<B, DEC, BITS, kVPL>(x1, f, acc, false, s_lut);
  }
  const size_t o = (size_t)u * kUnit + lane * kVPL;
  store_lane_out<OutT, kVPL>(reinterpret_cast<OutT*>(P.out) + o, kVPL, acc,
                             P.residual ? reinterpret_cast<const OutT*>(P.residual) + o
                                        : nullptr);
}

template <int B, int ENC, int BITS, int KB>
__device__ __forceinline__ void requant_unit(const P2Args& P, unsigned int e, uint32_t q,
                                             int lane, const float* s_lut) {
  constexpr int DEC = dec_of(ENC, BITS);
  constexpr int NSB = Geo<B>::NSB;
  using RL = RankLoad<B, BITS, kVPL>;
  const int nr = P.nranks;
  const int64_t slot = (int64_t)(e & 1u) * P.slot_stride;
  const uint8_t* rs = P.buf + slot;
  const Fmt f = P.f;
  float acc[kVPL];
#pragma unroll
  for (int i = 0; i < kVPL; ++i) acc[i] = 0.f;  // +0.0 (mx/netbench.py:332)
  for (int r = 0; r < nr; r += 2) {
    RL x0, x1;
    load_rank<B, BITS, kVPL, true>(x0, rs + (int64_t)r * P.shard_stride, P.scale_off, P.elem_off,
                                   (int64_t)q * kUnit, lane, kVPL, KB);
    if (r + 1 < nr)
      load_rank<B, BITS, kVPL, true>(x1, rs + (int64_t)(r + 1) * P.shard_stride, P.scale_off,
                                     P.elem_off, (int64_t)q * kUnit, lane, kVPL, KB);
    decode_rank<B, DEC, BITS, kVPL>(x0, f, acc, false, s_lut);
    if (r + 1 < nr) decode_rank<B, DEC, BITS, kVPL>(x1, f, acc, false, s_lut);
  }
  Raw<float> raw;
#pragma unroll
  for (int i = 0; i < kVPL; ++i) raw.w[i] = __float_as_uint(acc[i]);
  int stored[NSB];
  bool bad;
  LaneCodes<BITS> cc = quant_lane<float, B, ENC, BITS>(raw, f, stored, bad);
  if (bad)
    report_nonfinite_raw<float>(raw, kVPL, (int64_t)P.rank * P.c + (int64_t)q * kUnit + lane * kVPL,
                                P.nonfinite);
  const int64_t ag = slot + (int64_t)nr * P.shard_stride + (int64_t)P.rank * P.shard_stride;
  [[maybe_unused]] uint64_t pk = 0;
  if constexpr (KB != 8) pk = pack_unit_scales_k<B>(stored, lane, KB);  // warp-collective
  for (int j = 0; j < nr; ++j) {
    uint8_t* dst = P.peer_bufs[j] + ag;
    store_lane_codes<BITS>(dst + P.elem_off + (int64_t)q * (kUnit / 8 * BITS) + lane * (4 * BITS),
                           cc, kVPL);
    if constexpr (KB != 8) {
      constexpr int G = scale_group_lanes<B>();
      if (lane % G == 0) {
        uint8_t* sp = dst + P.scale_off + ((int64_t)q * (kUnit / B) / 8 + lane / G) * KB;
#pragma unroll
        for (int i = 0; i < KB; ++i) sp[i] = (uint8_t)(pk >> (8 * i));
      }
    } else {
      uint8_t* sp = dst + P.scale_off + (int64_t)q * (kUnit / B) + lane * NSB;
      if constexpr (NSB == 4)
        *reinterpret_cast<uint32_t*>(sp) = (uint32_t)stored[0] | ((uint32_t)stored[1] << 8) |
                                           ((uint32_t)stored[2] << 16) |
                                           ((uint32_t)stored[3] << 24);
      else if constexpr (NSB == 2)
        *reinterpret_cast<uint16_t*>(sp) = (uint16_t)(stored[0] | (stored[1] << 8));
      else
        *sp = (uint8_t)stored[0];
    }
  }
}

// reduce-scatter leg done everywhere -> this rank's chunk: N shards decoded
// in rank order, fp32 sum from +0.0, re-quantised (K3's arithmetic) and
// pushed into every rank's all-gather region
template <int B, int ENC, int BITS, int KB>
__global__ void __launch_bounds__(kLeanThreads2) k_push2_requant(const P2Args P) {
  constexpr int DEC = dec_of(ENC, BITS);
  __shared__ float s_lut[DEC == ENC_E2M1 ? 1 : 256];
  if constexpr (DEC != ENC_E2M1) fill_lut(s_lut, P.f);  // visible after the wait's barrier
  pdl_prologue();
  __shared__ unsigned int s_e;
  if (threadIdx.x == 0) s_e = *reinterpret_cast<const volatile unsigned int*>(P.state);
  __syncthreads();
  const unsigned int e = s_e;
  const int nr = P.nranks;
  wait_flags(P.flags, nr, e, P.status, P.timeout_ns);  // RS flags [0, nr): every GEMM's chunk
  const int lane = threadIdx.x & 31;
  const uint32_t q = blockIdx.x * kLeanWarps2 + (threadIdx.x >> 5);
  if (q < (uint32_t)(P.c / kUnit)) requant_unit<B, ENC, BITS, KB>(P, e, q, lane, s_lut);
  // the last CTA to finish publishes the all-gather leg: AG flag [nr + rank]
  // of every rank, one system fence (the GEMM's pattern)
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int prev;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;"
                 : "=r"(prev) : "l"(P.state + 2) : "memory");
    if (prev == gridDim.x - 1) {
      P.state[2] = 0u;
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      for (int j = 0; j < nr; ++j)
        asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(P.peer_flags[j] + nr + P.rank),
                     "r"(e)
                     : "memory");
    }
  }
}

// all-gather leg done everywhere -> decode every owner's reduced chunk
template <typename OutT, int B, int ENC, int BITS, int KB>
__global__ void __launch_bounds__(kLeanThreads2, 8) k_push2_decode(const P2Args P) {
  constexpr int DEC = dec_of(ENC, BITS);
  using RL = RankLoad<B, BITS, kVPL>;
  __shared__ float s_lut[DEC == ENC_E2M1 ? 1 : 256];
  if constexpr (DEC != ENC_E2M1) fill_lut(s_lut, P.f);  // visible after the wait's barrier
  pdl_prologue();
  __shared__ unsigned int s_e;
  if (threadIdx.x == 0) s_e = *reinterpret_cast<const volatile unsigned int*>(P.state);
  __syncthreads();
  const unsigned int e = s_e;
  const int nr = P.nranks;
  wait_flags(P.flags + nr, nr, e, P.status, P.timeout_ns);  // AG flags [nr, 2 nr)
  const int lane = threadIdx.x & 31;
  const uint32_t u = blockIdx.x * kLeanWarps2 + (threadIdx.x >> 5);
  if (u >= (uint32_t)(P.n / kUnit)) return;
  const uint32_t upc = (uint32_t)(P.c / kUnit);
  const uint32_t j = u / upc, q = u - j * upc;
  const uint8_t* base = P.buf + (int64_t)(e & 1u) * P.slot_stride +
                        (int64_t)(nr + (int)j) * P.shard_stride;
  RL x;
  load_rank<B, BITS, kVPL, true>(x, base, P.scale_off, P.elem_off, (int64_t)q * kUnit, lane, kVPL,
                                 KB);
  float acc[kVPL];
#pragma unroll
  for (int i = 0; i < kVPL; ++i) acc[i] = 0.f;  // K2's two-shot final decode: from +0.0
  decode_rank<B, DEC, BITS, kVPL>(x, P.f, acc, false, s_lut);
  const size_t o = (size_t)u * kUnit + lane * kVPL;
  store_lane_out<OutT, kVPL>(reinterpret_cast<OutT*>(P.out) + o, kVPL, acc,
                             P.residual ? reinterpret_cast<const OutT*>(P.residual) + o
                                        : nullptr);
}

// the push set: (block, element encoding, bits, scale bits)
#define MXB_PUSH_SET(X)        \
  X(32, ENC_E2M1, 4, 8)        \
  X(16, ENC_E2M1, 4, 8)        \
  X(32, ENC_E2M1, 4, 5)        \
  X(16, ENC_E2M1, 4, 5)        \
  X(8, ENC_E2M1, 4, 5)         \
  X(32, ENC_E2M2, 5, 5)

template <typename OutT>
bool go_dqsum(const PArgs& a, int block, int enc, cudaStream_t st) {
  const dim3 grid((unsigned)((a.n / kUnit + kLeanWarps2 - 1) / kLeanWarps2));
  const int kb = a.f.kbits, bits = a.f.bits;
#define X(B_, E_, BT_, KB_)                                                              \
  if (block == B_ && enc == E_ && bits == BT_ && kb == KB_) {                            \
    launch_pdl(k_push_dqsum<OutT, B_, E_, BT_, KB_>, grid, dim3(kLeanThreads2), 0, st, a); \
    return true;                                                                         \
  }
  MXB_PUSH_SET(X)
#undef X
  return false;
}

template <typename OutT>
bool go_decode(const P2Args& a, int block, int enc, cudaStream_t st) {
  const dim3 grid((unsigned)((a.n / kUnit + kLeanWarps2 - 1) / kLeanWarps2));
  const int kb = a.f.kbits, bits = a.f.bits;
#define X(B_, E_, BT_, KB_)                                                                \
  if (block == B_ && enc == E_ && bits == BT_ && kb == KB_) {                              \
    launch_pdl(k_push2_decode<OutT, B_, E_, BT_, KB_>, grid, dim3(kLeanThreads2), 0, st, a); \
    return true;                                                                           \
  }
  MXB_PUSH_SET(X)
#undef X
  return false;
}
}  // namespace

bool launch_push_dqsum(const PArgs& a, int out_is_bf16, int block, int enc, cudaStream_t st) {
  return out_is_bf16 ? go_dqsum<__nv_bfloat16>(a, block, enc, st)
                     : go_dqsum<float>(a, block, enc, st);
}

bool launch_push2_requant(const P2Args& a, int block, int enc, cudaStream_t st) {
  const dim3 grid((unsigned)((a.c / kUnit + kLeanWarps2 - 1) / kLeanWarps2));
  const int kb = a.f.kbits, bits = a.f.bits;
#define X(B_, E_, BT_, KB_)                                                           \
  if (block == B_ && enc == E_ && bits == BT_ && kb == KB_) {                         \
    launch_pdl(k_push2_requant<B_, E_, BT_, KB_>, grid, dim3(kLeanThreads2), 0, st, a); \
    return true;                                                                      \
  }
  MXB_PUSH_SET(X)
#undef X
  return false;
}

bool launch_push2_decode(const P2Args& a, int out_is_bf16, int block, int enc, cudaStream_t st) {
  return out_is_bf16 ? go_decode<__nv_bfloat16>(a, block, enc, st)
                     : go_decode<float>(a, block, enc, st);
}

}  // namespace mxb
