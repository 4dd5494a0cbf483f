// Fused one-shot compressed all-reduce in ONE persistent kernel (templates;
// instantiated per output type x block size by k_fused_inst.cu, dispatched
// by k_fused.cu):
//   phase 1  K1: every local partial is quantised into its slot of the
//            gather buffer (the bytes an all-gather would deliver),
//   barrier  grid-wide (all CTAs resident: the grid is one occupancy wave),
//   phase 2  K2: the N shards are decoded and summed in fp32 rank order.
// Two kernel boundaries (~2 us of launch/ramp/drain each at these sizes)
// disappear.  This is the single-device form of the NVLink-pull fused
// collective (peer shards read in phase 2); the per-phase code is exactly the
// K1/K2 code of mx_kernels.cuh, so results are bit-identical to
// quantise -> all-gather -> dequant-sum (mx/netbench.py:323-334).
#pragma once
#include "mx_kernels.cuh"

namespace mxb {

namespace fz {

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Sense-free generation barrier across all CTAs of the grid.
__device__ __forceinline__ void grid_barrier(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int gen = ld_acquire(bar + 1);
    __threadfence();  // release this CTA's phase-1 stores
    const unsigned int arrived = atomicAdd(bar, 1u) + 1u;
    if (arrived == gridDim.x) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (ld_acquire(bar + 1) == gen) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

template <typename InT, typename OutT, int B, int ENC, int BITS>
__global__ void __launch_bounds__(kThreads, 3) k_fused_oneshot(const FArgs F) {
  constexpr int DEC = dec_of(ENC, BITS);
  __shared__ __align__(16) uint8_t s_stage[kWarps][kUnit / 8];
  __shared__ float s_lut[DEC == ENC_E2M1 ? 1 : 256];
  const Fmt f = F.f;
  if constexpr (DEC != ENC_E2M1) fill_lut(s_lut, f);  // visible after the grid barrier
  const int lane = threadIdx.x & 31;
  const uint32_t nw = (uint32_t)(gridDim.x * kWarps);
  const uint32_t gw = blockIdx.x * kWarps + (threadIdx.x >> 5);

  // ---- phase 1: quantise every local partial (K1) ----------------------
  {
    QArgs A;
    A.n = F.n;
    A.cv = F.n;
    A.units_per_chunk = (F.n + kUnit - 1) / kUnit;
    A.total_units = A.units_per_chunk;
    A.chunk_stride = 0;
    A.nonfinite = F.nonfinite;
    A.flat_off = 0;
    A.f = f;
    const uint32_t upp = (uint32_t)A.units_per_chunk;
    const uint32_t nfull = (uint32_t)(F.n / kUnit);
    uint8_t* stage = s_stage[threadIdx.x >> 5];
    // units of all partials in one round-robin sequence u -> (rank, unit);
    // taken in pairs whose loads are both in flight before any math
    const uint32_t total = upp * (uint32_t)F.nranks;
    for (uint32_t u0 = gw; u0 < total; u0 += 2 * nw) {
      const uint32_t u1 = u0 + nw;
      const bool has1 = u1 < total;
      const uint32_t r0 = u0 / upp, q0 = u0 - r0 * upp;
      const uint32_t r1 = has1 ? u1 / upp : r0, q1 = has1 ? u1 - r1 * upp : q0;
      const InT* x0 = reinterpret_cast<const InT*>(F.partials[r0]);
      const InT* x1 = reinterpret_cast<const InT*>(F.partials[r1]);
      const bool full0 = q0 < nfull && f.kbits == 8, full1 = has1 && q1 < nfull && f.kbits == 8;
      Raw<InT> w0, w1;
      if (full0) load_raw<InT>(x0 + (size_t)q0 * kUnit + lane * kVPL, w0);
      if (full1) load_raw<InT>(x1 + (size_t)q1 * kUnit + lane * kVPL, w1);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1 && !has1) break;
        const uint32_t r = h ? r1 : r0, q = h ? q1 : q0;
        A.x = F.partials[r];
        A.scale_base = F.shards + r * F.shard_stride + F.scale_off;
        A.elem_base = F.shards + r * F.shard_stride + F.elem_off;
        if (h ? full1 : full0) {
          quant_full_unit<InT, B, ENC, BITS>(A, f, q, h ? w1 : w0, lane);
        } else {
          UnitPos p = unit_pos(q, upp, true, A.cv, A.n);
          Raw<InT> raw;
          load_unit<InT>(reinterpret_cast<const InT*>(A.x), p, lane, raw);
          quant_unit<InT, B, ENC, BITS>(A, f, p, raw, lane, stage);
        }
      }
    }
  }

  grid_barrier(F.bar);

  // ---- phase 2: decode the N shards in rank order, fp32 sum (K2) -------
  // ranks 0/1 of the next unit are prefetched while this unit decodes;
  // ld.global.cg: the shards were written by other CTAs of this kernel
  {
    using RL = RankLoad<B, BITS, kVPL2>;
    const uint32_t total = (uint32_t)((F.n + kUnit2 - 1) / kUnit2);
    const int nr = F.nranks;
    uint32_t u = gw;
    if (u < total) {
      int64_t uoff = (int64_t)u * kUnit2;
      int valid = max(0, min(kVPL2, (int)min((int64_t)kUnit2, F.n - uoff) - lane * kVPL2));
      RL c0, c1;
      load_rank<B, BITS, kVPL2, true>(c0, F.shards, F.scale_off, F.elem_off, uoff, lane, valid,
                                      f.kbits);
      if (nr > 1)
        load_rank<B, BITS, kVPL2, true>(c1, F.shards + F.shard_stride, F.scale_off, F.elem_off,
                                        uoff, lane, valid, f.kbits);
      while (true) {
        const uint32_t un = u + nw;
        const bool more = un < total;
        int64_t uoffn = uoff;
        int validn = 0;
        RL n0, n1;
        if (more) {
          uoffn = (int64_t)un * kUnit2;
          validn = max(0, min(kVPL2, (int)min((int64_t)kUnit2, F.n - uoffn) - lane * kVPL2));
          load_rank<B, BITS, kVPL2, true>(n0, F.shards, F.scale_off, F.elem_off, uoffn, lane,
                                          validn, f.kbits);
          if (nr > 1)
            load_rank<B, BITS, kVPL2, true>(n1, F.shards + F.shard_stride, F.scale_off,
                                            F.elem_off, uoffn, lane, validn, f.kbits);
        }
        float acc[kVPL2];
#pragma unroll
        for (int i = 0; i < kVPL2; ++i) acc[i] = 0.f;  // +0.0 (mx/netbench.py:332)
        decode_rank<B, DEC, BITS, kVPL2>(c0, f, acc, false, s_lut);
        if (nr > 1) decode_rank<B, DEC, BITS, kVPL2>(c1, f, acc, false, s_lut);
        const uint8_t* b = F.shards + 2 * F.shard_stride;
        for (int rk = 2; rk < nr; ++rk, b += F.shard_stride) {
          RL r;
          load_rank<B, BITS, kVPL2, true>(r, b, F.scale_off, F.elem_off, uoff, lane, valid,
                                          f.kbits);
          decode_rank<B, DEC, BITS, kVPL2>(r, f, acc, false, s_lut);
        }
        if (valid > 0)
          store_lane_out<OutT, kVPL2>(reinterpret_cast<OutT*>(F.out) + uoff + lane * kVPL2,
                                      valid, acc);
        if (!more) break;
        u = un;
        uoff = uoffn;
        valid = validn;
        c0 = n0;
        c1 = n1;
      }
    }
  }
}

// Units per warp of k_fused_flow: enough that a warp's E8M0 scale bytes of
// one shard fill a 32-byte sector (B = 64: 16 bytes per unit), so its
// read-back never hits a partially written sector.
// (measured: helps FP4 only; the heavier formats keep one unit per warp)
__host__ __device__ constexpr int flow_units_per_warp(int B, int ENC) {
  return (B >= 64 && ENC == ENC_E2M1) ? 32 * B / kUnit : 1;
}

// Dataflow variant for the common case (bf16 partials, n % 1024 == 0, E8M0
// scales): no grid barrier.  The reduction of unit u depends only on unit u
// of every rank's shard, and on one device the warp that quantises unit u of
// every partial is the natural owner of its reduction: it writes the N shard
// slices of u into the gather buffer (exactly the bytes the all-gather would
// deliver), then reads them back (ld.global.cg, lane-for-lane the bytes it
// wrote, plus a __syncwarp for the B = 64 scale shared by two lanes) and
// decodes + sums them in rank order.  Quantise and dequant-sum of different
// units overlap across warps instead of being separated by a grid barrier;
// every warp owns one unit, the grid is sized to the work (several waves).
template <typename OutT, int B, int ENC, int BITS, int TH = kThreads, int KB = 8>
__device__ __forceinline__ void k_flow_one_unit(const FArgs& F) {
  using InT = __nv_bfloat16;
  constexpr int DEC = dec_of(ENC, BITS);
  constexpr int NSB = Geo<B>::NSB;
  constexpr int LPB = Geo<B>::LPB;
  constexpr int UBYTES = kUnit / 8 * BITS;  // element-stream bytes per unit
  constexpr int USCALES = kUnit / B;         // scale bytes per unit (k = 8)
  __shared__ float s_lut[DEC == ENC_E2M1 ? 1 : 256];
  const Fmt f = F.f;
  if constexpr (DEC != ENC_E2M1) {
    fill_lut(s_lut, f);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const uint32_t q = blockIdx.x * (TH / 32) + (threadIdx.x >> 5);
  if (q >= (uint32_t)(F.n / kUnit)) return;
  const int nr = F.nranks;
  const size_t xoff = (size_t)q * kUnit + lane * kVPL;
  const size_t eoff = F.elem_off + (size_t)q * UBYTES;
  const size_t soff = F.scale_off + (size_t)q * USCALES;

  auto quantise = [&](const Raw<InT>& raw, int r) {
    int stored[NSB];
    bool bad;
    LaneCodes<BITS> c = quant_lane<InT, B, ENC, BITS>(raw, f, stored, bad);
    if (bad) report_nonfinite_raw<InT>(raw, kVPL, (int64_t)xoff, F.nonfinite);
    uint8_t* shard = F.shards + (size_t)r * F.shard_stride;
    store_lane_codes<BITS>(shard + eoff + lane * (4 * BITS), c, kVPL);
    if constexpr (KB != 8) {  // E5M0 etc.: packed k-bit codes, group leaders store
      store_unit_scales_k<B>(shard + F.scale_off, (int64_t)q * USCALES, stored, lane, KB);
      return;
    }
    uint8_t* sp = shard + soff + (lane / LPB) * NSB;
    if constexpr (NSB == 4) {
      *reinterpret_cast<uint32_t*>(sp) = (uint32_t)stored[0] | ((uint32_t)stored[1] << 8) |
                                         ((uint32_t)stored[2] << 16) |
                                         ((uint32_t)stored[3] << 24);
    } else if constexpr (NSB == 2) {
      *reinterpret_cast<uint16_t*>(sp) = (uint16_t)(stored[0] | (stored[1] << 8));
    } else {
      if (lane % LPB == 0) *sp = (uint8_t)stored[0];
    }
  };

  if constexpr (KB != 8) {
    // Packed k-bit scale codes (E5M0): a unit's scale segment (e.g. 20 B at
    // B = 32) straddles 32-byte sectors that neighbouring warps write too,
    // so the codes are not read back -- rank pair by rank pair, the warp
    // quantises into the shard, reads the element codes back and decodes
    // them with the scale codes from the registers that produced (and
    // stored) them: the same bits the shard holds.  Rank order is kept.
    using RL = RankLoad<B, BITS, kVPL>;
    float acc[kVPL];
#pragma unroll
    for (int i = 0; i < kVPL; ++i) acc[i] = 0.f;  // +0.0 (mx/netbench.py:332)
    auto quantise_k = [&](const Raw<InT>& raw, int r, RL& x) {
      bool bad;
      LaneCodes<BITS> c = quant_lane<InT, B, ENC, BITS>(raw, f, x.st, bad);
      if (bad) report_nonfinite_raw<InT>(raw, kVPL, (int64_t)xoff, F.nonfinite);
      uint8_t* shard = F.shards + (size_t)r * F.shard_stride;
      store_lane_codes<BITS>(shard + eoff + lane * (4 * BITS), c, kVPL);
      store_unit_scales_k<B>(shard + F.scale_off, (int64_t)q * USCALES, x.st, lane, KB);
    };
    for (int r = 0; r < nr; r += 2) {
      Raw<InT> a, b;
      load_raw<InT>(reinterpret_cast<const InT*>(F.partials[r]) + xoff, a);
      if (r + 1 < nr) load_raw<InT>(reinterpret_cast<const InT*>(F.partials[r + 1]) + xoff, b);
      RL x0, x1;
      quantise_k(a, r, x0);
      if (r + 1 < nr) quantise_k(b, r + 1, x1);
      __syncwarp();
      x0.c = load_lane_codes<BITS, true>(F.shards + (size_t)r * F.shard_stride + eoff +
                                         lane * (4 * BITS), kVPL);
      if (r + 1 < nr)
        x1.c = load_lane_codes<BITS, true>(F.shards + (size_t)(r + 1) * F.shard_stride + eoff +
                                           lane * (4 * BITS), kVPL);
      decode_rank<B, DEC, BITS, kVPL>(x0, f, acc, false, s_lut);
      if (r + 1 < nr) decode_rank<B, DEC, BITS, kVPL>(x1, f, acc, false, s_lut);
    }
    store_lane_out<OutT, kVPL>(reinterpret_cast<OutT*>(F.out) + xoff, kVPL, acc);
    return;
  }

  // ---- quantise unit q of every partial, two ranks' loads in flight ------
  for (int r = 0; r < nr; r += 2) {
    Raw<InT> a, b;
    load_raw<InT>(reinterpret_cast<const InT*>(F.partials[r]) + xoff, a);
    if (r + 1 < nr) load_raw<InT>(reinterpret_cast<const InT*>(F.partials[r + 1]) + xoff, b);
    quantise(a, r);
    if (r + 1 < nr) quantise(b, r + 1);
  }
  __syncwarp();

  // ---- read the N shard slices back, decode, fp32 rank-order sum ---------
  using RL = RankLoad<B, BITS, kVPL>;
  float acc[kVPL];
#pragma unroll
  for (int i = 0; i < kVPL; ++i) acc[i] = 0.f;  // +0.0 (mx/netbench.py:332)
  for (int r = 0; r < nr; r += 2) {
    RL x0, x1;
    load_rank<B, BITS, kVPL, true>(x0, F.shards + (size_t)r * F.shard_stride, F.scale_off,
                                   F.elem_off, (int64_t)q * kUnit, lane, kVPL, KB);
    if (r + 1 < nr)
      load_rank<B, BITS, kVPL, true>(x1, F.shards + (size_t)(r + 1) * F.shard_stride,
                                     F.scale_off, F.elem_off, (int64_t)q * kUnit, lane, kVPL,
                                     KB);
    decode_rank<B, DEC, BITS, kVPL>(x0, f, acc, false, s_lut);
    if (r + 1 < nr) decode_rank<B, DEC, BITS, kVPL>(x1, f, acc, false, s_lut);
  }
  store_lane_out<OutT, kVPL>(reinterpret_cast<OutT*>(F.out) + xoff, kVPL, acc);
}

template <typename OutT, int B, int ENC, int BITS, int TH = kThreads, int KB = 8>
__device__ __forceinline__ void k_flow_multi_unit(const FArgs& F) {
  using InT = __nv_bfloat16;
  constexpr int DEC = dec_of(ENC, BITS);
  constexpr int NSB = Geo<B>::NSB;
  constexpr int LPB = Geo<B>::LPB;
  constexpr int UBYTES = kUnit / 8 * BITS;  // element-stream bytes per unit
  constexpr int USCALES = kUnit / B;         // scale bytes per unit (k = 8)
  __shared__ float s_lut[DEC == ENC_E2M1 ? 1 : 256];
  const Fmt f = F.f;
  if constexpr (DEC != ENC_E2M1) {
    fill_lut(s_lut, f);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  constexpr int UPW = flow_units_per_warp(B, ENC);
  const uint32_t nunits = (uint32_t)(F.n / kUnit);
  const uint32_t q0 = (blockIdx.x * (TH / 32) + (threadIdx.x >> 5)) * UPW;
  if (q0 >= nunits) return;
  const int nr = F.nranks;

  auto quantise = [&](const Raw<InT>& raw, int r, uint32_t q) {
    int stored[NSB];
    bool bad;
    LaneCodes<BITS> c = quant_lane<InT, B, ENC, BITS>(raw, f, stored, bad);
    if (bad)
      report_nonfinite_raw<InT>(raw, kVPL, (int64_t)q * kUnit + lane * kVPL, F.nonfinite);
    uint8_t* shard = F.shards + (size_t)r * F.shard_stride;
    store_lane_codes<BITS>(shard + F.elem_off + (size_t)q * UBYTES + lane * (4 * BITS), c, kVPL);
    if constexpr (KB != 8) {
      store_unit_scales_k<B>(shard + F.scale_off, (int64_t)q * USCALES, stored, lane, KB);
      return;
    }
    uint8_t* sp = shard + F.scale_off + (size_t)q * USCALES + (lane / LPB) * NSB;
    if constexpr (NSB == 4) {
      *reinterpret_cast<uint32_t*>(sp) = (uint32_t)stored[0] | ((uint32_t)stored[1] << 8) |
                                         ((uint32_t)stored[2] << 16) |
                                         ((uint32_t)stored[3] << 24);
    } else if constexpr (NSB == 2) {
      *reinterpret_cast<uint16_t*>(sp) = (uint16_t)(stored[0] | (stored[1] << 8));
    } else {
      if (lane % LPB == 0) *sp = (uint8_t)stored[0];
    }
  };

  // ---- quantise the warp's units of every partial, two ranks in flight ---
#pragma unroll
  for (int u = 0; u < UPW; ++u) {
    const uint32_t q = q0 + u;
    if (UPW > 1 && q >= nunits) break;
    const size_t xoff = (size_t)q * kUnit + lane * kVPL;
    for (int r = 0; r < nr; r += 2) {
      Raw<InT> a, b;
      load_raw<InT>(reinterpret_cast<const InT*>(F.partials[r]) + xoff, a);
      if (r + 1 < nr) load_raw<InT>(reinterpret_cast<const InT*>(F.partials[r + 1]) + xoff, b);
      quantise(a, r, q);
      if (r + 1 < nr) quantise(b, r + 1, q);
    }
  }
  __syncwarp();

  // ---- read the N shard slices back, decode, fp32 rank-order sum ---------
  using RL = RankLoad<B, BITS, kVPL>;
#pragma unroll
  for (int u = 0; u < UPW; ++u) {
    const uint32_t q = q0 + u;
    if (UPW > 1 && q >= nunits) break;
    float acc[kVPL];
#pragma unroll
    for (int i = 0; i < kVPL; ++i) acc[i] = 0.f;  // +0.0 (mx/netbench.py:332)
    for (int r = 0; r < nr; r += 2) {
      RL x0, x1;
      load_rank<B, BITS, kVPL, true>(x0, F.shards + (size_t)r * F.shard_stride, F.scale_off,
                                     F.elem_off, (int64_t)q * kUnit, lane, kVPL, KB);
      if (r + 1 < nr)
        load_rank<B, BITS, kVPL, true>(x1, F.shards + (size_t)(r + 1) * F.shard_stride,
                                       F.scale_off, F.elem_off, (int64_t)q * kUnit, lane, kVPL,
                                       KB);
      decode_rank<B, DEC, BITS, kVPL>(x0, f, acc, false, s_lut);
      if (r + 1 < nr) decode_rank<B, DEC, BITS, kVPL>(x1, f, acc, false, s_lut);
    }
    store_lane_out<OutT, kVPL>(reinterpret_cast<OutT*>(F.out) + (size_t)q * kUnit + lane * kVPL,
                               kVPL, acc);
  }
}

template <typename OutT, int B, int ENC, int BITS, int TH = kThreads, int KB = 8>
__device__ __forceinline__ void k_fused_flow_body(const FArgs& F) {
  if constexpr (flow_units_per_warp(B, ENC) == 1 || KB != 8)
    k_flow_one_unit<OutT, B, ENC, BITS, TH, KB>(F);
  else
    k_flow_multi_unit<OutT, B, ENC, BITS, TH, KB>(F);
}

template <typename OutT, int B, int ENC, int BITS, int TH = kThreads, int KB = 8>
__global__ void __launch_bounds__(TH, (ENC == ENC_E2M1 && B == 64) ? 1024 / TH : 0) k_fused_flow(const FArgs F) {
  // programmatic dependent launch: the producer grid (e.g. the o_proj GEMM
  // writing the partials) completes and flushes before any partial is read
  pdl_prologue();
  k_fused_flow_body<OutT, B, ENC, BITS, TH, KB>(F);
}

// ---------------------------------------------------------------------------
// Multi-GPU fused one-shot over symmetric (peer-mapped) memory: the NVLink
// form of k_fused_flow, with per-CTA dataflow instead of grid barriers.
// CTA b owns the same 8 units on every rank.  It quantises its units of the
// local partial into ITS shard slot (slot = epoch parity) of its symmetric
// buffer, publishes "CTA b of rank r is ready at epoch e" by a system-scope
// release store into every peer's flag array, waits (acquire) for the N
// flags of CTA b, then decodes its units of the N shards straight out of
// the peers' memory over NVLink in rank order (fp32 from +0.0).  No gather
// buffer, no NCCL kernel, no grid-wide barrier: CTAs of different ranks
// pipeline against each other.  Per-CTA epochs (local memory) make every
// launch -- and every CUDA-graph replay -- use the next epoch.  Double
// buffering: rank r writes slot e&1 at epoch e only after its epoch e-1
// launch saw every peer's epoch e-1 flag for the same CTA, i.e. after every
// peer had finished epoch e-2, the last reader of slot e&1.  A wait that
// exceeds the timeout (MXB200_SYMM_TIMEOUT_MS, default 30 s) sets *status
// and proceeds (no hang); the host raises on it (check_status(), which the
// TP hook calls once per forward).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <typename OutT, int B, int ENC, int BITS, int KB = 8>
__global__ void __launch_bounds__(kThreads) k_symm_flow(const SArgs S) {
  using InT = __nv_bfloat16;
  constexpr int DEC = dec_of(ENC, BITS);
  constexpr int NSB = Geo<B>::NSB;
  constexpr int LPB = Geo<B>::LPB;
  constexpr int UBYTES = kUnit / 8 * BITS;
  constexpr int USCALES = kUnit / B;
  __shared__ float s_lut[DEC == ENC_E2M1 ? 1 : 256];
  __shared__ unsigned int s_e;
  const Fmt f = S.f;
  if constexpr (DEC != ENC_E2M1) fill_lut(s_lut, f);
  pdl_prologue();  // the previous call's epochs, flags and outputs are final
  const uint32_t b = blockIdx.x, G = gridDim.x;
  if (threadIdx.x == 0) s_e = S.epoch[b] + 1u;
  __syncthreads();
  const unsigned int e = s_e;
  const int lane = threadIdx.x & 31;
  // CTA b owns unit rows b*U .. b*U+U-1 (kWarps units each): one flag
  // exchange (one release fence) per U*kWarps units.
  const uint32_t units = (uint32_t)(S.n / kUnit);
  const uint32_t U = (units + G * kWarps - 1) / (G * kWarps);
  const int nr = S.nranks;
  const int64_t slot = (int64_t)(e & 1u) * S.slot_stride;

  // ---- quantise my units of the local partial into my shard slot ---------
  for (uint32_t u = 0; u < U; ++u) {
    const uint32_t q = (b * U + u) * kWarps + (threadIdx.x >> 5);
    if (q >= units) break;
    Raw<InT> raw;
    load_raw<InT>(reinterpret_cast<const InT*>(S.x) + (size_t)q * kUnit + lane * kVPL, raw);
    int stored[NSB];
    bool bad;
    LaneCodes<BITS> c = quant_lane<InT, B, ENC, BITS>(raw, f, stored, bad);
    if (bad) report_nonfinite_raw<InT>(raw, kVPL, (int64_t)q * kUnit + lane * kVPL, S.nonfinite);
    uint8_t* shard = S.bufs[S.rank] + slot;
    store_lane_codes<BITS>(shard + S.elem_off + (size_t)q * UBYTES + lane * (4 * BITS), c, kVPL);
    if constexpr (KB != 8) {  // packed k-bit scale codes (group leaders store)
      store_unit_scales_k<B>(shard + S.scale_off, (int64_t)q * USCALES, stored, lane, KB);
      continue;
    }
    uint8_t* sp = shard + S.scale_off + (size_t)q * USCALES + (lane / LPB) * NSB;
    if constexpr (NSB == 4) {
      *reinterpret_cast<uint32_t*>(sp) = (uint32_t)stored[0] | ((uint32_t)stored[1] << 8) |
                                         ((uint32_t)stored[2] << 16) | ((uint32_t)stored[3] << 24);
    } else if constexpr (NSB == 2) {
      *reinterpret_cast<uint16_t*>(sp) = (uint16_t)(stored[0] | (stored[1] << 8));
    } else {
      if (lane % LPB == 0) *sp = (uint8_t)stored[0];
    }
  }
  __syncthreads();

  // ---- publish to every peer, then wait for every peer's CTA b -----------
  if ((int)threadIdx.x < nr) {
    const int j = threadIdx.x;
    // The release store is cumulative over the CTA's shard writes ordered
    // before it by __syncthreads (the acquire side mirrors it), so no
    // fence.sc.sys is needed; MXB200_SYMM_FENCE=1 adds one on both sides.
    if (S.full_fence) __threadfence_system();
    st_release_sys(S.flags[j] + (size_t)S.rank * G + b, e);
    const unsigned int* mine = S.flags[S.rank] + (size_t)j * G + b;
    const unsigned long long t0 = globaltimer_ns();
    while ((int)(ld_acquire_sys(mine) - e) < 0) {
      __nanosleep(32);
      if (globaltimer_ns() - t0 > S.timeout_ns) {  // report, do not hang
        atomicExch(S.status, 1u);
        break;
      }
    }
    if (S.full_fence) __threadfence_system();
  }
  __syncthreads();

  // ---- pull-decode my units of the N shards over NVLink, rank order ------
  for (uint32_t u = 0; u < U; ++u) {
    const uint32_t q = (b * U + u) * kWarps + (threadIdx.x >> 5);
    if (q >= units) break;
    using RL = RankLoad<B, BITS, kVPL>;
    float acc[kVPL];
#pragma unroll
    for (int i = 0; i < kVPL; ++i) acc[i] = 0.f;  // +0.0 (mx/netbench.py:332)
    for (int r = 0; r < nr; r += 2) {
      RL x0, x1;
      load_rank<B, BITS, kVPL, true>(x0, S.bufs[r] + slot, S.scale_off, S.elem_off,
                                     (int64_t)q * kUnit, lane, kVPL, KB);
      if (r + 1 < nr)
        load_rank<B, BITS, kVPL, true>(x1, S.bufs[r + 1] + slot, S.scale_off, S.elem_off,
                                       (int64_t)q * kUnit, lane, kVPL, KB);
      decode_rank<B, DEC, BITS, kVPL>(x0, f, acc, false, s_lut);
      if (r + 1 < nr) decode_rank<B, DEC, BITS, kVPL>(x1, f, acc, false, s_lut);
    }
    const size_t o = (size_t)q * kUnit + lane * kVPL;
    store_lane_out<OutT, kVPL>(reinterpret_cast<OutT*>(S.out) + o, kVPL, acc,
                               S.residual ? reinterpret_cast<const OutT*>(S.residual) + o
                                          : nullptr);
  }
  if (threadIdx.x == 0) S.epoch[b] = e;
}

// ---------------------------------------------------------------------------
// Two-shot over NVLink peer memory (the TP >= 4 algorithm), one launch per
// rank, per-CTA dataflow.  Chunk j (c = n/N values) is owned by rank j.
// CTA b owns unit rows [b*U, b*U+U) (8 units each) of EVERY chunk:
//   A1  quantise those units of the local partial, chunk by chunk, into this
//       rank's send shards (slot e&1: N chunk shards);  publish flag A(b)
//   A2  wait for A(b) of every peer; pull the N peers' send shards of MY
//       chunk over NVLink, fp32 rank-order sum from +0.0, re-quantise into
//       this rank's reduced shard (k_requant's arithmetic);  publish B(b)
//   B   wait for B(b) of every peer; pull each owner's reduced shard of its
//       chunk and decode it (one rank, +0.0 start) into out.
// Same bytes and same arithmetic as quantise -> all_to_all -> K3 ->
// all_gather -> K2 (collective.py two-shot), so the result is bit-identical
// to it; no NCCL kernel, no grid barrier.
// ---------------------------------------------------------------------------

template <typename OutT, int B, int ENC, int BITS, int KB = 8>
__global__ void __launch_bounds__(kThreads) k_symm2_flow(const S2Args S) {
  using InT = __nv_bfloat16;
  constexpr int DEC = dec_of(ENC, BITS);
  constexpr int NSB = Geo<B>::NSB;
  constexpr int LPB = Geo<B>::LPB;
  constexpr int UBYTES = kUnit / 8 * BITS;
  constexpr int USCALES = kUnit / B;
  using RL = RankLoad<B, BITS, kVPL>;
  __shared__ float s_lut[DEC == ENC_E2M1 ? 1 : 256];
  __shared__ unsigned int s_e;
  const Fmt f = S.f;
  if constexpr (DEC != ENC_E2M1) fill_lut(s_lut, f);
  pdl_prologue();  // the previous call's epochs, flags and outputs are final
  const uint32_t b = blockIdx.x, G = gridDim.x;
  if (threadIdx.x == 0) s_e = S.epoch[b] + 1u;
  __syncthreads();
  const unsigned int e = s_e;
  const int lane = threadIdx.x & 31;
  // CTA b owns unit rows b*U .. b*U+U-1 (kWarps units each) of every chunk
  const uint32_t cu = (uint32_t)(S.c / kUnit);
  const uint32_t U = (cu + G * kWarps - 1) / (G * kWarps);
  const int nr = S.nranks, me = S.rank;
  const int64_t slot = (int64_t)(e & 1u) * S.slot_stride;
  uint8_t* const mine = S.bufs[me] + slot;

  auto put = [&](uint8_t* shard, uint32_t q, const LaneCodes<BITS>& cc, const int* stored) {
    store_lane_codes<BITS>(shard + S.elem_off + (size_t)q * UBYTES + lane * (4 * BITS), cc, kVPL);
    if constexpr (KB != 8) {
      store_unit_scales_k<B>(shard + S.scale_off, (int64_t)q * USCALES, stored, lane, KB);
      return;
    }
    uint8_t* sp = shard + S.scale_off + (size_t)q * USCALES + (lane / LPB) * NSB;
    if constexpr (NSB == 4) {
      *reinterpret_cast<uint32_t*>(sp) = (uint32_t)stored[0] | ((uint32_t)stored[1] << 8) |
                                         ((uint32_t)stored[2] << 16) | ((uint32_t)stored[3] << 24);
    } else if constexpr (NSB == 2) {
      *reinterpret_cast<uint16_t*>(sp) = (uint16_t)(stored[0] | (stored[1] << 8));
    } else {
      if (lane % LPB == 0) *sp = (uint8_t)stored[0];
    }
  };
  auto publish_wait = [&](int which) {
    __syncthreads();
    if ((int)threadIdx.x < nr) {
      const int j = threadIdx.x;
      if (S.full_fence) __threadfence_system();
      st_release_sys(S.flags[j] + ((size_t)which * nr + me) * G + b, e);
      const unsigned int* w = S.flags[me] + ((size_t)which * nr + j) * G + b;
      const unsigned long long t0 = globaltimer_ns();
      while ((int)(ld_acquire_sys(w) - e) < 0) {
        __nanosleep(32);
        if (globaltimer_ns() - t0 > S.timeout_ns) {
          atomicExch(S.status, 1u);
          break;
        }
      }
      if (S.full_fence) __threadfence_system();
    }
    __syncthreads();
  };

  // ---- A1: my partial's unit q of every chunk -> my send shards ----------
  for (uint32_t u = 0; u < U; ++u) {
    const uint32_t q = (b * U + u) * kWarps + (threadIdx.x >> 5);  // unit inside every chunk
    if (q >= cu) break;
    const InT* x = reinterpret_cast<const InT*>(S.x) + (size_t)q * kUnit + lane * kVPL;
    for (int j = 0; j < nr; j += 2) {
      Raw<InT> r0, r1;
      load_raw<InT>(x + (size_t)j * S.c, r0);
      if (j + 1 < nr) load_raw<InT>(x + (size_t)(j + 1) * S.c, r1);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (j + h >= nr) break;
        int stored[NSB];
        bool bad;
        LaneCodes<BITS> cc = quant_lane<InT, B, ENC, BITS>(h ? r1 : r0, f, stored, bad);
        if (bad)
          report_nonfinite_raw<InT>(h ? r1 : r0, kVPL,
                                    (int64_t)(j + h) * S.c + (int64_t)q * kUnit + lane * kVPL,
                                    S.nonfinite);
        put(mine + (size_t)(j + h) * S.shard_stride, q, cc, stored);
      }
    }
  }
  publish_wait(0);

  // ---- A2: sum my chunk's N send shards (NVLink), re-quantise -----------
  for (uint32_t u = 0; u < U; ++u) {
    const uint32_t q = (b * U + u) * kWarps + (threadIdx.x >> 5);  // unit inside every chunk
    if (q >= cu) break;
    float acc[kVPL];
#pragma unroll
    for (int i = 0; i < kVPL; ++i) acc[i] = 0.f;  // +0.0 (mx/netbench.py:332)
    for (int r = 0; r < nr; r += 2) {
      RL a0, a1;
      load_rank<B, BITS, kVPL, true>(a0, S.bufs[r] + slot + (size_t)me * S.shard_stride,
                                     S.scale_off, S.elem_off, (int64_t)q * kUnit, lane, kVPL, KB);
      if (r + 1 < nr)
        load_rank<B, BITS, kVPL, true>(a1, S.bufs[r + 1] + slot + (size_t)me * S.shard_stride,
                                       S.scale_off, S.elem_off, (int64_t)q * kUnit, lane, kVPL,
                                       KB);
      decode_rank<B, DEC, BITS, kVPL>(a0, f, acc, false, s_lut);
      if (r + 1 < nr) decode_rank<B, DEC, BITS, kVPL>(a1, f, acc, false, s_lut);
    }
    Raw<float> raw;
#pragma unroll
    for (int i = 0; i < kVPL; ++i) raw.w[i] = __float_as_uint(acc[i]);
    int stored[NSB];
    bool bad;
    LaneCodes<BITS> cc = quant_lane<float, B, ENC, BITS>(raw, f, stored, bad);
    if (bad)
      report_nonfinite_raw<float>(raw, kVPL, (int64_t)me * S.c + (int64_t)q * kUnit + lane * kVPL,
                                  S.nonfinite);
    put(mine + (size_t)nr * S.shard_stride, q, cc, stored);
  }
  publish_wait(1);

  // ---- B: every owner's reduced shard -> out ------------------------------
  for (uint32_t u = 0; u < U; ++u) {
    const uint32_t q = (b * U + u) * kWarps + (threadIdx.x >> 5);  // unit inside every chunk
    if (q >= cu) break;
    for (int j = 0; j < nr; ++j) {
      RL a;
      load_rank<B, BITS, kVPL, true>(a, S.bufs[j] + slot + (size_t)nr * S.shard_stride,
                                     S.scale_off, S.elem_off, (int64_t)q * kUnit, lane, kVPL, KB);
      float acc[kVPL];
#pragma unroll
      for (int i = 0; i < kVPL; ++i) acc[i] = 0.f;
      decode_rank<B, DEC, BITS, kVPL>(a, f, acc, false, s_lut);
      const size_t o = (size_t)j * S.c + (size_t)q * kUnit + lane * kVPL;
      store_lane_out<OutT, kVPL>(reinterpret_cast<OutT*>(S.out) + o, kVPL, acc,
                                 S.residual ? reinterpret_cast<const OutT*>(S.residual) + o
                                            : nullptr);
    }
  }
  if (threadIdx.x == 0) S.epoch[b] = e;
}

template <typename OutT, int B, int ENC, int BITS>
bool go_symm2(const S2Args& a, cudaStream_t st) {
  const int64_t g = symm_ctas(a.c);
  if (a.f.kbits == 8) {
    launch_pdl(k_symm2_flow<OutT, B, ENC, BITS, 8>, dim3((unsigned)g), dim3(kThreads), 0, st, a);
    return true;
  }
  if constexpr (lean_k_ok(ENC)) {  // E5M0 scales (the paper's selected schemes)
    if (a.f.kbits == 5) {
      launch_pdl(k_symm2_flow<OutT, B, ENC, BITS, 5>, dim3((unsigned)g), dim3(kThreads), 0, st,
                 a);
      return true;
    }
  }
  return false;
}

template <typename OutT, int B>
bool symm2_by_enc(const S2Args& a, int enc, int bits, cudaStream_t st) {
  switch (enc) {
    case ENC_E2M1: return go_symm2<OutT, B, ENC_E2M1, 4>(a, st);
    case ENC_E2M3: return go_symm2<OutT, B, ENC_E2M3, 6>(a, st);
    case ENC_E3M2: return go_symm2<OutT, B, ENC_E3M2, 6>(a, st);
    case ENC_INT:
      if (bits == 8) return go_symm2<OutT, B, ENC_INT, 8>(a, st);
      return false;
  }
  if (enc == ENC_E2M2) return go_symm2<OutT, B, ENC_E2M2, 5>(a, st);
  if (bits == 5) return go_symm2<OutT, B, ENC_GEN, 5>(a, st);
  return false;
}

template <typename OutT, int B, int ENC, int BITS>
bool go_symm(const SArgs& a, cudaStream_t st) {
  const dim3 grid((unsigned)symm_ctas(a.n));
  if (a.f.kbits == 8) {
    launch_pdl(k_symm_flow<OutT, B, ENC, BITS, 8>, grid, dim3(kThreads), 0, st, a);
    return true;
  }
  if constexpr (lean_k_ok(ENC)) {  // E5M0 scales (the paper's selected schemes)
    if (a.f.kbits == 5) {
      launch_pdl(k_symm_flow<OutT, B, ENC, BITS, 5>, grid, dim3(kThreads), 0, st, a);
      return true;
    }
  }
  return false;
}

template <typename InT, typename OutT, int B, int ENC, int BITS>
void go(const FArgs& a, cudaStream_t st) {
  if (a.n % kUnit == 0) {
    // dataflow kernel: one warp per unit, no grid barrier.  E8M0 scale
    // bytes, or (the paper's formats) packed k-bit codes stored by the
    // warp's group leaders and read back after the __syncwarp that orders
    // the warp's shard writes
    constexpr int UPW = flow_units_per_warp(B, ENC);
    const int64_t units = a.n / kUnit;
    const dim3 grid((unsigned)((units + kWarps * UPW - 1) / (kWarps * UPW)));
    if (a.f.kbits == 8) {
      launch_pdl(k_fused_flow<OutT, B, ENC, BITS, kThreads, 8>, grid, dim3(kThreads), 0, st, a);
      return;
    }
    if constexpr (lean_k_ok(ENC)) {  // E5M0 scales (the paper's selected schemes)
      if (a.f.kbits == 5) {  // one unit per warp
        launch_pdl(k_fused_flow<OutT, B, ENC, BITS, kThreads, 5>,
                   dim3((unsigned)((units + kWarps - 1) / kWarps)), dim3(kThreads), 0, st, a);
        return;
      }
    }
  }
  auto k = k_fused_oneshot<InT, OutT, B, ENC, BITS>;
  static thread_local int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kThreads, 0);
  if (occ < 1) occ = 1;
  // every CTA must be resident for the grid barrier: at most one wave, and
  // no more CTAs than the larger phase has warp units for
  const int64_t units = std::max<int64_t>((a.n + kUnit2 - 1) / kUnit2,
                                          a.nranks * ((a.n + kUnit - 1) / kUnit));
  const int64_t need = (units + kWarps - 1) / kWarps;
  k<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * occ, need)), kThreads, 0,
      st>>>(a);
}

template <typename InT, typename OutT, int B>
void by_enc(const FArgs& a, int enc, int bits, cudaStream_t st) {
  switch (enc) {
    case ENC_E2M1: go<InT, OutT, B, ENC_E2M1, 4>(a, st); return;
    case ENC_E2M3: go<InT, OutT, B, ENC_E2M3, 6>(a, st); return;
    case ENC_E3M2: go<InT, OutT, B, ENC_E3M2, 6>(a, st); return;
    case ENC_E2M2: go<InT, OutT, B, ENC_E2M2, 5>(a, st); return;
    case ENC_INT:
      if (bits == 4) go<InT, OutT, B, ENC_INT, 4>(a, st);
      else if (bits == 5) go<InT, OutT, B, ENC_INT, 5>(a, st);
      else go<InT, OutT, B, ENC_INT, 8>(a, st);
      return;
  }
  switch (bits) {
    case 4: go<InT, OutT, B, ENC_GEN, 4>(a, st); return;
    case 5: go<InT, OutT, B, ENC_GEN, 5>(a, st); return;
    case 6: go<InT, OutT, B, ENC_GEN, 6>(a, st); return;
    default: go<InT, OutT, B, ENC_GEN, 8>(a, st); return;
  }
}

template <typename OutT, int B>
bool symm_by_enc(const SArgs& a, int enc, int bits, cudaStream_t st) {
  switch (enc) {
    case ENC_E2M1: return go_symm<OutT, B, ENC_E2M1, 4>(a, st);
    case ENC_E2M3: return go_symm<OutT, B, ENC_E2M3, 6>(a, st);
    case ENC_E3M2: return go_symm<OutT, B, ENC_E3M2, 6>(a, st);
    case ENC_INT:
      if (bits == 8) return go_symm<OutT, B, ENC_INT, 8>(a, st);
      return false;
  }
  if (enc == ENC_E2M2) return go_symm<OutT, B, ENC_E2M2, 5>(a, st);
  if (bits == 5) return go_symm<OutT, B, ENC_GEN, 5>(a, st);
  return false;
}

}  // namespace fz

}  // namespace mxb
