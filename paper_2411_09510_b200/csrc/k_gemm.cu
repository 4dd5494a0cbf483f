// Row-parallel GEMM with the MX quantiser fused into its epilogue (sm_100a).
//
//   partial[M, N] = x[M, K] . W[N, K]^T     (F.linear of the o_proj /
//                                            down_proj shard, fp32 accumulate)
//   shard         = MX codes + E8M0 scales of bf16(partial)
//
// This is the producer of the compressed TP all-reduce: the reference encodes
// each rank's partial right after its matmul (mx/tpsim.py:263-265:
// `partial = x_shard @ shards[rank]` -> `wire.encode(partial)`).  Fusing the
// encode into the GEMM epilogue removes the 2-byte/value write of the bf16
// partial and K1's read of it; the shard bytes come straight out of the
// accumulator.  The codes are exactly K1's codes of the bf16-rounded partial
// (same quant_lane, mx/codec.py:140-172), which the tests check byte for
// byte against the oracle.
//
// Kernel structure (persistent, one CTA per SM, warp-specialised):
//   warp 0      TMA producer: x and W tiles (BK = 64 bf16 = one 128-byte
//               swizzle row) into a 4-stage shared-memory ring, completion on
//               mbarriers (expect_tx)
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma.cta_group::1
//               .kind::f16 (M = 128, N = BN, K = 16) from shared-memory
//               descriptors into a TMEM accumulator; tcgen05.commit frees the
//               smem stage and, after the last k-block, signals the epilogue
//   warps 2-5   epilogue: tcgen05.ld 32x32b.x32 -- thread t of the four warps
//               owns accumulator row t, 32 consecutive columns per load,
//               which is exactly one lane's 32 values of the MX layout (a
//               block of B <= 32 never crosses threads) -- round to bf16,
//               quantise in registers, store codes + scales (+ optionally
//               the bf16 partial), then release the accumulator
// The accumulator is double-buffered in TMEM (2 x BN columns), so tile i's
// epilogue overlaps tile i+1's main loop.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "mx_kernels.cuh"
#include "mxb200.h"

namespace mxb {
namespace gm {

constexpr int BM = 128;
constexpr int BK = 64;  // bf16: 128 bytes, one SW128 row
constexpr int kStages = 4;
// epilogue warps: 4 (one per TMEM lane quarter) or 8 (two per quarter, each
// owning half of the tile's columns); MXB200_GEMM_EPI picks, default 8
template <int EPI>
constexpr int gemm_threads() { return 64 + 32 * EPI; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// Shared-memory matrix descriptor, K-major, 128-byte swizzle: rows of 128 B,
// 8-row (1024 B) swizzle atoms stacked at SBO = 1024 B; LBO unused (1);
// descriptor version 1 (sm_100); layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// Instruction descriptor, kind::f16: D f32, A/B bf16, both K-major, M x N.
template <int N>
__host__ __device__ constexpr uint32_t idesc_bf16(int m) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct GArgs {
  int64_t M, N, K;
  int64_t cv;             // values per chunk (M*N: one tensor)
  int64_t chunk_stride;   // bytes between chunk shards (two-shot send buffer)
  uint8_t* scale_out;     // chunk 0's scale stream (nullable: plain GEMM)
  uint8_t* elem_out;      // chunk 0's element stream
  void* partial_out;      // bf16 [M, N] (nullable)
  unsigned long long* nonfinite;
  float* ws;              // stream-K partial tiles: gridDim.x slots of BM x BN fp32 (nullable)
  unsigned int* flags;    // gridDim.x u32, zero between launches (the kernel resets them)
  Fmt f;
  // all-gather push (2-CTA form, PUSH = true): the epilogue writes this
  // rank's shard into slot (epoch & 1) of EVERY rank's symmetric buffer over
  // NVLink, tile by tile as the accumulators drain; the last CTA (GPU-scope
  // arrival counter) publishes the epoch into every rank's flag array with
  // one system-scope fence, and records it locally
  uint8_t* const* push_peers;       // device [npush]: peer buffer bases
  int npush, push_rank;
  int push_scatter;                 // 1: chunk j (cv values) goes to rank j only (two-shot
                                    // reduce-scatter leg); 0: the whole shard to every rank
  int64_t push_slot_stride;         // bytes per slot (npush shards)
  int64_t push_off;                 // this rank's shard inside a slot
  int64_t push_scale_off, push_elem_off;  // shard layout
  unsigned int* push_state;         // local: [0] epoch, [1] CTA arrival counter
  int64_t push_flags_off;           // flag array inside every peer buffer (u32 [npush])
};
constexpr int kMaxPush = 8;


// Work distribution.  With a workspace: stream-K -- the T tiles x KB
// k-blocks are cut into gridDim.x contiguous ranges of (nearly) equal
// length, so every CTA does the same MMA work (no 1.73-wave tail when T is
// not a multiple of the SM count).  Ranges are >= KB long (T >= grid), so a
// tile is split between at most two CTAs: CTA p+1 runs the tile's TAIL
// k-blocks first (start of its range) and parks the fp32 partial in
// workspace slot p+1; CTA p runs the HEAD at the end of its range and
// finalises: acc(head) + ws(tail), a fixed order, so results are
// deterministic.  Without a workspace: whole tiles, grid-stride.
struct Sched {
  int64_t u, e;
  int KB, T, t;
  bool dp;
  __device__ __forceinline__ Sched(int T_, int KB_, bool streamk) : KB(KB_), T(T_) {
    dp = !streamk;
    t = blockIdx.x;
    const int64_t W = (int64_t)T_ * KB_;
    u = W * blockIdx.x / gridDim.x;
    e = W * (blockIdx.x + 1) / gridDim.x;
  }
  __device__ __forceinline__ bool next(int& tile, int& kb0, int& kb1) {
    if (dp) {
      if (t >= T) return false;
      tile = t;
      kb0 = 0;
      kb1 = KB;
      t += gridDim.x;
      return true;
    }
    if (u >= e) return false;
    tile = (int)(u / KB);
    kb0 = (int)(u - (int64_t)tile * KB);
    kb1 = (int)min((int64_t)KB, kb0 + (e - u));
    u += kb1 - kb0;
    return true;
  }
};

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <int EPI>
__device__ __forceinline__ void epi_bar() {  // the epilogue warps only
  asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI) : "memory");
}

// One thread's 32 accumulator columns -> bf16(partial) (RNE, the tensor
// F.linear returns) -> [bf16 partial] + [MX codes + scales at flat index
// `flat` (a multiple of 32) of the row-major partial].
// KB = 8: E8M0 scale bytes stored here; KB = 5 (E5M0, the paper's scales):
// the chunk's scale codes go back through stored_out and the caller packs
// a whole group of 8 blocks (5 bytes) once its last chunk is done
template <int MODE, int B, int ENC, int BITS, int KB = 8, bool PUSH = false>
__device__ __forceinline__ void epi_chunk(const GArgs& A, const Fmt& f, const uint32_t* v,
                                          int64_t flat, int* stored_out = nullptr,
                                          uint8_t* const* pdst = nullptr) {
  Raw<__nv_bfloat16> raw;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[2 * i]),
                                             __uint_as_float(v[2 * i + 1]));
    raw.w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  if (MODE == 0 || A.partial_out) {
    uint4* p = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(A.partial_out) + flat);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      p[j] = make_uint4(raw.w[4 * j], raw.w[4 * j + 1], raw.w[4 * j + 2], raw.w[4 * j + 3]);
  }
  if constexpr (MODE == 1) {
    constexpr int NSB = Geo<B>::NSB;
    int stored[NSB];
    bool bad;
    LaneCodes<BITS> cw = quant_lane<__nv_bfloat16, B, ENC, BITS>(raw, f, stored, bad);
    if (bad) report_nonfinite_raw<__nv_bfloat16>(raw, kVPL, flat, A.nonfinite);
    if constexpr (PUSH) {  // the shard (or chunk j of it) to the ranks
      // two-shot: a 32-value group (an 8-block scale group) never straddles
      // a chunk; KB < 8: the scale codes go back to the caller, which packs
      // and pushes whole groups
      auto put = [&](uint8_t* base, int64_t v) {
        store_lane_codes<BITS>(base + A.push_elem_off + v / 8 * BITS, cw, kVPL);
        if constexpr (KB == 8) {
          uint8_t* sp = base + A.push_scale_off + v / B;
          if constexpr (NSB == 4)
            *reinterpret_cast<uint32_t*>(sp) = (uint32_t)stored[0] | ((uint32_t)stored[1] << 8) |
                                               ((uint32_t)stored[2] << 16) |
                                               ((uint32_t)stored[3] << 24);
          else if constexpr (NSB == 2)
            *reinterpret_cast<uint16_t*>(sp) = (uint16_t)(stored[0] | (stored[1] << 8));
          else
            *sp = (uint8_t)stored[0];
        }
      };
      if (A.push_scatter) {
        const int64_t j = flat / A.cv;
        put(pdst[j], flat - j * A.cv);
      } else {
#pragma unroll 1
        for (int j = 0; j < A.npush; ++j) put(pdst[j], flat);
      }
      if constexpr (KB != 8) {
#pragma unroll
        for (int sb = 0; sb < NSB; ++sb) stored_out[sb] = stored[sb];
      }
      return;
    }
    // chunked shards (two-shot): a 32-value group never straddles a chunk
    // (chunk sizes are multiples of 8B >= 128 values)
    const int64_t chunk = flat / A.cv, local = flat - chunk * A.cv;
    const int64_t cofs = chunk * A.chunk_stride;
    store_lane_codes<BITS>(A.elem_out + cofs + local / 8 * BITS, cw, kVPL);
    if constexpr (KB != 8) {
#pragma unroll
      for (int sb = 0; sb < NSB; ++sb) stored_out[sb] = stored[sb];
      return;
    }
    uint8_t* sp = A.scale_out + cofs + local / B;
    if constexpr (NSB == 4) {
      *reinterpret_cast<uint32_t*>(sp) = (uint32_t)stored[0] | ((uint32_t)stored[1] << 8) |
                                         ((uint32_t)stored[2] << 16) |
                                         ((uint32_t)stored[3] << 24);
    } else if constexpr (NSB == 2) {
      *reinterpret_cast<uint16_t*>(sp) = (uint16_t)(stored[0] | (stored[1] << 8));
    } else {
      *sp = (uint8_t)stored[0];
    }
  }
}

// MODE 0: bf16 partial only (plain GEMM, the unfused baseline's producer)
// MODE 1: MX shard (+ bf16 partial when partial_out != nullptr)
template <int BN, int EPI, int MODE, int B, int ENC, int BITS>
__global__ void __launch_bounds__(gemm_threads<EPI>(), 1)
    k_gemm_mx(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
              const GArgs A) {
  constexpr int A_BYTES = BM * BK * 2;
  constexpr int B_BYTES = BN * BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN;  // double-buffered accumulator
  constexpr uint32_t IDESC = idesc_bf16<BN>(BM);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t M = A.M, N = A.N, K = A.K;
  const int num_m = (int)((M + BM - 1) / BM);
  const int num_n = (int)(N / BN);
  const int num_tiles = num_m * num_n;
  const int num_kb = (int)(K / BK);
  const bool streamk = A.ws != nullptr;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
  }
  if (warp == 1) {  // whole warp: allocate the accumulator columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  // x is produced by the previous kernel (attention / activation): wait for
  // it under programmatic dependent launch, release our own dependents
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");

  Sched sch(num_tiles, num_kb, streamk);
  int tile, kb0, kb1;
  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      while (sch.next(tile, kb0, kb1)) {
        const int mb = tile % num_m, nb = tile / num_m;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1u);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          mbar_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_2d(sa, &map_x, &full[stage], kb * BK, mb * BM);
          tma_load_2d(sa + A_BYTES, &map_w, &full[stage], kb * BK, nb * BN);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    while (sch.next(tile, kb0, kb1)) {
      const int acc = it & 1;
      const uint32_t aphase = (uint32_t)(it >> 1) & 1u;
      ++it;
      mbar_wait(&tempty[acc], aphase ^ 1u);
      tc_fence_after();
      const uint32_t d = tmem_base + (uint32_t)(acc * BN);
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {  // +32 bytes per K = 16 step
            mma_bf16(d, smem_desc_sw128(sa + 32 * k), smem_desc_sw128(sb + 32 * k), IDESC,
                     (kb > kb0 || k > 0) ? 1u : 0u);
          }
          mma_commit(&empty[stage]);  // frees the stage when these MMAs finish
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1u;
        }
      }
      if (lane == 0) mma_commit(&tfull[acc]);  // accumulator complete
      __syncwarp();
    }
  } else {
    // ---------------- epilogue (EPI warps) ----------------
    // warp w: TMEM lane quarter w % 4 (hardware rule), column part
    // (w - 2) / 4 of the tile; thread = one accumulator row
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    constexpr int CPH = BN / 32 / (EPI / 4);  // 32-column chunks per part
    const int r_in_tile = 32 * q + lane;
    const bool leader = threadIdx.x == 64;
    const Fmt f = A.f;
    int it = 0;
    while (sch.next(tile, kb0, kb1)) {
      const int mb = tile % num_m, nb = tile / num_m;
      const int acc = it & 1;
      const uint32_t aphase = (uint32_t)(it >> 1) & 1u;
      ++it;
      const bool tail = kb0 > 0;          // partial for the CTA before us
      const bool head = kb1 < num_kb;     // we finalise: + the next CTA's tail
      if (head) {  // wait for the tail partial (published long ago, typically)
        if (leader)
          while (ld_acquire_gpu(A.flags + blockIdx.x + 1) == 0u) __nanosleep(64);
        epi_bar<EPI>();
      }
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const int64_t row = (int64_t)mb * BM + r_in_tile;
      const bool live = row < M;
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * BN);
      float* wrow = A.ws + ((size_t)(tail ? blockIdx.x : blockIdx.x + 1) * BM + r_in_tile) * BN;
#pragma unroll 1
      for (int c = half * CPH; c < (half + 1) * CPH; ++c) {
        uint32_t v[32];
        tmem_ld32(taddr + 32 * c, v);
        tmem_ld_wait();
        if (tail) {  // park the fp32 partial (L2-resident, read once)
          float4* wp = reinterpret_cast<float4*>(wrow + 32 * c);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            __stcg(wp + j, make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                       __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3])));
          continue;
        }
        if (head) {
          const float4* wp = reinterpret_cast<const float4*>(wrow + 32 * c);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 t4 = __ldcg(wp + j);
            v[4 * j] = __float_as_uint(__uint_as_float(v[4 * j]) + t4.x);
            v[4 * j + 1] = __float_as_uint(__uint_as_float(v[4 * j + 1]) + t4.y);
            v[4 * j + 2] = __float_as_uint(__uint_as_float(v[4 * j + 2]) + t4.z);
            v[4 * j + 3] = __float_as_uint(__uint_as_float(v[4 * j + 3]) + t4.w);
          }
        }
        if (live) epi_chunk<MODE, B, ENC, BITS>(A, f, v, row * N + (int64_t)nb * BN + 32 * c);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (tail) {  // publish the parked partial to the CTA before us
        __threadfence();
        epi_bar<EPI>();
        if (leader) st_release_gpu(A.flags + blockIdx.x, 1u);
      }
      if (head && leader) A.flags[blockIdx.x + 1] = 0u;  // consumed: ready for the next launch
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(TMEM_COLS)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// 2-CTA form (cta_group::2): a cluster of two CTAs on an SM pair computes a
// 256 x BN tile.  CTA r loads rows [128r, 128r+128) of the x tile and rows
// [128r, 128r+128) of the BN-row W tile (its half of N); the leader's single
// thread issues tcgen05.mma.cta_group::2 (M = 256), which reads A from each
// CTA's own smem and B from both, and accumulates each CTA's 128 rows x BN
// in that CTA's TMEM.  Per SM the ring stage is 32 KB (x 16 KB + half of W
// 16 KB, against 48 KB for the 1-CTA 128 x 256 tile), so 6 stages fit and a
// third less L2->SM traffic is needed per MMA.
//   full[s]   leader's: both CTAs' TMA bytes complete_tx on it
//   empty[s]  each CTA's: the leader's commit multicasts to both
//   tfull[a]  each CTA's: commit multicast
//   tempty[a] leader's: every epilogue warp of both CTAs arrives (remote)
// ---------------------------------------------------------------------------
constexpr int kStages2 = 6;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// both CTAs: data into the local smem, completion bytes on the LEADER's
// barrier (peer bit cleared, as CUTLASS's SM100_TMA_2SM_LOAD)
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void mma2_bf16(uint32_t tmem_d, uint64_t da, uint64_t db,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma2_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

template <int BN, int EPI, int MODE, int B, int ENC, int BITS, int KB = 8, bool PUSH = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(gemm_threads<EPI>(), 1)
    k_gemm_mx2(const __grid_constant__ CUtensorMap map_x,
               const __grid_constant__ CUtensorMap map_w, const GArgs A) {
  constexpr int A_BYTES = 128 * BK * 2;
  constexpr int B_BYTES = (BN / 2) * BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN;
  constexpr uint32_t IDESC = idesc_bf16<BN>(256);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t full[kStages2], empty[kStages2], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int64_t M = A.M, N = A.N, K = A.K;
  const int num_m = (int)((M + 255) / 256);
  const int num_n = (int)(N / BN);
  const int num_tiles = num_m * num_n;
  const int num_kb = (int)(K / BK);
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * EPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
  }
  if (warp == 1) {  // paired allocation: the same warp in both CTAs
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_sh)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  // push: this call's epoch (the previous launch's last CTA stored epoch - 1
  // and completed before griddepcontrol.wait returned) picks the slot
  __shared__ uint8_t* s_dst[PUSH ? kMaxPush : 1];
  __shared__ unsigned int s_epoch;
  if constexpr (PUSH) {
    if (threadIdx.x == 0)
      s_epoch = *reinterpret_cast<volatile unsigned int*>(A.push_state) + 1u;
    __syncthreads();
    if ((int)threadIdx.x < A.npush)
      s_dst[threadIdx.x] = A.push_peers[threadIdx.x] +
                           (int64_t)(s_epoch & 1u) * A.push_slot_stride + A.push_off;
    __syncthreads();
  }

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < num_tiles; t += ncl) {
        const int mb = t % num_m, nb = t / num_m;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1u);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          if (leader) mbar_expect_tx(&full[stage], 2 * STAGE_BYTES);
          tma_load_2d_2sm(sa, &map_x, &full[stage], kb * BK, mb * 256 + 128 * (int)rank);
          tma_load_2d_2sm(sa + A_BYTES, &map_w, &full[stage], kb * BK,
                          nb * BN + (BN / 2) * (int)rank);
          if (++stage == kStages2) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA only) ----------------
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = cid; t < num_tiles; t += ncl, ++it) {
        const int acc = it & 1;
        const uint32_t aphase = (uint32_t)(it >> 1) & 1u;
        mbar_wait(&tempty[acc], aphase ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
            const uint32_t sb = sa + A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma2_bf16(d, smem_desc_sw128(sa + 32 * k), smem_desc_sw128(sb + 32 * k), IDESC,
                        (kb | k) != 0);
            mma2_commit_both(&empty[stage]);  // both CTAs' producers may refill
          }
          __syncwarp();
          if (++stage == kStages2) {
            stage = 0;
            phase ^= 1u;
          }
        }
        if (lane == 0) mma2_commit_both(&tfull[acc]);
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue (both CTAs: their own 128 rows) ----------------
    const int q = warp & 3;
    const int part = (warp - 2) >> 2;
    constexpr int CPP = BN / 32 / (EPI / 4);
    const Fmt f = A.f;
    const uint32_t tempty_leader0 = mapa(smem_u32(&tempty[0]), 0);
    const uint32_t tempty_leader1 = mapa(smem_u32(&tempty[1]), 0);
    int it = 0;
    for (int t = cid; t < num_tiles; t += ncl, ++it) {
      const int mb = t % num_m, nb = t / num_m;
      const int acc = it & 1;
      const uint32_t aphase = (uint32_t)(it >> 1) & 1u;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const int64_t row = (int64_t)mb * 256 + 128 * rank + 32 * q + lane;
      const bool live = row < M;
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * BN);
      // KB < 8: this thread's consecutive chunks cover whole groups of 8
      // blocks (B = 8: 2 chunks, 16: 4, 32: 8 -- EPI = 4 gives 8 chunks per
      // thread; N % 256 == 0 keeps groups inside one row); the group's k-bit
      // codes are packed in registers and stored by this thread alone
      [[maybe_unused]] uint64_t pk = 0;
      [[maybe_unused]] int nbk = 0;
#pragma unroll 1
      for (int c = part * CPP; c < (part + 1) * CPP; ++c) {
        uint32_t v[32];
        tmem_ld32(taddr + 32 * c, v);
        tmem_ld_wait();
        const int64_t flat = row * N + (int64_t)nb * BN + 32 * c;
        if constexpr (PUSH && KB == 8) {
          if (live) epi_chunk<MODE, B, ENC, BITS, 8, true>(A, f, v, flat, nullptr, s_dst);
        } else if constexpr (PUSH) {  // E5M0 push: whole groups, to every destination
          constexpr int NSB = Geo<B>::NSB;
          if (live) {
            int st[NSB];
            epi_chunk<MODE, B, ENC, BITS, KB, true>(A, f, v, flat, st, s_dst);
#pragma unroll
            for (int sb = 0; sb < NSB; ++sb) pk |= (uint64_t)st[sb] << ((nbk + sb) * KB);
            nbk += NSB;
            if (nbk == 8) {
              const int64_t g0 = flat + 32 - 8 * B;  // the group's first value
              const int j0 = A.push_scatter ? (int)(g0 / A.cv) : 0;
              const int j1 = A.push_scatter ? j0 + 1 : A.npush;
              const int64_t local = A.push_scatter ? g0 - j0 * A.cv : g0;
#pragma unroll 1
              for (int j = j0; j < j1; ++j) {
                uint8_t* sp = s_dst[j] + A.push_scale_off + (local / B / 8) * KB;
#pragma unroll
                for (int i = 0; i < KB; ++i) sp[i] = (uint8_t)(pk >> (8 * i));
              }
              pk = 0;
              nbk = 0;
            }
          }
        } else if constexpr (KB == 8) {
          if (live) epi_chunk<MODE, B, ENC, BITS>(A, f, v, flat);
        } else {
          constexpr int NSB = Geo<B>::NSB;
          if (live) {
            int st[NSB];
            epi_chunk<MODE, B, ENC, BITS, KB>(A, f, v, flat, st);
#pragma unroll
            for (int sb = 0; sb < NSB; ++sb) pk |= (uint64_t)st[sb] << ((nbk + sb) * KB);
            nbk += NSB;
            if (nbk == 8) {
              const int64_t g0 = flat + 32 - 8 * B;  // the group's first value
              const int64_t chunk = g0 / A.cv, local = g0 - chunk * A.cv;
              uint8_t* sp = A.scale_out + chunk * A.chunk_stride + (local / B / 8) * KB;
#pragma unroll
              for (int i = 0; i < KB; ++i) sp[i] = (uint8_t)(pk >> (8 * i));
              pk = 0;
              nbk = 0;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(acc ? tempty_leader1 : tempty_leader0);
    }
  }
  tc_fence_before();
  cluster_sync();  // no remote arrive or MMA is in flight past this point
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(TMEM_COLS)
                 : "memory");
  }
  if constexpr (PUSH) {
    // threadfence-reduction at two scopes: every CTA's epilogue stores are
    // ordered before its GPU-scope acq_rel arrival (bar.sync above, then
    // cumulativity); the last CTA to arrive has acquired them all, and ONE
    // system-scope fence then makes them visible before its relaxed flag
    // stores reach the peers -- no per-CTA system fence on the tail
    if (threadIdx.x == 0) {
      unsigned int prev;
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;"
                   : "=r"(prev) : "l"(A.push_state + 1) : "memory");
      if (prev == gridDim.x - 1) {
        A.push_state[1] = 0u;
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        for (int j = 0; j < A.npush; ++j)
          asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(
                           A.push_peers[j] + A.push_flags_off + 4 * (int64_t)A.push_rank),
                       "r"(s_epoch)
                       : "memory");
        *reinterpret_cast<volatile unsigned int*>(A.push_state) = s_epoch;
      }
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D bf16 K-major operand [rows, K] (row stride K * 2 bytes), box {64, box_rows}
bool make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t K, int box_rows) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int num_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

inline int tile_n(int64_t N) { return N % 256 == 0 ? 256 : 128; }

// one CTA per SM (at most one per tile)
inline int grid_ctas(int64_t M, int64_t N, int BN) {
  const int64_t tiles = (M + BM - 1) / BM * (N / BN);
  return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, num_sms()));
}

// stream-K workspace: one BM x BN fp32 slot per CTA, then one u32 flag per CTA
inline int64_t ws_bytes(int64_t M, int64_t N) {
  const int BN = tile_n(N);
  const int64_t g = grid_ctas(M, N, BN);
  return g * BM * BN * 4 + (g * 4 + 255) / 256 * 256;
}

inline int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

template <int BN, int EPI, int MODE, int B, int ENC, int BITS>
cudaError_t go_epi(const GArgs& a, const void* x, const void* w, cudaStream_t st) {
  CUtensorMap mx, mw;
  if (!make_map(&mx, x, a.M, a.K, BM) || !make_map(&mw, w, a.N, a.K, BN))
    return cudaErrorInvalidValue;
  auto k = k_gemm_mx<BN, EPI, MODE, B, ENC, BITS>;
  constexpr int smem = kStages * (BM * BK * 2 + BN * BK * 2) + 1024;
  static bool attr = false;  // per instantiation
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  launch_pdl(k, dim3(grid_ctas(a.M, a.N, BN)), dim3(gemm_threads<EPI>()), smem, st, mx, mw, a);
  return cudaGetLastError();
}

template <int BN, int EPI, int MODE, int B, int ENC, int BITS, int KB = 8, bool PUSH = false>
cudaError_t go_2cta(const GArgs& a, const void* x, const void* w, cudaStream_t st) {
  CUtensorMap mx, mw;
  if (!make_map(&mx, x, a.M, a.K, 128) || !make_map(&mw, w, a.N, a.K, BN / 2))
    return cudaErrorInvalidValue;
  auto k = k_gemm_mx2<BN, EPI, MODE, B, ENC, BITS, KB, PUSH>;
  constexpr int smem = kStages2 * (128 * BK * 2 + (BN / 2) * BK * 2) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int64_t tiles = (a.M + 255) / 256 * (a.N / BN);
  const int clusters = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, num_sms() / 2));
  launch_pdl(k, dim3(2 * clusters), dim3(gemm_threads<EPI>()), smem, st, mx, mw, a);
  return cudaGetLastError();
}

template <int BN, int MODE, int B, int ENC, int BITS>
cudaError_t go(const GArgs& a, const void* x, const void* w, cudaStream_t st) {
  static const int epi = env_int("MXB200_GEMM_EPI", 8);
  static const int two = env_int("MXB200_GEMM_2CTA", 1);
  if (two && a.ws == nullptr)
    return epi == 8 ? go_2cta<BN, 8, MODE, B, ENC, BITS>(a, x, w, st)
                    : go_2cta<BN, 4, MODE, B, ENC, BITS>(a, x, w, st);
  return epi == 8 ? go_epi<BN, 8, MODE, B, ENC, BITS>(a, x, w, st)
                  : go_epi<BN, 4, MODE, B, ENC, BITS>(a, x, w, st);
}

// E5M0 scales (the paper's selected schemes): 2-CTA form only, 256-wide
// tiles; B = 32 takes 4 epilogue warps so one thread owns a whole group
template <int BN, int B, int ENC, int BITS>
cudaError_t go_k5(const GArgs& a, const void* x, const void* w, cudaStream_t st) {
  static const int two = env_int("MXB200_GEMM_2CTA", 1);
  if constexpr (BN != 256) {
    return cudaErrorNotSupported;
  } else {
    if (!two || a.ws != nullptr) return cudaErrorNotSupported;
    return go_2cta<BN, B == 32 ? 4 : 8, 1, B, ENC, BITS, 5>(a, x, w, st);
  }
}

template <int BN>
cudaError_t by_fmt(const GArgs& a, const void* x, const void* w, int mode, int block, int enc,
                   int bits, cudaStream_t st) {
  if (mode == 0) return go<BN, 0, 32, ENC_E2M1, 4>(a, x, w, st);
  if (a.f.kbits == 5) {
    if (block == 8 && enc == ENC_E2M1 && bits == 4) return go_k5<BN, 8, ENC_E2M1, 4>(a, x, w, st);
    if (block == 16 && enc == ENC_E2M1 && bits == 4) return go_k5<BN, 16, ENC_E2M1, 4>(a, x, w, st);
    if (block == 32 && enc == ENC_E2M1 && bits == 4) return go_k5<BN, 32, ENC_E2M1, 4>(a, x, w, st);
    if (block == 32 && enc == ENC_E2M2 && bits == 5) return go_k5<BN, 32, ENC_E2M2, 5>(a, x, w, st);
    return cudaErrorNotSupported;
  }
#define MXB_GEMM_CASE(BLK, E, BT)                                   \
  if (block == BLK && enc == E && bits == BT) return go<BN, 1, BLK, E, BT>(a, x, w, st);
  MXB_GEMM_CASE(32, ENC_E2M1, 4)
  MXB_GEMM_CASE(16, ENC_E2M1, 4)
  MXB_GEMM_CASE(8, ENC_E2M1, 4)
  MXB_GEMM_CASE(32, ENC_E2M3, 6)
  MXB_GEMM_CASE(32, ENC_E3M2, 6)
  MXB_GEMM_CASE(32, ENC_E2M2, 5)
  MXB_GEMM_CASE(32, ENC_INT, 8)
  MXB_GEMM_CASE(16, ENC_INT, 8)
#undef MXB_GEMM_CASE
  return cudaErrorNotSupported;
}

}  // namespace gm

int64_t gemm_workspace_bytes(int64_t M, int64_t N) { return gm::ws_bytes(M, N); }

// returns cudaErrorNotSupported for shapes / schemes outside the fused path
cudaError_t launch_gemm_mx(const void* x, const void* w, int64_t M, int64_t N, int64_t K,
                           const Fmt* fmt, int enc_id, int64_t chunk_values, int64_t chunk_stride,
                           uint8_t* scale_out, uint8_t* elem_out, void* partial_out,
                           unsigned long long* nonfinite, void* workspace, int64_t workspace_bytes,
                           cudaStream_t st) {
  using namespace gm;
  if (M < 1 || N < 128 || K < BK || K % BK != 0 || N % 128 != 0) return cudaErrorNotSupported;
  if (chunk_values < 1 || (chunk_values % 32 != 0 && chunk_values < M * N))
    return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 15)
    return cudaErrorNotSupported;
  GArgs a;
  memset(&a, 0, sizeof(a));  // push fields off
  a.M = M; a.N = N; a.K = K;
  a.cv = chunk_values; a.chunk_stride = chunk_stride;
  a.scale_out = scale_out; a.elem_out = elem_out; a.partial_out = partial_out;
  a.nonfinite = nonfinite;
  // stream-K when a big enough workspace is given (else whole tiles)
  a.ws = nullptr;
  a.flags = nullptr;
  static const int streamk = env_int("MXB200_GEMM_STREAMK", 0);
  if (streamk && workspace && workspace_bytes >= ws_bytes(M, N)) {
    const int BN = tile_n(N);
    a.ws = reinterpret_cast<float*>(workspace);
    a.flags = reinterpret_cast<unsigned int*>(reinterpret_cast<uint8_t*>(workspace) +
                                              (int64_t)grid_ctas(M, N, BN) * BM * BN * 4);
  }
  int mode = 0, block = 32, enc = ENC_E2M1, bits = 4;
  memset(&a.f, 0, sizeof(a.f));
  if (fmt) {
    if (fmt->kbits != 8 && fmt->kbits != 5) return cudaErrorNotSupported;
    if (fmt->block != 8 && fmt->block != 16 && fmt->block != 32) return cudaErrorNotSupported;
    // E5M0: whole 8-block groups per thread inside one row (256-wide tiles)
    if (fmt->kbits == 5 &&
        (N % 256 != 0 || (chunk_values < M * N && chunk_values % (8 * fmt->block) != 0)))
      return cudaErrorNotSupported;
    if (!scale_out || !elem_out) return cudaErrorInvalidValue;
    a.f = *fmt;
    mode = 1;
    block = fmt->block;
    enc = enc_id;
    bits = a.f.bits;
  } else if (!partial_out) {
    return cudaErrorInvalidValue;
  }
  if (tile_n(N) == 256) return by_fmt<256>(a, x, w, mode, block, enc, bits, st);
  return by_fmt<128>(a, x, w, mode, block, enc, bits, st);
}

// The GEMM with the quantiser AND the all-gather in its epilogue (2-CTA
// form, one tensor; fp4_e2m1 E8M0 B in {16, 32}, fp4_e2m1 E5M0 B in
// {8, 16, 32}, fp5_e2m2 E5M0 B = 32): returns cudaErrorNotSupported outside it.
cudaError_t launch_gemm_mx_push(const void* x, const void* w, int64_t M, int64_t N, int64_t K,
                                const Fmt* fmt, int enc_id, uint8_t* const* peers, int npush,
                                int rank, int64_t slot_stride, int64_t push_off,
                                int64_t scale_off, int64_t elem_off, int64_t scatter_chunk,
                                int64_t flags_off, unsigned int* state,
                                unsigned long long* nonfinite, cudaStream_t st) {
  using namespace gm;
  static const int two = env_int("MXB200_GEMM_2CTA", 1);
  if (!two || !fmt || M < 1 || N < 256 || N % 256 != 0 || K < BK || K % BK != 0)
    return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 15)
    return cudaErrorNotSupported;
  if (npush < 1 || npush > kMaxPush || rank < 0 || rank >= npush) return cudaErrorNotSupported;
  const int blk = fmt->block;
  const bool fp4 = enc_id == ENC_E2M1 && fmt->bits == 4;
  const bool fp5 = enc_id == ENC_E2M2 && fmt->bits == 5;
  if (fmt->kbits == 8 ? !(fp4 && (blk == 16 || blk == 32))
                      : !(fmt->kbits == 5 && ((fp4 && (blk == 8 || blk == 16 || blk == 32)) ||
                                              (fp5 && blk == 32))))
    return cudaErrorNotSupported;
  GArgs a;
  memset(&a, 0, sizeof(a));
  a.M = M; a.N = N; a.K = K;
  a.cv = scatter_chunk > 0 ? scatter_chunk : M * N; a.chunk_stride = 0;
  if (scatter_chunk > 0 && (scatter_chunk % (8 * blk) != 0 || scatter_chunk * npush != M * N))
    return cudaErrorNotSupported;
  a.push_scatter = scatter_chunk > 0;
  a.nonfinite = nonfinite;
  a.f = *fmt;
  a.push_peers = peers; a.npush = npush; a.push_rank = rank;
  a.push_slot_stride = slot_stride; a.push_off = push_off;
  a.push_scale_off = scale_off; a.push_elem_off = elem_off; a.push_state = state;
  a.push_flags_off = flags_off;
  if (fmt->kbits == 5) {  // E5M0: B = 32 takes 4 epilogue warps (one thread, one group)
    if (fp5) return go_2cta<256, 4, 1, 32, ENC_E2M2, 5, 5, true>(a, x, w, st);
    if (blk == 32) return go_2cta<256, 4, 1, 32, ENC_E2M1, 4, 5, true>(a, x, w, st);
    if (blk == 16) return go_2cta<256, 8, 1, 16, ENC_E2M1, 4, 5, true>(a, x, w, st);
    return go_2cta<256, 8, 1, 8, ENC_E2M1, 4, 5, true>(a, x, w, st);
  }
  if (blk == 32) return go_2cta<256, 8, 1, 32, ENC_E2M1, 4, 8, true>(a, x, w, st);
  return go_2cta<256, 8, 1, 16, ENC_E2M1, 4, 8, true>(a, x, w, st);
}

}  // namespace mxb
