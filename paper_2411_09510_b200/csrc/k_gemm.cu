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
constexpr int kEpiWarps = 4;
constexpr int kGemmThreads = 64 + 32 * kEpiWarps;

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
  Fmt f;
};

// MODE 0: bf16 partial only (plain GEMM, the unfused baseline's producer)
// MODE 1: MX shard (+ bf16 partial when partial_out != nullptr)
template <int BN, int MODE, int B, int ENC, int BITS>
__global__ void __launch_bounds__(kGemmThreads, 1)
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

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps);
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

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int mb = t % num_m, nb = t / num_m;
        for (int kb = 0; kb < num_kb; ++kb) {
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
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
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
          for (int k = 0; k < BK / 16; ++k) {  // +32 bytes per K = 16 step
            mma_bf16(d, smem_desc_sw128(sa + 32 * k), smem_desc_sw128(sb + 32 * k), IDESC,
                     (kb | k) != 0);
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
    // ---------------- epilogue ----------------
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const Fmt f = A.f;
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      const int mb = t % num_m, nb = t / num_m;
      const int acc = it & 1;
      const uint32_t aphase = (uint32_t)(it >> 1) & 1u;
      mbar_wait(&tfull[acc], aphase);
      tc_fence_after();
      const int64_t row = (int64_t)mb * BM + 32 * q + lane;
      const bool live = row < M;
      const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * BN);
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(taddr + 32 * c, v);
        tmem_ld_wait();
        Raw<__nv_bfloat16> raw;  // bf16(partial), RNE: the tensor F.linear returns
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[2 * i]),
                                                   __uint_as_float(v[2 * i + 1]));
          raw.w[i] = *reinterpret_cast<uint32_t*>(&h);
        }
        if (!live) continue;
        const int64_t flat = row * N + (int64_t)nb * BN + 32 * c;  // multiple of 32
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
          // chunked shards (two-shot): a 32-value group never straddles a
          // chunk (chunk sizes are multiples of 8B >= 128 values)
          const int64_t chunk = flat / A.cv, local = flat - chunk * A.cv;
          const int64_t cofs = chunk * A.chunk_stride;
          store_lane_codes<BITS>(A.elem_out + cofs + local / 8 * BITS, cw, kVPL);
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
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
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

template <int BN, int MODE, int B, int ENC, int BITS>
cudaError_t go(const GArgs& a, const void* x, const void* w, cudaStream_t st) {
  CUtensorMap mx, mw;
  if (!make_map(&mx, x, a.M, a.K, BM) || !make_map(&mw, w, a.N, a.K, BN))
    return cudaErrorInvalidValue;
  auto k = k_gemm_mx<BN, MODE, B, ENC, BITS>;
  constexpr int smem = kStages * (BM * BK * 2 + BN * BK * 2) + 1024;
  static bool attr = false;  // per instantiation
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int tiles = (int)((a.M + BM - 1) / BM) * (int)(a.N / BN);
  const int grid = std::max(1, std::min(tiles, num_sms()));
  launch_pdl(k, dim3(grid), dim3(kGemmThreads), smem, st, mx, mw, a);
  return cudaGetLastError();
}

template <int BN>
cudaError_t by_fmt(const GArgs& a, const void* x, const void* w, int mode, int block, int enc,
                   int bits, cudaStream_t st) {
  if (mode == 0) return go<BN, 0, 32, ENC_E2M1, 4>(a, x, w, st);
#define MXB_GEMM_CASE(BLK, E, BT)                                   \
  if (block == BLK && enc == E && bits == BT) return go<BN, 1, BLK, E, BT>(a, x, w, st);
  MXB_GEMM_CASE(32, ENC_E2M1, 4)
  MXB_GEMM_CASE(16, ENC_E2M1, 4)
  MXB_GEMM_CASE(32, ENC_E2M3, 6)
  MXB_GEMM_CASE(32, ENC_E3M2, 6)
  MXB_GEMM_CASE(32, ENC_E2M2, 5)
  MXB_GEMM_CASE(32, ENC_INT, 8)
  MXB_GEMM_CASE(16, ENC_INT, 8)
#undef MXB_GEMM_CASE
  return cudaErrorNotSupported;
}

}  // namespace gm

// returns cudaErrorNotSupported for shapes / schemes outside the fused path
cudaError_t launch_gemm_mx(const void* x, const void* w, int64_t M, int64_t N, int64_t K,
                           const Fmt* fmt, int enc_id, int64_t chunk_values, int64_t chunk_stride,
                           uint8_t* scale_out, uint8_t* elem_out, void* partial_out,
                           unsigned long long* nonfinite, cudaStream_t st) {
  using namespace gm;
  if (M < 1 || N < 128 || K < BK || K % BK != 0 || N % 128 != 0) return cudaErrorNotSupported;
  if (chunk_values < 1 || (chunk_values % 32 != 0 && chunk_values < M * N))
    return cudaErrorNotSupported;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w)) & 15)
    return cudaErrorNotSupported;
  GArgs a;
  a.M = M; a.N = N; a.K = K;
  a.cv = chunk_values; a.chunk_stride = chunk_stride;
  a.scale_out = scale_out; a.elem_out = elem_out; a.partial_out = partial_out;
  a.nonfinite = nonfinite;
  int mode = 0, block = 32, enc = ENC_E2M1, bits = 4;
  memset(&a.f, 0, sizeof(a.f));
  if (fmt) {
    if (fmt->kbits != 8 || (fmt->block != 16 && fmt->block != 32)) return cudaErrorNotSupported;
    if (!scale_out || !elem_out) return cudaErrorInvalidValue;
    a.f = *fmt;
    mode = 1;
    block = fmt->block;
    enc = enc_id;
    bits = a.f.bits;
  } else if (!partial_out) {
    return cudaErrorInvalidValue;
  }
  if (N % 256 == 0) return by_fmt<256>(a, x, w, mode, block, enc, bits, st);
  return by_fmt<128>(a, x, w, mode, block, enc, bits, st);
}

}  // namespace mxb
