// K1 on the TMA path (sm_100a): bulk-tensor loads into a 4-stage shared
// memory ring, then the same per-lane quantiser as mx_kernels.cuh.
//
// The input (bf16/f16, 16 B aligned, n_main = multiple of 8192 values) is
// viewed as a 2-D tensor of rows of 64 values = 128 bytes.  One tile = 128
// rows = 8192 values = 16 KB, loaded by a single cp.async.bulk.tensor with
// 128-byte swizzle, completion signalled on an mbarrier (expect_tx).  Warp w
// owns rows [16w, 16w+16) of a tile; lane L owns the 32 consecutive values
// [32L, 32L+32) of the warp's 1024 (row 16w+L/2, half L&1) -- one block of
// 32 per lane, so no shuffles for B <= 32.  Its four 16-byte chunks c live at
// physical chunk c ^ (row & 7) of the row, which makes every LDS.128 of the
// warp bank-conflict free.  A persistent grid walks the tiles round-robin;
// thread 0 refills a stage as soon as all warps have copied it to registers,
// so up to 4 x 16 KB per CTA are in flight while the warps compute.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "mx_kernels.cuh"

namespace mxb {
namespace {

constexpr int kRowV = 64;                  // values per tensor row (128 B)
constexpr int kTileRows = 128;             // rows per tile
constexpr int kTileV = kRowV * kTileRows;  // 8192 values per tile
constexpr int kTileBytes = kTileV * 2;     // 16 KB (16-bit inputs)
constexpr int kStages = 4;

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

template <typename InT, int B, int ENC, int BITS>
__global__ void __launch_bounds__(kThreads) k_quant_tma(const __grid_constant__ CUtensorMap map,
                                                        const QArgs A, int ntiles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // stage buffers must be 1024-byte aligned for the 128-byte swizzle
  uint8_t* stages = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ __align__(8) uint64_t full[kStages];
  const Fmt f = A.f;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int grid = gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      int t = blockIdx.x + s * grid;
      if (t < ntiles) {
        mbar_expect_tx(&full[s], kTileBytes);
        tma_load_2d(stages + s * kTileBytes, &map, &full[s], 0, t * kTileRows);
      }
    }
  }
  const int row = warp * 16 + (lane >> 1);  // tensor row inside the tile
  const int half = lane & 1;
  for (int i = 0;; ++i) {
    const int t = blockIdx.x + i * grid;
    if (t >= ntiles) break;
    const int s = i % kStages;
    mbar_wait(&full[s], (uint32_t)(i / kStages) & 1u);
    Raw<InT> raw;
    const uint8_t* rowp = stages + s * kTileBytes + row * 128;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = (4 * half + j) ^ (row & 7);  // 128-byte swizzle
      uint4 v = *reinterpret_cast<const uint4*>(rowp + c * 16);
      raw.w[4 * j] = v.x; raw.w[4 * j + 1] = v.y; raw.w[4 * j + 2] = v.z; raw.w[4 * j + 3] = v.w;
    }
    __syncthreads();  // every warp holds its copy: the stage can be refilled
    if (tid == 0) {
      const int tn = t + kStages * grid;
      if (tn < ntiles) {
        mbar_expect_tx(&full[s], kTileBytes);
        tma_load_2d(stages + s * kTileBytes, &map, &full[s], 0, tn * kTileRows);
      }
    }
    // unit u = 8t + w has exactly the layout quant_full_unit expects
    quant_full_unit<InT, B, ENC, BITS>(A, f, (uint32_t)t * kWarps + warp, raw, lane);
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

template <typename InT, int B, int ENC, int BITS>
bool go(const CUtensorMap& map, const QArgs& a, int ntiles, cudaStream_t st) {
  auto k = k_quant_tma<InT, B, ENC, BITS>;
  const int smem = kStages * kTileBytes + 1024;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return false;
    attr = true;
  }
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kThreads, smem);
  if (occ < 1) occ = 1;
  int grid = std::min(ntiles, sms * occ);
  k<<<grid, kThreads, smem, st>>>(map, a, ntiles);
  return true;
}

template <typename InT, int B>
bool by_enc(const CUtensorMap& map, const QArgs& a, int ntiles, int enc, int bits,
            cudaStream_t st) {
  switch (enc) {
    case ENC_E2M1: return go<InT, B, ENC_E2M1, 4>(map, a, ntiles, st);
    case ENC_E2M3: return go<InT, B, ENC_E2M3, 6>(map, a, ntiles, st);
    case ENC_E3M2: return go<InT, B, ENC_E3M2, 6>(map, a, ntiles, st);
    case ENC_INT:
      if (bits == 4) return go<InT, B, ENC_INT, 4>(map, a, ntiles, st);
      if (bits == 8) return go<InT, B, ENC_INT, 8>(map, a, ntiles, st);
      break;
  }
  switch (bits) {
    case 2: return go<InT, B, ENC_GEN, 2>(map, a, ntiles, st);
    case 3: return go<InT, B, ENC_GEN, 3>(map, a, ntiles, st);
    case 4: return go<InT, B, ENC_GEN, 4>(map, a, ntiles, st);
    case 5: return go<InT, B, ENC_GEN, 5>(map, a, ntiles, st);
    case 6: return go<InT, B, ENC_GEN, 6>(map, a, ntiles, st);
    case 7: return go<InT, B, ENC_GEN, 7>(map, a, ntiles, st);
    default: return go<InT, B, ENC_GEN, 8>(map, a, ntiles, st);
  }
}

template <typename InT>
bool by_block(const CUtensorMap& map, const QArgs& a, int ntiles, int block, int enc, int bits,
              cudaStream_t st) {
  switch (block) {
    case 8: return by_enc<InT, 8>(map, a, ntiles, enc, bits, st);
    case 16: return by_enc<InT, 16>(map, a, ntiles, enc, bits, st);
    case 32: return by_enc<InT, 32>(map, a, ntiles, enc, bits, st);
    case 64: return by_enc<InT, 64>(map, a, ntiles, enc, bits, st);
  }
  return false;
}

}  // namespace

// Quantise the first floor(n / 8192) * 8192 values of a single-chunk,
// E8M0-scaled bf16/f16 tensor through TMA.  Returns the number of values
// handled (0 = not applicable; the caller's kernels do the rest).
int64_t launch_quant_tma(const QArgs& a, int dtype_is_bf16, int block, int enc, int bits,
                         cudaStream_t st) {
  const int64_t ntiles64 = a.n / kTileV;
  if (ntiles64 < 1 || ntiles64 > (1 << 30) / kTileRows) return 0;
  PFN_cuTensorMapEncodeTiled_v12000 enc_fn = encode_fn();
  if (!enc_fn) return 0;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)kRowV, (cuuint64_t)(ntiles64 * kTileRows)};
  cuuint64_t strides[1] = {(cuuint64_t)kRowV * 2};
  cuuint32_t box[2] = {(cuuint32_t)kRowV, (cuuint32_t)kTileRows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc_fn(&map,
                      dtype_is_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                    : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                      2, const_cast<void*>(a.x), dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return 0;
  const int ntiles = (int)ntiles64;
  bool ok = dtype_is_bf16 ? by_block<__nv_bfloat16>(map, a, ntiles, block, enc, bits, st)
                          : by_block<__half>(map, a, ntiles, block, enc, bits, st);
  return ok ? ntiles64 * kTileV : 0;
}

}  // namespace mxb
