// Fast quantise kernels, __nv_bfloat16 input (instantiations).
#include "mx_kernels.cuh"

namespace mxb {
namespace {
template <int LPB, int ENC, int BITS>
void go(const QArgs& a, int64_t nchunks, cudaStream_t st) {
  dim3 grid((unsigned)a.tiles_per_chunk, (unsigned)nchunks);
  k_quant<__nv_bfloat16, LPB, ENC, BITS, kU><<<grid, kThreads, 0, st>>>(a);
}
template <int LPB>
void by_enc(const QArgs& a, int64_t nchunks, int enc, int bits, cudaStream_t st) {
  switch (enc) {
    case ENC_E2M1: go<LPB, ENC_E2M1, 4>(a, nchunks, st); return;
    case ENC_E2M3: go<LPB, ENC_E2M3, 6>(a, nchunks, st); return;
    case ENC_E3M2: go<LPB, ENC_E3M2, 6>(a, nchunks, st); return;
    default:
      if (bits == 8) go<LPB, ENC_GEN, 8>(a, nchunks, st);
      else go<LPB, ENC_GEN, 0>(a, nchunks, st);
  }
}
}  // namespace

void launch_quant_bf16(const QArgs& a, int64_t nchunks, int lpb, int enc, int bits, cudaStream_t st) {
  switch (lpb) {
    case 1: by_enc<1>(a, nchunks, enc, bits, st); return;
    case 2: by_enc<2>(a, nchunks, enc, bits, st); return;
    case 4: by_enc<4>(a, nchunks, enc, bits, st); return;
    case 8: by_enc<8>(a, nchunks, enc, bits, st); return;
  }
}
}  // namespace mxb
