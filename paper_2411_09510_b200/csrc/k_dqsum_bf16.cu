// Fast dequant-sum kernels, __nv_bfloat16 output (instantiations).
#include "mx_kernels.cuh"

namespace mxb {
namespace {
template <int LPB>
void by_dec(const DArgs& a, int64_t nchunks, int enc, int bits, cudaStream_t st) {
  dim3 grid((unsigned)a.tiles_per_chunk, (unsigned)nchunks);
  if (enc == ENC_E2M1) k_dqsum<__nv_bfloat16, LPB, ENC_E2M1, 4, kU><<<grid, kThreads, 0, st>>>(a);
  else if (bits == 8) k_dqsum<__nv_bfloat16, LPB, ENC_GEN, 8, kU><<<grid, kThreads, 0, st>>>(a);
  else if (bits == 4) k_dqsum<__nv_bfloat16, LPB, ENC_GEN, 4, kU><<<grid, kThreads, 0, st>>>(a);
  else k_dqsum<__nv_bfloat16, LPB, ENC_GEN, 0, kU><<<grid, kThreads, 0, st>>>(a);
}
}  // namespace

void launch_dqsum_bf16(const DArgs& a, int64_t nchunks, int lpb, int enc, int bits, cudaStream_t st) {
  switch (lpb) {
    case 1: by_dec<1>(a, nchunks, enc, bits, st); return;
    case 2: by_dec<2>(a, nchunks, enc, bits, st); return;
    case 4: by_dec<4>(a, nchunks, enc, bits, st); return;
    case 8: by_dec<8>(a, nchunks, enc, bits, st); return;
  }
}
}  // namespace mxb
