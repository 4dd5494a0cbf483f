// Fast quantise kernels, __nv_bfloat16 input (instantiations).  build.py
// compiles this file once per -DMXB_B (block size slice); the MXB_B=8 slice
// also carries the dispatcher.
#include "mx_kernels.cuh"

#ifndef MXB_B
#error "compile with -DMXB_B=<8|16|32|64>"
#endif

namespace mxb {
namespace qb {
template <int B, int ENC, int BITS>
void go(const QArgs& a, cudaStream_t st) {
  launch_quant<__nv_bfloat16, B, ENC, BITS>(a, st);
}
template <int B>
void by_enc(const QArgs& a, int enc, int bits, cudaStream_t st) {
  switch (enc) {
    case ENC_E2M1: go<B, ENC_E2M1, 4>(a, st); return;
    case ENC_E2M3: go<B, ENC_E2M3, 6>(a, st); return;
    case ENC_E3M2: go<B, ENC_E3M2, 6>(a, st); return;
    case ENC_E2M2: go<B, ENC_E2M2, 5>(a, st); return;
    case ENC_INT:
      switch (bits) {
        case 3: go<B, ENC_INT, 3>(a, st); return;
        case 4: go<B, ENC_INT, 4>(a, st); return;
        case 5: go<B, ENC_INT, 5>(a, st); return;
        default: go<B, ENC_INT, 8>(a, st); return;
      }
  }
  switch (bits) {
    case 2: go<B, ENC_GEN, 2>(a, st); return;
    case 3: go<B, ENC_GEN, 3>(a, st); return;
    case 4: go<B, ENC_GEN, 4>(a, st); return;
    case 5: go<B, ENC_GEN, 5>(a, st); return;
    case 6: go<B, ENC_GEN, 6>(a, st); return;
    case 7: go<B, ENC_GEN, 7>(a, st); return;
    default: go<B, ENC_GEN, 8>(a, st); return;
  }
}
template void by_enc<MXB_B>(const QArgs&, int, int, cudaStream_t);
#if MXB_B == 8  // the dispatcher links to the other slices
extern template void by_enc<16>(const QArgs&, int, int, cudaStream_t);
extern template void by_enc<32>(const QArgs&, int, int, cudaStream_t);
extern template void by_enc<64>(const QArgs&, int, int, cudaStream_t);
#endif
}  // namespace qb

#if MXB_B == 8
void launch_quant_bf16(const QArgs& a, int block, int enc, int bits, cudaStream_t st) {
  using namespace qb;
  switch (block) {
    case 8: by_enc<8>(a, enc, bits, st); return;
    case 16: by_enc<16>(a, enc, bits, st); return;
    case 32: by_enc<32>(a, enc, bits, st); return;
    case 64: by_enc<64>(a, enc, bits, st); return;
  }
}
#endif
}  // namespace mxb
