// Fast quantise kernels, __half input (instantiations).
#include "mx_kernels.cuh"

namespace mxb {
namespace {
template <int B, int ENC, int BITS>
void go(const QArgs& a, cudaStream_t st) {
  launch_quant<__half, B, ENC, BITS>(a, st);
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
}  // namespace

void launch_quant_f16(const QArgs& a, int block, int enc, int bits, cudaStream_t st) {
  switch (block) {
    case 8: by_enc<8>(a, enc, bits, st); return;
    case 16: by_enc<16>(a, enc, bits, st); return;
    case 32: by_enc<32>(a, enc, bits, st); return;
    case 64: by_enc<64>(a, enc, bits, st); return;
  }
}
}  // namespace mxb
