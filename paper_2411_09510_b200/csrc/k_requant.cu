// Fast two-shot requantise kernels (instantiations).
#include "mx_kernels.cuh"

namespace mxb {
namespace {
template <int LPB>
void by_enc(const RArgs& a, int enc, int bits, cudaStream_t st) {
  unsigned tiles = (unsigned)((a.n + kTile - 1) / kTile);
  switch (enc) {
    case ENC_E2M1: k_requant<LPB, ENC_E2M1, 4, kU><<<tiles, kThreads, 0, st>>>(a); return;
    case ENC_E2M3: k_requant<LPB, ENC_E2M3, 6, kU><<<tiles, kThreads, 0, st>>>(a); return;
    case ENC_E3M2: k_requant<LPB, ENC_E3M2, 6, kU><<<tiles, kThreads, 0, st>>>(a); return;
    default:
      if (bits == 8) k_requant<LPB, ENC_GEN, 8, kU><<<tiles, kThreads, 0, st>>>(a);
      else k_requant<LPB, ENC_GEN, 0, kU><<<tiles, kThreads, 0, st>>>(a);
  }
}
}  // namespace

void launch_requant(const RArgs& a, int lpb, int enc, int bits, cudaStream_t st) {
  switch (lpb) {
    case 1: by_enc<1>(a, enc, bits, st); return;
    case 2: by_enc<2>(a, enc, bits, st); return;
    case 4: by_enc<4>(a, enc, bits, st); return;
    case 8: by_enc<8>(a, enc, bits, st); return;
  }
}
}  // namespace mxb
