// Fast dequant-sum kernels, __nv_bfloat16 output (instantiations).
#include "mx_kernels.cuh"

namespace mxb {
namespace {
template <int B, int DEC, int BITS>
void go(const DArgs& a, cudaStream_t st) {
  if (a.cv % kUnit == 0 && a.n % a.cv == 0 && (!a.plain || a.nranks == 1)) {
    const dim3 grid((unsigned)((a.n / kUnit + kLeanWarps2 - 1) / kLeanWarps2));
    if (a.f.kbits == 8) {
      launch_pdl(k_dqsum_lean<__nv_bfloat16, B, DEC, BITS, 8>, grid, dim3(kLeanThreads2), 0, st, a);
      return;
    }
    if constexpr (lean_k_ok(DEC)) {  // E5M0 scales (the paper's selected schemes)
      if (a.f.kbits == 5) {
        launch_pdl(k_dqsum_lean<__nv_bfloat16, B, DEC, BITS, 5>, grid, dim3(kLeanThreads2), 0, st, a);
        return;
      }
    }
  }
  auto k = k_dqsum<__nv_bfloat16, B, DEC, BITS>;
  k<<<work_grid(k, a.total_units, 2), kThreads, 0, st>>>(a);
}
template <int B>
void by_dec(const DArgs& a, int enc, int bits, cudaStream_t st) {
  if (enc == ENC_E2M1) {
    go<B, ENC_E2M1, 4>(a, st);
    return;
  }
  if (enc == ENC_E2M3) { go<B, ENC_E2M3, 6>(a, st); return; }
  if (enc == ENC_E3M2) { go<B, ENC_E3M2, 6>(a, st); return; }
  if (enc == ENC_E2M2) { go<B, ENC_E2M2, 5>(a, st); return; }
  if (enc == ENC_INT && bits == 8) { go<B, ENC_INT, 8>(a, st); return; }
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

void launch_dqsum_bf16(const DArgs& a, int block, int enc, int bits, cudaStream_t st) {
  switch (block) {
    case 8: by_dec<8>(a, enc, bits, st); return;
    case 16: by_dec<16>(a, enc, bits, st); return;
    case 32: by_dec<32>(a, enc, bits, st); return;
    case 64: by_dec<64>(a, enc, bits, st); return;
  }
}
}  // namespace mxb
