// Dispatch of the fused kernels (k_fused.cuh) to the slices instantiated by
// k_fused_inst.cu.
#include "mx_kernels.cuh"

namespace mxb {
namespace fz {
template <typename InT, typename OutT, int B>
void by_enc(const FArgs& a, int enc, int bits, cudaStream_t st);
template <typename OutT, int B>
bool symm_by_enc(const SArgs& a, int enc, int bits, cudaStream_t st);
template <typename OutT, int B>
bool symm2_by_enc(const S2Args& a, int enc, int bits, cudaStream_t st);

template <typename OutT>
void by_block(const FArgs& a, int block, int enc, int bits, cudaStream_t st) {
  switch (block) {
    case 8: by_enc<__nv_bfloat16, OutT, 8>(a, enc, bits, st); return;
    case 16: by_enc<__nv_bfloat16, OutT, 16>(a, enc, bits, st); return;
    case 32: by_enc<__nv_bfloat16, OutT, 32>(a, enc, bits, st); return;
    case 64: by_enc<__nv_bfloat16, OutT, 64>(a, enc, bits, st); return;
  }
}
}  // namespace fz

bool launch_symm_oneshot(const SArgs& a, int out_is_bf16, int block, int enc, int bits,
                         cudaStream_t st) {
  using namespace fz;
  switch (block) {
    case 16: return out_is_bf16 ? symm_by_enc<__nv_bfloat16, 16>(a, enc, bits, st)
                                : symm_by_enc<float, 16>(a, enc, bits, st);
    case 32: return out_is_bf16 ? symm_by_enc<__nv_bfloat16, 32>(a, enc, bits, st)
                                : symm_by_enc<float, 32>(a, enc, bits, st);
    case 64: return out_is_bf16 ? symm_by_enc<__nv_bfloat16, 64>(a, enc, bits, st)
                                : symm_by_enc<float, 64>(a, enc, bits, st);
  }
  return false;
}

bool launch_symm_twoshot(const S2Args& a, int out_is_bf16, int block, int enc, int bits,
                         cudaStream_t st) {
  using namespace fz;
  switch (block) {
    case 16: return out_is_bf16 ? symm2_by_enc<__nv_bfloat16, 16>(a, enc, bits, st)
                                : symm2_by_enc<float, 16>(a, enc, bits, st);
    case 32: return out_is_bf16 ? symm2_by_enc<__nv_bfloat16, 32>(a, enc, bits, st)
                                : symm2_by_enc<float, 32>(a, enc, bits, st);
    case 64: return out_is_bf16 ? symm2_by_enc<__nv_bfloat16, 64>(a, enc, bits, st)
                                : symm2_by_enc<float, 64>(a, enc, bits, st);
  }
  return false;
}

// bf16 partials -> bf16/f32 out; element widths 4/5/6/8 (the BASELINE sweep)
bool launch_fused_oneshot(const FArgs& a, int out_is_bf16, int block, int enc, int bits,
                          cudaStream_t st) {
  if (!(block == 8 || block == 16 || block == 32 || block == 64)) return false;
  if (!(bits == 4 || bits == 5 || bits == 6 || bits == 8)) return false;
  if (out_is_bf16) fz::by_block<__nv_bfloat16>(a, block, enc, bits, st);
  else fz::by_block<float>(a, block, enc, bits, st);
  return true;
}

}  // namespace mxb
