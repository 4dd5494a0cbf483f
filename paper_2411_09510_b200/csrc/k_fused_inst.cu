// One (output dtype, block size) slice of the fused kernels; build.py
// compiles this file once per -DMXB_OUT (0 bf16, 1 f32) x -DMXB_B so the
// slices build in parallel.
#include "k_fused.cuh"

#if !defined(MXB_OUT) || !defined(MXB_B)
#error "compile with -DMXB_OUT=<0|1> -DMXB_B=<8|16|32|64>"
#endif

namespace mxb {
namespace fz {
#if MXB_OUT == 0
using OutT = __nv_bfloat16;
#else
using OutT = float;
#endif
template void by_enc<__nv_bfloat16, OutT, MXB_B>(const FArgs&, int, int, cudaStream_t);
#if MXB_B != 8
template bool symm_by_enc<OutT, MXB_B>(const SArgs&, int, int, cudaStream_t);
template bool symm2_by_enc<OutT, MXB_B>(const S2Args&, int, int, cudaStream_t);
#endif
}  // namespace fz
}  // namespace mxb
