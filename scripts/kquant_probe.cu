// Standalone A/B probe (not part of the product) for K1 at the 8B shape:
// occupancy / units-per-warp variants of the single-chunk E8M0 quantiser
// body (quant_full_unit from mx_kernels.cuh), every variant checked
// byte-identical to the shipped k_quant, timed like bench.py (CUDA graph of
// R back-to-back PDL launches over buffer sets rotated > 3x L2).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v \
//        -I include -I paper_2411_09510_b200/csrc scripts/kquant_probe.cu -o scripts/bin/kquant_probe
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "mx_kernels.cuh"

using namespace mxb;

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

static Fmt fp4fmt() {
  Fmt f;
  memset(&f, 0, sizeof(f));
  f.bits = 4; f.kbits = 8; f.sbias = 127; f.s_min = -126; f.s_max = 128; f.block = 32;
  f.y = 1; f.lo = 0; f.emax = 2; f.gmax64 = 6.0; f.gmax = 6.f;
  f.ovf32 = (1u << 23) - (1u << 22);
  f.ovf64 = (1ull << 52) - (1ull << 51);
  f.s_fast_lo = -148; f.s_fast_hi = 125;
  return f;
}

template <int TH, int MINB, int UPW>
__global__ void __launch_bounds__(TH, MINB) kq(const QArgs A) {
  pdl_prologue();
  constexpr int W = TH / 32;
  const int lane = threadIdx.x & 31;
  const __nv_bfloat16* x = reinterpret_cast<const __nv_bfloat16*>(A.x);
  const uint32_t nfull = (uint32_t)(A.n / kUnit);
  const uint32_t nw = gridDim.x * W;
  const uint32_t gw = blockIdx.x * W + (threadIdx.x >> 5);
  const Fmt f = A.f;
  for (uint32_t u0 = gw; u0 < nfull; u0 += UPW * nw) {
    Raw<__nv_bfloat16> r[UPW];
#pragma unroll
    for (int k = 0; k < UPW; ++k)
      if (u0 + k * nw < nfull) load_raw<__nv_bfloat16>(x + (size_t)(u0 + k * nw) * kUnit + lane * kVPL, r[k]);
#pragma unroll
    for (int k = 0; k < UPW; ++k)
      if (u0 + k * nw < nfull) quant_full_unit<__nv_bfloat16, 32, ENC_E2M1, 4>(A, f, u0 + k * nw, r[k], lane);
  }
}

template <typename K, typename... A>
static void pdl(K k, unsigned grid, unsigned block, cudaStream_t s, A... a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k, a...));
}

template <typename F>
static double bench(const char* name, int R, F launch, double bytes, cudaStream_t st) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < R; ++i) launch(i, st);
  CK(cudaStreamEndCapture(st, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  for (int i = 0; i < 5; ++i) CK(cudaGraphLaunch(ge, st));
  CK(cudaStreamSynchronize(st));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 100;
  double best = 1e30;
  for (int t = 0; t < 3; ++t) {
    CK(cudaEventRecord(e0, st));
    for (int i = 0; i < reps; ++i) CK(cudaGraphLaunch(ge, st));
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms * 1e3 / (reps * R));
  }
  printf("{\"kernel\": \"%s\", \"us\": %.3f, \"gbs\": %.1f}\n", name, best, bytes / best / 1e3);
  fflush(stdout);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return best;
}

int main(int argc, char** argv) {
  int64_t n = argc > 1 ? atoll(argv[1]) : 2048LL * 4096;
  int sms = 148;
  CK(cudaSetDevice(0));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t xbytes = n * 2, sbytes = n / 32, ebytes = n / 2, S = sbytes + ebytes;
  const int R = (int)std::max<int64_t>(3, 3LL * 126 * 1024 * 1024 / (xbytes + S) + 1);
  std::vector<uint16_t> h(n);
  srand(1);
  for (int64_t i = 0; i < n; ++i) {
    float v = ((rand() & 0xffff) / 32768.f - 1.f) * ((rand() % 100) == 0 ? 100.f : 1.f);
    uint32_t u;
    memcpy(&u, &v, 4);
    h[i] = (uint16_t)(u >> 16);
  }
  std::vector<QArgs> qa(R);
  const Fmt f = fp4fmt();
  for (int r = 0; r < R; ++r) {
    void *x0, *sh;
    CK(cudaMalloc(&x0, xbytes));
    CK(cudaMalloc(&sh, S));
    CK(cudaMemcpy(x0, h.data(), xbytes, cudaMemcpyHostToDevice));
    QArgs& q = qa[r];
    memset(&q, 0, sizeof q);
    q.x = x0; q.n = n; q.cv = n; q.units_per_chunk = q.total_units = n / kUnit;
    q.scale_base = (uint8_t*)sh; q.elem_base = (uint8_t*)sh + sbytes; q.chunk_stride = S;
    q.nonfinite = nullptr; q.flat_off = 0; q.f = f;
  }
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const double bytes = 1.0 * xbytes + S;
  printf("# n=%lld R=%d sms=%d\n", (long long)n, R, sms);
  const unsigned units = (unsigned)(n / kUnit);
  std::vector<uint8_t> ref(S), got(S);
  auto check = [&](const char* nm) {
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(got.data(), qa[0].scale_base, S, cudaMemcpyDeviceToHost));
    printf("# %s %s\n", nm, got == ref ? "identical" : "DIFFER");
    CK(cudaMemset(qa[0].scale_base, 0, S));
  };
  auto shipped = k_quant<__nv_bfloat16, 32, ENC_E2M1, 4>;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, shipped, kThreads, 0);
  const unsigned gship = std::min<unsigned>(sms * occ, (units + 2 * kWarps - 1) / (2 * kWarps));
  bench("k_quant shipped", R, [&](int i, cudaStream_t s) { pdl(shipped, gship, kThreads, s, qa[i]); },
        bytes, st);
  CK(cudaStreamSynchronize(st));
  CK(cudaMemcpy(ref.data(), qa[0].scale_base, S, cudaMemcpyDeviceToHost));
  CK(cudaMemset(qa[0].scale_base, 0, S));
#define V(TH, MINB, UPW)                                                                       \
  {                                                                                            \
    auto k = kq<TH, MINB, UPW>;                                                                \
    int o = 0;                                                                                 \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, TH, 0);                               \
    for (unsigned g : {std::min<unsigned>(sms * o, (units + (TH / 32) * UPW - 1) / ((TH / 32) * UPW)), \
                       (unsigned)(units + (TH / 32) * UPW - 1) / ((TH / 32) * UPW)}) {          \
      char nm[96];                                                                             \
      snprintf(nm, sizeof nm, "kq th%d minb%d upw%d occ%d grid%u", TH, MINB, UPW, o, g);       \
      bench(nm, R, [&](int i, cudaStream_t s) { pdl(k, g, TH, s, qa[i]); }, bytes, st);       \
      check(nm);                                                                               \
    }                                                                                          \
  }
  V(256, 4, 2)
  V(256, 4, 1)
  V(256, 6, 1)
  V(256, 8, 1)
  V(256, 6, 2)
  V(128, 8, 2)
  V(128, 12, 1)
  V(128, 16, 1)
  V(512, 2, 2)
  V(512, 3, 1)
  V(1024, 1, 1)
  V(256, 8, 2)
  return 0;
}
