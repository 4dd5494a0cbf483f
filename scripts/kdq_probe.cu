// Standalone A/B probe (not part of the product) for K2 (one-shot
// dequant-sum of N shards -> bf16) at the 8B / 70B shapes: occupancy and
// values-per-lane variants of k_dqsum_lean's body, each checked
// bit-identical to the shipped kernel, timed like bench.py (CUDA graph of R
// back-to-back PDL launches over buffer sets rotated > 3x L2).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v \
//        -I include -I paper_2411_09510_b200/csrc scripts/kdq_probe.cu -o scripts/bin/kdq_probe
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

// the lean body with VPL values per lane, TH threads, MINB resident CTAs
template <int TH, int MINB, int VPL>
__global__ void __launch_bounds__(TH, MINB) kd(const DArgs A) {
  using RL = RankLoad<32, 4, VPL>;
  pdl_prologue();
  constexpr int U = 32 * VPL;
  const int lane = threadIdx.x & 31;
  const uint32_t u = blockIdx.x * (TH / 32) + (threadIdx.x >> 5);
  if (u >= (uint32_t)(A.n / U)) return;
  const int64_t uoff = (int64_t)u * U;
  const int nr = A.nranks;
  float acc[VPL];
#pragma unroll
  for (int i = 0; i < VPL; ++i) acc[i] = 0.f;
  const uint8_t* b = A.in;
  const Fmt f = A.f;
  for (int r = 0; r < nr; r += 2, b += 2 * A.rank_stride) {
    RL x0, x1;
    load_rank<32, 4, VPL>(x0, b, A.scale_off, A.elem_off, uoff, lane, VPL, 8);
    if (r + 1 < nr)
      load_rank<32, 4, VPL>(x1, b + A.rank_stride, A.scale_off, A.elem_off, uoff, lane, VPL, 8);
    decode_rank<32, ENC_E2M1, 4, VPL>(x0, f, acc, false, nullptr);
    if (r + 1 < nr) decode_rank<32, ENC_E2M1, 4, VPL>(x1, f, acc, false, nullptr);
  }
  store_lane_out<__nv_bfloat16, VPL>(reinterpret_cast<__nv_bfloat16*>(A.out) + uoff + lane * VPL,
                                     VPL, acc);
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
  const int N = argc > 2 ? atoi(argv[2]) : 2;
  int sms = 148;
  CK(cudaSetDevice(0));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t sbytes = n / 32, ebytes = n / 2;
  const int64_t S = ((sbytes + 31) / 32) * 32 + ebytes;
  const int64_t per = N * S + 2 * n;
  const int R = (int)std::max<int64_t>(3, 3LL * 126 * 1024 * 1024 / per + 1);
  std::vector<uint8_t> h(N * S);
  srand(3);
  for (auto& v : h) v = rand() & 0xff;
  for (int r = 0; r < N; ++r)  // sane scales: 2^-4..2^3
    for (int64_t i = 0; i < sbytes; ++i) h[r * S + i] = 123 + (rand() % 8);
  std::vector<DArgs> da(R);
  const Fmt f = fp4fmt();
  for (int r = 0; r < R; ++r) {
    void *in, *out;
    CK(cudaMalloc(&in, N * S));
    CK(cudaMalloc(&out, 2 * n));
    CK(cudaMemcpy(in, h.data(), N * S, cudaMemcpyHostToDevice));
    DArgs& a = da[r];
    memset(&a, 0, sizeof a);
    a.in = (const uint8_t*)in; a.rank_stride = S; a.nranks = N; a.chunk_stride = 0;
    a.scale_off = 0; a.elem_off = S - ebytes; a.n = n; a.cv = n;
    a.units_per_chunk = a.total_units = n / kUnit2; a.out = out; a.residual = nullptr;
    a.plain = 0; a.f = f;
  }
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const double bytes = 1.0 * N * (sbytes + ebytes) + 2.0 * n;
  printf("# n=%lld N=%d R=%d sms=%d\n", (long long)n, N, R, sms);
  std::vector<uint16_t> ref(n), got(n);
  auto check = [&](const char* nm) {
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(got.data(), da[0].out, 2 * n, cudaMemcpyDeviceToHost));
    printf("# %s %s\n", nm, got == ref ? "identical" : "DIFFER");
    CK(cudaMemset(da[0].out, 0, 2 * n));
  };
  auto shipped = k_dqsum_lean<__nv_bfloat16, 32, ENC_E2M1, 4>;
  const unsigned gs = (unsigned)((n / kUnit + kWarps - 1) / kWarps);
  bench("k_dqsum_lean shipped", R, [&](int i, cudaStream_t s) { pdl(shipped, gs, kThreads, s, da[i]); },
        bytes, st);
  CK(cudaStreamSynchronize(st));
  CK(cudaMemcpy(ref.data(), da[0].out, 2 * n, cudaMemcpyDeviceToHost));
  CK(cudaMemset(da[0].out, 0, 2 * n));
#define V(TH, MINB, VPL)                                                                   \
  {                                                                                        \
    auto k = kd<TH, MINB, VPL>;                                                            \
    int o = 0;                                                                             \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, TH, 0);                           \
    unsigned g = (unsigned)((n / (32 * VPL) + TH / 32 - 1) / (TH / 32));                   \
    char nm[96];                                                                           \
    snprintf(nm, sizeof nm, "kd th%d minb%d vpl%d occ%d grid%u", TH, MINB, VPL, o, g);     \
    bench(nm, R, [&](int i, cudaStream_t s) { pdl(k, g, TH, s, da[i]); }, bytes, st);     \
    check(nm);                                                                             \
  }
  V(256, 1, 32)
  V(256, 4, 32)
  V(256, 5, 32)
  V(256, 6, 32)
  V(256, 4, 16)
  V(256, 6, 16)
  V(256, 8, 16)
  V(128, 8, 32)
  V(128, 12, 16)
  V(128, 16, 16)
  return 0;
}
