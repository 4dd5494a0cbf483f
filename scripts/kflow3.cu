// Standalone A/B probe (not part of the product): a split-warp K4 -- two
// warps per unit, warp w of the pair quantises rank w's partial (one rank's
// registers per warp: fewer registers, more resident warps), a 64-thread
// named barrier, then each warp decodes + sums HALF of the unit (16 values
// per lane, the K2 VPL=16 layout) from both shards.  Shipped k_fused_flow
// for comparison; outputs checked bit-identical.  bf16
// (round-2 result: a variant that decoded the own rank from registers and hid
// rank 1's read-back behind rank 0's quantise measured SLOWER -- 12.65-13.4 us
// vs 12.19 us at 8B -- and was removed; profiles/r02/kflow2/).  Inputs:
// fp4_e2m1:32:e8m0, 2 ranks, inputs rotated through > 3x L2, every variant
// checked bit-identical to the shipped kernel's output.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        -I include -I paper_2411_09510_b200/csrc scripts/kflow3.cu -o scripts/bin/kflow3
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "k_fused.cuh"

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


// TH threads per CTA, MINB resident CTAs; 2 ranks only (the bench step)
template <int TH, int MINB>
__global__ void __launch_bounds__(TH, MINB) k_split(const FArgs F) {
  using InT = __nv_bfloat16;
  constexpr int B = 32, ENC = ENC_E2M1, BITS = 4, DEC = ENC_E2M1;
  constexpr int UBYTES = kUnit / 8 * BITS;
  constexpr int USCALES = kUnit / B;
  pdl_prologue();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int pair = warp >> 1, r = warp & 1;
  const uint32_t q = blockIdx.x * (TH / 64) + pair;
  const bool live = q < (uint32_t)(F.n / kUnit);
  const Fmt f = F.f;
  if (live) {
    Raw<InT> raw;
    const size_t xoff = (size_t)q * kUnit + lane * kVPL;
    load_raw<InT>(reinterpret_cast<const InT*>(F.partials[r]) + xoff, raw);
    int stored[1];
    bool bad;
    LaneCodes<BITS> c = quant_lane<InT, B, ENC, BITS>(raw, f, stored, bad);
    if (bad) report_nonfinite_raw<InT>(raw, kVPL, (int64_t)xoff, F.nonfinite);
    uint8_t* shard = F.shards + (size_t)r * F.shard_stride;
    store_lane_codes<BITS>(shard + F.elem_off + (size_t)q * UBYTES + lane * (4 * BITS), c, kVPL);
    shard[F.scale_off + (size_t)q * USCALES + lane] = (uint8_t)stored[0];
  }
  // the pair's two warps: named barrier 1 + pair (64 threads)
  asm volatile("bar.sync %0, 64;" ::"r"(1 + pair) : "memory");
  if (!live) return;
  using RL = RankLoad<B, BITS, kVPL2>;
  const int64_t uoff = (int64_t)q * kUnit + r * kUnit2;  // this warp's half
  RL x0, x1;
  load_rank<B, BITS, kVPL2, true>(x0, F.shards, F.scale_off, F.elem_off, uoff, lane, kVPL2, 8);
  load_rank<B, BITS, kVPL2, true>(x1, F.shards + F.shard_stride, F.scale_off, F.elem_off, uoff,
                                  lane, kVPL2, 8);
  float acc[kVPL2];
#pragma unroll
  for (int i = 0; i < kVPL2; ++i) acc[i] = 0.f;
  decode_rank<B, DEC, BITS, kVPL2>(x0, f, acc, false, nullptr);
  decode_rank<B, DEC, BITS, kVPL2>(x1, f, acc, false, nullptr);
  store_lane_out<__nv_bfloat16, kVPL2>(reinterpret_cast<__nv_bfloat16*>(F.out) + uoff +
                                           lane * kVPL2, kVPL2, acc);
}

// sequential ranks: one rank's raw registers live at a time (fewer
// registers -> more resident warps); read-back + decode as shipped
template <int TH, int MINB>
__global__ void __launch_bounds__(TH, MINB) k_seq(const FArgs F) {
  using InT = __nv_bfloat16;
  constexpr int B = 32, ENC = ENC_E2M1, BITS = 4, DEC = ENC_E2M1;
  constexpr int UBYTES = kUnit / 8 * BITS;
  constexpr int USCALES = kUnit / B;
  pdl_prologue();
  const int lane = threadIdx.x & 31;
  const uint32_t q = blockIdx.x * (TH / 32) + (threadIdx.x >> 5);
  if (q >= (uint32_t)(F.n / kUnit)) return;
  const Fmt f = F.f;
  const size_t xoff = (size_t)q * kUnit + lane * kVPL;
  const int nr = F.nranks;
  for (int r = 0; r < nr; ++r) {
    Raw<InT> raw;
    load_raw<InT>(reinterpret_cast<const InT*>(F.partials[r]) + xoff, raw);
    int stored[1];
    bool bad;
    LaneCodes<BITS> c = quant_lane<InT, B, ENC, BITS>(raw, f, stored, bad);
    if (bad) report_nonfinite_raw<InT>(raw, kVPL, (int64_t)xoff, F.nonfinite);
    uint8_t* shard = F.shards + (size_t)r * F.shard_stride;
    store_lane_codes<BITS>(shard + F.elem_off + (size_t)q * UBYTES + lane * (4 * BITS), c, kVPL);
    shard[F.scale_off + (size_t)q * USCALES + lane] = (uint8_t)stored[0];
  }
  __syncwarp();
  using RL = RankLoad<B, BITS, kVPL>;
  float acc[kVPL];
#pragma unroll
  for (int i = 0; i < kVPL; ++i) acc[i] = 0.f;
  for (int r = 0; r < nr; r += 2) {
    RL x0, x1;
    load_rank<B, BITS, kVPL, true>(x0, F.shards + (size_t)r * F.shard_stride, F.scale_off,
                                   F.elem_off, (int64_t)q * kUnit, lane, kVPL, 8);
    if (r + 1 < nr)
      load_rank<B, BITS, kVPL, true>(x1, F.shards + (size_t)(r + 1) * F.shard_stride,
                                     F.scale_off, F.elem_off, (int64_t)q * kUnit, lane, kVPL, 8);
    decode_rank<B, DEC, BITS, kVPL>(x0, f, acc, false, nullptr);
    if (r + 1 < nr) decode_rank<B, DEC, BITS, kVPL>(x1, f, acc, false, nullptr);
  }
  store_lane_out<__nv_bfloat16, kVPL>(reinterpret_cast<__nv_bfloat16*>(F.out) + xoff, kVPL, acc);
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
  const int reps = 60;
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
  const int64_t per_set = 2 * xbytes + 2 * S + xbytes;
  const int R = (int)std::max<int64_t>(3, 3LL * 126 * 1024 * 1024 / per_set + 1);
  std::vector<uint16_t> h(n);
  srand(1);
  for (int64_t i = 0; i < n; ++i) {
    float v = ((rand() & 0xffff) / 32768.f - 1.f) * ((rand() % 100) == 0 ? 100.f : 1.f);
    uint32_t u;
    memcpy(&u, &v, 4);
    h[i] = (uint16_t)(u >> 16);
  }
  std::vector<FArgs> args(R);
  std::vector<QArgs> qa(R);
  const Fmt f = fp4fmt();
  for (int r = 0; r < R; ++r) {
    void *x0, *x1, *sh, *out, **ptrs;
    CK(cudaMalloc(&x0, xbytes));
    CK(cudaMalloc(&x1, xbytes));
    CK(cudaMalloc(&sh, 2 * S));
    CK(cudaMalloc(&out, xbytes));
    CK(cudaMalloc(&ptrs, 2 * sizeof(void*)));
    CK(cudaMemcpy(x0, h.data(), xbytes, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(x1, h.data() + 7, xbytes - 14, cudaMemcpyHostToDevice));
    void* hp[2] = {x0, x1};
    CK(cudaMemcpy(ptrs, hp, sizeof hp, cudaMemcpyHostToDevice));
    FArgs& a = args[r];
    memset(&a, 0, sizeof a);
    a.partials = (const void* const*)ptrs; a.nranks = 2; a.n = n; a.shards = (uint8_t*)sh;
    a.shard_stride = S; a.scale_off = 0; a.elem_off = sbytes; a.out = out; a.bar = nullptr;
    a.nonfinite = nullptr; a.f = f;
    QArgs& q = qa[r];
    memset(&q, 0, sizeof q);
    q.x = x0; q.n = n; q.cv = n; q.units_per_chunk = q.total_units = n / kUnit;
    q.scale_base = (uint8_t*)sh; q.elem_base = (uint8_t*)sh + sbytes; q.chunk_stride = S;
    q.nonfinite = nullptr; q.flat_off = 0; q.f = f;
  }
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const double bytes = 2.0 * xbytes + 2.0 * S + xbytes;  // compulsory HBM bytes
  printf("# n=%lld R=%d sms=%d\n", (long long)n, R, sms);
  const unsigned units = (unsigned)(n / kUnit);
  std::vector<uint16_t> ref(n), got(n);
  auto check = [&](const char* nm) {
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(got.data(), args[0].out, xbytes, cudaMemcpyDeviceToHost));
    printf("# %s %s\n", nm, got == ref ? "identical" : "DIFFER");
    CK(cudaMemset(args[0].out, 0, xbytes));
  };
  bench("k_fused_flow shipped (pdl)", R, [&](int i, cudaStream_t s) {
    pdl(fz::k_fused_flow<__nv_bfloat16, 32, ENC_E2M1, 4>, units / kWarps, kThreads, s, args[i]); },
    bytes, st);
  CK(cudaStreamSynchronize(st));
  CK(cudaMemcpy(ref.data(), args[0].out, xbytes, cudaMemcpyDeviceToHost));
  CK(cudaMemset(args[0].out, 0, xbytes));
#define SPLIT(TH, MINB)                                                                       \
  bench("split th" #TH " minb" #MINB, R, [&](int i, cudaStream_t s) {                          \
    pdl(k_split<TH, MINB>, (units + TH / 64 - 1) / (TH / 64), TH, s, args[i]); }, bytes, st);  \
  check("split");
  SPLIT(256, 4)
  SPLIT(512, 3)
#define SEQ(TH, MINB)                                                                         \
  bench("seq th" #TH " minb" #MINB, R, [&](int i, cudaStream_t s) {                          \
    pdl(k_seq<TH, MINB>, (units + TH / 32 - 1) / (TH / 32), TH, s, args[i]); }, bytes, st);   \
  check("seq");
  SEQ(256, 4)
  SEQ(256, 5)
  SEQ(256, 6)
  SEQ(128, 8)
  SEQ(128, 10)
  SEQ(128, 12)
  return 0;
}
