// Standalone design-space microbenchmark for the single-device fused
// one-shot (not part of the product): the shipped barrier-free kernel
// (k_fused_flow) against software-pipelined persistent variants, bf16
// fp4_e2m1:32:e8m0, 2 ranks, inputs rotated through > 3x L2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        -I include -I paper_2411_09510_b200/csrc scripts/kflow.cu -o scripts/bin/kflow
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

// Persistent, software-pipelined: the next unit's partial loads are issued
// before the current unit's shards are read back and decoded (the L2
// read-back latency hides behind DRAM loads in flight).  Decode runs in two
// 512-value halves with 16 values per lane (lane mapping differs from the
// quantiser's, hence the __syncwarp).  nranks == 2.
template <int B, int ENC, int BITS, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_flow_pipe(const FArgs F) {
  using InT = __nv_bfloat16;
  using OutT = __nv_bfloat16;
  constexpr int DEC = ENC_E2M1;
  constexpr int NSB = Geo<B>::NSB;
  constexpr int LPB = Geo<B>::LPB;
  constexpr int UBYTES = kUnit / 8 * BITS;
  constexpr int USCALES = kUnit / B;
  const Fmt f = F.f;
  const int lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * kWarps;
  const uint32_t nunits = (uint32_t)(F.n / kUnit);
  const InT* x0 = reinterpret_cast<const InT*>(F.partials[0]) + lane * kVPL;
  const InT* x1 = reinterpret_cast<const InT*>(F.partials[1]) + lane * kVPL;
  auto quantise = [&](const Raw<InT>& raw, int r, uint32_t q) {
    int stored[NSB];
    bool bad;
    LaneCodes<BITS> c = quant_lane<InT, B, ENC, BITS>(raw, f, stored, bad);
    if (bad) report_nonfinite_raw<InT>(raw, kVPL, (int64_t)q * kUnit + lane * kVPL, F.nonfinite);
    uint8_t* shard = F.shards + (size_t)r * F.shard_stride;
    store_lane_codes<BITS>(shard + F.elem_off + (size_t)q * UBYTES + lane * (4 * BITS), c, kVPL);
    uint8_t* sp = shard + F.scale_off + (size_t)q * USCALES + (lane / LPB) * NSB;
    if constexpr (NSB == 4) {
      *reinterpret_cast<uint32_t*>(sp) = (uint32_t)stored[0] | ((uint32_t)stored[1] << 8) |
                                         ((uint32_t)stored[2] << 16) | ((uint32_t)stored[3] << 24);
    } else if constexpr (NSB == 2) {
      *reinterpret_cast<uint16_t*>(sp) = (uint16_t)(stored[0] | (stored[1] << 8));
    } else {
      if (lane % LPB == 0) *sp = (uint8_t)stored[0];
    }
  };
  using RL = RankLoad<B, BITS, kVPL2>;
  uint32_t u = blockIdx.x * kWarps + (threadIdx.x >> 5);
  Raw<InT> a, b;
  if (u < nunits) {
    load_raw<InT>(x0 + (size_t)u * kUnit, a);
    load_raw<InT>(x1 + (size_t)u * kUnit, b);
  }
  while (u < nunits) {
    quantise(a, 0, u);
    quantise(b, 1, u);
    const uint32_t un = u + nw;
    if (un < nunits) {
      load_raw<InT>(x0 + (size_t)un * kUnit, a);
      load_raw<InT>(x1 + (size_t)un * kUnit, b);
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t uoff = (int64_t)u * kUnit + h * kUnit2;
      RL r0, r1;
      load_rank<B, BITS, kVPL2, true>(r0, F.shards, F.scale_off, F.elem_off, uoff, lane, kVPL2, 8);
      load_rank<B, BITS, kVPL2, true>(r1, F.shards + F.shard_stride, F.scale_off, F.elem_off, uoff,
                                      lane, kVPL2, 8);
      float acc[kVPL2];
#pragma unroll
      for (int i = 0; i < kVPL2; ++i) acc[i] = 0.f;
      decode_rank<B, DEC, BITS, kVPL2>(r0, f, acc, false, nullptr);
      decode_rank<B, DEC, BITS, kVPL2>(r1, f, acc, false, nullptr);
      store_lane_out<OutT, kVPL2>(reinterpret_cast<OutT*>(F.out) + uoff + lane * kVPL2, kVPL2, acc);
    }
    u = un;
  }
}

// PDL form: identical body behind griddepcontrol.wait; the next launch is
// released at our start (launch_dependents), so its CTAs are scheduled and
// parked while this grid drains.
template <int WHERE>
__global__ void __launch_bounds__(kThreads) k_flow_pdl(const FArgs F) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (WHERE == 0) asm volatile("griddepcontrol.launch_dependents;");
  // same per-warp work as k_fused_flow (one unit per warp)
  fz::k_fused_flow_body<__nv_bfloat16, 32, ENC_E2M1, 4, kThreads>(F);
  if (WHERE == 1) asm volatile("griddepcontrol.launch_dependents;");
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
  const int reps = 40;
  CK(cudaEventRecord(e0, st));
  for (int i = 0; i < reps; ++i) CK(cudaGraphLaunch(ge, st));
  CK(cudaEventRecord(e1, st));
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double us = ms * 1e3 / (reps * R);
  printf("{\"kernel\": \"%s\", \"us\": %.3f, \"gbs\": %.1f}\n", name, us, bytes / us / 1e3);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return us;
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
  }
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const double bytes = 2.0 * xbytes + 2.0 * S + xbytes;  // compulsory HBM bytes
  printf("# n=%lld R=%d\n", (long long)n, R);
  const unsigned flat = (unsigned)(n / kUnit / kWarps);
  bench("k_fused_flow(shipped)", R, [&](int i, cudaStream_t s) {
    fz::k_fused_flow<__nv_bfloat16, 32, ENC_E2M1, 4><<<flat, kThreads, 0, s>>>(args[i]); }, bytes, st);
  std::vector<uint16_t> ref(n), got(n);
  CK(cudaStreamSynchronize(st));
  CK(cudaMemcpy(ref.data(), args[0].out, xbytes, cudaMemcpyDeviceToHost));
  auto check = [&](const char* nm) {
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(got.data(), args[0].out, xbytes, cudaMemcpyDeviceToHost));
    printf("# %s %s\n", nm, got == ref ? "identical" : "DIFFER");
    CK(cudaMemset(args[0].out, 0, xbytes));
  };
  CK(cudaMemset(args[0].out, 0, xbytes));
#define PIPE(MINB, C)                                                                        \
  bench("k_flow_pipe<minb" #MINB ",grid" #C "x148>", R, [&](int i, cudaStream_t s) {         \
    k_flow_pipe<32, ENC_E2M1, 4, MINB><<<sms * C, kThreads, 0, s>>>(args[i]); }, bytes, st); \
  check("pipe");
  PIPE(3, 3)
#define FLOWT(TH)                                                                             \
  bench("k_fused_flow<threads" #TH ">", R, [&](int i, cudaStream_t s) {                       \
    fz::k_fused_flow<__nv_bfloat16, 32, ENC_E2M1, 4, TH>                                      \
        <<<(unsigned)(n / kUnit / (TH / 32)), TH, 0, s>>>(args[i]); }, bytes, st);            \
  check("flowT");
  FLOWT(256)
  {
    // block 64 (two lanes per block): one E8M0 byte per 64 values
    std::vector<FArgs> a64 = args;
    for (auto& a : a64) { a.f.block = 64; a.scale_off = 0; a.elem_off = n / 64 + ((32 - (n / 64) % 32) % 32); }
    bench("k_fused_flow<B=64>", R, [&](int i, cudaStream_t s) {
      fz::k_fused_flow<__nv_bfloat16, 64, ENC_E2M1, 4><<<flat / fz::flow_units_per_warp(64, ENC_E2M1), kThreads, 0, s>>>(a64[i]); },
      bytes, st);
    bench("k_fused_flow<B=16>", R, [&](int i, cudaStream_t s) {
      fz::k_fused_flow<__nv_bfloat16, 16, ENC_E2M1, 4><<<flat, kThreads, 0, s>>>(args[i]); },
      bytes, st);
  }
  for (int where = 0; where < 2; ++where) {
    auto k = where == 0 ? k_flow_pdl<0> : k_flow_pdl<1>;
    bench(where == 0 ? "k_flow_pdl(launch_dependents at start)" : "k_flow_pdl(launch_dependents at end)",
          R, [&](int i, cudaStream_t s) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(flat);
            cfg.blockDim = dim3(kThreads);
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            CK(cudaLaunchKernelEx(&cfg, k, args[i]));
          }, bytes, st);
    check("pdl");
  }
  // result written straight to mapped pinned host memory (D2H by SM stores)
  {
    void* hout;
    CK(cudaHostAlloc(&hout, xbytes, cudaHostAllocMapped));
    FArgs a = args[0];
    a.out = hout;
    bench("k_fused_flow, device partials -> host result (SM stores over PCIe)", 1,
          [&](int i, cudaStream_t s) {
            fz::k_fused_flow<__nv_bfloat16, 32, ENC_E2M1, 4><<<flat, kThreads, 0, s>>>(a); },
          xbytes, st);
    void* dout;
    CK(cudaMalloc(&dout, xbytes));
    bench("cudaMemcpyAsync D2H 16.8 MB", 1, [&](int i, cudaStream_t s) {
      CK(cudaMemcpyAsync(hout, dout, xbytes, cudaMemcpyDeviceToHost, s)); }, xbytes, st);
  }
  return 0;
}
