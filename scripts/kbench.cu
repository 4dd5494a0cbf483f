// Standalone K1 design-space microbenchmark (not part of the product):
// times quantiser variants for bf16 fp4_e2m1:32:e8m0 against the read floor
// and an empty launch, every launch on data rotated through > 3x L2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        -I include -I paper_2411_09510_b200/csrc scripts/kbench.cu -o /tmp/kbench
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

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

__global__ void k_empty() {}

// read floor: every warp sums a contiguous balanced range with 256-bit loads
template <int T, bool HINT>
__global__ void __launch_bounds__(T) k_read(const uint32_t* x, int64_t nwords, uint32_t* sink) {
  // balanced over warps in 1 KB chunks (256 words)
  constexpr int W = T / 32;
  const uint32_t nw = gridDim.x * W, gw = blockIdx.x * W + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const uint32_t nch = (uint32_t)(nwords / 256), per = nch / nw, rem = nch % nw;
  const uint32_t c0 = gw * per + min(gw, rem), cnt = per + (gw < rem ? 1u : 0u);
  const uint32_t* p = x + (size_t)c0 * 256 + lane * 8;
  uint32_t acc = 0;
  for (uint32_t i = 0; i < cnt; i += 4) {
    uint32_t r[4][8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (i + j < cnt) {
        if (HINT)
          asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(r[j][0]), "=r"(r[j][1]), "=r"(r[j][2]), "=r"(r[j][3]), "=r"(r[j][4]),
                         "=r"(r[j][5]), "=r"(r[j][6]), "=r"(r[j][7])
                       : "l"(p + (size_t)(i + j) * 256));
        else
          ldg256(p + (size_t)(i + j) * 256, r[j]);
      } else {
        for (int t = 0; t < 8; ++t) r[j][t] = 0;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int t = 0; t < 8; ++t) acc ^= r[j][t];
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int T>
__global__ void __launch_bounds__(T) k_write(uint32_t* x, int64_t nwords) {
  constexpr int W = T / 32;
  const uint32_t nw = gridDim.x * W, gw = blockIdx.x * W + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const uint32_t nch = (uint32_t)(nwords / 256), per = nch / nw, rem = nch % nw;
  const uint32_t c0 = gw * per + min(gw, rem), cnt = per + (gw < rem ? 1u : 0u);
  uint32_t* p = x + (size_t)c0 * 256 + lane * 8;
  uint32_t v[8];
  for (int t = 0; t < 8; ++t) v[t] = gw + t;
  for (uint32_t i = 0; i < cnt; ++i) stg256(p + (size_t)i * 256, v);
}

// ---------------------------------------------------------------------------
// V1: register path, SM-balanced.  Grid = #SMs x CPS CTAs; CTA b owns a
// contiguous unit range (sizes differ by at most one unit); its warps take
// units round robin, all of a warp's loads (<= UPW units) issued up front.
// ---------------------------------------------------------------------------
template <int UPW, int THREADS>
__global__ void __launch_bounds__(THREADS) k_q_bal(const QArgs A) {
  const Fmt f = A.f;
  constexpr int W = THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t total = (uint32_t)A.total_units;
  const uint32_t per = total / gridDim.x, rem = total % gridDim.x;
  const uint32_t b = blockIdx.x;
  const uint32_t u_begin = b * per + min(b, rem), cnt = per + (b < rem ? 1u : 0u);
  const __nv_bfloat16* x = reinterpret_cast<const __nv_bfloat16*>(A.x);
  for (uint32_t i0 = warp; i0 < cnt; i0 += UPW * W) {
    Raw<__nv_bfloat16> r[UPW];
#pragma unroll
    for (int j = 0; j < UPW; ++j) {
      uint32_t i = i0 + j * W;
      if (i < cnt) load_raw<__nv_bfloat16>(x + (size_t)(u_begin + i) * kUnit + lane * kVPL, r[j]);
    }
#pragma unroll
    for (int j = 0; j < UPW; ++j) {
      uint32_t i = i0 + j * W;
      if (i < cnt) quant_full_unit<__nv_bfloat16, 32, ENC_E2M1, 4>(A, f, u_begin + i, r[j], lane);
    }
  }
}

// ---------------------------------------------------------------------------
// V2: bulk-copy path.  One CTA per SM owns a contiguous unit range and one
// thread requests ALL of it at t=0 with 1-D cp.async.bulk (PIECE units per
// request, one mbarrier each).  Warps consume units from shared memory with
// the lane reading 16-byte chunks k*512 + 16*lane (conflict-free): it holds
// values 256k + 8 lane + [0,8); a block of 32 spans 4 lanes (2 shuffles).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// 8 bf16 (one 16-byte chunk) of a 32-block spread over 4 lanes -> 4 code bytes
__device__ __forceinline__ uint32_t quant8_shfl(uint4 v, const Fmt& f, int& stored) {
  const uint32_t M = 0x7fff7fffu;
  uint32_t m = __vmaxu2(__vmaxu2(v.x & M, v.y & M), __vmaxu2(v.z & M, v.w & M));
  uint32_t h = max(m & 0xffffu, m >> 16);
  h = max(h, __shfl_xor_sync(0xffffffffu, h, 1));
  h = max(h, __shfl_xor_sync(0xffffffffu, h, 2));
  const uint32_t ab = h << 16;
  const bool bad = ab >= 0x7f800000u;
  const int s = shared_exp_fast(bad ? 0u : ab, f);
  const bool zero = (ab == 0u) | bad;
  stored = zero ? 0 : s + f.sbias;
  const uint32_t i16 = (uint32_t)(127 - s) << 7;
  const uint32_t inv2 = i16 | (i16 << 16);
  uint32_t w[4] = {v.x, v.y, v.z, v.w};
  float x[8];
#pragma unroll
  for (int hh = 0; hh < 4; ++hh) {
    __nv_bfloat162 y = __hmul2(*reinterpret_cast<const __nv_bfloat162*>(&w[hh]),
                               *reinterpret_cast<const __nv_bfloat162*>(&inv2));
    uint32_t yu = *reinterpret_cast<uint32_t*>(&y);
    x[2 * hh] = __uint_as_float(yu << 16);
    x[2 * hh + 1] = __uint_as_float(yu & 0xffff0000u);
  }
  uint32_t c = (uint32_t)encode8<ENC_E2M1, 4>(x, f);
  return zero ? 0u : c;
}

template <int THREADS, int PIECE>
__global__ void __launch_bounds__(THREADS, 1) k_q_bulk(const QArgs A) {
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr int W = THREADS / 32;
  constexpr int MAXP = 64;
  __shared__ __align__(8) uint64_t bar[MAXP];
  const Fmt f = A.f;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t total = (uint32_t)A.total_units;
  const uint32_t per = total / gridDim.x, rem = total % gridDim.x;
  const uint32_t b = blockIdx.x;
  const uint32_t u_begin = b * per + min(b, rem), cnt = per + (b < rem ? 1u : 0u);
  const uint32_t npiece = (cnt + PIECE - 1) / PIECE;
  const uint8_t* xb = reinterpret_cast<const uint8_t*>(A.x) + (size_t)u_begin * kUnit * 2;
  if (threadIdx.x == 0) {
    for (uint32_t p = 0; p < npiece; ++p) mbar_init(&bar[p], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (uint32_t p = 0; p < npiece; ++p) {
      uint32_t units = min((uint32_t)PIECE, cnt - p * PIECE);
      mbar_expect_tx(&bar[p], units * kUnit * 2);
      bulk_g2s(sm + (size_t)p * PIECE * kUnit * 2, xb + (size_t)p * PIECE * kUnit * 2,
               units * kUnit * 2, &bar[p]);
    }
  }
  __syncthreads();
  for (uint32_t i = warp; i < cnt; i += W) {
    mbar_wait(&bar[i / PIECE], 0);
    const uint8_t* up = sm + (size_t)i * kUnit * 2;
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = *reinterpret_cast<const uint4*>(up + k * 512 + lane * 16);
    const uint32_t u = u_begin + i;
    uint8_t* el = A.elem_base + (size_t)u * 512;
    uint8_t* sc = A.scale_base + (size_t)u * 32;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int st;
      uint32_t c = quant8_shfl(v[k], f, st);
      reinterpret_cast<uint32_t*>(el + k * 128)[lane] = c;
      // gather the 8 scale bytes of this k into lane 0..1 words
      uint32_t s0 = __shfl_sync(0xffffffffu, st, (lane & 1) * 16 + 0);
      uint32_t s1 = __shfl_sync(0xffffffffu, st, (lane & 1) * 16 + 4);
      uint32_t s2 = __shfl_sync(0xffffffffu, st, (lane & 1) * 16 + 8);
      uint32_t s3 = __shfl_sync(0xffffffffu, st, (lane & 1) * 16 + 12);
      if (lane < 2)
        reinterpret_cast<uint32_t*>(sc + k * 8)[lane] = s0 | (s1 << 8) | (s2 << 16) | (s3 << 24);
    }
  }
}

// ---------------------------------------------------------------------------
struct Bufs {
  std::vector<void*> x, sc, el, y, sh;
};

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
  int dev = 0, sms = 148;
  CK(cudaSetDevice(dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t xbytes = n * 2, sbytes = n / 32, ebytes = n / 2;
  const int R = (int)std::max<int64_t>(4, (3LL * 126 * 1024 * 1024) / (2 * xbytes + 3 * (sbytes + ebytes)) + 1);
  Bufs B;
  std::vector<uint16_t> h(n);
  srand(1);
  for (int64_t i = 0; i < n; ++i) {
    float v = ((rand() & 0xffff) / 32768.f - 1.f) * ((rand() % 100) == 0 ? 100.f : 1.f);
    uint32_t u;
    memcpy(&u, &v, 4);
    h[i] = (uint16_t)(u >> 16);
  }
  for (int r = 0; r < R; ++r) {
    void *x, *s, *e;
    CK(cudaMalloc(&x, xbytes));
    CK(cudaMalloc(&s, sbytes + 64));
    CK(cudaMalloc(&e, ebytes + 64));
    CK(cudaMemcpy(x, h.data(), xbytes, cudaMemcpyHostToDevice));
    B.x.push_back(x); B.sc.push_back(s); B.el.push_back(e);
    void *y, *sh;
    CK(cudaMalloc(&y, xbytes));
    CK(cudaMalloc(&sh, 2 * (sbytes + ebytes)));
    B.y.push_back(y); B.sh.push_back(sh);
  }
  uint32_t* sink;
  CK(cudaMalloc(&sink, 64));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  const Fmt f = fp4fmt();
  auto qa = [&](int i) {
    QArgs a;
    memset(&a, 0, sizeof(a));
    a.x = B.x[i]; a.n = n; a.cv = n; a.units_per_chunk = n / kUnit; a.total_units = n / kUnit;
    a.scale_base = (uint8_t*)B.sc[i]; a.elem_base = (uint8_t*)B.el[i]; a.chunk_stride = 0;
    a.nonfinite = nullptr; a.flat_off = 0; a.f = f;
    return a;
  };
  const double kbytes = xbytes + sbytes + ebytes;
  printf("# n=%lld R=%d sms=%d\n", (long long)n, R, sms);
  bench("empty<148x32>", R, [&](int i, cudaStream_t s) { k_empty<<<sms, 32, 0, s>>>(); }, 0, st);
#define RD(T, C, H)                                                                          \
  bench("read<t" #T ",cps" #C ",hint" #H ">", R, [&](int i, cudaStream_t s) {                 \
    k_read<T, H><<<sms * C, T, 0, s>>>((const uint32_t*)B.x[i], xbytes / 4, sink); }, xbytes, st);
  RD(512, 1, 0) RD(512, 2, 0) RD(512, 4, 0) RD(256, 4, 0) RD(256, 8, 0) RD(128, 16, 0)
  RD(1024, 2, 0) RD(512, 2, 1) RD(256, 8, 1) RD(1024, 2, 1)
#define WR(T, C)                                                                             \
  bench("write<t" #T ",cps" #C ">", R, [&](int i, cudaStream_t s) {                           \
    k_write<T><<<sms * C, T, 0, s>>>((uint32_t*)B.y[i], xbytes / 4); }, xbytes, st);
  WR(512, 2) WR(256, 8) WR(1024, 2)
  // restore inputs (copy test overwrote them with identical data; fine)
  // reference outputs of the current kernel
  {
    auto k = k_quant<__nv_bfloat16, 32, ENC_E2M1, 4>;
    unsigned g = work_grid(k, n / kUnit, kUPW);
    bench("k_quant(current)", R, [&](int i, cudaStream_t s) { k<<<g, kThreads, 0, s>>>(qa(i)); },
          kbytes, st);
  }
  std::vector<uint8_t> ref_s(sbytes), ref_e(ebytes), got_s(sbytes), got_e(ebytes);
  CK(cudaStreamSynchronize(st));
  CK(cudaMemcpy(ref_s.data(), B.sc[0], sbytes, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ref_e.data(), B.el[0], ebytes, cudaMemcpyDeviceToHost));
  auto check = [&](const char* name) {
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(got_s.data(), B.sc[0], sbytes, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(got_e.data(), B.el[0], ebytes, cudaMemcpyDeviceToHost));
    bool ok = got_s == ref_s && got_e == ref_e;
    printf("# %s bytes %s\n", name, ok ? "identical" : "DIFFER");
    CK(cudaMemset(B.sc[0], 0xAB, sbytes));
    CK(cudaMemset(B.el[0], 0xAB, ebytes));
  };
  CK(cudaMemset(B.sc[0], 0xAB, sbytes));
  CK(cudaMemset(B.el[0], 0xAB, ebytes));
#define BAL(UPW, T, CPS)                                                                   \
  bench("k_q_bal<upw" #UPW ",t" #T ",cps" #CPS ">", R,                                     \
        [&](int i, cudaStream_t s) { k_q_bal<UPW, T><<<sms * CPS, T, 0, s>>>(qa(i)); }, kbytes, \
        st);                                                                               \
  check("bal");
  BAL(2, 1024, 1)
  BAL(2, 512, 2)
  BAL(1, 512, 4)
  BAL(2, 256, 4)
  BAL(4, 256, 4)
  BAL(1, 256, 8)
#define BULK(T, P)                                                                          \
  {                                                                                         \
    auto k = k_q_bulk<T, P>;                                                                \
    int per = (int)((n / kUnit + sms - 1) / sms);                                           \
    int smem = per * kUnit * 2;                                                             \
    if (smem <= 220 * 1024) {                                                               \
      CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));       \
      bench("k_q_bulk<t" #T ",piece" #P ">", R,                                             \
            [&](int i, cudaStream_t s) { k<<<sms, T, smem, s>>>(qa(i)); }, kbytes, st);     \
      check("bulk");                                                                        \
    }                                                                                       \
  }
  BULK(512, 2)
  BULK(512, 4)
  BULK(1024, 4)
  BULK(1024, 1)
  BULK(256, 4)
  // K1 current kernel with other grids
  {
    auto k = k_quant<__nv_bfloat16, 32, ENC_E2M1, 4>;
    bench("k_quant(flat grid, 1 unit/warp)", R, [&](int i, cudaStream_t s) {
      k<<<(unsigned)(n / kUnit / kWarps), kThreads, 0, s>>>(qa(i)); }, kbytes, st);
    for (int c : {4}) {
      char nm[64];
      snprintf(nm, sizeof nm, "k_quant(grid=%dx148)", c);
      bench(nm, R, [&](int i, cudaStream_t s) { k<<<sms * c, kThreads, 0, s>>>(qa(i)); }, kbytes, st);
    }
  }
  // K2: two shards per set made by K1
  const int64_t S = sbytes + ebytes;
  for (int r = 0; r < R; ++r)
    for (int rk = 0; rk < 2; ++rk) {
      QArgs a = qa(r);
      a.scale_base = (uint8_t*)B.sh[r] + rk * S;
      a.elem_base = (uint8_t*)B.sh[r] + rk * S + sbytes;
      auto k = k_quant<__nv_bfloat16, 32, ENC_E2M1, 4>;
      k<<<sms * 4, kThreads, 0, st>>>(a);
    }
  CK(cudaStreamSynchronize(st));
  auto da = [&](int i) {
    DArgs a;
    memset(&a, 0, sizeof(a));
    a.in = (const uint8_t*)B.sh[i]; a.rank_stride = S; a.nranks = 2; a.chunk_stride = 0;
    a.scale_off = 0; a.elem_off = sbytes; a.n = n; a.cv = n;
    a.units_per_chunk = n / kUnit2; a.total_units = n / kUnit2; a.out = B.y[i]; a.plain = 0; a.f = f;
    return a;
  };
  const double k2bytes = 2.0 * S + xbytes;
  {
    auto k = k_dqsum<__nv_bfloat16, 32, ENC_E2M1, 4>;
    unsigned g = work_grid(k, n / kUnit2, 2);
    printf("# k_dqsum current grid %u\n", g);
    bench("k_dqsum(current)", R, [&](int i, cudaStream_t s) { k<<<g, kThreads, 0, s>>>(da(i)); }, k2bytes, st);
    auto kl = k_dqsum_lean<__nv_bfloat16, 32, ENC_E2M1, 4>;
    std::vector<uint16_t> r2(n), g2(n);
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(r2.data(), B.y[0], xbytes, cudaMemcpyDeviceToHost));
    CK(cudaMemset(B.y[0], 0, xbytes));
    bench("k_dqsum_lean", R, [&](int i, cudaStream_t s) {
      kl<<<(unsigned)(n / kUnit / kWarps), kThreads, 0, s>>>(da(i)); }, k2bytes, st);
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(g2.data(), B.y[0], xbytes, cudaMemcpyDeviceToHost));
    printf("# lean %s\n", g2 == r2 ? "identical" : "DIFFER");
    for (int c : {4}) {
      char nm[64];
      snprintf(nm, sizeof nm, "k_dqsum(grid=%dx148)", c);
      bench(nm, R, [&](int i, cudaStream_t s) { k<<<sms * c, kThreads, 0, s>>>(da(i)); }, k2bytes, st);
    }
  }
  return 0;
}
