// Size-matched HBM floor probe (not part of the product).  How fast can ANY
// kernel stream the K1 / K2 / K4 byte counts of the 8B shape on this B200,
// timed exactly like bench.py times the product kernels (CUDA graph of R
// back-to-back launches over buffer sets rotated beyond L2, PDL attribute,
// CUDA events)?  The answer separates the kernels' own inefficiency from the
// fixed ramp/drain cost every ~20 MB kernel pays.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/floor.cu -o scripts/bin/floor
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__device__ __forceinline__ void pdl() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
}
__device__ __forceinline__ void ld256(const void* p, uint32_t* r) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}
__device__ __forceinline__ void st128(void* p, uint4 v) {
  asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// "ideal K1": each lane reads RB bytes of input (RB/32 256-bit loads) and
// writes WB bytes (RB * wfrac) -- no math beyond an xor fold.  Unit = 32
// lanes x RB bytes; grid-stride over units, UPW units' loads in flight.
template <int RB, int WB, int UPW>
__global__ void __launch_bounds__(256) k_stream(const uint8_t* __restrict__ in,
                                                uint8_t* __restrict__ out, int64_t units) {
  pdl();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * 8;
  const int64_t gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  for (int64_t u0 = gw; u0 < units; u0 += UPW * nw) {
    uint32_t r[UPW][RB / 4];
#pragma unroll
    for (int k = 0; k < UPW; ++k) {
      int64_t u = u0 + k * nw;
      if (u < units) {
#pragma unroll
        for (int j = 0; j < RB / 32; ++j) ld256(in + (u * 32 + lane) * RB + 32 * j, &r[k][8 * j]);
      }
    }
#pragma unroll
    for (int k = 0; k < UPW; ++k) {
      int64_t u = u0 + k * nw;
      if (u >= units) break;
      uint32_t v[WB / 4];
#pragma unroll
      for (int i = 0; i < WB / 4; ++i) {
        uint32_t a = 0;
#pragma unroll
        for (int j = i; j < RB / 4; j += WB / 4) a ^= r[k][j];
        v[i] = a;
      }
#pragma unroll
      for (int i = 0; i < WB / 16; ++i)
        st128(out + (u * 32 + lane) * WB + 16 * i, make_uint4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
    }
  }
}

// pure read: xor-fold everything, one word per warp written
template <int RB, int UPW>
__global__ void __launch_bounds__(256) k_read(const uint8_t* __restrict__ in,
                                              uint32_t* __restrict__ out, int64_t units) {
  pdl();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * 8;
  const int64_t gw = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  uint32_t acc = 0;
  for (int64_t u0 = gw; u0 < units; u0 += UPW * nw) {
    uint32_t r[UPW][RB / 4];
#pragma unroll
    for (int k = 0; k < UPW; ++k) {
      int64_t u = u0 + k * nw;
      if (u < units) {
#pragma unroll
        for (int j = 0; j < RB / 32; ++j) ld256(in + (u * 32 + lane) * RB + 32 * j, &r[k][8 * j]);
      } else {
#pragma unroll
        for (int j = 0; j < RB / 4; ++j) r[k][j] = 0;
      }
    }
#pragma unroll
    for (int k = 0; k < UPW; ++k)
#pragma unroll
      for (int j = 0; j < RB / 4; ++j) acc ^= r[k][j];
  }
  if (acc == 0x12345678u) out[gw * 32 + lane] = acc;  // keeps the loads alive
}

// pure write
__global__ void __launch_bounds__(256) k_write(uint8_t* __restrict__ out, int64_t n16) {
  pdl();
  int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  for (; i < n16; i += (int64_t)gridDim.x * 256) st128(out + 16 * i, make_uint4(i, 1, 2, 3));
}

template <typename F>
static float time_graph(F launch_all, int reps) {
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  launch_all(s);
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  for (int i = 0; i < 5; ++i) CK(cudaGraphLaunch(ge, s));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaStreamSynchronize(s));
  CK(cudaEventRecord(a, s));
  for (int i = 0; i < reps; ++i) CK(cudaGraphLaunch(ge, s));
  CK(cudaEventRecord(b, s));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  CK(cudaGraphExecDestroy(ge));
  CK(cudaGraphDestroy(g));
  CK(cudaStreamDestroy(s));
  return ms / reps;
}

template <typename... KArgs, typename... Args>
static void launch(bool use_pdl, void (*k)(KArgs...), int grid, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = 256;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = use_pdl ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, k, args...));
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 8388608;  // bf16 values (8B shape)
  const int R = 24, reps = 200;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t rbytes = 2 * n;             // bf16 partial
  const int64_t wbytes = n / 2 + n / 32;    // fp4 codes + e8m0 scales (K1 writes)
  std::vector<uint8_t*> in(R), out(R);
  for (int i = 0; i < R; ++i) {
    CK(cudaMalloc(&in[i], rbytes * 2));
    CK(cudaMalloc(&out[i], rbytes * 2));
    CK(cudaMemset(in[i], i, rbytes * 2));
  }
  printf("# n=%lld read=%lld write=%lld R=%d sms=%d\n", (long long)n, (long long)rbytes,
         (long long)wbytes, R, sms);
  auto report = [&](const char* name, int grid, bool p, double bytes, float ms) {
    printf("{\"kernel\": \"%s\", \"grid\": %d, \"pdl\": %d, \"us\": %.3f, \"gbs\": %.1f}\n", name,
           grid, (int)p, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
  };
  for (int p = 0; p < 2; ++p) {
    // K1-shaped: 64 B in, 16 B out per lane  (2.5 B/value; scale bytes folded in)
    {
      const int64_t units = rbytes / (32 * 64);
      for (int grid : {sms * 2, sms * 4, sms * 8, (int)((units + 15) / 16)}) {
        float ms = time_graph([&](cudaStream_t s) {
          for (int i = 0; i < R; ++i) launch(p, k_stream<64, 16, 2>, grid, s, in[i], out[i], units);
        }, reps);
        report("stream 64B->16B upw2", grid, p, units * 32 * 80.0, ms / R);
      }
      for (int grid : {sms * 4, sms * 8}) {
        float ms = time_graph([&](cudaStream_t s) {
          for (int i = 0; i < R; ++i) launch(p, k_stream<64, 16, 1>, grid, s, in[i], out[i], units);
        }, reps);
        report("stream 64B->16B upw1", grid, p, units * 32 * 80.0, ms / R);
      }
      for (int grid : {sms * 4, sms * 8}) {
        float ms = time_graph([&](cudaStream_t s) {
          for (int i = 0; i < R; ++i) launch(p, k_read<64, 2>, grid, s, in[i], (uint32_t*)out[i], units);
        }, reps);
        report("read 64B upw2", grid, p, (double)rbytes, ms / R);
      }
      for (int grid : {sms * 4, sms * 8}) {
        float ms = time_graph([&](cudaStream_t s) {
          for (int i = 0; i < R; ++i) launch(p, k_write, grid, s, out[i], wbytes / 16);
        }, reps);
        report("write K1 bytes", grid, p, (double)wbytes, ms / R);
      }
    }
    // K2-shaped (2 shards -> bf16): 32 B of codes in, 64 B of output per lane
    {
      const int64_t units = rbytes / (32 * 64);  // one 64 B output per lane
      for (int grid : {sms * 4, sms * 8, (int)((units + 7) / 8)}) {
        float ms = time_graph([&](cudaStream_t s) {
          for (int i = 0; i < R; ++i) launch(p, k_stream<32, 64, 1>, grid, s, in[i], out[i], units);
        }, reps);
        report("K2-shaped 32B->64B", grid, p, units * 32 * 96.0, ms / R);
      }
    }
    // K4-shaped (2 ranks): 2 x 2n read, 2 shards + 2n written = one 128 B-in / 64+... lane
    {
      const int64_t units = 2 * rbytes / (32 * 128);
      for (int grid : {sms * 4, sms * 8}) {
        float ms = time_graph([&](cudaStream_t s) {
          for (int i = 0; i < R; ++i) launch(p, k_stream<128, 96, 1>, grid, s, in[i], out[i], units);
        }, reps);
        report("K4-shaped 128B->96B", grid, p, units * 32 * 224.0, ms / R);
      }
    }
    // copy (torch_copy equivalent): 32 B in, 32 B out
    {
      const int64_t units = 2 * rbytes / (32 * 64);
      for (int grid : {sms * 4, sms * 8}) {
        float ms = time_graph([&](cudaStream_t s) {
          for (int i = 0; i < R; ++i) launch(p, k_stream<64, 64, 1>, grid, s, in[i], out[i], units / 2);
        }, reps);
        report("copy 64B->64B", grid, p, units / 2 * 32 * 128.0, ms / R);
      }
    }
  }
  return 0;
}
