// Host side of libmxb200.so: scheme lowering, dispatch between the fast
// sm_100a kernels (mx_kernels.cuh, one TU per dtype) and the generic
// any-block-size kernels below, and the C ABI of include/mxb200.h.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <type_traits>

#include "../../include/mxb200.h"
#include "mx_kernels.cuh"

namespace mxb {

// ---------------------------------------------------------------------------
// Generic path: any block size, any alignment, f64 input.  Three passes
// through a one-byte-per-block workspace.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ double gen_load(const void* x, int64_t i) {
  if constexpr (std::is_same<T, double>::value) return reinterpret_cast<const double*>(x)[i];
  else return (double)InTraits<T>::to_f32(reinterpret_cast<const T*>(x)[i]);
}

// G1: one thread per block -> stored scale code in ws[global block]
template <typename T>
__global__ void g_scales(const void* x, int64_t n, int64_t cv, int64_t nbc, int64_t nb_total,
                         uint8_t* ws, unsigned long long* nonfinite, Fmt f) {
  int64_t gb = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gb >= nb_total) return;
  int64_t chunk = gb / nbc, lb = gb % nbc;
  int64_t cbase = chunk * cv;
  int64_t len = min(cv, n - cbase);
  int64_t i0 = lb * f.block, i1 = min(i0 + f.block, len);
  uint64_t ab = 0;
  bool bad = false;
  for (int64_t i = i0; i < i1; ++i) {
    double v = gen_load<T>(x, cbase + i);
    uint64_t u = (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffull;
    if (u >= 0x7ff0000000000000ull) {
      if (!bad && nonfinite) atomicMin(nonfinite, (unsigned long long)(cbase + i));
      bad = true;
    }
    ab = max(ab, u);
  }
  int stored = 0;
  if (!bad && ab != 0) stored = shared_exp64(ab, f) + f.sbias;
  ws[gb] = (uint8_t)stored;
}

// G2: one thread per 8-value group -> b bytes of the element stream
template <typename T>
__global__ void g_elems(const void* x, int64_t n, int64_t cv, int64_t gpc, int64_t ng_total,
                        int64_t nbc, const uint8_t* ws, uint8_t* elem_base, int64_t chunk_stride,
                        Fmt f) {
  int64_t gg = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gg >= ng_total) return;
  int64_t chunk = gg / gpc, lg = gg % gpc;
  int64_t cbase = chunk * cv;
  int64_t len = min(cv, n - cbase);
  int64_t i0 = lg * 8;
  if (i0 >= len) return;
  int valid = (int)min((int64_t)8, len - i0);
  uint64_t w = 0;
  for (int t = 0; t < valid; ++t) {
    int64_t li = i0 + t;
    int stored = ws[chunk * nbc + li / f.block];
    if (stored == 0) continue;
    int s = stored - f.sbias;
    double v = gen_load<T>(x, cbase + li);
    uint32_t code;
    if constexpr (std::is_same<T, double>::value) {
      // scale in f64 exactly, encode in f64
      double xs = v * pow2d(-s);
      code = encode_gen(xs, f);
    } else {
      float xs = (float)v * pow2f(-s);
      code = encode_gen(xs, f);
    }
    w |= (uint64_t)code << (t * f.bits);
  }
  uint8_t* p = elem_base + chunk * chunk_stride + lg * f.bits;
  int nbytes = (valid * f.bits + 7) / 8;
  for (int i = 0; i < nbytes; ++i) p[i] = (uint8_t)(w >> (8 * i));
}

// G3: pack the workspace scale codes (k bits each)
__global__ void g_pack_scales(const uint8_t* ws, int64_t n, int64_t cv, int64_t block,
                               int64_t nbc, int64_t gpc8, int64_t ng_total, uint8_t* scale_base,
                               int64_t chunk_stride, int k) {
  int64_t gg = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gg >= ng_total) return;
  int64_t chunk = gg / gpc8, lg = gg % gpc8;
  int64_t len = min(cv, n - chunk * cv);
  int64_t nblocks = (len + block - 1) / block;
  int64_t b0 = lg * 8;
  if (b0 >= nblocks) return;
  int cnt = (int)min((int64_t)8, nblocks - b0);
  uint64_t w = 0;
  for (int i = 0; i < cnt; ++i) w |= (uint64_t)ws[chunk * nbc + b0 + i] << (i * k);
  uint8_t* p = scale_base + chunk * chunk_stride + lg * k;
  int nbytes = (cnt * k + 7) / 8;
  for (int i = 0; i < nbytes; ++i) p[i] = (uint8_t)(w >> (8 * i));
}

// G4: generic decode / rank-order sum, one thread per 8-value group
template <typename OutT>
__global__ void g_dqsum(DArgs A, int64_t gpc, int64_t ng_total) {
  int64_t gg = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gg >= ng_total) return;
  int64_t chunk = gg / gpc, lg = gg % gpc;
  int64_t cbase = chunk * A.cv;
  int64_t len = min(A.cv, A.n - cbase);
  int64_t i0 = lg * 8;
  if (i0 >= len) return;
  int valid = (int)min((int64_t)8, len - i0);
  const Fmt& f = A.f;
  const uint32_t mask = (1u << f.bits) - 1u;
  OutT* out = reinterpret_cast<OutT*>(A.out) + cbase;
  if constexpr (std::is_same<OutT, double>::value) {
    const uint8_t* base = A.in + chunk * A.chunk_stride;
    for (int t = 0; t < valid; ++t) {
      int64_t li = i0 + t;
      int stored = read_scale(base + A.scale_off, li / f.block, f.kbits);
      uint64_t bit = (uint64_t)li * f.bits;
      const uint8_t* e = base + A.elem_off + (bit >> 3);
      int sh = (int)(bit & 7);
      uint32_t wv = e[0];
      if (sh + f.bits > 8) wv |= (uint32_t)e[1] << 8;
      uint32_t code = (wv >> sh) & mask;
      out[li] = decode_gen64(code, stored - f.sbias, stored == 0, f);
    }
  } else {
    float acc[8];
    for (int t = 0; t < 8; ++t) acc[t] = 0.f;
    for (int rk = 0; rk < A.nranks; ++rk) {
      const uint8_t* base = A.in + rk * A.rank_stride + chunk * A.chunk_stride;
      for (int t = 0; t < valid; ++t) {
        int64_t li = i0 + t;
        int stored = read_scale(base + A.scale_off, li / f.block, f.kbits);
        uint64_t bit = (uint64_t)li * f.bits;
        const uint8_t* e = base + A.elem_off + (bit >> 3);
        int sh = (int)(bit & 7);
        uint32_t wv = e[0];
        if (sh + f.bits > 8) wv |= (uint32_t)e[1] << 8;
        uint32_t code = (wv >> sh) & mask;
        float val = decode_gen(code, stored - f.sbias, stored == 0, f);
        acc[t] = A.plain ? val : __fadd_rn(acc[t], val);
      }
    }
    const OutT* res = reinterpret_cast<const OutT*>(A.residual);
    for (int t = 0; t < valid; ++t)
      out[i0 + t] = from_f32<OutT>(
          res ? __fadd_rn(InTraits<OutT>::to_f32(from_f32<OutT>(acc[t])),
                          InTraits<OutT>::to_f32(res[cbase + i0 + t]))
              : acc[t]);
  }
}

__global__ void g_unpack(const uint8_t* packed, int64_t count, int width, uint8_t* codes) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  uint64_t bit = (uint64_t)i * width;
  const uint8_t* e = packed + (bit >> 3);
  int sh = (int)(bit & 7);
  uint32_t w = e[0];
  if (sh + width > 8) w |= (uint32_t)e[1] << 8;
  codes[i] = (uint8_t)((w >> sh) & ((1u << width) - 1u));
}

__global__ void g_pack(const uint8_t* codes, int64_t count, int width, uint8_t* packed) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // 8-code group
  int64_t i0 = g * 8;
  if (i0 >= count) return;
  int cnt = (int)min((int64_t)8, count - i0);
  uint64_t w = 0;
  for (int i = 0; i < cnt; ++i) w |= (uint64_t)(codes[i0 + i] & ((1u << width) - 1u)) << (i * width);
  uint8_t* p = packed + g * width;
  int nbytes = (cnt * width + 7) / 8;
  for (int i = 0; i < nbytes; ++i) p[i] = (uint8_t)(w >> (8 * i));
}

__global__ void g_fill_u64(unsigned long long* p, unsigned long long v) { *p = v; }

// MXC1 container on the device (mx/codec.py:340-348): header (a kernel
// parameter, so the launch is graph-capturable with no host buffer) +
// scale stream + element stream concatenated at arbitrary byte offsets.
// Thread t owns output bytes [16t, 16t+16): a 128-bit store when aligned,
// its source bytes gathered with byte loads (neighbouring lanes share the
// 32 B sectors, so the gather is L1-served; the streams are read once from
// HBM).  Also the realigning copy of deserialize (no header, one segment).
constexpr int kMaxHeader = 544;  // 20 + 8 * 64: numpy's 64 dimensions
struct CatArgs {
  uint8_t hdr[kMaxHeader];
  int hlen;
  const uint8_t* s0;
  int64_t n0;
  const uint8_t* s1;
  int64_t n1;
  uint8_t* out;
  int64_t total;
};

__global__ void __launch_bounds__(256) k_mxc1_cat(const __grid_constant__ CatArgs A) {
  const int64_t o0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 16;
  if (o0 >= A.total) return;
  const int64_t e0 = A.hlen, e1 = e0 + A.n0;
  uint32_t w[4] = {0u, 0u, 0u, 0u};
  const int cnt = (int)min((int64_t)16, A.total - o0);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (i >= cnt) break;
    const int64_t o = o0 + i;
    uint32_t v;
    if (o < e0)
      v = A.hdr[o];
    else if (o < e1)
      v = __ldg(A.s0 + (o - e0));
    else
      v = __ldg(A.s1 + (o - e1));
    w[i >> 2] |= v << (8 * (i & 3));
  }
  uint8_t* d = A.out + o0;
  if (cnt == 16 && ((uintptr_t)d & 15) == 0) {
    *reinterpret_cast<uint4*>(d) = make_uint4(w[0], w[1], w[2], w[3]);
  } else {
    for (int i = 0; i < cnt; ++i) d[i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
  }
}

int launch_cat(const uint8_t* hdr, int hlen, const uint8_t* s0, int64_t n0, const uint8_t* s1,
               int64_t n1, uint8_t* out, cudaStream_t st) {
  CatArgs a;
  memset(&a, 0, sizeof(a));
  if (hlen) memcpy(a.hdr, hdr, hlen);
  a.hlen = hlen; a.s0 = s0; a.n0 = n0; a.s1 = s1; a.n1 = n1; a.out = out;
  a.total = hlen + n0 + n1;
  if (a.total == 0) return 0;
  const int64_t threads = (a.total + 15) / 16;
  k_mxc1_cat<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(a);
  return 1;
}

// k_gemm.cu
cudaError_t launch_gemm_mx(const void* x, const void* w, int64_t M, int64_t N, int64_t K,
                           const Fmt* f, int enc, int64_t chunk_values, int64_t chunk_stride,
                           uint8_t* scale_out, uint8_t* elem_out, void* partial_out,
                           unsigned long long* nonfinite, void* workspace, int64_t workspace_bytes,
                           cudaStream_t st);
int64_t gemm_workspace_bytes(int64_t M, int64_t N);
cudaError_t launch_gemm_mx_push(const void* x, const void* w, int64_t M, int64_t N, int64_t K,
                                const Fmt* fmt, int enc_id, uint8_t* const* peers, int npush,
                                int rank, int64_t slot_stride, int64_t push_off,
                                int64_t scale_off, int64_t elem_off, int64_t scatter_chunk,
                                int64_t flags_off, unsigned int* state,
                                unsigned long long* nonfinite, cudaStream_t st);

}  // namespace mxb

// ===========================================================================
// Host side
// ===========================================================================
namespace {

using namespace mxb;

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MX_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return MX_OK;
}

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
int64_t align16(int64_t v) { return (v + 15) & ~(int64_t)15; }
int64_t align32(int64_t v) { return (v + 31) & ~(int64_t)31; }

int check_scheme(const mx_scheme_t* s) {
  if (!s) return fail(MX_ERR_INVALID_ARGUMENT, "scheme is NULL");
  if (s->kind != MX_KIND_FLOAT && s->kind != MX_KIND_INT)
    return fail(MX_ERR_UNKNOWN_SCHEME, "unknown element kind %d", s->kind);
  if (s->exponent_bits < 0 || s->mantissa_bits < 0)
    return fail(MX_ERR_UNKNOWN_SCHEME, "bit counts must be non-negative");
  if (s->kind == MX_KIND_FLOAT && s->exponent_bits < 1)
    return fail(MX_ERR_UNKNOWN_SCHEME, "FloatMicro needs at least one exponent bit");
  if (s->kind == MX_KIND_INT && (s->exponent_bits != 0 || s->mantissa_bits < 1))
    return fail(MX_ERR_UNKNOWN_SCHEME, "IntSymmetric needs 0 exponent and >=1 magnitude bits");
  int tb = 1 + s->exponent_bits + s->mantissa_bits;
  if (tb < 2 || tb > 8)
    return fail(MX_ERR_UNKNOWN_SCHEME, "total width %d outside the supported [2, 8] range", tb);
  if (s->scale_bits < 4 || s->scale_bits > 8)
    return fail(MX_ERR_UNKNOWN_SCHEME, "scale exponent width must be in [4, 8]");
  if (s->block_size < 1) return fail(MX_ERR_UNKNOWN_SCHEME, "block size must be positive");
  return MX_OK;
}

Fmt make_fmt(const mx_scheme_t* s) {
  Fmt f;
  memset(&f, 0, sizeof(f));
  f.bits = 1 + s->exponent_bits + s->mantissa_bits;
  f.kbits = s->scale_bits;
  f.sbias = (1 << (s->scale_bits - 1)) - 1;
  f.s_min = 1 - f.sbias;
  f.s_max = (1 << s->scale_bits) - 1 - f.sbias;
  f.block = (int)s->block_size;
  f.y = s->mantissa_bits;
  if (s->kind == MX_KIND_FLOAT) {
    int bias = (1 << (s->exponent_bits - 1)) - 1;
    f.lo = 1 - bias;
    f.emax = (1 << s->exponent_bits) - 1 - bias;
    // grid max (2^(y+1)-1) * 2^(emax-y); ratio to 2^emax = 2 - 2^-y
    f.gmax64 = ldexp((double)((1 << (f.y + 1)) - 1), f.emax - f.y);
    f.ovf32 = (1u << 23) - (1u << (23 - f.y));
    f.ovf64 = (1ull << 52) - (1ull << (52 - f.y));
  } else {
    f.lo = f.y;
    f.emax = f.y - 1;
    f.gmax64 = (double)((1 << f.y) - 1);
    // ratio (2^y-1)/2^(y-1) = 2 - 2^(1-y)
    f.ovf32 = (1u << 23) - (1u << (24 - f.y));
    f.ovf64 = (1ull << 52) - (1ull << (53 - f.y));
  }
  f.gmax = (float)f.gmax64;
  // grid*2^s is an exact f32 iff its finest quantum 2^(lo-y+s) >= 2^-149 and
  // gmax*2^s < 2^128 (gmax < 2^(emax+1))
  f.s_fast_lo = max(-149, -149 - (f.lo - f.y));
  f.s_fast_hi = 127 - f.emax;
  return f;
}

int enc_of(const mx_scheme_t* s) {
  if (s->kind == MX_KIND_FLOAT) {
    if (s->exponent_bits == 2 && s->mantissa_bits == 1) return ENC_E2M1;
    if (s->exponent_bits == 2 && s->mantissa_bits == 3) return ENC_E2M3;
    if (s->exponent_bits == 3 && s->mantissa_bits == 2) return ENC_E3M2;
    if (s->exponent_bits == 2 && s->mantissa_bits == 2) return ENC_E2M2;
    return ENC_GEN;
  }
  int b = 1 + s->mantissa_bits;  // sign-magnitude INTb with a compiled width
  return (b == 3 || b == 4 || b == 5 || b == 8) ? ENC_INT : ENC_GEN;
}

// MXB200_TMA=1 routes whole tiles of single-chunk E8M0 16-bit inputs through
// the TMA quantiser (k_quant_tma.cu); the register-path kernel is the default
// because it measured faster at the 8B prefill size (profiles/ROUND1.md).
bool use_tma() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MXB200_TMA");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// MXB200_SYMM_FENCE=1 adds fence.sc.sys beside the release/acquire flag
// operations of the NVLink kernels (k_fused.cuh); off by default -- the
// release/acquire pair alone orders the shard bytes.
int symm_full_fence() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MXB200_SYMM_FENCE");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v;
}

// peer flag wait limit of the NVLink kernels before they report a timeout
// (status word) instead of hanging: MXB200_SYMM_TIMEOUT_MS, default 30 s
unsigned long long symm_timeout_ns() {
  static long long v = -1;
  if (v < 0) {
    const char* e = getenv("MXB200_SYMM_TIMEOUT_MS");
    v = e ? atoll(e) : 30000;
    if (v < 1) v = 1;
  }
  return (unsigned long long)v * 1000000ull;
}

// block sizes with a fast (template) kernel
bool fast_block(int64_t block) { return block == 8 || block == 16 || block == 32 || block == 64; }

bool aligned(const void* p, int a) { return ((uintptr_t)p % a) == 0; }

int in_size(int dtype) {
  switch (dtype) {
    case MX_F32: return 4;
    case MX_F16: return 2;
    case MX_BF16: return 2;
    case MX_F64: return 8;
    default: return 0;
  }
}

// ---- common quantise driver (plain and chunked) ----------------------------
int quantize_impl(const void* x, int dtype, int64_t n, int64_t cv, const mx_scheme_t* s,
                  uint8_t* scale_base, uint8_t* elem_base, int64_t chunk_stride,
                  uint64_t* nonfinite, void* ws, int64_t ws_bytes, cudaStream_t st) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (n < 0) return fail(MX_ERR_INVALID_ARGUMENT, "negative element count");
  if (in_size(dtype) == 0) return fail(MX_ERR_INVALID_ARGUMENT, "unknown input dtype %d", dtype);
  if (n == 0) return MX_OK;
  if (!x || !scale_base || !elem_base) return fail(MX_ERR_INVALID_ARGUMENT, "NULL buffer");
  Fmt f = make_fmt(s);
  int64_t nchunks = cdiv(n, cv);
  if (nchunks > 65535) return fail(MX_ERR_INVALID_ARGUMENT, "too many chunks (%lld)", (long long)nchunks);
  int bits = f.bits;
  int enc = enc_of(s);
  // fast kernels: 256-bit input loads (32-B aligned chunks), 16-B aligned
  // element streams, 8-B aligned scale streams
  bool fast = fast_block(s->block_size) && dtype != MX_F64 && aligned(x, 32) &&
              aligned(elem_base, bits == 8 ? 32 : 16) && aligned(scale_base, 8) &&
              (nchunks == 1 || (chunk_stride % 32 == 0 && (cv * in_size(dtype)) % 32 == 0));
  unsigned long long* nf = reinterpret_cast<unsigned long long*>(nonfinite);
  if (fast) {
    QArgs a;
    a.x = x; a.n = n; a.cv = cv;
    a.units_per_chunk = cdiv(cv, kUnit);
    a.total_units = a.units_per_chunk * nchunks;
    a.scale_base = scale_base; a.elem_base = elem_base; a.chunk_stride = chunk_stride;
    a.nonfinite = nf; a.f = f; a.flat_off = 0;
    int blk = (int)s->block_size;
    // single chunk, E8M0, 16-bit input: TMA pipeline for all whole 8192-value
    // tiles, the register-path kernel for the remainder
    if (nchunks == 1 && f.kbits == 8 && (dtype == MX_BF16 || dtype == MX_F16) && use_tma()) {
      int64_t m = launch_quant_tma(a, dtype == MX_BF16, blk, enc, bits, st);
      if (m > 0) {
        rc = cuda_check("k_quant_tma");
        if (rc || m == n) return rc;
        a.x = static_cast<const uint8_t*>(x) + m * 2;
        a.n = n - m; a.cv = a.n;
        a.units_per_chunk = cdiv(a.n, kUnit);
        a.total_units = a.units_per_chunk;
        a.elem_base = elem_base + m / 8 * bits;
        a.scale_base = scale_base + m / s->block_size;
        a.flat_off = m;
      }
    }
    switch (dtype) {
      case MX_BF16: launch_quant_bf16(a, blk, enc, bits, st); break;
      case MX_F16: launch_quant_f16(a, blk, enc, bits, st); break;
      default: launch_quant_f32(a, blk, enc, bits, st); break;
    }
    return cuda_check("k_quant");
  }
  // generic three-pass path
  int64_t nbc = cdiv(cv, s->block_size);
  int64_t nb_total = nbc * nchunks;
  if (!ws || ws_bytes < nb_total)
    return fail(MX_ERR_WORKSPACE, "generic path needs %lld workspace bytes", (long long)nb_total);
  uint8_t* w = reinterpret_cast<uint8_t*>(ws);
  const int T = 256;
  switch (dtype) {
    case MX_BF16: g_scales<__nv_bfloat16><<<cdiv(nb_total, T), T, 0, st>>>(x, n, cv, nbc, nb_total, w, nf, f); break;
    case MX_F16: g_scales<__half><<<cdiv(nb_total, T), T, 0, st>>>(x, n, cv, nbc, nb_total, w, nf, f); break;
    case MX_F32: g_scales<float><<<cdiv(nb_total, T), T, 0, st>>>(x, n, cv, nbc, nb_total, w, nf, f); break;
    default: g_scales<double><<<cdiv(nb_total, T), T, 0, st>>>(x, n, cv, nbc, nb_total, w, nf, f); break;
  }
  int64_t gpc = cdiv(cv, 8);
  int64_t ng_total = gpc * nchunks;
  switch (dtype) {
    case MX_BF16: g_elems<__nv_bfloat16><<<cdiv(ng_total, T), T, 0, st>>>(x, n, cv, gpc, ng_total, nbc, w, elem_base, chunk_stride, f); break;
    case MX_F16: g_elems<__half><<<cdiv(ng_total, T), T, 0, st>>>(x, n, cv, gpc, ng_total, nbc, w, elem_base, chunk_stride, f); break;
    case MX_F32: g_elems<float><<<cdiv(ng_total, T), T, 0, st>>>(x, n, cv, gpc, ng_total, nbc, w, elem_base, chunk_stride, f); break;
    default: g_elems<double><<<cdiv(ng_total, T), T, 0, st>>>(x, n, cv, gpc, ng_total, nbc, w, elem_base, chunk_stride, f); break;
  }
  int64_t gpc8 = cdiv(nbc, 8);
  int64_t ng8 = gpc8 * nchunks;
  g_pack_scales<<<cdiv(ng8, T), T, 0, st>>>(w, n, cv, s->block_size, nbc, gpc8, ng8, scale_base,
                                             chunk_stride, f.kbits);
  return cuda_check("generic quantise");
}

int dqsum_impl(const uint8_t* in, int64_t rank_stride, int nranks, int64_t n, int64_t cv,
               int64_t chunk_stride, int64_t scale_off, int64_t elem_off, const mx_scheme_t* s,
               void* out, int out_dtype, int plain, cudaStream_t st,
               const void* residual = nullptr) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (n < 0 || nranks < 1 || cv < 1)
    return fail(MX_ERR_INVALID_ARGUMENT, "bad sizes (n=%lld, nranks=%d)", (long long)n, nranks);
  if (n == 0) return MX_OK;
  if (!in || !out) return fail(MX_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (out_dtype == MX_F64 && !(plain && nranks == 1))
    return fail(MX_ERR_INVALID_ARGUMENT, "float64 output is only for plain decompression");
  Fmt f = make_fmt(s);
  DArgs a;
  a.in = in; a.rank_stride = rank_stride; a.nranks = nranks; a.chunk_stride = chunk_stride;
  a.scale_off = scale_off; a.elem_off = elem_off;
  a.n = n; a.cv = cv; a.out = out; a.plain = plain; a.f = f;
  a.residual = residual;
  if (residual && (plain || out_dtype == MX_F64))
    return fail(MX_ERR_INVALID_ARGUMENT, "a residual needs a bf16/f16/f32 sum");
  int64_t nchunks = cdiv(n, cv);
  if (nchunks > 65535) return fail(MX_ERR_INVALID_ARGUMENT, "too many chunks");
  int osz = out_dtype == MX_F32 ? 4 : 2;
  bool fast = fast_block(s->block_size) && out_dtype != MX_F64 && aligned(out, 32) &&
              (!residual || aligned(residual, 32)) &&
              aligned(in + elem_off, 16) && aligned(in + scale_off, 8) && rank_stride % 32 == 0 &&
              chunk_stride % 32 == 0 && (nchunks == 1 || (cv * osz) % 32 == 0);
  if (fast) {
    a.units_per_chunk = cdiv(cv, kUnit2);
    a.total_units = a.units_per_chunk * nchunks;
    int enc = enc_of(s);
    int blk = (int)s->block_size;
    switch (out_dtype) {
      case MX_BF16: launch_dqsum_bf16(a, blk, enc, f.bits, st); break;
      case MX_F16: launch_dqsum_f16(a, blk, enc, f.bits, st); break;
      case MX_F32: launch_dqsum_f32(a, blk, enc, f.bits, st); break;
      default: return fail(MX_ERR_INVALID_ARGUMENT, "unknown output dtype %d", out_dtype);
    }
    return cuda_check("k_dqsum");
  }
  int64_t gpc = cdiv(cv, 8);
  int64_t ng = gpc * nchunks;
  const int T = 256;
  switch (out_dtype) {
    case MX_BF16: g_dqsum<__nv_bfloat16><<<cdiv(ng, T), T, 0, st>>>(a, gpc, ng); break;
    case MX_F16: g_dqsum<__half><<<cdiv(ng, T), T, 0, st>>>(a, gpc, ng); break;
    case MX_F32: g_dqsum<float><<<cdiv(ng, T), T, 0, st>>>(a, gpc, ng); break;
    case MX_F64: g_dqsum<double><<<cdiv(ng, T), T, 0, st>>>(a, gpc, ng); break;
    default: return fail(MX_ERR_INVALID_ARGUMENT, "unknown output dtype %d", out_dtype);
  }
  return cuda_check("generic dequant-sum");
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int mx_abi_version(void) { return MXB200_ABI_VERSION; }

const char* mx_last_error(void) { return g_err; }

int mx_scheme_check(const mx_scheme_t* scheme) { return check_scheme(scheme); }

int mx_stream_nbytes(int64_t n, const mx_scheme_t* s, int64_t* scale_bytes, int64_t* element_bytes) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (n < 0) return fail(MX_ERR_INVALID_ARGUMENT, "negative element count");
  int64_t nb = cdiv(n, s->block_size);
  if (scale_bytes) *scale_bytes = (nb * s->scale_bits + 7) / 8;
  if (element_bytes) *element_bytes = (n * (1 + s->exponent_bits + s->mantissa_bits) + 7) / 8;
  return MX_OK;
}

int mx_shard_layout(int64_t n, const mx_scheme_t* s, int64_t* scale_offset, int64_t* element_offset,
                    int64_t* shard_bytes) {
  int64_t sb, eb;
  int rc = mx_stream_nbytes(n, s, &sb, &eb);
  if (rc) return rc;
  // 32-byte granules: every stream starts on a full sector (256-bit accesses)
  if (scale_offset) *scale_offset = 0;
  if (element_offset) *element_offset = align32(sb);
  if (shard_bytes) *shard_bytes = align32(align32(sb) + eb);
  return MX_OK;
}

int mx_workspace_bytes(int64_t n, const mx_scheme_t* s, int64_t* bytes) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (!bytes || n < 0) return fail(MX_ERR_INVALID_ARGUMENT, "bad arguments");
  // generic quantise: one byte per block
  *bytes = cdiv(n, s->block_size) + 64;
  return MX_OK;
}

int mx_requant_workspace_bytes(int64_t n, const mx_scheme_t* s, int64_t* bytes) {
  int rc = mx_workspace_bytes(n, s, bytes);
  if (rc) return rc;
  // generic requant: an fp32 sum buffer (16-byte aligned) in front of it
  *bytes += align16(4 * n) + 16;
  return MX_OK;
}

int mx_quantize(const void* x, int32_t dtype, int64_t n, const mx_scheme_t* s, uint8_t* scale_stream,
                uint8_t* element_stream, uint64_t* nonfinite, void* workspace,
                int64_t workspace_bytes, void* stream) {
  return quantize_impl(x, dtype, n, n > 0 ? n : 1, s, scale_stream, element_stream, 0, nonfinite,
                       workspace, workspace_bytes, (cudaStream_t)stream);
}

int mx_quantize_chunks(const void* x, int32_t dtype, int64_t n, int64_t chunk_values,
                       const mx_scheme_t* s, uint8_t* shards, int64_t shard_stride,
                       uint64_t* nonfinite, void* workspace, int64_t workspace_bytes, void* stream) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (chunk_values < 1 || chunk_values % (8 * s->block_size) != 0)
    return fail(MX_ERR_INVALID_ARGUMENT, "chunk_values must be a positive multiple of 8*block");
  int64_t so, eo, sbytes;
  mx_shard_layout(chunk_values, s, &so, &eo, &sbytes);
  if (shard_stride < sbytes) return fail(MX_ERR_INVALID_ARGUMENT, "shard_stride smaller than a shard");
  return quantize_impl(x, dtype, n, chunk_values, s, shards + so, shards + eo, shard_stride,
                       nonfinite, workspace, workspace_bytes, (cudaStream_t)stream);
}

int mx_dequantize(const uint8_t* scale_stream, const uint8_t* element_stream, int64_t n,
                  const mx_scheme_t* s, void* out, int32_t out_dtype, void* stream) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (n == 0) return MX_OK;
  if (!scale_stream || !element_stream) return fail(MX_ERR_INVALID_ARGUMENT, "NULL stream");
  // the two streams are addressed as one "shard": base = scale stream,
  // element offset = distance to the element stream (any value)
  int64_t off = (int64_t)(element_stream - scale_stream);
  return dqsum_impl(scale_stream, 0, 1, n, n, 0, 0, off, s, out, out_dtype, 1,
                    (cudaStream_t)stream);
}

int mx_dequant_sum(const uint8_t* shards, int64_t rank_stride, int32_t nranks, int64_t n,
                   int64_t chunk_values, int64_t chunk_stride, const mx_scheme_t* s, void* out,
                   int32_t out_dtype, void* stream) {
  if (out_dtype == MX_F64) return fail(MX_ERR_INVALID_ARGUMENT, "sums are fp32 (mx/netbench.py:332)");
  int64_t so, eo, sbytes;
  int rc = mx_shard_layout(chunk_values, s, &so, &eo, &sbytes);
  if (rc) return rc;
  return dqsum_impl(shards, rank_stride, nranks, n, chunk_values, chunk_stride, so, eo, s, out,
                    out_dtype, 0, (cudaStream_t)stream);
}

int mx_dequant_sum_residual(const uint8_t* shards, int64_t rank_stride, int32_t nranks,
                            int64_t n, int64_t chunk_values, int64_t chunk_stride,
                            const mx_scheme_t* s, const void* residual, void* out,
                            int32_t out_dtype, void* stream) {
  if (out_dtype == MX_F64) return fail(MX_ERR_INVALID_ARGUMENT, "sums are fp32 (mx/netbench.py:332)");
  if (!residual) return fail(MX_ERR_INVALID_ARGUMENT, "NULL residual");
  int64_t so, eo, sbytes;
  int rc = mx_shard_layout(chunk_values, s, &so, &eo, &sbytes);
  if (rc) return rc;
  return dqsum_impl(shards, rank_stride, nranks, n, chunk_values, chunk_stride, so, eo, s, out,
                    out_dtype, 0, (cudaStream_t)stream, residual);
}

int mx_dequant_sum_requant(const uint8_t* shards, int64_t rank_stride, int32_t nranks, int64_t n,
                           int64_t chunk_values, const mx_scheme_t* s, uint8_t* out_shard,
                           uint64_t* nonfinite, void* workspace, int64_t workspace_bytes,
                           void* stream) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (n < 0 || nranks < 1 || chunk_values < n) return fail(MX_ERR_INVALID_ARGUMENT, "bad sizes");
  if (n == 0) return MX_OK;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t so, eo, sbytes;
  mx_shard_layout(chunk_values, s, &so, &eo, &sbytes);
  Fmt f = make_fmt(s);
  if (fast_block(s->block_size) && aligned(shards, 32) && rank_stride % 32 == 0 &&
      aligned(out_shard, 32)) {
    RArgs a;
    a.in = shards; a.rank_stride = rank_stride; a.nranks = nranks;
    a.scale_off = so; a.elem_off = eo; a.n = n;
    a.total_units = cdiv(n, kUnit);
    a.out_scale = out_shard + so; a.out_elem = out_shard + eo;
    a.nonfinite = reinterpret_cast<unsigned long long*>(nonfinite); a.f = f;
    launch_requant(a, (int)s->block_size, enc_of(s), f.bits, st);
    return cuda_check("k_requant");
  }
  // generic: fp32 sum into the workspace, then the generic quantiser
  int64_t need;
  mx_requant_workspace_bytes(n, s, &need);
  if (!workspace || workspace_bytes < need)
    return fail(MX_ERR_WORKSPACE, "generic requant needs %lld workspace bytes", (long long)need);
  uint8_t* w = reinterpret_cast<uint8_t*>(workspace);
  uintptr_t p = ((uintptr_t)w + 15) & ~(uintptr_t)15;
  float* sum = reinterpret_cast<float*>(p);
  uint8_t* rest = reinterpret_cast<uint8_t*>(p + align16(4 * n));
  int64_t rest_bytes = workspace_bytes - (int64_t)((uint8_t*)rest - w);
  rc = dqsum_impl(shards, rank_stride, nranks, n, chunk_values, 0, so, eo, s, sum, MX_F32, 0, st);
  if (rc) return rc;
  return quantize_impl(sum, MX_F32, n, n, s, out_shard + so, out_shard + eo, 0, nonfinite, rest,
                       rest_bytes, st);
}

int mx_allreduce_fused(const void* const* partials, int32_t dtype, int32_t nranks, int64_t n,
                       const mx_scheme_t* s, uint8_t* shards, int64_t shard_stride, void* out,
                       int32_t out_dtype, uint32_t* barrier, uint64_t* nonfinite, void* stream) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (n <= 0 || nranks < 1) return fail(MX_ERR_INVALID_ARGUMENT, "bad sizes");
  if (!partials || !shards || !out || !barrier) return fail(MX_ERR_INVALID_ARGUMENT, "NULL buffer");
  int64_t so, eo, sbytes;
  mx_shard_layout(n, s, &so, &eo, &sbytes);
  if (shard_stride < sbytes || shard_stride % 32 != 0)
    return fail(MX_ERR_INVALID_ARGUMENT, "shard_stride must be >= shard bytes and 32-aligned");
  Fmt f = make_fmt(s);
  if (dtype != MX_BF16 || (out_dtype != MX_BF16 && out_dtype != MX_F32) || !aligned(shards, 32) ||
      !aligned(out, 32) || !fast_block(s->block_size))
    return fail(MX_ERR_UNSUPPORTED, "fused path: bf16 in, bf16/f32 out, B in {8,16,32,64}");
  FArgs a;
  a.partials = partials; a.nranks = nranks; a.n = n;
  a.shards = shards; a.shard_stride = shard_stride; a.scale_off = so; a.elem_off = eo;
  a.out = out; a.bar = barrier; a.nonfinite = reinterpret_cast<unsigned long long*>(nonfinite);
  a.f = f;
  if (!launch_fused_oneshot(a, out_dtype == MX_BF16, (int)s->block_size, enc_of(s), f.bits,
                            (cudaStream_t)stream))
    return fail(MX_ERR_UNSUPPORTED, "fused path: element width %d not instantiated", f.bits);
  return cuda_check("k_fused_oneshot");
}

static int gemm_impl(const void* x, const void* w, int64_t M, int64_t N, int64_t K,
                     const mx_scheme_t* s, int64_t cv, int64_t cs, uint8_t* scale_stream,
                     uint8_t* element_stream, void* partial, uint64_t* nonfinite, void* stream) {
  if (s) {
    int rc = check_scheme(s);
    if (rc) return rc;
    if (!scale_stream || !element_stream) return fail(MX_ERR_INVALID_ARGUMENT, "NULL stream buffer");
  } else if (!partial) {
    return fail(MX_ERR_INVALID_ARGUMENT, "plain GEMM needs a partial buffer");
  }
  if (!x || !w) return fail(MX_ERR_INVALID_ARGUMENT, "NULL operand");
  if (M < 1 || N < 1 || K < 1) return fail(MX_ERR_INVALID_ARGUMENT, "bad sizes");
  if (partial && !aligned(partial, 16)) return fail(MX_ERR_INVALID_ARGUMENT, "partial not 16-byte aligned");
  Fmt f;
  if (s) f = make_fmt(s);
  // opt-in stream-K (MXB200_GEMM_STREAMK=1, measured slower than whole tiles)
  // needs an fp32 fix-up workspace: grown on demand, never freed; not for
  // use under graph capture
  static void* ws = nullptr;
  static int64_t ws_cap = 0;
  int64_t ws_need = 0;
  if (const char* e = getenv("MXB200_GEMM_STREAMK"); e && atoi(e)) {
    ws_need = gemm_workspace_bytes(M, N);
    if (ws_need > ws_cap) {
      if (ws) cudaFree(ws);
      ws = nullptr; ws_cap = 0;
      if (cudaMalloc(&ws, ws_need) != cudaSuccess) return fail(MX_ERR_CUDA, "stream-K workspace");
      ws_cap = ws_need;
    }
  }
  cudaError_t e = launch_gemm_mx(x, w, M, N, K, s ? &f : nullptr, s ? enc_of(s) : 0, cv, cs,
                                 scale_stream, element_stream,
                                 partial, reinterpret_cast<unsigned long long*>(nonfinite),
                                 ws_need ? ws : nullptr, ws_need ? ws_cap : 0,
                                 (cudaStream_t)stream);
  if (e == cudaErrorNotSupported)
    return fail(MX_ERR_UNSUPPORTED,
                "fused GEMM: needs K %% 64 == 0, N %% 128 == 0, 16-byte aligned operands, "
                "E8M0 scales with B in {8, 16, 32} (fp4_e2m1 / fp6 / fp5_e2m2 / int8) or E5M0 "
                "scales (fp4_e2m1 B in {8, 16, 32}, fp5_e2m2 B = 32, N %% 256 == 0)");
  if (e != cudaSuccess) return fail(MX_ERR_CUDA, "k_gemm_mx: %s", cudaGetErrorString(e));
  return cuda_check("k_gemm_mx");
}

int mx_gemm_quantize(const void* x, const void* w, int64_t M, int64_t N, int64_t K,
                     const mx_scheme_t* s, uint8_t* scale_stream, uint8_t* element_stream,
                     void* partial, uint64_t* nonfinite, void* stream) {
  return gemm_impl(x, w, M, N, K, s, M * N, 0, scale_stream, element_stream, partial, nonfinite,
                   stream);
}

int mx_gemm_quantize_chunks(const void* x, const void* w, int64_t M, int64_t N, int64_t K,
                            int64_t chunk_values, const mx_scheme_t* s, uint8_t* shards,
                            int64_t shard_stride, void* partial, uint64_t* nonfinite,
                            void* stream) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (!shards) return fail(MX_ERR_INVALID_ARGUMENT, "NULL shards");
  if (chunk_values < 1 || (chunk_values < M * N && chunk_values % (8 * s->block_size) != 0))
    return fail(MX_ERR_INVALID_ARGUMENT,
                "chunk_values must be >= M*N or a positive multiple of 8*block_size");
  int64_t so, eo, sbytes;
  mx_shard_layout(chunk_values, s, &so, &eo, &sbytes);
  const int64_t nchunks = (M * N + chunk_values - 1) / chunk_values;
  if (nchunks > 1 && (shard_stride < sbytes || shard_stride % 32 != 0))
    return fail(MX_ERR_INVALID_ARGUMENT, "shard_stride must be >= shard bytes and 32-aligned");
  return gemm_impl(x, w, M, N, K, s, chunk_values, shard_stride, shards + so, shards + eo,
                   partial, nonfinite, stream);
}

#define PUSH_SET                                                                     \
  "fp4_e2m1 E8M0 with B in {16, 32}, fp4_e2m1 E5M0 with B in {8, 16, 32} or fp5_e2m2 " \
  "E5M0 with B = 32"

int mx_push_layout(int64_t n, const mx_scheme_t* s, int32_t nranks, int64_t* slot_stride,
                   int64_t* shard_stride, int64_t* flags_offset, int64_t* buffer_bytes) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (n <= 0 || nranks < 1) return fail(MX_ERR_INVALID_ARGUMENT, "bad sizes");
  int64_t so, eo, sb;
  mx_shard_layout(n, s, &so, &eo, &sb);
  const int64_t slot = (int64_t)nranks * sb;
  const int64_t foff = (2 * slot + 255) / 256 * 256;
  if (slot_stride) *slot_stride = slot;
  if (shard_stride) *shard_stride = sb;
  if (flags_offset) *flags_offset = foff;
  if (buffer_bytes) *buffer_bytes = foff + ((int64_t)nranks * 4 + 255) / 256 * 256;
  return MX_OK;
}

int mx_gemm_allgather_push(const void* x, const void* w, int64_t M, int64_t N, int64_t K,
                           const mx_scheme_t* s, uint8_t* const* peer_bufs, int32_t rank,
                           int32_t nranks, uint32_t* state, uint64_t* nonfinite, void* stream) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (!x || !w || !peer_bufs || !state)
    return fail(MX_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (M < 1 || N < 1 || K < 1 || rank < 0 || rank >= nranks)
    return fail(MX_ERR_INVALID_ARGUMENT, "bad sizes");
  int64_t slot, sb, foff, total, so, eo, sbytes;
  mx_push_layout(M * N, s, nranks, &slot, &sb, &foff, &total);
  mx_shard_layout(M * N, s, &so, &eo, &sbytes);
  Fmt f = make_fmt(s);
  cudaError_t e = launch_gemm_mx_push(x, w, M, N, K, &f, enc_of(s), peer_bufs, nranks,
                                      rank, slot, (int64_t)rank * sb, so, eo, 0, foff,
                                      reinterpret_cast<unsigned int*>(state),
                                      reinterpret_cast<unsigned long long*>(nonfinite),
                                      (cudaStream_t)stream);
  if (e == cudaErrorNotSupported)
    return fail(MX_ERR_UNSUPPORTED,
                "GEMM + all-gather push: " PUSH_SET ", N %% 256 == 0, K %% 64 == 0, at most "
                "8 ranks, 16-byte aligned operands");
  if (e != cudaSuccess) return fail(MX_ERR_CUDA, "k_gemm_mx2 push: %s", cudaGetErrorString(e));
  return cuda_check("k_gemm_mx2 push");
}

int mx_push_dequant_sum(const uint8_t* buf, int64_t n, const mx_scheme_t* s, int32_t rank,
                        int32_t nranks, const uint32_t* flags, const uint32_t* state,
                        uint32_t* status, void* out, int32_t out_dtype, const void* residual,
                        void* stream) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (!buf || !flags || !state || !status || !out || rank < 0 || rank >= nranks)
    return fail(MX_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (n <= 0 || n % 1024 != 0 || nranks < 1 || nranks > 8)
    return fail(MX_ERR_UNSUPPORTED, "push decode: n %% 1024 == 0, 1..8 ranks");
  Fmt f = make_fmt(s);
  if ((out_dtype != MX_BF16 && out_dtype != MX_F32) || !aligned(out, 32) ||
      !aligned(residual, 32))
    return fail(MX_ERR_UNSUPPORTED, "push decode: bf16/f32 out, 32-B aligned");
  int64_t slot, sb, foff, total, so, eo, sbytes;
  mx_push_layout(n, s, nranks, &slot, &sb, &foff, &total);
  mx_shard_layout(n, s, &so, &eo, &sbytes);
  PArgs a;
  a.buf = buf; a.slot_stride = slot; a.shard_stride = sb; a.scale_off = so; a.elem_off = eo;
  a.nranks = nranks; a.n = n; a.rank = rank;
  a.flags = reinterpret_cast<const unsigned int*>(flags);
  a.state = reinterpret_cast<const unsigned int*>(state);
  a.status = reinterpret_cast<unsigned int*>(status);
  a.timeout_ns = symm_timeout_ns();
  a.out = out; a.residual = residual; a.f = f;
  if (!launch_push_dqsum(a, out_dtype == MX_BF16, (int)s->block_size, enc_of(s),
                         (cudaStream_t)stream))
    return fail(MX_ERR_UNSUPPORTED, "push decode: " PUSH_SET);
  return cuda_check("k_push_dqsum");
}

int mx_push2_layout(int64_t n, const mx_scheme_t* s, int32_t nranks, int64_t* chunk_values,
                    int64_t* slot_stride, int64_t* shard_stride, int64_t* flags_offset,
                    int64_t* buffer_bytes) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (n <= 0 || nranks < 1 || n % (1024 * (int64_t)nranks) != 0)
    return fail(MX_ERR_UNSUPPORTED, "two-shot push: n %% (1024 * nranks) == 0");
  const int64_t c = n / nranks;
  int64_t so, eo, sb;
  mx_shard_layout(c, s, &so, &eo, &sb);
  const int64_t slot = 2 * (int64_t)nranks * sb;  // RS region, then AG region
  const int64_t foff = (2 * slot + 255) / 256 * 256;
  if (chunk_values) *chunk_values = c;
  if (slot_stride) *slot_stride = slot;
  if (shard_stride) *shard_stride = sb;
  if (flags_offset) *flags_offset = foff;
  if (buffer_bytes) *buffer_bytes = foff + ((int64_t)nranks * 8 + 255) / 256 * 256;
  return MX_OK;
}

int mx_gemm_reducescatter_push(const void* x, const void* w, int64_t M, int64_t N, int64_t K,
                               const mx_scheme_t* s, uint8_t* const* peer_bufs, int32_t rank,
                               int32_t nranks, uint32_t* state, uint64_t* nonfinite,
                               void* stream) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (!x || !w || !peer_bufs || !state) return fail(MX_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (M < 1 || N < 1 || K < 1 || rank < 0 || rank >= nranks)
    return fail(MX_ERR_INVALID_ARGUMENT, "bad sizes");
  int64_t c, slot, sb, foff, total, so, eo, sbytes;
  rc = mx_push2_layout(M * N, s, nranks, &c, &slot, &sb, &foff, &total);
  if (rc) return rc;
  mx_shard_layout(c, s, &so, &eo, &sbytes);
  Fmt f = make_fmt(s);
  cudaError_t e = launch_gemm_mx_push(x, w, M, N, K, &f, enc_of(s), peer_bufs, nranks, rank,
                                      slot, (int64_t)rank * sb, so, eo, c, foff,
                                      reinterpret_cast<unsigned int*>(state),
                                      reinterpret_cast<unsigned long long*>(nonfinite),
                                      (cudaStream_t)stream);
  if (e == cudaErrorNotSupported)
    return fail(MX_ERR_UNSUPPORTED,
                "GEMM + reduce-scatter push: " PUSH_SET ", N %% 256 == 0, K %% 64 == 0, "
                "M*N %% (1024 * nranks) == 0, at most 8 ranks");
  if (e != cudaSuccess) return fail(MX_ERR_CUDA, "k_gemm_mx2 push: %s", cudaGetErrorString(e));
  return cuda_check("k_gemm_mx2 reduce-scatter push");
}

static int push2_args(P2Args& a, const uint8_t* buf, int64_t n, const mx_scheme_t* s,
                      int32_t rank, int32_t nranks, uint8_t* const* peer_bufs,
                      uint32_t* const* peer_flags, uint32_t* state, uint32_t* status) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (!buf || !state || !status || rank < 0 || rank >= nranks || nranks > 8)
    return fail(MX_ERR_INVALID_ARGUMENT, "bad buffers or ranks");
  Fmt f = make_fmt(s);
  int64_t c, slot, sb, foff, total, so, eo, sbytes;
  rc = mx_push2_layout(n, s, nranks, &c, &slot, &sb, &foff, &total);
  if (rc) return rc;
  mx_shard_layout(c, s, &so, &eo, &sbytes);
  a.buf = buf; a.slot_stride = slot; a.shard_stride = sb; a.scale_off = so; a.elem_off = eo;
  a.nranks = nranks; a.rank = rank; a.n = n; a.c = c;
  a.peer_bufs = peer_bufs;
  a.peer_flags = reinterpret_cast<unsigned int* const*>(peer_flags);
  a.flags = reinterpret_cast<const unsigned int*>(buf + foff);
  a.state = state;
  a.status = reinterpret_cast<unsigned int*>(status);
  a.timeout_ns = symm_timeout_ns();
  a.nonfinite = nullptr; a.out = nullptr; a.residual = nullptr;
  a.f = f;
  return MX_OK;
}

int mx_push2_requant(const uint8_t* buf, int64_t n, const mx_scheme_t* s, int32_t rank,
                     int32_t nranks, uint8_t* const* peer_bufs, uint32_t* const* peer_flags,
                     uint32_t* state, uint32_t* status, uint64_t* nonfinite, void* stream) {
  P2Args a;
  int rc = push2_args(a, buf, n, s, rank, nranks, peer_bufs, peer_flags, state, status);
  if (rc) return rc;
  if (!peer_bufs || !peer_flags) return fail(MX_ERR_INVALID_ARGUMENT, "NULL peer buffers");
  a.nonfinite = reinterpret_cast<unsigned long long*>(nonfinite);
  if (!launch_push2_requant(a, (int)s->block_size, enc_of(s), (cudaStream_t)stream))
    return fail(MX_ERR_UNSUPPORTED, "two-shot push: " PUSH_SET);
  return cuda_check("k_push2_requant");
}

int mx_push2_decode(const uint8_t* buf, int64_t n, const mx_scheme_t* s, int32_t rank,
                    int32_t nranks, const uint32_t* state, uint32_t* status, void* out,
                    int32_t out_dtype, const void* residual, void* stream) {
  P2Args a;
  int rc = push2_args(a, buf, n, s, rank, nranks, nullptr, nullptr,
                      const_cast<uint32_t*>(state), status);
  if (rc) return rc;
  if (!out || (out_dtype != MX_BF16 && out_dtype != MX_F32) || !aligned(out, 32) ||
      !aligned(residual, 32))
    return fail(MX_ERR_UNSUPPORTED, "two-shot push decode: bf16/f32 out, 32-B aligned");
  a.out = out; a.residual = residual;
  if (!launch_push2_decode(a, out_dtype == MX_BF16, (int)s->block_size, enc_of(s),
                           (cudaStream_t)stream))
    return fail(MX_ERR_UNSUPPORTED, "two-shot push: " PUSH_SET);
  return cuda_check("k_push2_decode");
}

int mx_symm_layout(int64_t n, const mx_scheme_t* s, int32_t nranks, int64_t* slot_stride,
                   int64_t* flags_offset, int64_t* buffer_bytes, int64_t* ctas) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (n <= 0 || nranks < 1) return fail(MX_ERR_INVALID_ARGUMENT, "bad sizes");
  int64_t so, eo, sbytes;
  mx_shard_layout(n, s, &so, &eo, &sbytes);
  const int64_t slot = (sbytes + 255) / 256 * 256;
  const int64_t g = symm_ctas(n);
  if (slot_stride) *slot_stride = slot;
  if (flags_offset) *flags_offset = 2 * slot;
  if (buffer_bytes) *buffer_bytes = 2 * slot + ((int64_t)nranks * g * 4 + 255) / 256 * 256;
  if (ctas) *ctas = g;
  return MX_OK;
}

int mx_allreduce_symm(const void* x, int32_t dtype, int64_t n, const mx_scheme_t* s,
                      uint8_t* const* peer_bufs, uint32_t* const* peer_flags, int32_t rank,
                      int32_t nranks, int64_t slot_stride, void* out, int32_t out_dtype,
                      const void* residual, uint32_t* status, uint32_t* epochs,
                      uint64_t* nonfinite, void* stream) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (n <= 0 || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(MX_ERR_INVALID_ARGUMENT, "bad sizes");
  if (!x || !peer_bufs || !peer_flags || !out || !status || !epochs)
    return fail(MX_ERR_INVALID_ARGUMENT, "NULL buffer");
  int64_t so, eo, sbytes;
  mx_shard_layout(n, s, &so, &eo, &sbytes);
  Fmt f = make_fmt(s);
  if (dtype != MX_BF16 || (out_dtype != MX_BF16 && out_dtype != MX_F32) || n % 1024 != 0 ||
      slot_stride < sbytes || slot_stride % 32 != 0 || !aligned(x, 32) ||
      !aligned(out, 32) || !aligned(residual, 32))
    return fail(MX_ERR_UNSUPPORTED,
                "symmetric path: bf16 in, bf16/f32 out, n %% 1024 == 0, 32-B aligned");
  if (nranks > kThreads) return fail(MX_ERR_UNSUPPORTED, "at most %d ranks", kThreads);
  SArgs a;
  a.x = x; a.n = n;
  a.bufs = peer_bufs; a.flags = reinterpret_cast<unsigned int* const*>(peer_flags);
  a.rank = rank; a.nranks = nranks; a.slot_stride = slot_stride;
  a.scale_off = so; a.elem_off = eo; a.out = out; a.residual = residual; a.status = status;
  a.epoch = epochs; a.nonfinite = reinterpret_cast<unsigned long long*>(nonfinite); a.f = f;
  a.full_fence = symm_full_fence();
  a.timeout_ns = symm_timeout_ns();
  if (!launch_symm_oneshot(a, out_dtype == MX_BF16, (int)s->block_size, enc_of(s), f.bits,
                           (cudaStream_t)stream))
    return fail(MX_ERR_UNSUPPORTED, "symmetric path: scheme not instantiated");
  return cuda_check("k_symm_flow");
}

int mx_symm_twoshot_layout(int64_t n, const mx_scheme_t* s, int32_t nranks,
                           int64_t* slot_stride, int64_t* shard_stride, int64_t* flags_offset,
                           int64_t* buffer_bytes, int64_t* ctas) {
  int rc = check_scheme(s);
  if (rc) return rc;
  if (n <= 0 || nranks < 1 || n % (1024 * (int64_t)nranks) != 0)
    return fail(MX_ERR_UNSUPPORTED, "two-shot symmetric path needs n %% (1024*nranks) == 0");
  const int64_t c = n / nranks;
  int64_t so, eo, sc;
  mx_shard_layout(c, s, &so, &eo, &sc);
  const int64_t slot = ((nranks + 1) * sc + 255) / 256 * 256;
  const int64_t g = symm_ctas(c);
  if (slot_stride) *slot_stride = slot;
  if (shard_stride) *shard_stride = sc;
  if (flags_offset) *flags_offset = 2 * slot;
  if (buffer_bytes) *buffer_bytes = 2 * slot + (2 * (int64_t)nranks * g * 4 + 255) / 256 * 256;
  if (ctas) *ctas = g;
  return MX_OK;
}

int mx_allreduce_symm_twoshot(const void* x, int32_t dtype, int64_t n, const mx_scheme_t* s,
                              uint8_t* const* peer_bufs, uint32_t* const* peer_flags,
                              int32_t rank, int32_t nranks, void* out, int32_t out_dtype,
                              const void* residual, uint32_t* status, uint32_t* epochs,
                              uint64_t* nonfinite, void* stream) {
  int64_t slot, sc, foff, total, g;
  int rc = mx_symm_twoshot_layout(n, s, nranks, &slot, &sc, &foff, &total, &g);
  if (rc) return rc;
  if (rank < 0 || rank >= nranks) return fail(MX_ERR_INVALID_ARGUMENT, "bad rank");
  if (!x || !peer_bufs || !peer_flags || !out || !status || !epochs)
    return fail(MX_ERR_INVALID_ARGUMENT, "NULL buffer");
  Fmt f = make_fmt(s);
  if (dtype != MX_BF16 || (out_dtype != MX_BF16 && out_dtype != MX_F32) ||
      !aligned(x, 32) || !aligned(out, 32) || !aligned(residual, 32))
    return fail(MX_ERR_UNSUPPORTED, "two-shot symmetric path: bf16 in, bf16/f32 out");
  if (nranks > kThreads) return fail(MX_ERR_UNSUPPORTED, "at most %d ranks", kThreads);
  const int64_t c = n / nranks;
  int64_t so, eo, sb;
  mx_shard_layout(c, s, &so, &eo, &sb);
  S2Args a;
  a.x = x; a.n = n; a.c = c;
  a.bufs = peer_bufs; a.flags = reinterpret_cast<unsigned int* const*>(peer_flags);
  a.rank = rank; a.nranks = nranks; a.slot_stride = slot; a.shard_stride = sc;
  a.scale_off = so; a.elem_off = eo; a.out = out; a.residual = residual; a.status = status;
  a.epoch = epochs;
  a.nonfinite = reinterpret_cast<unsigned long long*>(nonfinite); a.f = f;
  a.full_fence = symm_full_fence();
  a.timeout_ns = symm_timeout_ns();
  if (!launch_symm_twoshot(a, out_dtype == MX_BF16, (int)s->block_size, enc_of(s), f.bits,
                           (cudaStream_t)stream))
    return fail(MX_ERR_UNSUPPORTED, "two-shot symmetric path: scheme not instantiated");
  return cuda_check("k_symm2_flow");
}

int mx_unpack_codes(const uint8_t* packed, int64_t count, int32_t width, uint8_t* codes, void* stream) {
  if (width < 1 || width > 8) return fail(MX_ERR_INVALID_ARGUMENT, "width %d outside [1, 8]", width);
  if (count <= 0) return MX_OK;
  g_unpack<<<cdiv(count, 256), 256, 0, (cudaStream_t)stream>>>(packed, count, width, codes);
  return cuda_check("g_unpack");
}

int mx_pack_codes(const uint8_t* codes, int64_t count, int32_t width, uint8_t* packed, void* stream) {
  if (width < 1 || width > 8) return fail(MX_ERR_INVALID_ARGUMENT, "width %d outside [1, 8]", width);
  if (count <= 0) return MX_OK;
  int64_t groups = cdiv(count, 8);
  g_pack<<<cdiv(groups, 256), 256, 0, (cudaStream_t)stream>>>(codes, count, width, packed);
  return cuda_check("g_pack");
}

int mx_serialize(const uint8_t* header, int32_t header_bytes, const uint8_t* scale_stream,
                 int64_t scale_bytes, const uint8_t* element_stream, int64_t element_bytes,
                 uint8_t* out, void* stream) {
  if (header_bytes < 0 || header_bytes > kMaxHeader)
    return fail(MX_ERR_INVALID_ARGUMENT, "header of %d bytes (at most %d: 64 dimensions)",
                header_bytes, kMaxHeader);
  if (scale_bytes < 0 || element_bytes < 0) return fail(MX_ERR_INVALID_ARGUMENT, "bad sizes");
  if ((header_bytes && !header) || (scale_bytes && !scale_stream) ||
      (element_bytes && !element_stream) || !out)
    return fail(MX_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (launch_cat(header, header_bytes, scale_stream, scale_bytes, element_stream, element_bytes,
                 out, (cudaStream_t)stream))
    return cuda_check("k_mxc1_cat");
  return MX_OK;
}

int mx_copy_bytes(const uint8_t* src, int64_t nbytes, uint8_t* dst, void* stream) {
  if (nbytes < 0 || (nbytes && (!src || !dst))) return fail(MX_ERR_INVALID_ARGUMENT, "bad copy");
  if (launch_cat(nullptr, 0, src, nbytes, nullptr, 0, dst, (cudaStream_t)stream))
    return cuda_check("k_mxc1_cat");
  return MX_OK;
}

int mx_memset_async(void* ptr, int32_t value, int64_t bytes, void* stream) {
  if (!ptr || bytes < 0) return fail(MX_ERR_INVALID_ARGUMENT, "bad memset");
  if (cudaMemsetAsync(ptr, value, (size_t)bytes, (cudaStream_t)stream) != cudaSuccess)
    return cuda_check("cudaMemsetAsync");
  return MX_OK;
}

int mx_nonfinite_reset(uint64_t* nonfinite, void* stream) {
  if (!nonfinite) return fail(MX_ERR_INVALID_ARGUMENT, "NULL flag");
  g_fill_u64<<<1, 1, 0, (cudaStream_t)stream>>>(reinterpret_cast<unsigned long long*>(nonfinite),
                                                ~0ull);
  return cuda_check("mx_nonfinite_reset");
}

int mx_chanint_compress(const void* x, int32_t dtype, int64_t rows, int64_t channels,
                        int32_t bits, uint16_t* scales, uint8_t* codes, void* workspace,
                        int64_t workspace_bytes, uint64_t* nonfinite, void* stream) {
  if (bits < 2 || bits > 8) return fail(MX_ERR_INVALID_ARGUMENT, "bits must be in [2, 8], got %d", bits);
  if (rows < 0 || channels < 1) return fail(MX_ERR_SHAPE, "bad shape (%lld x %lld)", (long long)rows, (long long)channels);
  if (in_size(dtype) == 0) return fail(MX_ERR_INVALID_ARGUMENT, "unknown input dtype %d", dtype);
  if (rows == 0) return MX_OK;
  if (!x || !scales || !codes) return fail(MX_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (!workspace || workspace_bytes < 8 * channels)
    return fail(MX_ERR_WORKSPACE, "channel INT needs %lld workspace bytes", (long long)(8 * channels));
  launch_chanint_compress(x, dtype, rows, channels, bits, scales, codes, workspace,
                          reinterpret_cast<unsigned long long*>(nonfinite), (cudaStream_t)stream);
  return cuda_check("chanint compress");
}

int mx_chanint_decompress(const uint16_t* scales, const uint8_t* codes, int64_t rows,
                          int64_t channels, int32_t bits, void* out, int32_t out_dtype,
                          void* stream) {
  if (bits < 2 || bits > 8) return fail(MX_ERR_INVALID_ARGUMENT, "bits must be in [2, 8], got %d", bits);
  if (rows < 0 || channels < 1) return fail(MX_ERR_SHAPE, "bad shape");
  if (out_dtype != MX_F64 && out_dtype != MX_F32 && out_dtype != MX_BF16)
    return fail(MX_ERR_INVALID_ARGUMENT, "out dtype must be f64, f32 or bf16");
  if (rows == 0) return MX_OK;
  if (!scales || !codes || !out) return fail(MX_ERR_INVALID_ARGUMENT, "NULL buffer");
  launch_chanint_decompress(scales, codes, rows * channels, channels, bits, out, out_dtype,
                            (cudaStream_t)stream);
  return cuda_check("chanint decompress");
}

int mx_topk_workspace_bytes(int64_t n, int64_t* bytes) {
  if (n < 0 || !bytes) return fail(MX_ERR_INVALID_ARGUMENT, "bad arguments");
  *bytes = topk_workspace_bytes(n);
  return MX_OK;
}

int mx_topk_compress(const void* x, int32_t dtype, int64_t n, int64_t k, uint32_t* indices,
                     uint16_t* values, void* workspace, int64_t workspace_bytes,
                     uint64_t* nonfinite, void* stream) {
  if (n < 0 || k < 0 || k > n) return fail(MX_ERR_INVALID_ARGUMENT, "need 0 <= k <= n");
  if (n > 0xffffffffLL) return fail(MX_ERR_UNSUPPORTED, "TopK indices are u32");
  if (in_size(dtype) == 0) return fail(MX_ERR_INVALID_ARGUMENT, "unknown input dtype %d", dtype);
  if (k == 0) return MX_OK;
  if (!x || !indices || !values) return fail(MX_ERR_INVALID_ARGUMENT, "NULL buffer");
  if (!workspace || workspace_bytes < topk_workspace_bytes(n))
    return fail(MX_ERR_WORKSPACE, "TopK needs %lld workspace bytes", (long long)topk_workspace_bytes(n));
  if (((uintptr_t)workspace) % 256 != 0) return fail(MX_ERR_INVALID_ARGUMENT, "workspace must be 256-B aligned");
  launch_topk_compress(x, dtype, n, k, indices, values, workspace,
                       reinterpret_cast<unsigned long long*>(nonfinite), (cudaStream_t)stream);
  return cuda_check("topk compress");
}

int mx_topk_decompress(const uint32_t* indices, const uint16_t* values, int64_t k, int64_t n,
                       void* out, int32_t out_dtype, void* stream) {
  if (n < 0 || k < 0 || k > n) return fail(MX_ERR_INVALID_ARGUMENT, "need 0 <= k <= n");
  if (out_dtype != MX_F64 && out_dtype != MX_F32 && out_dtype != MX_BF16)
    return fail(MX_ERR_INVALID_ARGUMENT, "out dtype must be f64, f32 or bf16");
  if (n == 0) return MX_OK;
  if (!out || (k > 0 && (!indices || !values))) return fail(MX_ERR_INVALID_ARGUMENT, "NULL buffer");
  launch_topk_decompress(indices, values, k, n, out, out_dtype, (cudaStream_t)stream);
  return cuda_check("topk decompress");
}

}  // extern "C"
