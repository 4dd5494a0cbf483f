/*
 * mxb200.h -- C ABI of the B200 (sm_100a) compressed tensor-parallel
 * all-reduce path of arXiv 2411.09510 ("mxcomm" reference).
 *
 * The reference is pure Python/numpy; its hot path is the block codec
 * (mx/codec.py:140-188, mx/bitpack.py:22-58) driven by the compressed
 * collective (mx/netbench.py:307-339) and the row-parallel hook
 * (mx/tpsim.py:234-302).  Each entry point below replaces one of those
 * reference interfaces (cited per function; `mx/` = pkg/src/mxcomm/).
 *
 * Conventions
 *  - Plain C types only; every pointer marked "device" is device memory
 *    owned by the caller (e.g. the torch caching allocator).
 *  - Every compute call is asynchronous on `stream` (a cudaStream_t passed
 *    as void*; NULL = legacy default stream), performs no host sync and no
 *    allocation, and is safe to capture into a CUDA graph.
 *  - Return value: MX_OK (0) or a negative MX_ERR_* code.  Codes map 1:1 to
 *    the reference exception classes of mx/errors.py; a thread-local
 *    message is available from mx_last_error().
 *  - Streams: "scale stream" = one k-bit scale code per block, "element
 *    stream" = one b-bit code per value, both LSB-first within each byte,
 *    zero-padded only at their end (mx/bitpack.py:3-7, mx/codec.py:27-43).
 *    Byte-identical to the reference's CompressedTensor streams.
 *  - Shard ("wire message") layout used by the collectives:
 *      [scale stream | pad to 32 B | element stream | pad to 32 B]
 *    see mx_shard_layout().
 */
#ifndef MXB200_H
#define MXB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MXB200_ABI_VERSION 1

/* FormatKind (mx/formats.py:54-56) */
enum { MX_KIND_FLOAT = 0, MX_KIND_INT = 1 };

/* element dtypes of dense tensors crossing the ABI */
enum { MX_F32 = 0, MX_F16 = 1, MX_BF16 = 2, MX_F64 = 3 };

/* status codes <-> mx/errors.py */
enum {
  MX_OK = 0,
  MX_ERR_INVALID_ARGUMENT = -1, /* ValueError                         */
  MX_ERR_NONFINITE = -2,        /* NonFiniteInput       (errors.py:8)  */
  MX_ERR_MALFORMED_CODE = -3,   /* MalformedCode        (errors.py:16) */
  MX_ERR_TRUNCATED = -4,        /* TruncatedStream      (errors.py:32) */
  MX_ERR_UNKNOWN_SCHEME = -5,   /* UnknownScheme        (errors.py:36) */
  MX_ERR_SHAPE = -6,            /* ShapeMismatch        (errors.py:40) */
  MX_ERR_CUDA = -7,             /* CUDA launch / runtime failure       */
  MX_ERR_UNSUPPORTED = -8,      /* valid scheme, path not implemented  */
  MX_ERR_WORKSPACE = -9         /* workspace too small                 */
};

/* SchemeDescriptor (mx/formats.py:157-175) lowered to a POD.
 * element: ElementFormat(kind, exponent_bits, mantissa_bits)
 *          (mx/formats.py:59-103; INTn has exponent_bits 0, mantissa n-1)
 * scale:   ScaleFormat(scale_bits) = EkM0, k in [4,8] (mx/formats.py:106-132) */
typedef struct mx_scheme {
  int32_t kind;
  int32_t exponent_bits;
  int32_t mantissa_bits;
  int32_t scale_bits;
  int64_t block_size;
} mx_scheme_t;

int mx_abi_version(void);
const char* mx_last_error(void);

/* Validates a scheme like ElementFormat/ScaleFormat/SchemeDescriptor
 * __post_init__ (mx/formats.py:68-83,112-114,165-167). */
int mx_scheme_check(const mx_scheme_t* scheme);

/* packed_nbytes for both streams (mx/bitpack.py:17-19, as used by
 * serialized_nbytes mx/codec.py:291-299 minus the header). */
int mx_stream_nbytes(int64_t n, const mx_scheme_t* scheme, int64_t* scale_bytes,
                     int64_t* element_bytes);

/* Wire-message layout of one shard holding n values (no MXC1 header on the
 * NCCL wire; serialize() adds it on the host). */
int mx_shard_layout(int64_t n, const mx_scheme_t* scheme, int64_t* scale_offset,
                    int64_t* element_offset, int64_t* shard_bytes);

/* Bytes of device workspace mx_quantize / mx_quantize_chunks may need
 * (generic path only: any block size, unaligned or float64 input).  For the
 * chunked call pass n = nchunks * chunk_values. */
int mx_workspace_bytes(int64_t n, const mx_scheme_t* scheme, int64_t* bytes);

/* Same for mx_dequant_sum_requant on an n-value chunk. */
int mx_requant_workspace_bytes(int64_t n, const mx_scheme_t* scheme, int64_t* bytes);

/* compress_tensor (mx/codec.py:238-263) incl. _quantize_block_matrix
 * (140-172), _round_to_grid (127-137) and pack_bits (mx/bitpack.py:22-34).
 *   x              device, n values of `dtype` (row-major flattened)
 *   scale_stream   device, mx_stream_nbytes().scale_bytes
 *   element_stream device, mx_stream_nbytes().element_bytes
 *   nonfinite      device u64, nullable.  Caller initialises it to
 *                  UINT64_MAX (mx_nonfinite_reset); the kernel atomically
 *                  lowers it to the flat index of the first NaN/Inf, which
 *                  the host turns into NonFiniteInput(block_index =
 *                  index // block_size) exactly like _check_finite
 *                  (mx/codec.py:191-199).  Outputs are unspecified then. */
int mx_quantize(const void* x, int32_t dtype, int64_t n, const mx_scheme_t* scheme,
                uint8_t* scale_stream, uint8_t* element_stream, uint64_t* nonfinite,
                void* workspace, int64_t workspace_bytes, void* stream);

/* decompress_tensor (mx/codec.py:266-284) incl. unpack_bits
 * (mx/bitpack.py:37-58) and _dequantize_block_matrix (175-188).
 * out_dtype MX_F64 is exact; MX_F32/F16/BF16 round the exact value once
 * (RNE), like ndarray.astype. */
int mx_dequantize(const uint8_t* scale_stream, const uint8_t* element_stream, int64_t n,
                  const mx_scheme_t* scheme, void* out, int32_t out_dtype, void* stream);

/* Chunked compress for the collectives: x (n values) is cut into
 * ceil(n / chunk_values) chunks, each compressed as an independent tensor
 * into the shard at  shards + j * shard_stride  with mx_shard_layout(
 * chunk_values) offsets.  chunk_values must be a multiple of 8*block_size
 * (blocks never straddle chunks, so codes equal whole-tensor codes). */
int mx_quantize_chunks(const void* x, int32_t dtype, int64_t n, int64_t chunk_values,
                       const mx_scheme_t* scheme, uint8_t* shards, int64_t shard_stride,
                       uint64_t* nonfinite, void* workspace, int64_t workspace_bytes,
                       void* stream);

/* The compressed-collective reduction (mx/netbench.py:329-334): decode
 * `nranks` shards and sum them in fp32 in rank order starting from +0.0,
 * then cast once to out_dtype (MX_F32/F16/BF16).
 * Shard of (rank r, chunk j) lives at  shards + r*rank_stride + j*chunk_stride
 * with mx_shard_layout(chunk_values) offsets; output value i of chunk j is
 * out[j*chunk_values + i].
 *   one-shot all-gather : nranks=N, rank_stride=shard bytes, chunk_values=n
 *   two-shot all-gather : nranks=1, chunk_stride=shard bytes, chunk_values=c */
int mx_dequant_sum(const uint8_t* shards, int64_t rank_stride, int32_t nranks, int64_t n,
                   int64_t chunk_values, int64_t chunk_stride, const mx_scheme_t* scheme,
                   void* out, int32_t out_dtype, void* stream);

/* mx_dequant_sum with the Llama residual add fused into the store (the
 * row-parallel consumer `h + all_reduce(partial)`, tpsim's hook output fed
 * to the residual stream): out[i] = round(residual[i] + round(sum[i])) in
 * out_dtype -- bit-identical to mx_dequant_sum followed by an elementwise
 * add in out_dtype, without writing and re-reading the sum.  `residual` has
 * out_dtype and out's layout and may alias `out` (in-place h += ...). */
int mx_dequant_sum_residual(const uint8_t* shards, int64_t rank_stride, int32_t nranks, int64_t n,
                            int64_t chunk_values, int64_t chunk_stride,
                            const mx_scheme_t* scheme, const void* residual, void* out,
                            int32_t out_dtype, void* stream);

/* Two-shot middle step (not in the reference; restated from the same codec
 * calls): decode `nranks` shards of one n-value chunk, fp32 rank-order sum
 * from +0.0, re-quantise the sum into the shard at `out_shard`.  All shards
 * use mx_shard_layout(chunk_values) offsets (chunk_values >= n; the last
 * chunk of a tensor is shorter than the others). */
int mx_dequant_sum_requant(const uint8_t* shards, int64_t rank_stride, int32_t nranks,
                           int64_t n, int64_t chunk_values, const mx_scheme_t* scheme,
                           uint8_t* out_shard, uint64_t* nonfinite, void* workspace,
                           int64_t workspace_bytes, void* stream);

/* The whole one-shot compressed all-reduce of `nranks` partials that live on
 * THIS device, fused into one persistent kernel: quantise each partial into
 * its shard (shards + r*shard_stride, mx_shard_layout(n) offsets), grid-wide
 * barrier, fp32 rank-order dequant-sum into `out`.  Bit-identical to
 * mx_quantize x nranks + mx_dequant_sum.  `partials` is a DEVICE array of
 * nranks pointers (bf16, 32-byte aligned); `barrier` is 2 device uint32
 * zeroed once (reusable across calls on one stream).  Returns
 * MX_ERR_UNSUPPORTED outside bf16-in, bf16/f32-out, B in {8,16,32,64} (any scale width),
 * element widths 4/5/6/8. */
int mx_allreduce_fused(const void* const* partials, int32_t dtype, int32_t nranks, int64_t n,
                       const mx_scheme_t* scheme, uint8_t* shards, int64_t shard_stride,
                       void* out, int32_t out_dtype, uint32_t* barrier, uint64_t* nonfinite,
                       void* stream);

/* Row-parallel GEMM with the MX quantiser fused into its epilogue -- the
 * producer side of the compressed all-reduce: the reference computes the
 * rank's partial and encodes it (mx/tpsim.py:263-265, `partial = x_shard @
 * shards[rank]` -> `wire.encode(partial)` = compress_tensor, mx/codec.py:
 * 238-263).  partial[M, N] = x[M, K] . w[N, K]^T (F.linear of a row-parallel
 * weight shard; bf16 operands, row-major, fp32 accumulation on the tcgen05
 * tensor cores); the MX streams of bf16(partial) (flat row-major order) are
 * written to scale_stream / element_stream -- byte-identical to
 * mx_quantize of that bf16 tensor.  `partial` (bf16 [M, N], nullable)
 * additionally receives the bf16 partial.  scheme == NULL: plain GEMM,
 * `partial` required.  Requires K % 64 == 0, N % 128 == 0, 16-byte aligned
 * operands, and E8M0 scales with B in {8, 16, 32} or E5M0 scales (the paper's
 * selected schemes: fp4_e2m1 B in {8, 16, 32}, fp5_e2m2 B = 32) with
 * N % 256 == 0; else MX_ERR_UNSUPPORTED. */
int mx_gemm_quantize(const void* x, const void* w, int64_t M, int64_t N, int64_t K,
                     const mx_scheme_t* scheme, uint8_t* scale_stream, uint8_t* element_stream,
                     void* partial, uint64_t* nonfinite, void* stream);

/* The same GEMM writing chunked shards like mx_quantize_chunks (the
 * two-shot send buffer, or one shard slot of the one-shot gather buffer with
 * chunk_values >= M*N): chunk j of the flat partial goes to
 * shards + j*shard_stride with mx_shard_layout(chunk_values) offsets. */
int mx_gemm_quantize_chunks(const void* x, const void* w, int64_t M, int64_t N, int64_t K,
                            int64_t chunk_values, const mx_scheme_t* scheme, uint8_t* shards,
                            int64_t shard_stride, void* partial, uint64_t* nonfinite,
                            void* stream);

/* Sizes of the symmetric-memory collective for n values and nranks ranks:
 * every rank allocates one symmetric buffer of *buffer_bytes holding two
 * shard slots of *slot_stride bytes (double buffering) followed, at
 * *flags_offset, by the flag array (nranks x *ctas u32, zero-initialised
 * before first use); the local per-CTA epoch array is *ctas u32. */
int mx_symm_layout(int64_t n, const mx_scheme_t* scheme, int32_t nranks, int64_t* slot_stride,
                   int64_t* flags_offset, int64_t* buffer_bytes, int64_t* ctas);

/* Multi-GPU one-shot fused over symmetric (peer-mapped) memory, ONE launch
 * per rank, per-CTA dataflow (no grid barrier): CTA b quantises its 8 units
 * of `x` into this rank's shard slot, publishes a ready flag for CTA b into
 * every peer's flag array (system-scope release), waits for the nranks
 * flags of CTA b (acquire), then decodes its units of all nranks shards
 * straight from the peers' buffers in rank order (fp32 from +0.0) into
 * `out`.  Replaces all-gather + dequant-sum (mx/netbench.py:323-334) with
 * no gather buffer and no NCCL kernel.
 *   peer_bufs     device array [nranks] of peer buffer bases
 *   peer_flags    device array [nranks] of peer flag arrays (buffer base +
 *                 flags_offset of mx_symm_layout)
 *   status        local device u32 (zeroed once): set to 1 if a peer wait
 *                 timed out (~2 s) instead of hanging
 *   epochs        local device u32 x ctas (zeroed once)
 *   residual      nullable, out_dtype, n values, may alias out: the residual
 *                 add fused into the store as in mx_dequant_sum_residual
 * MX_ERR_UNSUPPORTED outside bf16 in, n % 1024 == 0, B in {16,32,64}. */
int mx_allreduce_symm(const void* x, int32_t dtype, int64_t n, const mx_scheme_t* scheme,
                      uint8_t* const* peer_bufs, uint32_t* const* peer_flags, int32_t rank,
                      int32_t nranks, int64_t slot_stride, void* out, int32_t out_dtype,
                      const void* residual, uint32_t* status, uint32_t* epochs,
                      uint64_t* nonfinite, void* stream);

/* Sizes of the two-shot symmetric-memory collective (n % (1024*nranks) == 0):
 * one buffer per rank of *buffer_bytes = two slots of *slot_stride bytes
 * (each: nranks send chunk shards + one reduced chunk shard, *shard_stride
 * bytes apiece) followed, at *flags_offset, by 2 x nranks x *ctas u32 flags
 * (zero-initialised); local epochs are *ctas u32. */
int mx_symm_twoshot_layout(int64_t n, const mx_scheme_t* scheme, int32_t nranks,
                           int64_t* slot_stride, int64_t* shard_stride, int64_t* flags_offset,
                           int64_t* buffer_bytes, int64_t* ctas);

/* Two-shot compressed all-reduce over NVLink peer memory, ONE launch per
 * rank, per-CTA dataflow: quantise the local partial's N chunks into this
 * rank's send shards -> flag -> pull the N peers' shards of this rank's
 * chunk, fp32 rank-order sum, re-quantise into the reduced shard -> flag ->
 * pull every owner's reduced shard and decode into `out`.  Bit-identical
 * to quantise_chunks -> all_to_all -> dequant_sum_requant -> all_gather ->
 * dequant_sum.  Arguments as mx_allreduce_symm, sizes from
 * mx_symm_twoshot_layout.  MX_ERR_UNSUPPORTED outside bf16 in,
 * n % (1024*nranks) == 0, B in {16,32,64}. */
int mx_allreduce_symm_twoshot(const void* x, int32_t dtype, int64_t n,
                              const mx_scheme_t* scheme, uint8_t* const* peer_bufs,
                              uint32_t* const* peer_flags, int32_t rank, int32_t nranks,
                              void* out, int32_t out_dtype, const void* residual,
                              uint32_t* status, uint32_t* epochs, uint64_t* nonfinite,
                              void* stream);

/* unpack_bits (mx/bitpack.py:37-58) on the device: `count` codes of
 * `width` bits -> one uint8 per code (quantize_block's return value). */
int mx_unpack_codes(const uint8_t* packed, int64_t count, int32_t width, uint8_t* codes,
                    void* stream);

/* pack_bits (mx/bitpack.py:22-34) on the device: the inverse of
 * mx_unpack_codes (dequantize_block's input path). */
int mx_pack_codes(const uint8_t* codes, int64_t count, int32_t width, uint8_t* packed,
                  void* stream);

/* ---- GEMM + quantise + all-gather push over NVLink (one kernel) ----------
 * The row-parallel GEMM of mx/tpsim.py:263-265 (`partial = x_shard @ W_r`,
 * `wire.encode(partial)`) and the all-gather of mx/netbench.py:323-328 in
 * ONE kernel per rank: the tcgen05 GEMM's epilogue quantises each drained
 * accumulator tile and stores the shard bytes straight into slot
 * (epoch & 1) of EVERY rank's symmetric buffer (peer memory, NVLink), so the
 * transfer overlaps the remaining tiles' math; its last CTA (GPU-scope
 * arrival counter) issues one system-scope fence and stores the epoch into
 * flag [rank] of every rank's flag array.  mx_push_dequant_sum waits for the
 * N local flags (`flags`, this rank's array) and decodes the N local shards
 * in rank order (bit-identical to the NCCL one-shot).  Buffer: mx_push_layout
 * bytes per rank (two slots of nranks shards, then nranks u32 flags, zeroed
 * once); state: 2 local u32 zeroed once ([0] epoch, [1] CTA counter);
 * status: one local u32 (1 = a peer wait timed out after
 * MXB200_SYMM_TIMEOUT_MS).
 * The push set: fp4_e2m1 E8M0 with B in {16, 32}, and the paper's E5M0
 * schemes -- fp4_e2m1 with B in {8, 16, 32}, fp5_e2m2 with B = 32; N % 256
 * == 0, at most 8 ranks (MX_ERR_UNSUPPORTED outside it). */
int mx_push_layout(int64_t n, const mx_scheme_t* scheme, int32_t nranks, int64_t* slot_stride,
                   int64_t* shard_stride, int64_t* flags_offset, int64_t* buffer_bytes);
int mx_gemm_allgather_push(const void* x, const void* w, int64_t M, int64_t N, int64_t K,
                           const mx_scheme_t* scheme, uint8_t* const* peer_bufs, int32_t rank,
                           int32_t nranks, uint32_t* state, uint64_t* nonfinite, void* stream);
int mx_push_dequant_sum(const uint8_t* buf, int64_t n, const mx_scheme_t* scheme, int32_t rank,
                        int32_t nranks, const uint32_t* flags, const uint32_t* state,
                        uint32_t* status, void* out, int32_t out_dtype, const void* residual,
                        void* stream);

/* Two-shot form (the TP >= 4 algorithm; n % (1024*nranks) == 0): the GEMM's
 * epilogue scatters chunk j of its shard to rank j (the reduce-scatter leg,
 * one store per value group) and its last CTA publishes RS flag [rank]
 * everywhere; mx_push2_requant waits for every rank's chunk, sums the N
 * shards of this rank's chunk in rank order, re-quantises (K3's arithmetic),
 * pushes the reduced chunk shard into every rank (the all-gather leg) and
 * its last CTA publishes AG flag [nranks + rank] everywhere (one system
 * fence); mx_push2_decode waits for the AG flags and decodes every owner's
 * reduced chunk, residual fused.  Bit-identical to the NCCL two-shot.
 * Buffer: mx_push2_layout bytes (two slots of 2 x nranks chunk shards;
 * flags: nranks RS then nranks AG u32, zeroed once); peer_flags: device
 * array of every rank's flag array; state: 3 local u32 zeroed once ([0]
 * epoch, [1] GEMM CTA counter, [2] requantiser CTA counter). */
int mx_push2_layout(int64_t n, const mx_scheme_t* scheme, int32_t nranks, int64_t* chunk_values,
                    int64_t* slot_stride, int64_t* shard_stride, int64_t* flags_offset,
                    int64_t* buffer_bytes);
int mx_gemm_reducescatter_push(const void* x, const void* w, int64_t M, int64_t N, int64_t K,
                               const mx_scheme_t* scheme, uint8_t* const* peer_bufs,
                               int32_t rank, int32_t nranks, uint32_t* state, uint64_t* nonfinite,
                               void* stream);
int mx_push2_requant(const uint8_t* buf, int64_t n, const mx_scheme_t* scheme, int32_t rank,
                     int32_t nranks, uint8_t* const* peer_bufs, uint32_t* const* peer_flags,
                     uint32_t* state, uint32_t* status, uint64_t* nonfinite, void* stream);
int mx_push2_decode(const uint8_t* buf, int64_t n, const mx_scheme_t* scheme, int32_t rank,
                    int32_t nranks, const uint32_t* state, uint32_t* status, void* out,
                    int32_t out_dtype, const void* residual, void* stream);

/* serialize (mx/codec.py:340-348) on the device: out = header || scale
 * stream || element stream, one launch, any byte alignment.  `header` is a
 * HOST pointer to the pack_header bytes (mx/codec.py:300-308), at most 544
 * bytes (64 dimensions), copied into the kernel's parameters -- so the call
 * is CUDA-graph capturable; out holds serialized_nbytes(scheme, shape). */
int mx_serialize(const uint8_t* header, int32_t header_bytes, const uint8_t* scale_stream,
                 int64_t scale_bytes, const uint8_t* element_stream, int64_t element_bytes,
                 uint8_t* out, void* stream);

/* Device byte copy at any source / destination alignment (deserialize's
 * payload slices, mx/codec.py:351-380, moved to aligned stream buffers so
 * the decode takes the vectorised kernels). */
int mx_copy_bytes(const uint8_t* src, int64_t nbytes, uint8_t* dst, void* stream);

/* ---- comparison codecs (mx/baselines.py), the paper's Table 4 baselines ---- */

/* channelwise_int_compress (mx/baselines.py:138-168): x is `rows` x
 * `channels` (channels = trailing dimension, row-major); per-channel scale
 * = f16_RNE(max|x| / (2^(bits-1)-1)) written as IEEE half bits to
 * `scales[channels]`; sign-magnitude codes rounded half-to-even against the
 * stored scale, clamped, LSB-first packed into `codes`
 * (ceil(rows*channels*bits/8) bytes).  bits in [2, 8].  `workspace` >=
 * 8*channels bytes.  dtype MX_F32/F16/BF16/F64.  Non-finite inputs lower
 * *nonfinite to their flat index (NonFiniteInput). */
int mx_chanint_compress(const void* x, int32_t dtype, int64_t rows, int64_t channels,
                        int32_t bits, uint16_t* scales, uint8_t* codes, void* workspace,
                        int64_t workspace_bytes, uint64_t* nonfinite, void* stream);

/* channelwise_int_decompress (mx/baselines.py:171-178): level * scale in
 * float64, cast once to out_dtype (MX_F64 exact, MX_F32, MX_BF16). */
int mx_chanint_decompress(const uint16_t* scales, const uint8_t* codes, int64_t rows,
                          int64_t channels, int32_t bits, void* out, int32_t out_dtype,
                          void* stream);

/* Workspace bytes of mx_topk_compress for n values. */
int mx_topk_workspace_bytes(int64_t n, int64_t* bytes);

/* topk_compress (mx/baselines.py:95-128) with an explicit K (the caller
 * computes topk_budget, mx/baselines.py:88-92): the K largest |x|, ties
 * toward the lower index, written in ascending index order as u32
 * `indices[K]` and IEEE half bits `values[K]` (RNE, overflow -> inf).
 * Radix select + stable compaction, no host synchronisation. */
int mx_topk_compress(const void* x, int32_t dtype, int64_t n, int64_t k, uint32_t* indices,
                     uint16_t* values, void* workspace, int64_t workspace_bytes,
                     uint64_t* nonfinite, void* stream);

/* topk_decompress (mx/baselines.py:131-135): zeros, then the K f16 values
 * scattered to their indices; out_dtype MX_F64 / MX_F32 / MX_BF16. */
int mx_topk_decompress(const uint32_t* indices, const uint16_t* values, int64_t k, int64_t n,
                       void* out, int32_t out_dtype, void* stream);

/* cudaMemsetAsync on `stream` (e.g. zeroing a symmetric-memory signal pad
 * without pulling the CUDA runtime into the host language). */
int mx_memset_async(void* ptr, int32_t value, int64_t bytes, void* stream);

/* Sets *nonfinite = UINT64_MAX on `stream`. */
int mx_nonfinite_reset(uint64_t* nonfinite, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MXB200_H */
