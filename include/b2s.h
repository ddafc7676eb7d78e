/*
 * b2s.h — C-ABI of the B200-native (sm_100a) Modalities training-step library.
 *
 * Plain pointers, sizes and a cudaStream_t passed as void*; no torch types.
 * Every entry point returns 0 (B2S_OK) or a negative status; the text of the
 * last failure on the calling thread is available from b2s_last_error().
 * All device buffers are caller-owned. Kernels are stateless and ordered only
 * by the stream argument. Device pointers are marked `d_`, host pointers `h_`.
 *
 * Reference interfaces replaced (reference = /root/reference, read-only):
 *   packed_data.py:49-59   token_width_for_vocab      -> b2s_token_width_for_vocab
 *   packed_data.py:188-194 PackedReader.sample_count  -> b2s_sample_count
 *   packed_data.py:196-203 PackedReader.get_sample    -> b2s_gather_samples (batched, on device)
 *   packed_data.py:226-238 splitmix64                 -> b2s_splitmix64
 *   packed_data.py:257-282 make_permutation           -> b2s_make_permutation
 *   packed_data.py:322-333 chunk                      -> b2s_chunk_bounds
 * The model/optimizer/FSDP kernels below have no reference implementation
 * (SPEC.md:12 puts the training step out of the reference's scope); their
 * callers are the registered `model`, `optimizer` and `trainer` components
 * (SPEC.md:24-123 registry/factory boundary).
 */
#ifndef B2S_H_
#define B2S_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* b2s_stream_t; /* cudaStream_t */

enum {
  B2S_OK = 0,
  B2S_EINVAL = -1,      /* bad argument (maps to ValueError)            */
  B2S_ERANGE = -2,      /* ordinal out of range (maps to OutOfRangeError) */
  B2S_ECUDA = -3,       /* CUDA runtime/driver failure                   */
  B2S_EUNSUPPORTED = -4 /* shape/dtype the kernel does not implement     */
};

const char* b2s_last_error(void);
int b2s_abi_version(void);

/* ------------------------------------------------------------------ */
/* Packed data path (CFPKD001)                                         */
/* ------------------------------------------------------------------ */

/* packed_data.py:49-59. Smallest of {1,2,4} bytes holding vocab_size-1. */
int b2s_token_width_for_vocab(uint64_t vocab_size, int* h_width);

/* packed_data.py:188-194. (token_count-1)//seq_len, 0 if token_count==0;
 * B2S_EINVAL if seq_len < 1. */
int b2s_sample_count(uint64_t token_count, int64_t seq_len, uint64_t* h_count);

/* packed_data.py:226-238. First `count` outputs of SplitMix64(seed). Host. */
int b2s_splitmix64(uint64_t seed, uint64_t count, uint64_t* h_out);

/* packed_data.py:257-282. Fisher-Yates over [0,n) driven by SplitMix64 with
 * rejection-sampled bounded draws; bit-exact with the reference. Host. */
int b2s_make_permutation(uint64_t n, uint64_t seed, uint64_t* h_order);

/* packed_data.py:322-333. Chunk c of a k-way split of n items is
 * [h_lo[c], h_lo[c+1]); h_lo has k+1 entries. B2S_EINVAL unless 1<=k<=max(1,n). */
int b2s_chunk_bounds(uint64_t n, uint64_t k, uint64_t* h_lo);

/* packed_data.py:196-203, batched on the GPU. For b in [0,batch):
 *   d_inputs [b, t] = payload[s_b*L + t]      t in [0, L)
 *   d_targets[b, t] = payload[s_b*L + t + 1]
 * with s_b = d_sample_ids[b], widened from the little-endian `width`-byte
 * token to int64. `d_payload` holds `token_count` tokens. Any s_b outside
 * [0, sample_count(L)) leaves its rows untouched and sets *d_status to 1
 * (caller maps it to OutOfRangeError); *d_status is not cleared. */
int b2s_gather_samples(const void* d_payload, int width, uint64_t token_count,
                       const uint64_t* d_sample_ids, int batch, int64_t seq_len,
                       int64_t* d_inputs, int64_t* d_targets, int32_t* d_status,
                       b2s_stream_t stream);


/* ------------------------------------------------------------------ */
/* Dense contractions (K5): tcgen05 + TMEM + TMA, persistent           */
/* ------------------------------------------------------------------ */

/* C[M,N] = epi( sum_k A(m,k) B(n,k) ), bf16 operands, fp32 accumulation.
 * A: a_mn_major=0 -> row-major [M][lda] (K contiguous); 1 -> [K][lda] (M contiguous).
 * B: b_mn_major=0 -> row-major [N][ldb];                 1 -> [K][ldb] (N contiguous).
 * C: row-major [M][ldc], fp32 if c_f32 else bf16; accumulate!=0 adds into C.
 * d_bias: optional bf16 [N] added before the activation.
 * act: 0 none; 1 GELU-tanh (pre-activation written to d_aux as bf16);
 *      2 multiply by GELU-tanh'(d_aux) (fused activation backward).
 * Strides must keep rows 16-byte aligned (multiples of 8 bf16). */
int b2s_gemm(const void* d_A, int a_mn_major, int64_t lda, const void* d_B, int b_mn_major,
             int64_t ldb, void* d_C, int64_t ldc, int c_f32, int M, int N, int K, int accumulate,
             const void* d_bias, int act, void* d_aux, int64_t ld_aux, b2s_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* B2S_H_ */
