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
 *   packed_data.py:336-344 materialize_chunk          -> b2s_gather_documents (device copy)
 *   corpus_index.py:68-107 build_index (newline scan) -> b2s_newline_count / b2s_newline_positions
 *   pipeline.py:264-422    run_pipeline (+ tokenizers) -> b2s_tokenize_corpus (host C++ thread pool)
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
/* Number of CUDA kernels this library has launched since it was loaded. */
uint64_t b2s_launch_count(void);
/* cudaMemsetAsync of `bytes` bytes at device pointer `dst` to `value` on `stream` (a memset
   node, not a kernel: zeroes the gradient / residual-gradient accumulators inside the step). */
int b2s_memset_async(void* dst, int value, uint64_t bytes, void* stream);
/* Native CUDA-graph capture of the work issued to `stream` between begin and end (thread-local
 * capture mode); end instantiates it into *h_exec, launched by b2s_graph_launch and freed by
 * b2s_graph_destroy. Used for the single-GPU training step. */
int b2s_graph_capture_begin(void* stream);
int b2s_graph_capture_end(void* stream, void** h_exec);
int b2s_graph_launch(void* exec, void* stream);
int b2s_graph_destroy(void* exec);

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

/* packed_data.py:336-344 (materialize_chunk), on the device: for i < n_docs,
 * copy source tokens [d_src_start[i], d_src_start[i] + d_len[i]) of the
 * `width`-byte payload to token offset d_dst_start[i] of d_out. The caller
 * validates document ordinals (OutOfRangeError) and lays out the output
 * spans (exclusive prefix sum of the lengths). */
int b2s_gather_documents(const void* d_payload, int width, const uint64_t* d_src_start, const uint64_t* d_len,
                         const uint64_t* d_dst_start, int64_t n_docs, void* d_out, b2s_stream_t stream);

/* corpus_index.py:68-107 (build_index), the O(bytes) part on the GPU: the
 * newline (0x0A) byte positions of a raw buffer (16-byte aligned, n bytes)
 * split into nblocks chunks of `chunk` bytes (multiple of 16, nblocks*chunk >= n).
 * Pass 1: d_counts[b] = newlines in chunk b. The caller forms exclusive offsets
 * d_offsets[b] = sum_{c<b} d_counts[c]. Pass 2: writes base + position of every
 * newline, ascending, to d_pos[d_offsets[b] ...]. Spans follow on the host. */
int b2s_newline_count(const void* d_buf, uint64_t n, uint64_t chunk, uint32_t* d_counts, int nblocks,
                      b2s_stream_t stream);
int b2s_newline_positions(const void* d_buf, uint64_t n, uint64_t chunk, const uint64_t* d_offsets, int nblocks,
                          uint64_t base, uint64_t* d_pos, b2s_stream_t stream);

/* tokenizers.py (ByteTokenizer / WhitespaceTokenizer / BpeTokenizer), host C++.
 * kind: 0 byte, 1 whitespace, 2 bpe; h_pieces = n_pieces x (u32 length, UTF-8
 * bytes) vocabulary (id = index); h_merges = n_merges x (left, right) in the same
 * encoding (rank = index); unk / eod ids (-1: none). Returns a handle (null on error). */
void* b2s_tokenizer_create(int kind, const void* h_pieces, int64_t n_pieces, const void* h_merges, int64_t n_merges,
                           int64_t unk_id, int64_t eod_id);
void b2s_tokenizer_destroy(void* tokenizer);
/* encode one text given as UTF-8 ('surrogatepass' for lone surrogates) into at
 * most cap ids; *h_n = number of ids (B2S_ERANGE if > cap). B2S_EINVAL when the
 * byte / bpe tokenizer meets a lone surrogate (reference: UnicodeEncodeError). */
int b2s_tokenizer_encode(void* tokenizer, const char* h_text, int64_t len, uint32_t* h_out, int64_t cap,
                         int64_t* h_n);

/* pipeline.py:264-422 run_pipeline, as a host C++ thread pool (SURVEY §8(f)
 * rank 1): tokenize documents h_spans[2*i] (byte offset), h_spans[2*i+1]
 * (length) of raw_path, in index order, with `workers` threads over batches of
 * batch_size documents, into the CFPKD001 file out_path -- byte-identical for
 * any `workers` (order restored by the writer). h_stats (optional, 4 x i64):
 * documents, skipped, malformed, tokens. B2S_EINVAL on a lone surrogate under
 * the byte / bpe tokenizers (the reference run fails there too). */
int b2s_tokenize_corpus(const char* raw_path, const uint64_t* h_spans, int64_t n_docs, void* tokenizer,
                        const char* text_key, int append_eod, int width, int workers, int batch_size,
                        const char* out_path, int64_t* h_stats);

/* Same widening split for `batch` host-staged windows of seq_len+1 tokens
 * stored back to back in d_windows (window b starts at token b*(seq_len+1)):
 * the end-to-end feed that copies each step's windows from host memory. */
int b2s_unpack_windows(const void* d_windows, int width, int batch, int64_t seq_len, int64_t* d_inputs,
                       int64_t* d_targets, b2s_stream_t stream);


/* ------------------------------------------------------------------ */
/* Dense contractions (K5): tcgen05 + TMEM + TMA, persistent           */
/* ------------------------------------------------------------------ */

/* C[M,N] = epi( sum_k A(m,k) B(n,k) ), bf16 operands, fp32 accumulation.
 * A: a_mn_major=0 -> row-major [M][lda] (K contiguous); 1 -> [K][lda] (M contiguous).
 * B: b_mn_major=0 -> row-major [N][ldb];                 1 -> [K][ldb] (N contiguous).
 * C: row-major [M][ldc], fp32 if c_f32 else bf16; accumulate=1 adds into C; accumulate=2
 *    (fp32 C, act 0, no bias) overwrites C whatever it held -- a plain store, or when the
 *    host splits K a memset of C then the add-reduce (weight gradients written once per step).
 * d_bias: optional bf16 [N] added before the activation.
 * act: 0 none; 1 GELU-tanh (pre-activation written to d_aux as bf16);
 *      2 multiply by GELU-tanh'(d_aux) (fused activation backward);
 *      5 GELU-tanh with GELU-tanh'(pre-activation) written to d_aux (bf16), so that
 *      the backward is 6: multiply by d_aux (a plain product epilogue).
 * Strides must keep rows 16-byte aligned (multiples of 8 bf16). */
int b2s_gemm(const void* d_A, int a_mn_major, int64_t lda, const void* d_B, int b_mn_major,
             int64_t ldb, void* d_C, int64_t ldc, int c_f32, int M, int N, int K, int accumulate,
             const void* d_bias, int act, void* d_aux, int64_t ld_aux, b2s_stream_t stream);

/* b2s_gemm (bf16 C, act 0 / 2 / 6) that also writes the per-32-row column sums of the
 * stored (bf16-rounded) C: d_colsum_part [ceil(M/32)][N] fp32. Summing its rows
 * (b2s_colsum_accumulate, fp32) gives the bias gradient of a dgrad without re-reading C --
 * the reference's autograd bias grad, dbias = dY.sum(0). */
int b2s_gemm_colsum(const void* d_A, int a_mn_major, int64_t lda, const void* d_B, int b_mn_major, int64_t ldb,
                    void* d_C, int64_t ldc, int M, int N, int K, int act, void* d_aux, int64_t ld_aux,
                    float* d_colsum_part, b2s_stream_t stream);

/* Llama MLP with the SwiGLU fused into the GEMM epilogues (bf16).
 * Forward: gu = x @ W13^T ([M, 2F] = gate | up, kept for the backward) and
 * h = silu(gate) * up ([M, F]) from one GEMM -- each CTA-pair tile holds 128
 * gate columns and the matching 128 up columns. x [M][ldx] (K contiguous),
 * W13 [2F][ldw]; F % 128 == 0.
 * Backward: dgu = [dgate | dup] ([M, 2F]) from dh = dy @ W2 (dy [M][ld_dy],
 * W2 [K = d][ldw] rows of F) and the saved gu, without materialising dh. */
int b2s_gemm_swiglu_fwd(const void* d_x, int64_t ldx, const void* d_w13, int64_t ldw, void* d_gu, int64_t ld_gu,
                        void* d_h, int64_t ld_h, int M, int F, int K, b2s_stream_t stream);
int b2s_gemm_swiglu_bwd(const void* d_dy, int64_t ld_dy, const void* d_w2, int64_t ldw, const void* d_gu,
                        int64_t ld_gu, void* d_dgu, int64_t ld_dgu, int M, int F, int K, b2s_stream_t stream);
/* Fused QKV projection + rotary embedding (Llama): out = x @ W^T ([M, N], bf16) with columns
 * [0, rope_cols) -- the q and k heads, width dh in {64, 128} -- rotated in the epilogue
 * (rotate-half pairs j, j + dh/2; fp32 tables cos / sin [T, dh/2] at position row % T), the
 * same result as b2s_gemm followed by b2s_rope. N % 256 == 0. */
int b2s_gemm_rope(const void* d_x, int64_t ldx, const void* d_w, int64_t ldw, void* d_out, int64_t ldo, int M,
                  int N, int K, const float* d_cos, const float* d_sin, int T, int dh, int rope_cols,
                  b2s_stream_t stream);

/* ------------------------------------------------------------------ */
/* Bandwidth-bound kernels (K2-K4, K8-K11); no reference counterpart    */
/* ------------------------------------------------------------------ */
/* Hidden sizes D in {128, 768, 1024, 2048, 4096}. x is the fp32 residual
 * stream [M, D]; normalised outputs are bf16. d_x_copy (optional) receives a
 * copy of x (forwarding the residual into the next stream buffer). */
int b2s_layernorm_fwd(const float* d_x, const void* d_g, const void* d_b, void* d_y, float* d_mean,
                      float* d_rstd, float* d_x_copy, int64_t M, int D, float eps, b2s_stream_t stream);
int b2s_rmsnorm_fwd(const float* d_x, const void* d_g, void* d_y, float* d_rstd, float* d_x_copy,
                    int64_t M, int D, float eps, b2s_stream_t stream);
/* Residual-add forms: x_out = x + res (res = the previous sublayer's output,
 * bf16 [M, D]; x_out the new fp32 residual stream, may alias nothing else),
 * then y = norm(x_out). Replaces an fp32 add-reduce in the producing GEMM. */
int b2s_layernorm_fwd_res(const float* d_x, const void* d_res, const void* d_g, const void* d_b, void* d_y,
                          float* d_mean, float* d_rstd, float* d_x_out, int64_t M, int D, float eps,
                          b2s_stream_t stream);
int b2s_rmsnorm_fwd_res(const float* d_x, const void* d_res, const void* d_g, void* d_y, float* d_rstd,
                        float* d_x_out, int64_t M, int D, float eps, b2s_stream_t stream);
/* dx (fp32) += norm backward of dy (bf16); d_dx_bf16 (optional) <- bf16(dx);
 * d_dg / d_db (fp32 [D], optional) += parameter grads; d_dxsum (optional)
 * += column sums of the updated dx (the bias gradient of the linear layer
 * whose output gradient dx is). d_work: b2s_norm_work_floats(D) floats. */
int b2s_layernorm_bwd(const float* d_x, const void* d_dy, const void* d_g, const float* d_mean,
                      const float* d_rstd, float* d_dx, void* d_dx_bf16, float* d_dg, float* d_db,
                      float* d_dxsum, float* d_work, int64_t M, int D, b2s_stream_t stream);
int b2s_rmsnorm_bwd(const float* d_x, const void* d_dy, const void* d_g, const float* d_rstd, float* d_dx,
                    void* d_dx_bf16, float* d_dg, float* d_dxsum, float* d_work, int64_t M, int D,
                    b2s_stream_t stream);
int64_t b2s_norm_work_floats(int D);

/* d_out[c] (fp32) += sum_r x[r, c] over M rows of a bf16 (x_f32=0) or fp32
 * [M, ld] array (bias gradients). d_work: b2s_colsum_work_floats(N) floats. */
int b2s_colsum_accumulate(const void* d_x, int x_f32, int64_t M, int N, int64_t ld, float* d_out,
                          float* d_work, b2s_stream_t stream);
int64_t b2s_colsum_work_floats(int N);

/* x[m] = wte[tok[m]] (+ wpe[m % T]) -> fp32 [M, D]; backward scatters dx
 * into fp32 dwte (atomics) and sums positions into dwpe (optional). */
int b2s_embedding_fwd(const int64_t* d_tok, const void* d_wte, const void* d_wpe, float* d_x, int64_t M,
                      int T, int D, b2s_stream_t stream);
int b2s_embedding_bwd(const int64_t* d_tok, const float* d_dx, float* d_dwte, float* d_dwpe, int B, int T,
                      int D, b2s_stream_t stream);

/* Rotary embedding in place on the first `nheads` heads (dh wide) of each
 * [M, ld] bf16 row; rotate-half pairing; tables [T, dh/2] fp32; inverse=1
 * applies the transposed rotation (backward). */
int b2s_rope(void* d_qkv, int64_t M, int T, int64_t ld, int nheads, int dh, const float* d_cos,
             const float* d_sin, int inverse, b2s_stream_t stream);

/* h = silu(gate) * up with gu = [gate | up] (bf16 [M, 2F]); backward writes [dgate | dup]. */
int b2s_swiglu_fwd(const void* d_gu, void* d_h, int64_t M, int F, b2s_stream_t stream);
int b2s_swiglu_bwd(const void* d_gu, const void* d_dh, void* d_dgu, int64_t M, int F, b2s_stream_t stream);

/* Per-row softmax cross-entropy over the first V of ld bf16 logits:
 * d_loss_rows[m] = logsumexp - logit[target]; if write_grad, the logits are
 * overwritten by (softmax - onehot) * grad_scale (padding columns zeroed). */
int b2s_cross_entropy(void* d_logits, int64_t ld, int V, const int64_t* d_target, float* d_loss_rows,
                      float grad_scale, int64_t M, int write_grad, b2s_stream_t stream);

/* d_out[0] = scale * sum(x or x^2), single block, deterministic. */
int b2s_sum(const float* d_x, int64_t n, int squares, float* d_out, float scale, b2s_stream_t stream);
/* d_part[b] = partial sum of squares (b < nparts), deterministic stage 1. */
int b2s_sumsq_partial(const float* d_x, int64_t n, float* d_part, int nparts, b2s_stream_t stream);
/* Same over nseg buffers in one launch (the global gradient norm over every FSDP
 * unit's shard): d_ptrs / d_lens are device arrays of nseg fp32 buffer addresses
 * (16-byte aligned) and element counts; d_part[b] sums all segments. Replaces the
 * reference's per-parameter torch.nn.utils.clip_grad_norm_ norm pass
 * (gradient clipping in the optimizer step). */
int b2s_sumsq_partial_multi(const uint64_t* d_ptrs, const int64_t* d_lens, int nseg, float* d_part, int nparts,
                            b2s_stream_t stream);

/* Fused AdamW over a flat fp32 shard (K10). Gradient clipping by the global
 * norm is applied on the device: clip = min(1, max_norm/(sqrt(*d_gn2)+1e-6))
 * (d_gn2 = all-reduced squared grad norm; null or max_norm<=0 disables).
 * Writes the updated bf16 copy of p (the next all-gather source). d_wd_mask:
 * per-element u8 (1 = decay) or null (decay all). step is 1-based. */
int b2s_adamw(float* d_p, float* d_m, float* d_v, const float* d_g, void* d_p_bf16, const uint8_t* d_wd_mask,
              int64_t n, const float* d_gn2, float max_norm, float lr, float beta1, float beta2, float eps,
              float wd, int step, b2s_stream_t stream);

int b2s_f32_to_bf16(const float* d_x, void* d_y, int64_t n, float scale, b2s_stream_t stream);
int b2s_scale_f32(float* d_x, int64_t n, float scale, b2s_stream_t stream);

/* ------------------------------------------------------------------ */
/* Causal attention (K7): tcgen05 + TMEM + TMA, head dim 64            */
/* ------------------------------------------------------------------ */
/* q/k/v read in place from the fused projection output d_qkv, bf16
 * [B*T, (Hq + 2*Hkv)*dh] (q heads, then k heads, then v heads). Writes
 * d_o bf16 [B*T, Hq*dh] and d_lse fp32 [B, Hq, T] (natural-log softmax
 * normaliser of the scaled scores). T % 128 == 0, Hq % Hkv == 0. */
int b2s_attn_fwd(const void* d_qkv, void* d_o, float* d_lse, int B, int T, int Hq, int Hkv, int dh,
                 b2s_stream_t stream);
/* Backward of b2s_attn_fwd: writes dq, dk, dv into d_dqkv (same layout as
 * d_qkv). d_do: bf16 [B*T, Hq*dh]. d_work: b2s_attn_bwd_work_floats() floats
 * (fp32 dQ accumulator, scaled rowsum(dO*O), log2-unit LSE). */
int b2s_attn_bwd(const void* d_qkv, const void* d_o, const void* d_do, const float* d_lse, void* d_dqkv,
                 float* d_work, int B, int T, int Hq, int Hkv, int dh, b2s_stream_t stream);
int64_t b2s_attn_bwd_work_floats(int B, int T, int Hq, int dh);
/* b2s_attn_bwd for rotary-embedded q / k: also rotates the q and k heads of d_dqkv back
 * (inverse of b2s_rope with the same tables), i.e. the gradient w.r.t. the projection output.
 * dh 64 folds the dq rotation into the dq conversion pass. */
int b2s_attn_bwd_rope(const void* d_qkv, const void* d_o, const void* d_do, const float* d_lse, void* d_dqkv,
                      float* d_work, int B, int T, int Hq, int Hkv, int dh, const float* d_cos, const float* d_sin,
                      b2s_stream_t stream);

/* ------------------------------------------------------------------ */
/* fp32 mode (north star: per-step losses/gradients within 1e-4 of the  */
/* CPU fp32 reference). Same contracts as the bf16 entry points above   */
/* with every activation / weight operand fp32; GEMM and attention run  */
/* true-fp32 FFMA on the CUDA cores (not TF32).   */
/* ------------------------------------------------------------------ */
/* C[M,N] (fp32) = epi(sum_k A(m,k) B(n,k)); layouts, bias, act, aux and
 * accumulate as b2s_gemm (aux fp32). Any M, N, K >= 0. */
int b2s_gemm_f32(const float* d_A, int a_mn_major, int64_t lda, const float* d_B, int b_mn_major, int64_t ldb,
                 float* d_C, int64_t ldc, int M, int N, int K, int accumulate, const float* d_bias, int act,
                 float* d_aux, int64_t ld_aux, b2s_stream_t stream);
int b2s_layernorm_fwd_f32(const float* d_x, const float* d_g, const float* d_b, float* d_y, float* d_mean,
                          float* d_rstd, float* d_x_copy, int64_t M, int D, float eps, b2s_stream_t stream);
int b2s_rmsnorm_fwd_f32(const float* d_x, const float* d_g, float* d_y, float* d_rstd, float* d_x_copy,
                        int64_t M, int D, float eps, b2s_stream_t stream);
/* d_dx_copy: optional second copy of the updated dx (usually null in fp32 mode). */
int b2s_layernorm_fwd_res_f32(const float* d_x, const float* d_res, const float* d_g, const float* d_b, float* d_y,
                              float* d_mean, float* d_rstd, float* d_x_out, int64_t M, int D, float eps,
                              b2s_stream_t stream);
int b2s_rmsnorm_fwd_res_f32(const float* d_x, const float* d_res, const float* d_g, float* d_y, float* d_rstd,
                            float* d_x_out, int64_t M, int D, float eps, b2s_stream_t stream);
int b2s_layernorm_bwd_f32(const float* d_x, const float* d_dy, const float* d_g, const float* d_mean,
                          const float* d_rstd, float* d_dx, float* d_dx_copy, float* d_dg, float* d_db,
                          float* d_dxsum, float* d_work, int64_t M, int D, b2s_stream_t stream);
int b2s_rmsnorm_bwd_f32(const float* d_x, const float* d_dy, const float* d_g, const float* d_rstd, float* d_dx,
                        float* d_dx_copy, float* d_dg, float* d_dxsum, float* d_work, int64_t M, int D,
                        b2s_stream_t stream);
int b2s_embedding_fwd_f32(const int64_t* d_tok, const float* d_wte, const float* d_wpe, float* d_x, int64_t M,
                          int T, int D, b2s_stream_t stream);
int b2s_rope_f32(float* d_qkv, int64_t M, int T, int64_t ld, int nheads, int dh, const float* d_cos,
                 const float* d_sin, int inverse, b2s_stream_t stream);
int b2s_swiglu_fwd_f32(const float* d_gu, float* d_h, int64_t M, int F, b2s_stream_t stream);
int b2s_swiglu_bwd_f32(const float* d_gu, const float* d_dh, float* d_dgu, int64_t M, int F, b2s_stream_t stream);
int b2s_cross_entropy_f32(float* d_logits, int64_t ld, int V, const int64_t* d_target, float* d_loss_rows,
                          float grad_scale, int64_t M, int write_grad, b2s_stream_t stream);
/* d_p_copy: optional fp32 copy of the updated p (null when p is itself the
 * all-gather source / compute buffer). */
int b2s_adamw_f32(float* d_p, float* d_m, float* d_v, const float* d_g, float* d_p_copy, const uint8_t* d_wd_mask,
                  int64_t n, const float* d_gn2, float max_norm, float lr, float beta1, float beta2, float eps,
                  float wd, int step, b2s_stream_t stream);
/* Causal attention, fp32 [B*T, (Hq+2Hkv)*dh] fused projection, head dims
 * 32 / 64 / 128, any T >= 1. d_work: b2s_attn_bwd_work_floats() floats. */
int b2s_attn_fwd_f32(const float* d_qkv, float* d_o, float* d_lse, int B, int T, int Hq, int Hkv, int dh,
                     b2s_stream_t stream);
int b2s_attn_bwd_f32(const float* d_qkv, const float* d_o, const float* d_do, const float* d_lse, float* d_dqkv,
                     float* d_work, int B, int T, int Hq, int Hkv, int dh, b2s_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* B2S_H_ */
