// Packed-dataset sample indexer (K1) and the host-side seeded shuffle.
//
// Device: b2s_gather_samples is the batched GPU form of
//   PackedReader.get_sample  (reference packed_data.py:196-203)
// followed by the inputs = ids[:L], targets = ids[1:] split.
// Host:   SplitMix64 / make_permutation / chunk restated in C++ so the sampler
//   never runs the O(n) Python loop (packed_data.py:257-282, :322-333).
#include <stdlib.h>
#include <string.h>
#include <atomic>
#include <thread>
#include <type_traits>
#include "common.cuh"

namespace b2s {

static thread_local char g_err[512];
static std::atomic<unsigned long long> g_launches{0};
void count_launches(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

template <int W>
__device__ __forceinline__ int64_t load_token(const uint8_t* __restrict__ p, uint64_t i) {
  if constexpr (W == 1) return (int64_t)p[i];
  if constexpr (W == 2) return (int64_t)reinterpret_cast<const uint16_t*>(p)[i];
  return (int64_t)reinterpret_cast<const uint32_t*>(p)[i];
}

// One thread produces a pair of consecutive outputs of the flattened [B*L]
// input/target arrays and stores each pair as one 16-byte vector. The payload
// read for output (b,t) is token s_b*L+t (+1 for targets): consecutive threads
// read consecutive tokens, so loads and stores are both coalesced.
// Sample s starts at token s * stride: stride = L for the packed stream
// (consecutive samples overlap by one token), L + 1 for staged windows.
template <int W>
__global__ void __launch_bounds__(256) gather_samples_kernel(
    const uint8_t* __restrict__ payload, uint64_t nsamples, const uint64_t* __restrict__ ids,
    int batch, int64_t L, int64_t stride, int64_t* __restrict__ inputs, int64_t* __restrict__ targets,
    int32_t* __restrict__ status) {
  const uint64_t total = (uint64_t)batch * (uint64_t)L;
  const uint64_t npairs = (total + 1) / 2;
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < npairs;
       p += (uint64_t)gridDim.x * blockDim.x) {
    int64_t in2[2], tg2[2];
    bool ok[2] = {false, false};
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const uint64_t idx = 2 * p + e;
      if (idx >= total) break;
      const uint64_t b = idx / (uint64_t)L, t = idx - b * (uint64_t)L;
      const uint64_t s = ids ? __ldg(ids + b) : b;
      if (s >= nsamples) {
        if (t == 0) atomicExch(status, 1);
        continue;
      }
      const uint64_t base = s * (uint64_t)stride + t;  // 64-bit token offset
      in2[e] = load_token<W>(payload, base);
      tg2[e] = load_token<W>(payload, base + 1);
      ok[e] = true;
    }
    const uint64_t idx0 = 2 * p;
    if (ok[0] && ok[1] && idx0 + 1 < total) {
      *reinterpret_cast<longlong2*>(inputs + idx0) = make_longlong2(in2[0], in2[1]);
      *reinterpret_cast<longlong2*>(targets + idx0) = make_longlong2(tg2[0], tg2[1]);
    } else {
      if (ok[0]) { inputs[idx0] = in2[0]; targets[idx0] = tg2[0]; }
      if (ok[1] && idx0 + 1 < total) { inputs[idx0 + 1] = in2[1]; targets[idx0 + 1] = tg2[1]; }
    }
  }
}


// Document-level segmented copy (materialize_chunk on the device, reference
// packed_data.py:336-344): document i of the output is source tokens
// [src_start[i], src_start[i] + len[i]) written at token dst_start[i]. One warp
// per document (grid-stride), lanes on consecutive tokens: loads and stores are
// coalesced within a document and no per-token search is needed.
template <int W>
__global__ void __launch_bounds__(256) gather_documents_kernel(const uint8_t* __restrict__ payload,
                                                               const uint64_t* __restrict__ src_start,
                                                               const uint64_t* __restrict__ len,
                                                               const uint64_t* __restrict__ dst_start, int64_t n,
                                                               uint8_t* __restrict__ out) {
  using Tok = typename std::conditional<W == 1, uint8_t, typename std::conditional<W == 2, uint16_t, uint32_t>::type>::type;
  const Tok* src = reinterpret_cast<const Tok*>(payload);
  Tok* dst = reinterpret_cast<Tok*>(out);
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t d = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; d < n; d += warps) {
    const uint64_t s0 = __ldg(src_start + d), l = __ldg(len + d), o0 = __ldg(dst_start + d);
    uint64_t t = lane;
    for (; t + 96 < l; t += 128) {  // four independent loads in flight per lane
      const Tok a0 = src[s0 + t], a1 = src[s0 + t + 32], a2 = src[s0 + t + 64], a3 = src[s0 + t + 96];
      dst[o0 + t] = a0; dst[o0 + t + 32] = a1; dst[o0 + t + 64] = a2; dst[o0 + t + 96] = a3;
    }
    for (; t < l; t += 32) dst[o0 + t] = src[s0 + t];
  }
}

static inline uint64_t splitmix_next(uint64_t& state) {
  state += 0x9E3779B97F4A7C15ull;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace b2s

extern "C" {

const char* b2s_last_error(void) { return b2s::g_err; }
int b2s_abi_version(void) { return 1; }
uint64_t b2s_launch_count(void) { return b2s::g_launches.load(); }

int b2s_memset_async(void* dst, int value, uint64_t bytes, void* stream) {
  B2S_REQUIRE(dst || bytes == 0, B2S_EINVAL, "dst is null");
  if (bytes == 0) return B2S_OK;
  const cudaError_t e = cudaMemsetAsync(dst, value, (size_t)bytes, (cudaStream_t)stream);
  B2S_REQUIRE(e == cudaSuccess, B2S_ECUDA, "cudaMemsetAsync: %s", cudaGetErrorString(e));
  return B2S_OK;
}

// Native CUDA-graph capture of a stream's work (the W = 1 training step): the replay is a bare
// cudaGraphLaunch, so the step's launch list holds only this library's kernels and memsets
// (torch.cuda.CUDAGraph's replay adds two RNG-offset fill kernels per launch).
int b2s_graph_capture_begin(void* stream) {
  const cudaError_t e = cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeThreadLocal);
  B2S_REQUIRE(e == cudaSuccess, B2S_ECUDA, "cudaStreamBeginCapture: %s", cudaGetErrorString(e));
  return B2S_OK;
}
int b2s_graph_capture_end(void* stream, void** h_exec) {
  B2S_REQUIRE(h_exec, B2S_EINVAL, "h_exec is null");
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture((cudaStream_t)stream, &g);
  B2S_REQUIRE(e == cudaSuccess && g, B2S_ECUDA, "cudaStreamEndCapture: %s", cudaGetErrorString(e));
  cudaGraphExec_t x = nullptr;
  e = cudaGraphInstantiate(&x, g, 0);
  cudaGraphDestroy(g);
  B2S_REQUIRE(e == cudaSuccess, B2S_ECUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(e));
  *h_exec = (void*)x;
  return B2S_OK;
}
int b2s_graph_launch(void* exec, void* stream) {
  B2S_REQUIRE(exec, B2S_EINVAL, "exec is null");
  const cudaError_t e = cudaGraphLaunch((cudaGraphExec_t)exec, (cudaStream_t)stream);
  B2S_REQUIRE(e == cudaSuccess, B2S_ECUDA, "cudaGraphLaunch: %s", cudaGetErrorString(e));
  return B2S_OK;
}
int b2s_graph_destroy(void* exec) {
  if (exec) cudaGraphExecDestroy((cudaGraphExec_t)exec);
  return B2S_OK;
}

int b2s_token_width_for_vocab(uint64_t vocab_size, int* h_width) {
  B2S_REQUIRE(h_width, B2S_EINVAL, "h_width is null");
  B2S_REQUIRE(vocab_size >= 1, B2S_EINVAL, "vocab_size must be positive, got %llu",
              (unsigned long long)vocab_size);
  if (vocab_size <= (1ull << 8)) *h_width = 1;
  else if (vocab_size <= (1ull << 16)) *h_width = 2;
  else if (vocab_size <= (1ull << 32)) *h_width = 4;
  else B2S_REQUIRE(false, B2S_EINVAL, "vocab_size %llu exceeds the 4-byte token width",
                   (unsigned long long)vocab_size);
  return B2S_OK;
}

int b2s_sample_count(uint64_t token_count, int64_t seq_len, uint64_t* h_count) {
  B2S_REQUIRE(h_count, B2S_EINVAL, "h_count is null");
  B2S_REQUIRE(seq_len >= 1, B2S_EINVAL, "seq_len must be >= 1, got %lld", (long long)seq_len);
  *h_count = token_count == 0 ? 0 : (token_count - 1) / (uint64_t)seq_len;
  return B2S_OK;
}

int b2s_splitmix64(uint64_t seed, uint64_t count, uint64_t* h_out) {
  B2S_REQUIRE(h_out || count == 0, B2S_EINVAL, "h_out is null");
  uint64_t state = seed;
  for (uint64_t i = 0; i < count; ++i) h_out[i] = b2s::splitmix_next(state);
  return B2S_OK;
}

int b2s_make_permutation(uint64_t n, uint64_t seed, uint64_t* h_order) {
  B2S_REQUIRE(h_order || n == 0, B2S_EINVAL, "h_order is null");
  for (uint64_t i = 0; i < n; ++i) h_order[i] = i;
  uint64_t state = seed;  // seed already masked to 64 bits (packed_data.py:268)
  for (uint64_t i = n ? n - 1 : 0; i >= 1; --i) {
    const uint64_t bound = i + 1;
    // floor(2^64 / bound) * bound, in uint64: 2^64 - (2^64 mod bound); 0 encodes 2^64.
    const uint64_t rem = (UINT64_MAX % bound + 1) % bound;  // 2^64 mod bound
    const uint64_t threshold = 0ull - rem;                  // wraps to 0 when rem == 0
    uint64_t x;
    do {
      x = b2s::splitmix_next(state);
    } while (threshold != 0 && x >= threshold);
    const uint64_t j = x % bound;
    const uint64_t t = h_order[i];
    h_order[i] = h_order[j];
    h_order[j] = t;
  }
  return B2S_OK;
}

int b2s_chunk_bounds(uint64_t n, uint64_t k, uint64_t* h_lo) {
  B2S_REQUIRE(h_lo, B2S_EINVAL, "h_lo is null");
  const uint64_t kmax = n > 1 ? n : 1;
  B2S_REQUIRE(k >= 1 && k <= kmax, B2S_EINVAL, "k must be in [1, %llu], got %llu",
              (unsigned long long)kmax, (unsigned long long)k);
  const uint64_t q = n / k, r = n % k;
  uint64_t lo = 0;
  for (uint64_t c = 0; c < k; ++c) {
    h_lo[c] = lo;
    lo += q + (c < r ? 1 : 0);
  }
  h_lo[k] = lo;
  return B2S_OK;
}

int b2s_gather_samples(const void* d_payload, int width, uint64_t token_count,
                       const uint64_t* d_sample_ids, int batch, int64_t seq_len,
                       int64_t* d_inputs, int64_t* d_targets, int32_t* d_status,
                       b2s_stream_t stream) {
  B2S_REQUIRE(width == 1 || width == 2 || width == 4, B2S_EINVAL,
              "token width must be 1, 2 or 4, got %d", width);
  B2S_REQUIRE(seq_len >= 1, B2S_EINVAL, "seq_len must be >= 1, got %lld", (long long)seq_len);
  B2S_REQUIRE(batch >= 0, B2S_EINVAL, "batch must be >= 0");
  if (batch == 0) return B2S_OK;
  B2S_REQUIRE(d_payload && d_sample_ids && d_inputs && d_targets && d_status, B2S_EINVAL,
              "null device pointer");
  B2S_REQUIRE(((uintptr_t)d_inputs % 16) == 0 && ((uintptr_t)d_targets % 16) == 0, B2S_EINVAL,
              "inputs/targets must be 16-byte aligned");
  const uint64_t nsamples = token_count == 0 ? 0 : (token_count - 1) / (uint64_t)seq_len;
  const uint64_t npairs = ((uint64_t)batch * (uint64_t)seq_len + 1) / 2;
  unsigned grid = b2s::ceil_div(npairs, 256);
  if (grid > b2s::kNumSMs * 16) grid = b2s::kNumSMs * 16;
  cudaStream_t st = (cudaStream_t)stream;
  const uint8_t* p = (const uint8_t*)d_payload;
  switch (width) {
    case 1: b2s::gather_samples_kernel<1><<<grid, 256, 0, st>>>(p, nsamples, d_sample_ids, batch, seq_len, seq_len, d_inputs, d_targets, d_status); break;
    case 2: b2s::gather_samples_kernel<2><<<grid, 256, 0, st>>>(p, nsamples, d_sample_ids, batch, seq_len, seq_len, d_inputs, d_targets, d_status); break;
    default: b2s::gather_samples_kernel<4><<<grid, 256, 0, st>>>(p, nsamples, d_sample_ids, batch, seq_len, seq_len, d_inputs, d_targets, d_status); break;
  }
  return b2s::check_launch("gather_samples");
}

int b2s_unpack_windows(const void* d_windows, int width, int batch, int64_t seq_len, int64_t* d_inputs,
                       int64_t* d_targets, b2s_stream_t stream) {
  B2S_REQUIRE(width == 1 || width == 2 || width == 4, B2S_EINVAL, "token width must be 1, 2 or 4, got %d", width);
  B2S_REQUIRE(seq_len >= 1 && batch >= 0, B2S_EINVAL, "bad shape");
  if (batch == 0) return B2S_OK;
  B2S_REQUIRE(((uintptr_t)d_inputs % 16) == 0 && ((uintptr_t)d_targets % 16) == 0, B2S_EINVAL,
              "inputs/targets must be 16-byte aligned");
  const uint64_t npairs = ((uint64_t)batch * (uint64_t)seq_len + 1) / 2;
  unsigned grid = b2s::ceil_div(npairs, 256);
  if (grid > b2s::kNumSMs * 16) grid = b2s::kNumSMs * 16;
  cudaStream_t st = (cudaStream_t)stream;
  const uint8_t* p = (const uint8_t*)d_windows;
  switch (width) {
    case 1: b2s::gather_samples_kernel<1><<<grid, 256, 0, st>>>(p, batch, nullptr, batch, seq_len, seq_len + 1, d_inputs, d_targets, nullptr); break;
    case 2: b2s::gather_samples_kernel<2><<<grid, 256, 0, st>>>(p, batch, nullptr, batch, seq_len, seq_len + 1, d_inputs, d_targets, nullptr); break;
    default: b2s::gather_samples_kernel<4><<<grid, 256, 0, st>>>(p, batch, nullptr, batch, seq_len, seq_len + 1, d_inputs, d_targets, nullptr); break;
  }
  return b2s::check_launch("unpack_windows");
}

int b2s_gather_documents(const void* d_payload, int width, const uint64_t* d_src_start, const uint64_t* d_len,
                         const uint64_t* d_dst_start, int64_t n_docs, void* d_out, b2s_stream_t stream) {
  B2S_REQUIRE(width == 1 || width == 2 || width == 4, B2S_EINVAL, "token width must be 1, 2 or 4, got %d", width);
  B2S_REQUIRE(n_docs >= 0, B2S_EINVAL, "n_docs must be >= 0");
  if (n_docs == 0) return B2S_OK;
  B2S_REQUIRE(d_payload && d_src_start && d_len && d_dst_start && d_out, B2S_EINVAL, "null device pointer");
  int64_t blocks = (n_docs * 32 + 255) / 256;
  if (blocks > b2s::kNumSMs * 16) blocks = b2s::kNumSMs * 16;
  cudaStream_t st = (cudaStream_t)stream;
  const uint8_t* p = (const uint8_t*)d_payload;
  uint8_t* o = (uint8_t*)d_out;
  switch (width) {
    case 1: b2s::gather_documents_kernel<1><<<(unsigned)blocks, 256, 0, st>>>(p, d_src_start, d_len, d_dst_start, n_docs, o); break;
    case 2: b2s::gather_documents_kernel<2><<<(unsigned)blocks, 256, 0, st>>>(p, d_src_start, d_len, d_dst_start, n_docs, o); break;
    default: b2s::gather_documents_kernel<4><<<(unsigned)blocks, 256, 0, st>>>(p, d_src_start, d_len, d_dst_start, n_docs, o); break;
  }
  return b2s::check_launch("gather_documents");
}

}  // extern "C"
