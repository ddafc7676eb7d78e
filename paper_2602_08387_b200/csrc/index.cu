// Corpus indexing: the newline scan of
// corpus_index.build_index (reference corpus_index.py:68-107) on the GPU.
//
// A raw JSONL buffer resident in HBM is split into `nblocks` equal chunks
// (multiples of 16 bytes). Pass 1 counts the 0x0A bytes of each chunk; the
// caller turns the counts into exclusive offsets; pass 2 writes the absolute
// byte position of every newline, in file order, at its offset. 16-byte
// vector loads, warp-ballot ranks within a 512-byte step, one block-wide scan
// per step -- the output is ordered, so spans follow with one host diff.
#include "common.cuh"

namespace b2s {
namespace idx {

constexpr int kThreads = 256;  // 8 warps; a step covers 256 * 16 = 4 KB

__device__ __forceinline__ int nl_mask16(const uint4 v) {
  // bit k set iff byte k of the 16-byte vector is '\n'
  int m = 0;
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t x = w[i] ^ 0x0A0A0A0Au;  // zero byte where '\n'
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (((x >> (8 * b)) & 0xFFu) == 0u) m |= 1 << (4 * i + b);
  }
  return m;
}

__device__ __forceinline__ int load_mask(const uint8_t* __restrict__ buf, uint64_t n, uint64_t off) {
  if (off + 16 <= n) return nl_mask16(*reinterpret_cast<const uint4*>(buf + off));
  int m = 0;
  for (int k = 0; off + k < n && k < 16; ++k)
    if (buf[off + k] == 0x0A) m |= 1 << k;
  return m;
}

__global__ void __launch_bounds__(kThreads) count_kernel(const uint8_t* __restrict__ buf, uint64_t n,
                                                         uint64_t chunk, uint32_t* __restrict__ counts) {
  __shared__ uint32_t red[kThreads / 32];
  const uint64_t lo = (uint64_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
  uint32_t c = 0;
  for (uint64_t off = lo + 16ull * threadIdx.x; off < hi; off += 16ull * kThreads) c += __popc(load_mask(buf, hi, off));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
    counts[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kThreads) positions_kernel(const uint8_t* __restrict__ buf, uint64_t n,
                                                             uint64_t chunk, const uint64_t* __restrict__ offsets,
                                                             uint64_t base, uint64_t* __restrict__ pos) {
  __shared__ uint32_t wsum[kThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t lo = (uint64_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
  uint64_t out = offsets[blockIdx.x];
  for (uint64_t step = lo; step < hi; step += 16ull * kThreads) {
    const uint64_t off = step + 16ull * threadIdx.x;
    const int m = off < hi ? load_mask(buf, hi, off) : 0;
    const uint32_t c = __popc(m);
    // exclusive prefix of c over the block (thread order = byte order)
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    uint32_t before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
      const uint32_t s = wsum[w];
      before += (w < wid) ? s : 0u;
      total += s;
    }
    __syncthreads();
    uint64_t o = out + before + incl - c;
    int mm = m;
    while (mm) {
      const int k = __ffs(mm) - 1;
      pos[o++] = base + off + (uint64_t)k;
      mm &= mm - 1;
    }
    out += total;
  }
}

}  // namespace idx
}  // namespace b2s

extern "C" {

int b2s_newline_count(const void* d_buf, uint64_t n, uint64_t chunk, uint32_t* d_counts, int nblocks,
                      b2s_stream_t stream) {
  B2S_REQUIRE(chunk % 16 == 0 && chunk > 0 && nblocks > 0 && (uint64_t)nblocks * chunk >= n, B2S_EINVAL,
              "newline_count: chunk must be a positive multiple of 16 covering n");
  B2S_REQUIRE(((uintptr_t)d_buf % 16) == 0, B2S_EINVAL, "newline_count: buffer must be 16-byte aligned");
  b2s::idx::count_kernel<<<nblocks, b2s::idx::kThreads, 0, (cudaStream_t)stream>>>((const uint8_t*)d_buf, n, chunk,
                                                                                 d_counts);
  return b2s::check_launch("newline_count");
}

int b2s_newline_positions(const void* d_buf, uint64_t n, uint64_t chunk, const uint64_t* d_offsets, int nblocks,
                          uint64_t base, uint64_t* d_pos, b2s_stream_t stream) {
  B2S_REQUIRE(chunk % 16 == 0 && chunk > 0 && nblocks > 0 && (uint64_t)nblocks * chunk >= n, B2S_EINVAL,
              "newline_positions: chunk must be a positive multiple of 16 covering n");
  B2S_REQUIRE(((uintptr_t)d_buf % 16) == 0, B2S_EINVAL, "newline_positions: buffer must be 16-byte aligned");
  b2s::idx::positions_kernel<<<nblocks, b2s::idx::kThreads, 0, (cudaStream_t)stream>>>(
      (const uint8_t*)d_buf, n, chunk, d_offsets, base, d_pos);
  return b2s::check_launch("newline_positions");
}

}  // extern "C"
