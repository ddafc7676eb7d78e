// Bandwidth-bound kernels of the training step (K2-K4, K8-K11): embedding,
// LayerNorm / RMSNorm, RoPE, SwiGLU, cross-entropy, column sums, AdamW,
// grad-norm, casts. All HBM-bound: 16-byte vector accesses, one warp per row
// for the row-wise ops with the hidden size a compile-time constant (so the
// row lives in registers), warp-shuffle reductions, deterministic two-stage
// column reductions (no floating-point atomics except the embedding scatter).
#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "sm100.cuh"

namespace b2s {
namespace ew {

constexpr int kRowThreads = 256;  // 8 warps, one row per warp at a time

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ void ld_bf4(const __nv_bfloat16* p, float* f) {
  uint2 u = *reinterpret_cast<const uint2*>(p);
  float2 a = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.x));
  float2 b = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&u.y));
  f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
}
__device__ __forceinline__ void st_bf4(__nv_bfloat16* p, const float* f) {
  uint2 u;
  u.x = pack_bf16x2(f[0], f[1]);
  u.y = pack_bf16x2(f[2], f[3]);
  *reinterpret_cast<uint2*>(p) = u;
}
// Activation-type generic 4- and 8-element vectors: T = __nv_bfloat16 (the
// training precision) or float (fp32 mode, the 1e-4 parity configuration).
__device__ __forceinline__ void ld_v4(const __nv_bfloat16* p, float* f) { ld_bf4(p, f); }
__device__ __forceinline__ void ld_v4(const float* p, float* f) {
  const float4 v = ld4(p);
  f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
}
__device__ __forceinline__ void st_v4(__nv_bfloat16* p, const float* f) { st_bf4(p, f); }
__device__ __forceinline__ void st_v4(float* p, const float* f) { st4(p, make_float4(f[0], f[1], f[2], f[3])); }
__device__ __forceinline__ void ld_v8(const __nv_bfloat16* p, float* f) {
  unpack8(*reinterpret_cast<const bf16x8*>(p), f);
}
__device__ __forceinline__ void ld_v8(const float* p, float* f) { ld_v4(p, f); ld_v4(p + 4, f + 4); }
__device__ __forceinline__ void st_v8(__nv_bfloat16* p, const float* f) { *reinterpret_cast<bf16x8*>(p) = pack8(f); }
__device__ __forceinline__ void st_v8(float* p, const float* f) { st_v4(p, f); st_v4(p + 4, f + 4); }
// streaming (evict-first) variants: data read / written once that should not push
// still-needed lines out of L2
__device__ __forceinline__ void st_v8_cs(__nv_bfloat16* p, const float* f) {
  const bf16x8 v = pack8(f);
  __stcs(reinterpret_cast<uint4*>(p), *reinterpret_cast<const uint4*>(&v));
}
__device__ __forceinline__ void st_v8_cs(float* p, const float* f) {
  __stcs(reinterpret_cast<float4*>(p), make_float4(f[0], f[1], f[2], f[3]));
  __stcs(reinterpret_cast<float4*>(p + 4), make_float4(f[4], f[5], f[6], f[7]));
}
__device__ __forceinline__ void ld_v8_cs(const __nv_bfloat16* p, float* f) {
  const uint4 u = __ldcs(reinterpret_cast<const uint4*>(p));
  unpack8(*reinterpret_cast<const bf16x8*>(&u), f);
}
__device__ __forceinline__ void ld_v8_cs(const float* p, float* f) {
  const float4 a = __ldcs(reinterpret_cast<const float4*>(p)), b = __ldcs(reinterpret_cast<const float4*>(p + 4));
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return bf2f(v); }
__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ void from_f(__nv_bfloat16& d, float v) { d = f2bf(v); }
__device__ __forceinline__ void from_f(float& d, float v) { d = v; }


// Four elements loaded without conversion (bf16: one 8-byte load), converted at first use, so
// the load can stay in flight across other work.
template <typename T>
struct Raw4;
template <>
struct Raw4<__nv_bfloat16> {
  uint2 v;
  __device__ __forceinline__ void ld(const __nv_bfloat16* p) { v = *reinterpret_cast<const uint2*>(p); }
  __device__ __forceinline__ void get(float* f) const {
    f[0] = __uint_as_float(v.x << 16); f[1] = __uint_as_float(v.x & 0xffff0000u);
    f[2] = __uint_as_float(v.y << 16); f[3] = __uint_as_float(v.y & 0xffff0000u);
  }
};
template <>
struct Raw4<float> {
  float4 v;
  __device__ __forceinline__ void ld(const float* p) { v = ld4(p); }
  __device__ __forceinline__ void get(float* f) const { f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w; }
};

// ------------------------------------------------------------------ norms
// y = (x - mean) * rstd * g (+ b)  [LayerNorm]   or   y = x * rstd * g  [RMSNorm]
// x fp32 [M, D] (the residual stream), y bf16; optional x_copy (forward the
// residual into the next stream buffer while it is in registers).
// TPR threads cooperate on a row (32 = one warp for D <= 1024, 256 = the whole
// block for D >= 2048) so the row stays in registers at every hidden size.
// Sum over the TPR threads sharing a row. TPR = 64 / 128: the row's 2 / 4 warps
// exchange through double-buffered smem slots and a named barrier per row group
// (ids 1..4), so row groups of one block never wait on each other.
template <int TPR>
__device__ __forceinline__ float row_sum(float v, float* scratch, int& toggle) {
  if constexpr (TPR == 32) {
    return warp_sum(v);
  } else if constexpr (TPR == 64 || TPR == 128) {
    constexpr int NW = TPR / 32;
    v = warp_sum(v);
    const int wid = threadIdx.x >> 5;
    float* sl = scratch + toggle * 8;
    if ((threadIdx.x & 31) == 0) sl[wid] = v;
    asm volatile("bar.sync %0, %1;" ::"r"(1 + wid / NW), "n"(TPR) : "memory");
    toggle ^= 1;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < NW; ++k) s += sl[(wid / NW) * NW + k];
    return s;
  } else {
    return block_sum(v, scratch);
  }
}

// res (optional): the sublayer output y_prev [M, D] (activation type) to add to x
// first -- the residual add of the previous GEMM; x_copy then receives x + res
// (the new residual stream), which is what gets normalised.
// Block-per-row form (TPR 256, D >= 2048): the next row's loads are prefetched and the kernel
// is held to 64 registers (4 blocks per SM): Llama-1B RMSNorm 62.1 -> 56.1 us (0.82 -> 0.91 of
// HBM), with the residual add 68.5 -> 67.1 us. The warp-per-row form (D <= 1024) loads the
// current row as before: prefetching there measured slower (GPT-2 LayerNorm 23.6 -> 29.5 us).
template <int D, int TPR, bool RMS, typename T = __nv_bfloat16>
__global__ void __launch_bounds__(kRowThreads, TPR >= 256 ? 4 : 1) norm_fwd_kernel(
    const float* __restrict__ x, const T* __restrict__ g, const T* __restrict__ b,
    T* __restrict__ y, float* __restrict__ mean_out, float* __restrict__ rstd_out,
    float* __restrict__ x_copy, int64_t M, float eps, const T* __restrict__ res) {
  constexpr int V = D / (TPR * 4);  // float4 vectors per thread
  static_assert(V * TPR * 4 == D, "hidden size must tile the row threads");
  __shared__ float scratch[32];
  int tog = 0;
  const int t = threadIdx.x % TPR;
  const int64_t r0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / TPR;
  const int64_t nr = ((int64_t)gridDim.x * blockDim.x) / TPR;
  float gv[V][4], bv[V][4];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    ld_v4(g + t * 4 + j * TPR * 4, gv[j]);
    if (!RMS) ld_v4(b + t * 4 + j * TPR * 4, bv[j]);
  }
  // PF: the next row's x / res loads are issued before this row's reductions and stores (kept
  // raw in registers until then), so a block keeps HBM reads in flight through its two row syncs
  constexpr bool PF = TPR >= 256;
  float4 xn[V];
  Raw4<T> rn[V];
  auto fetch = [&](int64_t row) {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      xn[j] = ld4(x + row * D + t * 4 + j * TPR * 4);
      if (res) rn[j].ld(res + row * D + t * 4 + j * TPR * 4);
    }
  };
  if (PF && r0 < M) fetch(r0);
  for (int64_t row = r0; row < M; row += nr) {
    if (!PF) fetch(row);
    float4 xv[V];
    float s = 0.f, ss = 0.f;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      xv[j] = xn[j];
      if (res) {
        float r4[4];
        rn[j].get(r4);
        xv[j].x += r4[0]; xv[j].y += r4[1]; xv[j].z += r4[2]; xv[j].w += r4[3];
      }
      s += xv[j].x + xv[j].y + xv[j].z + xv[j].w;
    }
    if (PF && row + nr < M) fetch(row + nr);
    if (x_copy) {
#pragma unroll
      for (int j = 0; j < V; ++j) st4(x_copy + row * D + t * 4 + j * TPR * 4, xv[j]);
    }
    float mean = 0.f;
    if (!RMS) mean = row_sum<TPR>(s, scratch, tog) * (1.f / D);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      float a = xv[j].x - mean, c = xv[j].y - mean, d = xv[j].z - mean, e = xv[j].w - mean;
      ss += a * a + c * c + d * d + e * e;
    }
    const float rstd = rsqrtf(row_sum<TPR>(ss, scratch, tog) * (1.f / D) + eps);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      float o[4] = {(xv[j].x - mean) * rstd, (xv[j].y - mean) * rstd, (xv[j].z - mean) * rstd,
                    (xv[j].w - mean) * rstd};
#pragma unroll
      for (int u = 0; u < 4; ++u) o[u] = RMS ? o[u] * gv[j][u] : o[u] * gv[j][u] + bv[j][u];
      st_v4(y + row * D + t * 4 + j * TPR * 4, o);
    }
    if (t == 0) {
      if (!RMS) mean_out[row] = mean;
      rstd_out[row] = rstd;
    }
  }
}

// Backward. dy bf16 [M,D]; dx fp32 accumulated in place (dx += ...), with a
// bf16 copy of the updated dx (the next GEMM operand) when dx_bf16 != null.
// dg/db partial sums per block into part[blockIdx][3][D] (db only for LN).
// Each row group (TPR threads) owns an S-stage shared-memory ring: one thread
// bulk-copies (cp.async.bulk, mbarrier-tracked) the x, dx and dy rows of the
// group's row S iterations ahead, so every SM keeps ~S x rows x 10 D bytes of
// HBM reads in flight while the group reduces and writes the current row.
template <int D, int TPR, bool RMS, typename T>
struct NormBwd {
  static constexpr int kGroups = kRowThreads / TPR;  // rows processed concurrently by the block
  static constexpr int kStage = D * 8 + D * (int)sizeof(T);  // x fp32, dx fp32, dy
  // ring stages per group: 3 while two blocks per SM still fit, else 2
  static constexpr int S = 2 * kGroups * 3 * kStage <= 200 * 1024 ? 3 : 2;
  static constexpr int kSmem = kGroups * S * kStage;
  static constexpr int kChunk = D < 1024 ? D : 1024;  // columns reduced per smem pass (reuses the ring)
  static_assert(kGroups * kChunk * 4 <= kSmem, "reduction scratch must fit in the ring");
};
template <int D, int TPR, bool RMS, typename T = __nv_bfloat16>
__global__ void __launch_bounds__(kRowThreads) norm_bwd_kernel(
    const float* __restrict__ x, const T* __restrict__ dy, const T* __restrict__ g,
    const float* __restrict__ mean_in, const float* __restrict__ rstd_in, float* __restrict__ dx,
    T* __restrict__ dx_bf16, float* __restrict__ part, int64_t M, int want_dxsum) {
  using K = NormBwd<D, TPR, RMS, T>;
  constexpr int V = D / (TPR * 4);
  constexpr int kGroups = K::kGroups, S = K::S, kChunk = K::kChunk;
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ __align__(8) uint64_t full[kGroups][S];
  __shared__ float scratch[32];
  int tog = 0;
  const int t = threadIdx.x % TPR, grp = threadIdx.x / TPR;
  const int64_t r0 = (int64_t)blockIdx.x * kGroups + grp;
  const int64_t nr = (int64_t)gridDim.x * kGroups;
  uint8_t* const mine = ring + grp * S * K::kStage;
  if (t < S) sm100::mbar_init(&full[grp][t], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  auto issue = [&](int64_t row, int s) {
    uint8_t* b = mine + s * K::kStage;
    sm100::mbar_arrive_expect_tx(&full[grp][s], K::kStage);
    sm100::bulk_load_1d(b, x + row * D, D * 4, &full[grp][s]);
    sm100::bulk_load_1d(b + D * 4, dx + row * D, D * 4, &full[grp][s]);
    sm100::bulk_load_1d(b + D * 8, dy + row * D, D * sizeof(T), &full[grp][s]);
  };
  auto group_sync = [&]() {
    if constexpr (TPR == 32) __syncwarp();
    else if constexpr (TPR == kRowThreads) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "n"(TPR) : "memory");
  };
  if (t == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s)
      if (r0 + s * nr < M) issue(r0 + s * nr, s);
  }
  float gv[V][4], dg[V][4], db[V][4], ds[V][4];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    ld_v4(g + t * 4 + j * TPR * 4, gv[j]);
#pragma unroll
    for (int u = 0; u < 4; ++u) { dg[j][u] = 0.f; db[j][u] = 0.f; ds[j][u] = 0.f; }
  }
  // row statistics one row ahead, so their load latency overlaps the current row
  float mean_n = 0.f, rstd_n = 0.f;
  if (r0 < M) { mean_n = RMS ? 0.f : mean_in[r0]; rstd_n = rstd_in[r0]; }
  int it = 0;
  // the loop bound is uniform across the block when TPR spans the block (block_sum syncs)
  for (int64_t row = r0; row < M; row += nr, ++it) {
    const float mean = mean_n, rstd = rstd_n;
    if (row + nr < M) { mean_n = RMS ? 0.f : mean_in[row + nr]; rstd_n = rstd_in[row + nr]; }
    const int s = it % S;
    sm100::mbar_wait(&full[grp][s], (it / S) & 1);
    const uint8_t* b = mine + s * K::kStage;
    const float* xs = reinterpret_cast<const float*>(b);
    const float* dxs = reinterpret_cast<const float*>(b + D * 4);
    const T* dys = reinterpret_cast<const T*>(b + D * 8);
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const float4 xv = ld4(xs + t * 4 + j * TPR * 4);
      float d4[4];
      ld_v4(dys + t * 4 + j * TPR * 4, d4);
      const float xq[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float dyg = d4[u] * gv[j][u];
        s1 += dyg;
        s2 += dyg * (xq[u] - mean) * rstd;
      }
    }
    s2 = row_sum<TPR>(s2, scratch, tog) * (1.f / D);
    if (!RMS) s1 = row_sum<TPR>(s1, scratch, tog) * (1.f / D);
    else s1 = 0.f;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int c = t * 4 + j * TPR * 4;
      const float4 xv = ld4(xs + c);
      const float4 o = ld4(dxs + c);
      float d4[4];
      ld_v4(dys + c, d4);
      const float xq[4] = {xv.x, xv.y, xv.z, xv.w};
      float os[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float xh = (xq[u] - mean) * rstd;
        os[u] += rstd * (d4[u] * gv[j][u] - s1 - xh * s2);
        dg[j][u] += d4[u] * xh;
        db[j][u] += d4[u];
        ds[j][u] += os[u];
      }
      st4(dx + row * D + c, make_float4(os[0], os[1], os[2], os[3]));
      if (dx_bf16) st_v4(dx_bf16 + row * D + c, os);
    }
    group_sync();  // every thread of the group is done reading stage s
    if (t == 0 && row + S * nr < M) issue(row + S * nr, s);
  }
  // block-level reduction of dg, db, sum(dx) over the row groups -> part[block][pass]
  float(*red)[kChunk] = reinterpret_cast<float(*)[kChunk]>(ring);
  for (int pass = 0; pass < 3; ++pass) {
    if ((pass == 1 && RMS) || (pass == 2 && !want_dxsum)) continue;
    for (int c0 = 0; c0 < D; c0 += kChunk) {
      __syncthreads();
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int col = t * 4 + j * TPR * 4;
        if (col >= c0 && col < c0 + kChunk) {
#pragma unroll
          for (int u = 0; u < 4; ++u) red[grp][col - c0 + u] = pass == 0 ? dg[j][u] : pass == 1 ? db[j][u] : ds[j][u];
        }
      }
      __syncthreads();
      for (int c = threadIdx.x; c < kChunk && c0 + c < D; c += blockDim.x) {
        float acc = 0.f;
#pragma unroll
        for (int w = 0; w < kGroups; ++w) acc += red[w][c];
        part[((int64_t)blockIdx.x * 3 + pass) * D + c0 + c] = acc;
      }
    }
  }
}

// out[c] += sum_b part[b][which][c]  (deterministic second stage): block =
// 32 columns x 32 row groups (enough independent loads in flight to hide L2
// latency), fixed summation order.
__global__ void __launch_bounds__(1024) reduce_parts_kernel(const float* __restrict__ part, int nblocks, int D,
                                                            float* __restrict__ out0, float* __restrict__ out1,
                                                            float* __restrict__ out2) {
  __shared__ float red[32][33];
  const int which = blockIdx.y;
  float* out = which == 0 ? out0 : which == 1 ? out1 : out2;
  if (out == nullptr) return;
  const int c = blockIdx.x * 32 + (threadIdx.x & 31), rg = threadIdx.x >> 5;
  float acc = 0.f;
  if (c < D) {
#pragma unroll 4
    for (int b = rg; b < nblocks; b += 32) acc += part[((int64_t)b * 3 + which) * D + c];
  }
  red[rg][threadIdx.x & 31] = acc;
  __syncthreads();
  if (rg == 0 && c < D) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 32; ++k) s += red[k][threadIdx.x & 31];
    out[c] += s;
  }
}

// ------------------------------------------------------------------ column sums
// out[c] += sum over rows of x[r][c] (bf16 or fp32 x), one launch. Block
// (strip, part) sums rows [part * rows_per, ...) of a 32-vector column strip
// into part[part][c]; the last block of each strip to finish (per-strip arrival
// counter) adds the strip's partials in part order -- deterministic -- and
// re-arms the counter. 8 warps stride the rows; each lane owns one 16-byte
// column vector, so a warp reads 512 contiguous bytes per row. Requires N, ld
// multiples of the vector.
template <typename T>
__global__ void __launch_bounds__(256) colsum_kernel(const T* __restrict__ x, int64_t M, int N, int64_t ld,
                                                     int rows_per, float* __restrict__ part,
                                                     float* __restrict__ out, unsigned* __restrict__ arrivals) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int COLS = 32 * VEC;
  __shared__ float red[8][COLS];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * COLS + lane * VEC;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per;
  const int64_t r1 = min(M, r0 + rows_per);
  float acc[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) acc[i] = 0.f;
  if (c < N) {
    // four rows' 16-byte loads issued back to back before they are summed: the
    // loop is latency-bound otherwise (one load in flight per lane)
    constexpr int U = 16;
    int64_t r = r0 + w;
    for (; r + 8 * (U - 1) < r1; r += 8 * U) {
      uint4 q[U];
#pragma unroll
      for (int u = 0; u < U; ++u) q[u] = __ldcs(reinterpret_cast<const uint4*>(x + (r + 8 * u) * ld + c));
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if constexpr (sizeof(T) == 2) {
          float f[8];
          unpack8(*reinterpret_cast<const bf16x8*>(&q[u]), f);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] += f[i];
        } else {
          acc[0] += __uint_as_float(q[u].x); acc[1] += __uint_as_float(q[u].y);
          acc[2] += __uint_as_float(q[u].z); acc[3] += __uint_as_float(q[u].w);
        }
      }
    }
    for (; r < r1; r += 8) {
      const uint4 q = __ldcs(reinterpret_cast<const uint4*>(x + r * ld + c));
      if constexpr (sizeof(T) == 2) {
        float f[8];
        unpack8(*reinterpret_cast<const bf16x8*>(&q), f);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += f[i];
      } else {
        acc[0] += __uint_as_float(q.x); acc[1] += __uint_as_float(q.y);
        acc[2] += __uint_as_float(q.z); acc[3] += __uint_as_float(q.w);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < VEC; ++i) red[w][lane * VEC + i] = acc[i];
  __syncthreads();
  for (int k = threadIdx.x; k < COLS; k += blockDim.x) {
    const int cc = blockIdx.x * COLS + k;
    if (cc < N) {
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) s += red[j][k];
      part[(int64_t)blockIdx.y * N + cc] = s;
    }
  }
  __threadfence();  // publish this block's partials before counting its arrival
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&arrivals[blockIdx.x], 1u) == gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // COLS columns x 8 part groups (fixed order within and across the groups)
  const int nparts = gridDim.y;
  constexpr int PG = 256 / COLS;  // part groups: 1 (bf16) or 2 (fp32)
  const int k = threadIdx.x % COLS, g = threadIdx.x / COLS;
  const int cc = blockIdx.x * COLS + k;
  float s = 0.f;
  if (cc < N) {
    // 16 partials' loads in flight per batch (a serial chain of L2 round trips otherwise)
    int q = g;
    for (; q + 15 * PG < nparts; q += 16 * PG) {
      float v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = __ldcg(part + (int64_t)(q + u * PG) * N + cc);
#pragma unroll
      for (int u = 0; u < 16; ++u) s += v[u];
    }
    for (; q < nparts; q += PG) s += __ldcg(part + (int64_t)q * N + cc);
  }
  if constexpr (PG > 1) {
    red[g][k] = s;
    __syncthreads();
    if (g == 0) {
#pragma unroll
      for (int j = 1; j < PG; ++j) s += red[j][k];
    }
  }
  if (g == 0 && cc < N) out[cc] += s;
  if (threadIdx.x == 0) arrivals[blockIdx.x] = 0u;  // re-armed for the next launch using this slot
}

// ------------------------------------------------------------------ embedding
// x[m, :] = wte[tok[m], :] (+ wpe[m % T, :]), fp32 out.
template <typename E>
__global__ void embed_fwd_kernel(const int64_t* __restrict__ tok, const E* __restrict__ wte,
                                 const E* __restrict__ wpe, float* __restrict__ x, int64_t M,
                                 int T, int D) {
  const int vec = D / 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * vec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / vec;
    const int c = (int)(i - m * vec) * 4;
    float f[4];
    ld_v4(wte + tok[m] * D + c, f);
    if (wpe) {
      float p[4];
      ld_v4(wpe + (int64_t)(m % T) * D + c, p);
      f[0] += p[0]; f[1] += p[1]; f[2] += p[2]; f[3] += p[3];
    }
    st4(x + m * D + c, make_float4(f[0], f[1], f[2], f[3]));
  }
}
// dwte[tok[m]] += dx[m]  (fp32 atomics: rows collide only on repeated tokens)
__global__ void embed_bwd_tok_kernel(const int64_t* __restrict__ tok, const float* __restrict__ dx,
                                     float* __restrict__ dwte, int64_t M, int D) {
  const int vec = D / 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * vec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / vec;
    const int c = (int)(i - m * vec) * 4;
    float4 v = ld4(dx + m * D + c);
    float* o = dwte + tok[m] * D + c;
    atomicAdd(reinterpret_cast<float4*>(o), v);
  }
}
// dwpe[t] += sum_b dx[b*T + t]  (deterministic)
__global__ void embed_bwd_pos_kernel(const float* __restrict__ dx, float* __restrict__ dwpe, int B, int T, int D) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)T * D;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / D;
    const int c = (int)(i - t * D);
    float acc = 0.f;
    for (int b = 0; b < B; ++b) acc += dx[((int64_t)b * T + t) * D + c];
    dwpe[i] += acc;
  }
}

// ------------------------------------------------------------------ RoPE
// In place on the q and k heads of a [M, ld] bf16 buffer, rotate-half pairing
// (i, i + dh/2) as in Llama: (a, b) -> (a cos - b sin, b cos + a sin).
// inverse=1 applies the transpose rotation (backward).
template <typename E>
__global__ void rope_kernel(E* __restrict__ qkv, int64_t M, int T, int64_t ld, int nheads,
                            int dh, const float* __restrict__ cos_t, const float* __restrict__ sin_t,
                            int inverse) {
  // one thread = 8 consecutive rotation pairs of one head of one row (16-byte vectors)
  const int half = dh / 2;
  const int vph = half / 8;  // vectors per head
  const int64_t per_row = (int64_t)nheads * vph;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * per_row;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / per_row;
    const int r = (int)(i - m * per_row);
    const int h = r / vph, j0 = (r - h * vph) * 8;
    const int t = (int)(m % T);
    E* p = qkv + m * ld + (int64_t)h * dh + j0;
    float a[8], b[8], c[8], sn[8];
    ld_v8(p, a);
    ld_v8(p + half, b);
    const float4* cp = reinterpret_cast<const float4*>(cos_t + (int64_t)t * half + j0);
    const float4* sp = reinterpret_cast<const float4*>(sin_t + (int64_t)t * half + j0);
    float4 c0 = cp[0], c1 = cp[1], s0 = sp[0], s1 = sp[1];
    c[0] = c0.x; c[1] = c0.y; c[2] = c0.z; c[3] = c0.w; c[4] = c1.x; c[5] = c1.y; c[6] = c1.z; c[7] = c1.w;
    sn[0] = s0.x; sn[1] = s0.y; sn[2] = s0.z; sn[3] = s0.w; sn[4] = s1.x; sn[5] = s1.y; sn[6] = s1.z; sn[7] = s1.w;
    float oa[8], ob[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float s_ = inverse ? -sn[k] : sn[k];
      oa[k] = a[k] * c[k] - b[k] * s_;
      ob[k] = b[k] * c[k] + a[k] * s_;
    }
    st_v8(p, oa);
    st_v8(p + half, ob);
  }
}

// ------------------------------------------------------------------ SwiGLU
// sigmoid: fast MUFU exp / reciprocal for bf16 activations (the kernel is then
// HBM-bound instead of bound by IEEE expf + division), exact libm forms in fp32 mode.
template <typename T>
__device__ __forceinline__ float sigmoid(float x) {
  if constexpr (sizeof(T) == 4) return 1.f / (1.f + expf(-x));
  else return __frcp_rn(1.f + __expf(-x));
}
// gu [M, 2F] (gate | up), h [M, F] = silu(gate) * up
template <typename T>
__global__ void swiglu_fwd_kernel(const T* __restrict__ gu, T* __restrict__ h,
                                  int64_t M, int F) {
  const int vec = F / 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * vec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / vec;
    const int c = (int)(i - m * vec) * 8;
    float g[8], u[8], o[8];
    ld_v8(gu + m * 2 * F + c, g);
    ld_v8(gu + m * 2 * F + F + c, u);
#pragma unroll
    for (int t = 0; t < 8; ++t) o[t] = g[t] * sigmoid<T>(g[t]) * u[t];
    st_v8(h + m * F + c, o);
  }
}
// dgu = [dgate | dup] from dh and the saved gu
template <typename T>
__global__ void swiglu_bwd_kernel(const T* __restrict__ gu, const T* __restrict__ dh,
                                  T* __restrict__ dgu, int64_t M, int F) {
  const int vec = F / 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * vec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / vec;
    const int c = (int)(i - m * vec) * 8;
    float g[8], u[8], d[8], dg[8], du[8];
    ld_v8(gu + m * 2 * F + c, g);
    ld_v8(gu + m * 2 * F + F + c, u);
    ld_v8(dh + m * F + c, d);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const float sg = sigmoid<T>(g[t]);
      const float silu = g[t] * sg;
      du[t] = d[t] * silu;
      dg[t] = d[t] * u[t] * sg * (1.f + g[t] * (1.f - sg));
    }
    st_v8(dgu + m * 2 * F + c, dg);
    st_v8(dgu + m * 2 * F + F + c, du);
  }
}

// ------------------------------------------------------------------ cross-entropy
// One block per row of bf16 logits [M, ld] (first V columns valid). Writes
// loss[m] = logsumexp - logit[target] (fp32) and, in place over the logits,
// dlogits = (softmax - onehot) * gscale (columns >= V zeroed).
// The first pass keeps U row vectors in flight per thread before their exponentials (GPT-2
// logits: 659 / 665 / 648 / 720 us for U = 1 / 2 / 4 / 8, profiles/r1_xent_smem_ab.jsonl).
template <typename T, int U = 4>
__global__ void __launch_bounds__(512) xent_kernel(T* __restrict__ logits, int64_t ld, int V,
                                                   const int64_t* __restrict__ target, float* __restrict__ loss,
                                                   float gscale, int64_t M, int write_grad) {
  // log2 units throughout (y = x log2 e): one FFMA + one ex2 per element; the target
  // column is corrected once per row instead of a compare-select per element
  constexpr float L2E = 1.4426950408889634f;
  __shared__ float scratch[32];
  const int nvec = V / 8;  // full 8-wide vectors
  const int64_t m = blockIdx.x;
  T* row = logits + m * ld;
  // one pass: per-thread online (max, sum of 2^(y - max)), then a block-wide merge
  float mx = -INFINITY, se = 0.f;
  auto absorb = [&](const float* f) {
    const float lm = fmax3(fmax3(f[0], f[1], f[2]), fmax3(f[3], f[4], f[5]), fmaxf(f[6], f[7]));
    const float mn = fmaxf(mx, lm * L2E);
    float acc = 0.f;
#pragma unroll
    for (int t = 0; t < 8; ++t) acc += ex2f(fmaf(f[t], L2E, -mn));
    se = se * ex2f(mx - mn) + acc;
    mx = mn;
  };
  int i0 = threadIdx.x;
  if (U > 1) {  // U row vectors in flight per thread before their exponentials
    for (; i0 + (U - 1) * (int)blockDim.x < nvec; i0 += U * blockDim.x) {
      float f[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u) ld_v8(row + (int64_t)(i0 + u * blockDim.x) * 8, f[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) absorb(f[u]);
    }
  }
  for (int i = i0; i < nvec; i += blockDim.x) {
    float f[8];
    ld_v8(row + i * 8, f);
    absorb(f);
  }
  for (int c = nvec * 8 + threadIdx.x; c < V; c += blockDim.x) {
    const float y = to_f(row[c]) * L2E;
    const float mn = fmaxf(mx, y);
    se = se * ex2f(mx - mn) + ex2f(y - mn);
    mx = mn;
  }
  const float bmx = block_max(mx, scratch);
  se = (mx == -INFINITY) ? 0.f : se * ex2f(mx - bmx);
  mx = bmx;
  se = block_sum(se, scratch);
  const float lse = (mx + __log2f(se)) * (1.f / L2E);
  const int64_t tgt = target[m];
  const float xt = to_f(row[tgt]);
  __syncthreads();
  if (threadIdx.x == 0) loss[m] = lse - xt;
  if (!write_grad) return;
  const float inv = gscale / se;  // softmax * gscale = 2^(y - max) * gscale / sum
  const int j0 = threadIdx.x;
  for (int i = j0; i < nvec; i += blockDim.x) {
    float f[8];
    ld_v8_cs(row + i * 8, f);  // last read of the row (pass 1 left it in L2)
#pragma unroll
    for (int t = 0; t < 8; ++t) f[t] = ex2f(fmaf(f[t], L2E, -mx)) * inv;
    if ((uint64_t)(tgt - (int64_t)i * 8) < 8) f[tgt - (int64_t)i * 8] -= gscale;
    st_v8_cs(row + i * 8, f);  // written once: keep other rows' pass-2 reads in L2
  }
  for (int c = nvec * 8 + threadIdx.x; c < ld; c += blockDim.x) {
    float g = 0.f;
    if (c < V) g = ex2f(fmaf(to_f(row[c]), L2E, -mx)) * inv - (c == tgt ? gscale : 0.f);
    from_f(row[c], g);
  }
}


// ------------------------------------------------------------------ reductions
// Deterministic sum of n floats (optionally of squares) into out[0] (overwrite).
__global__ void __launch_bounds__(1024) sum_kernel(const float* __restrict__ x, int64_t n, int squares,
                                                   float* __restrict__ out, float scale) {
  __shared__ float scratch[32];
  float acc = 0.f;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += squares ? x[i] * x[i] : x[i];
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) out[0] = acc * scale;
}
// Stage 1 of the gradient norm over several buffers in one launch: every block
// grid-strides over each segment in turn (four 16-byte loads in flight per
// thread), part[block] = its sum of squares over all segments (fixed order).
__global__ void __launch_bounds__(256) sumsq_multi_kernel(const uint64_t* __restrict__ ptrs,
                                                          const int64_t* __restrict__ lens, int nseg,
                                                          float* __restrict__ part) {
  __shared__ float scratch[32];
  float acc = 0.f;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  for (int sgi = 0; sgi < nseg; ++sgi) {
    const float* x = reinterpret_cast<const float*>(ptrs[sgi]);
    const int64_t n = lens[sgi], nv = n / 4;
    int64_t i = tid;
    for (; i + 3 * nth < nv; i += 4 * nth) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(reinterpret_cast<const float4*>(x) + i + u * nth);
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += v[u].x * v[u].x + v[u].y * v[u].y + v[u].z * v[u].z + v[u].w * v[u].w;
    }
    for (; i < nv; i += nth) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(x) + i);
      acc += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    for (int64_t j = nv * 4 + tid; j < n; j += nth) acc += x[j] * x[j];
  }
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}
// Stage 1 of a deterministic large sum of squares: part[block] = sum x^2.
__global__ void __launch_bounds__(256) sumsq_part_kernel(const float* __restrict__ x, int64_t n,
                                                         float* __restrict__ part) {
  __shared__ float scratch[32];
  float acc = 0.f;
  const int64_t nv = n / 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = ld4(x + i * 4);
    acc += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  for (int64_t i = nv * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc += x[i] * x[i];
  acc = block_sum(acc, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// ------------------------------------------------------------------ AdamW
// Fused over one flat shard: fp32 master p, m, v, grad g; writes the bf16
// copy of p (the next step's all-gather source). The global clip factor is
// computed on the device from the all-reduced grad-norm^2 (no host sync):
//   clip = min(1, max_norm / (sqrt(gn2) + 1e-6)).
// Weight decay is applied where wd_mask (per-element u8, or null = all) is set.
template <typename T>
__global__ void __launch_bounds__(256) adamw_kernel(
    float* __restrict__ p, float* __restrict__ m, float* __restrict__ v, const float* __restrict__ g,
    T* __restrict__ p_bf16, const uint8_t* __restrict__ wd_mask, int64_t n,
    const float* __restrict__ gn2, float max_norm, float lr, float beta1, float beta2, float eps,
    float wd, float bc1, float bc2) {
  float clip = 1.f;
  if (gn2 && max_norm > 0.f) clip = fminf(1.f, max_norm / (sqrtf(gn2[0]) + 1e-6f));
  const int64_t nv = n / 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    float4 pp = ld4(p + 4 * i), mm = ld4(m + 4 * i), vv = ld4(v + 4 * i), gg = ld4(g + 4 * i);
    float P[4] = {pp.x, pp.y, pp.z, pp.w}, Mv[4] = {mm.x, mm.y, mm.z, mm.w};
    float Vv[4] = {vv.x, vv.y, vv.z, vv.w}, G[4] = {gg.x, gg.y, gg.z, gg.w};
    uint32_t mask = wd_mask ? *reinterpret_cast<const uint32_t*>(wd_mask + 4 * i) : 0x01010101u;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float gt = G[t] * clip;
      Mv[t] = beta1 * Mv[t] + (1.f - beta1) * gt;
      Vv[t] = beta2 * Vv[t] + (1.f - beta2) * gt * gt;
      const float dec = ((mask >> (8 * t)) & 0xff) ? wd : 0.f;
      P[t] = P[t] - lr * dec * P[t];
      P[t] = P[t] - lr * (Mv[t] / bc1) / (sqrtf(Vv[t] / bc2) + eps);
    }
    st4(p + 4 * i, make_float4(P[0], P[1], P[2], P[3]));
    st4(m + 4 * i, make_float4(Mv[0], Mv[1], Mv[2], Mv[3]));
    st4(v + 4 * i, make_float4(Vv[0], Vv[1], Vv[2], Vv[3]));
    if (p_bf16) st_v4(p_bf16 + 4 * i, P);
  }
  for (int64_t i = nv * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gt = g[i] * clip;
    const float mi = beta1 * m[i] + (1.f - beta1) * gt;
    const float vi = beta2 * v[i] + (1.f - beta2) * gt * gt;
    float pi = p[i];
    const float dec = (wd_mask ? wd_mask[i] : 1) ? wd : 0.f;
    pi = pi - lr * dec * pi;
    pi = pi - lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
    p[i] = pi; m[i] = mi; v[i] = vi;
    if (p_bf16) from_f(p_bf16[i], pi);
  }
}

// ------------------------------------------------------------------ casts / scale
__global__ void f32_to_bf16_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, int64_t n, float scale) {
  const int64_t nv = n / 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = ld4(x + 4 * i);
    float f[4] = {v.x * scale, v.y * scale, v.z * scale, v.w * scale};
    st_bf4(y + 4 * i, f);
  }
  for (int64_t i = nv * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = f2bf(x[i] * scale);
}
__global__ void scale_f32_kernel(float* __restrict__ x, int64_t n, float scale) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= scale;
}

static unsigned flat_grid(int64_t n, int per_thread = 4) {
  int64_t blocks = (n / per_thread + 255) / 256;
  if (blocks < 1) blocks = 1;
  int64_t cap = (int64_t)kNumSMs * 16;
  return (unsigned)(blocks < cap ? blocks : cap);
}

template <bool RMS, typename T = __nv_bfloat16>
static int norm_fwd(const float* x, const void* g, const void* b, void* y, float* mean, float* rstd,
                    float* x_copy, int64_t M, int D, float eps, cudaStream_t st, const void* res = nullptr) {
  auto go = [&](auto kern, int tpr) {
    int64_t blocks = (M * tpr + kRowThreads - 1) / kRowThreads;
    const int64_t cap = (int64_t)kNumSMs * 8;
    kern<<<(unsigned)(blocks < cap ? blocks : cap), kRowThreads, 0, st>>>(
        x, (const T*)g, (const T*)b, (T*)y, mean, rstd, x_copy, M, eps, (const T*)res);
    return check_launch("norm_fwd");
  };
  switch (D) {
    case 128: return go(norm_fwd_kernel<128, 32, RMS, T>, 32);
    case 256: return go(norm_fwd_kernel<256, 32, RMS, T>, 32);
    case 512: return go(norm_fwd_kernel<512, 32, RMS, T>, 32);
    case 768: return go(norm_fwd_kernel<768, 32, RMS, T>, 32);
    case 1024: return go(norm_fwd_kernel<1024, 32, RMS, T>, 32);
    case 2048: return go(norm_fwd_kernel<2048, 256, RMS, T>, 256);
    case 4096: return go(norm_fwd_kernel<4096, 256, RMS, T>, 256);
  }
  set_error("norm: unsupported hidden size %d", D);
  return B2S_EUNSUPPORTED;
}

constexpr int kNormBwdMaxBlocks = kNumSMs * 4;

// Per-device pool of zeroed colsum arrival counters (kColsumStrips per slot);
// launches rotate through the slots so column sums in flight on different
// streams never share one. Each launch leaves its counters at zero.
constexpr int kColsumStrips = 1024, kColsumSlots = 64;
static unsigned* colsum_slot() {
  static unsigned* pool[64] = {};
  static int next[64] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (!pool[dev]) {
    const size_t bytes = (size_t)kColsumSlots * kColsumStrips * sizeof(unsigned);
    if (cudaMalloc(&pool[dev], bytes) != cudaSuccess) return nullptr;
    cudaMemset(pool[dev], 0, bytes);
    cudaDeviceSynchronize();
  }
  unsigned* p = pool[dev] + (size_t)kColsumStrips * next[dev];
  next[dev] = (next[dev] + 1) % kColsumSlots;
  return p;
}

template <bool RMS, typename T = __nv_bfloat16>
static int norm_bwd(const float* x, const void* dy, const void* g, const float* mean, const float* rstd,
                    float* dx, void* dx_bf16, float* dg, float* db, float* dxsum, float* work, int64_t M, int D,
                    cudaStream_t st) {
  B2S_REQUIRE((((uintptr_t)x | (uintptr_t)dy | (uintptr_t)dx) & 15) == 0, B2S_EUNSUPPORTED,
              "norm_bwd: x, dy and dx must be 16-byte aligned");
  unsigned grid = 0;
  // persistent grid: as many blocks as are co-resident (the ring is the smem bound)
  auto go = [&](auto kern, auto traits) {
    using K = decltype(traits);
    static int occ = 0;  // per instantiation
    if (occ == 0) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, K::kSmem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kRowThreads, K::kSmem);
      if (occ < 1) occ = 1;
    }
    const int64_t blocks = (M + K::kGroups - 1) / K::kGroups;
    int64_t cap = (int64_t)kNumSMs * occ;
    if (cap > kNormBwdMaxBlocks) cap = kNormBwdMaxBlocks;
    grid = (unsigned)(blocks < cap ? blocks : cap);  // partial buffer: grid * 3 * D floats
    if (grid == 0) grid = 1;
    kern<<<grid, kRowThreads, K::kSmem, st>>>(x, (const T*)dy, (const T*)g, mean, rstd, dx, (T*)dx_bf16, work, M,
                                              dxsum != nullptr);
    return check_launch("norm_bwd");
  };
#define B2S_NB(D_, TPR_) go(norm_bwd_kernel<D_, TPR_, RMS, T>, NormBwd<D_, TPR_, RMS, T>{})
  int rc;
  switch (D) {
    case 128: rc = B2S_NB(128, 32); break;
    case 256: rc = B2S_NB(256, 32); break;
    case 512: rc = B2S_NB(512, 32); break;
    case 768: rc = B2S_NB(768, 64); break;
    case 1024: rc = B2S_NB(1024, 32); break;
    case 2048: rc = B2S_NB(2048, 128); break;  // 2 rows in flight per block
    case 4096: rc = B2S_NB(4096, 256); break;
    default:
      set_error("norm_bwd: unsupported hidden size %d", D);
      return B2S_EUNSUPPORTED;
  }
#undef B2S_NB
  if (rc) return rc;
  if (!dg && !(db && !RMS) && !dxsum) return B2S_OK;
  reduce_parts_kernel<<<dim3((D + 31) / 32, 3), 1024, 0, st>>>(work, grid, D, dg, RMS ? nullptr : db, dxsum);
  return check_launch("norm_bwd_reduce");
}

}  // namespace ew
}  // namespace b2s

using namespace b2s;

namespace {
// Host launchers shared by the bf16 and fp32 entry points (T = activation type).
template <typename T>
int embedding_fwd(const int64_t* d_tok, const void* d_wte, const void* d_wpe, float* d_x, int64_t M, int T_,
                  int D, cudaStream_t st) {
  B2S_REQUIRE(D % 4 == 0, B2S_EUNSUPPORTED, "embedding: D %% 4 != 0");
  ew::embed_fwd_kernel<T><<<ew::flat_grid(M * D), 256, 0, st>>>(d_tok, (const T*)d_wte, (const T*)d_wpe, d_x, M,
                                                                 T_, D);
  return check_launch("embedding_fwd");
}
template <typename T>
int rope(void* d_qkv, int64_t M, int T_, int64_t ld, int nheads, int dh, const float* d_cos, const float* d_sin,
         int inverse, cudaStream_t st) {
  B2S_REQUIRE(dh % 16 == 0 && ld % 8 == 0 && ((uintptr_t)d_qkv % 16) == 0, B2S_EUNSUPPORTED,
              "rope: head dim must be a multiple of 16 and rows 16-byte aligned");
  ew::rope_kernel<T><<<ew::flat_grid(M * nheads * dh / 16, 1), 256, 0, st>>>((T*)d_qkv, M, T_, ld, nheads, dh,
                                                                           d_cos, d_sin, inverse);
  return check_launch("rope");
}
template <typename T>
int swiglu_fwd(const void* d_gu, void* d_h, int64_t M, int F, cudaStream_t st) {
  B2S_REQUIRE(F % 8 == 0, B2S_EUNSUPPORTED, "swiglu: F %% 8 != 0");
  ew::swiglu_fwd_kernel<T><<<ew::flat_grid(M * F, 8), 256, 0, st>>>((const T*)d_gu, (T*)d_h, M, F);
  return check_launch("swiglu_fwd");
}
template <typename T>
int swiglu_bwd(const void* d_gu, const void* d_dh, void* d_dgu, int64_t M, int F, cudaStream_t st) {
  B2S_REQUIRE(F % 8 == 0, B2S_EUNSUPPORTED, "swiglu: F %% 8 != 0");
  ew::swiglu_bwd_kernel<T><<<ew::flat_grid(M * F, 8), 256, 0, st>>>((const T*)d_gu, (const T*)d_dh, (T*)d_dgu, M,
                                                                    F);
  return check_launch("swiglu_bwd");
}
template <typename T>
int cross_entropy(void* d_logits, int64_t ld, int V, const int64_t* d_target, float* d_loss_rows,
                  float grad_scale, int64_t M, int write_grad, cudaStream_t st) {
  B2S_REQUIRE(ld % 8 == 0 && V <= ld, B2S_EUNSUPPORTED, "cross_entropy: ld must be a multiple of 8 >= V");
  auto kern = ew::xent_kernel<T, 4>;
  kern<<<(unsigned)M, 512, 0, st>>>((T*)d_logits, ld, V, d_target, d_loss_rows, grad_scale, M, write_grad);
  return check_launch("cross_entropy");
}
template <typename T>
int adamw(float* d_p, float* d_m, float* d_v, const float* d_g, void* d_p_out, const uint8_t* d_wd_mask, int64_t n,
          const float* d_gn2, float max_norm, float lr, float beta1, float beta2, float eps, float wd, int step,
          cudaStream_t st) {
  B2S_REQUIRE(((uintptr_t)d_p | (uintptr_t)d_m | (uintptr_t)d_v | (uintptr_t)d_g) % 16 == 0 &&
                  ((uintptr_t)d_p_out % (4 * sizeof(T))) == 0 && (!d_wd_mask || ((uintptr_t)d_wd_mask % 4) == 0),
              B2S_EUNSUPPORTED, "adamw: misaligned shard");
  const float bc1 = 1.f - powf(beta1, (float)step), bc2 = 1.f - powf(beta2, (float)step);
  ew::adamw_kernel<T><<<ew::flat_grid(n), 256, 0, st>>>(d_p, d_m, d_v, d_g, (T*)d_p_out, d_wd_mask, n, d_gn2,
                                                        max_norm, lr, beta1, beta2, eps, wd, bc1, bc2);
  return check_launch("adamw");
}
}  // namespace

#define B2S_ST(s) ((cudaStream_t)(s))

extern "C" {

int b2s_layernorm_fwd(const float* d_x, const void* d_g, const void* d_b, void* d_y, float* d_mean,
                      float* d_rstd, float* d_x_copy, int64_t M, int D, float eps, b2s_stream_t stream) {
  return ew::norm_fwd<false>(d_x, d_g, d_b, d_y, d_mean, d_rstd, d_x_copy, M, D, eps, B2S_ST(stream));
}
int b2s_rmsnorm_fwd(const float* d_x, const void* d_g, void* d_y, float* d_rstd, float* d_x_copy,
                    int64_t M, int D, float eps, b2s_stream_t stream) {
  return ew::norm_fwd<true>(d_x, d_g, nullptr, d_y, nullptr, d_rstd, d_x_copy, M, D, eps, B2S_ST(stream));
}
int b2s_layernorm_bwd(const float* d_x, const void* d_dy, const void* d_g, const float* d_mean,
                      const float* d_rstd, float* d_dx, void* d_dx_bf16, float* d_dg, float* d_db,
                      float* d_dxsum, float* d_work, int64_t M, int D, b2s_stream_t stream) {
  return ew::norm_bwd<false>(d_x, d_dy, d_g, d_mean, d_rstd, d_dx, d_dx_bf16, d_dg, d_db, d_dxsum, d_work, M, D,
                             B2S_ST(stream));
}
int b2s_rmsnorm_bwd(const float* d_x, const void* d_dy, const void* d_g, const float* d_rstd, float* d_dx,
                    void* d_dx_bf16, float* d_dg, float* d_dxsum, float* d_work, int64_t M, int D,
                    b2s_stream_t stream) {
  return ew::norm_bwd<true>(d_x, d_dy, d_g, nullptr, d_rstd, d_dx, d_dx_bf16, d_dg, nullptr, d_dxsum, d_work, M,
                            D, B2S_ST(stream));
}
int b2s_layernorm_fwd_f32(const float* d_x, const float* d_g, const float* d_b, float* d_y, float* d_mean,
                          float* d_rstd, float* d_x_copy, int64_t M, int D, float eps, b2s_stream_t stream) {
  return ew::norm_fwd<false, float>(d_x, d_g, d_b, d_y, d_mean, d_rstd, d_x_copy, M, D, eps, B2S_ST(stream));
}
int b2s_rmsnorm_fwd_f32(const float* d_x, const float* d_g, float* d_y, float* d_rstd, float* d_x_copy,
                        int64_t M, int D, float eps, b2s_stream_t stream) {
  return ew::norm_fwd<true, float>(d_x, d_g, nullptr, d_y, nullptr, d_rstd, d_x_copy, M, D, eps, B2S_ST(stream));
}
int b2s_layernorm_bwd_f32(const float* d_x, const float* d_dy, const float* d_g, const float* d_mean,
                          const float* d_rstd, float* d_dx, float* d_dx_copy, float* d_dg, float* d_db,
                          float* d_dxsum, float* d_work, int64_t M, int D, b2s_stream_t stream) {
  return ew::norm_bwd<false, float>(d_x, d_dy, d_g, d_mean, d_rstd, d_dx, d_dx_copy, d_dg, d_db, d_dxsum, d_work,
                                    M, D, B2S_ST(stream));
}
int b2s_rmsnorm_bwd_f32(const float* d_x, const float* d_dy, const float* d_g, const float* d_rstd, float* d_dx,
                        float* d_dx_copy, float* d_dg, float* d_dxsum, float* d_work, int64_t M, int D,
                        b2s_stream_t stream) {
  return ew::norm_bwd<true, float>(d_x, d_dy, d_g, nullptr, d_rstd, d_dx, d_dx_copy, d_dg, nullptr, d_dxsum,
                                   d_work, M, D, B2S_ST(stream));
}
int b2s_layernorm_fwd_res(const float* d_x, const void* d_res, const void* d_g, const void* d_b, void* d_y,
                          float* d_mean, float* d_rstd, float* d_x_out, int64_t M, int D, float eps,
                          b2s_stream_t stream) {
  return ew::norm_fwd<false>(d_x, d_g, d_b, d_y, d_mean, d_rstd, d_x_out, M, D, eps, B2S_ST(stream), d_res);
}
int b2s_rmsnorm_fwd_res(const float* d_x, const void* d_res, const void* d_g, void* d_y, float* d_rstd,
                        float* d_x_out, int64_t M, int D, float eps, b2s_stream_t stream) {
  return ew::norm_fwd<true>(d_x, d_g, nullptr, d_y, nullptr, d_rstd, d_x_out, M, D, eps, B2S_ST(stream), d_res);
}
int b2s_layernorm_fwd_res_f32(const float* d_x, const float* d_res, const float* d_g, const float* d_b, float* d_y,
                              float* d_mean, float* d_rstd, float* d_x_out, int64_t M, int D, float eps,
                              b2s_stream_t stream) {
  return ew::norm_fwd<false, float>(d_x, d_g, d_b, d_y, d_mean, d_rstd, d_x_out, M, D, eps, B2S_ST(stream), d_res);
}
int b2s_rmsnorm_fwd_res_f32(const float* d_x, const float* d_res, const float* d_g, float* d_y, float* d_rstd,
                            float* d_x_out, int64_t M, int D, float eps, b2s_stream_t stream) {
  return ew::norm_fwd<true, float>(d_x, d_g, nullptr, d_y, nullptr, d_rstd, d_x_out, M, D, eps, B2S_ST(stream),
                                   d_res);
}
int64_t b2s_norm_work_floats(int D) { return (int64_t)ew::kNormBwdMaxBlocks * 3 * D; }

int b2s_colsum_accumulate(const void* d_x, int x_f32, int64_t M, int N, int64_t ld, float* d_out,
                          float* d_work, b2s_stream_t stream) {
  const int vec = x_f32 ? 4 : 8;
  B2S_REQUIRE(N % vec == 0 && ld % vec == 0 && ((uintptr_t)d_x % 16) == 0, B2S_EUNSUPPORTED,
              "colsum: N and ld must be multiples of %d and x 16-byte aligned", vec);
  cudaStream_t st = (cudaStream_t)stream;
  const int cols = 32 * vec;
  const int nblk = (N + cols - 1) / cols;
  B2S_REQUIRE(nblk <= ew::kColsumStrips, B2S_EUNSUPPORTED, "colsum: N = %d exceeds %d column strips", N,
              ew::kColsumStrips);
  unsigned* arrivals = ew::colsum_slot();
  B2S_REQUIRE(arrivals != nullptr, B2S_ECUDA, "colsum: arrival counter allocation failed");
  // about four blocks per SM (2..8 measured: 2-4 best, profiles/r1_colsum_bps_sweep.jsonl). No
  // block waits on another -- the last block of a column strip to arrive reduces the strip's
  // partials -- so co-residency is not required
  int nparts = 4 * kNumSMs / nblk;
  if (nparts > 256) nparts = 256;
  if (nparts < 1) nparts = 1;
  const int rows_per = (int)((M + nparts - 1) / nparts);
  dim3 grid(nblk, nparts);
  if (x_f32)
    ew::colsum_kernel<float><<<grid, 256, 0, st>>>((const float*)d_x, M, N, ld, rows_per, d_work, d_out, arrivals);
  else
    ew::colsum_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)d_x, M, N, ld, rows_per, d_work,
                                                           d_out, arrivals);
  return check_launch("colsum");
}
int64_t b2s_colsum_work_floats(int N) { return 256LL * N; }

int b2s_embedding_fwd(const int64_t* d_tok, const void* d_wte, const void* d_wpe, float* d_x, int64_t M,
                      int T, int D, b2s_stream_t stream) {
  return embedding_fwd<__nv_bfloat16>(d_tok, d_wte, d_wpe, d_x, M, T, D, B2S_ST(stream));
}
int b2s_embedding_fwd_f32(const int64_t* d_tok, const float* d_wte, const float* d_wpe, float* d_x, int64_t M,
                          int T, int D, b2s_stream_t stream) {
  return embedding_fwd<float>(d_tok, d_wte, d_wpe, d_x, M, T, D, B2S_ST(stream));
}
int b2s_embedding_bwd(const int64_t* d_tok, const float* d_dx, float* d_dwte, float* d_dwpe, int B, int T,
                      int D, b2s_stream_t stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t M = (int64_t)B * T;
  ew::embed_bwd_tok_kernel<<<ew::flat_grid(M * D), 256, 0, st>>>(d_tok, d_dx, d_dwte, M, D);
  if (d_dwpe) ew::embed_bwd_pos_kernel<<<ew::flat_grid((int64_t)T * D, 1), 256, 0, st>>>(d_dx, d_dwpe, B, T, D);
  return check_launch("embedding_bwd", d_dwpe ? 2 : 1);
}

int b2s_rope(void* d_qkv, int64_t M, int T, int64_t ld, int nheads, int dh, const float* d_cos,
             const float* d_sin, int inverse, b2s_stream_t stream) {
  return rope<__nv_bfloat16>(d_qkv, M, T, ld, nheads, dh, d_cos, d_sin, inverse, B2S_ST(stream));
}
int b2s_rope_f32(float* d_qkv, int64_t M, int T, int64_t ld, int nheads, int dh, const float* d_cos,
                 const float* d_sin, int inverse, b2s_stream_t stream) {
  return rope<float>(d_qkv, M, T, ld, nheads, dh, d_cos, d_sin, inverse, B2S_ST(stream));
}

int b2s_swiglu_fwd(const void* d_gu, void* d_h, int64_t M, int F, b2s_stream_t stream) {
  return swiglu_fwd<__nv_bfloat16>(d_gu, d_h, M, F, B2S_ST(stream));
}
int b2s_swiglu_bwd(const void* d_gu, const void* d_dh, void* d_dgu, int64_t M, int F, b2s_stream_t stream) {
  return swiglu_bwd<__nv_bfloat16>(d_gu, d_dh, d_dgu, M, F, B2S_ST(stream));
}
int b2s_swiglu_fwd_f32(const float* d_gu, float* d_h, int64_t M, int F, b2s_stream_t stream) {
  return swiglu_fwd<float>(d_gu, d_h, M, F, B2S_ST(stream));
}
int b2s_swiglu_bwd_f32(const float* d_gu, const float* d_dh, float* d_dgu, int64_t M, int F, b2s_stream_t stream) {
  return swiglu_bwd<float>(d_gu, d_dh, d_dgu, M, F, B2S_ST(stream));
}

int b2s_cross_entropy(void* d_logits, int64_t ld, int V, const int64_t* d_target, float* d_loss_rows,
                      float grad_scale, int64_t M, int write_grad, b2s_stream_t stream) {
  return cross_entropy<__nv_bfloat16>(d_logits, ld, V, d_target, d_loss_rows, grad_scale, M, write_grad,
                                      B2S_ST(stream));
}
int b2s_cross_entropy_f32(float* d_logits, int64_t ld, int V, const int64_t* d_target, float* d_loss_rows,
                          float grad_scale, int64_t M, int write_grad, b2s_stream_t stream) {
  return cross_entropy<float>(d_logits, ld, V, d_target, d_loss_rows, grad_scale, M, write_grad, B2S_ST(stream));
}

int b2s_sum(const float* d_x, int64_t n, int squares, float* d_out, float scale, b2s_stream_t stream) {
  ew::sum_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(d_x, n, squares, d_out, scale);
  return check_launch("sum");
}
int b2s_sumsq_partial_multi(const uint64_t* d_ptrs, const int64_t* d_lens, int nseg, float* d_part, int nparts,
                            b2s_stream_t stream) {
  B2S_REQUIRE(nseg >= 0 && nparts > 0, B2S_EINVAL, "sumsq_partial_multi: bad sizes");
  ew::sumsq_multi_kernel<<<nparts, 256, 0, (cudaStream_t)stream>>>(d_ptrs, d_lens, nseg, d_part);
  return check_launch("sumsq_partial_multi");
}
int b2s_sumsq_partial(const float* d_x, int64_t n, float* d_part, int nparts, b2s_stream_t stream) {
  ew::sumsq_part_kernel<<<nparts, 256, 0, (cudaStream_t)stream>>>(d_x, n, d_part);
  return check_launch("sumsq_partial");
}

int b2s_adamw(float* d_p, float* d_m, float* d_v, const float* d_g, void* d_p_bf16, const uint8_t* d_wd_mask,
              int64_t n, const float* d_gn2, float max_norm, float lr, float beta1, float beta2, float eps,
              float wd, int step, b2s_stream_t stream) {
  return adamw<__nv_bfloat16>(d_p, d_m, d_v, d_g, d_p_bf16, d_wd_mask, n, d_gn2, max_norm, lr, beta1, beta2, eps,
                              wd, step, B2S_ST(stream));
}
int b2s_adamw_f32(float* d_p, float* d_m, float* d_v, const float* d_g, float* d_p_copy, const uint8_t* d_wd_mask,
                  int64_t n, const float* d_gn2, float max_norm, float lr, float beta1, float beta2, float eps,
                  float wd, int step, b2s_stream_t stream) {
  return adamw<float>(d_p, d_m, d_v, d_g, d_p_copy, d_wd_mask, n, d_gn2, max_norm, lr, beta1, beta2, eps, wd, step,
                      B2S_ST(stream));
}

int b2s_f32_to_bf16(const float* d_x, void* d_y, int64_t n, float scale, b2s_stream_t stream) {
  ew::f32_to_bf16_kernel<<<ew::flat_grid(n), 256, 0, (cudaStream_t)stream>>>(d_x, (__nv_bfloat16*)d_y, n, scale);
  return check_launch("f32_to_bf16");
}
int b2s_scale_f32(float* d_x, int64_t n, float scale, b2s_stream_t stream) {
  ew::scale_f32_kernel<<<ew::flat_grid(n, 1), 256, 0, (cudaStream_t)stream>>>(d_x, n, scale);
  return check_launch("scale_f32");
}

}  // extern "C"
