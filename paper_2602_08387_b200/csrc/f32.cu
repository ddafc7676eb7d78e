// fp32 mode (north star: "per-step losses and gradients within 1e-4 relative
// in fp32 mode"): true-fp32 SIMT kernels for the two tensor-core ops of the
// step -- the dense contraction and causal attention. Appendix C of SURVEY.md
// fixes the policy: fp32 mode is IEEE fp32 FFMA, not TF32, so these run on the
// CUDA cores. They carry the same operand-layout / epilogue contract as the
// bf16 tcgen05 kernels (gemm.cu, attn.cu) so the model runs either precision
// through the same call sequence.
#include "common.cuh"

namespace b2s {
namespace f32 {

// ------------------------------------------------------------------ GEMM
// C[M,N] (+)= epi(sum_k A(m,k) B(n,k)); A(m,k) = a_mn ? A[k*lda+m] : A[m*lda+k],
// B(n,k) = b_mn ? B[k*ldb+n] : B[n*ldb+k]. 128x128 CTA tile, BK=16, 256 threads,
// 8x8 register micro-tile (two 4-row x two 4-col quads so the smem reads are
// float4 and conflict-free), next K-slice staged in registers while the
// current one is consumed from shared memory.
constexpr int BM = 128, BN = 128, BK = 16, NT = 256;
constexpr int LDS = BM + 4;

__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.f + tanhf(k0 * (x + k1 * x * x * x)));
}
__device__ __forceinline__ float gelu_tanh_grad(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float t = tanhf(k0 * (x + k1 * x * x * x));
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x * x);
}

// Loads this thread's 8 elements of a BK x 128 operand slice starting at (row0, k0).
// mn_major: element (k, r) at P[k*ld + r]; else at P[r*ld + k]. Consecutive
// threads walk the contiguous dimension (coalesced); out-of-range -> 0.
__device__ __forceinline__ void load_slice(const float* __restrict__ P, int mn_major, int64_t ld, int rows,
                                           int K, int row0, int k0, float (&v)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int e = threadIdx.x + i * NT;
    int kk, rr;
    if (mn_major) { kk = e / BM; rr = e % BM; } else { kk = e % BK; rr = e / BK; }
    const int r = row0 + rr, k = k0 + kk;
    v[i] = (r < rows && k < K) ? (mn_major ? P[(int64_t)k * ld + r] : P[(int64_t)r * ld + k]) : 0.f;
  }
}
__device__ __forceinline__ void store_slice(float (*S)[LDS], int mn_major, const float (&v)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int e = threadIdx.x + i * NT;
    if (mn_major) S[e / BM][e % BM] = v[i];
    else S[e % BK][e / BK] = v[i];
  }
}

__global__ void __launch_bounds__(NT) gemm_kernel(const float* __restrict__ A, int a_mn, int64_t lda,
                                                  const float* __restrict__ B, int b_mn, int64_t ldb,
                                                  float* __restrict__ C, int64_t ldc, int M, int N, int K,
                                                  int accumulate, const float* __restrict__ bias, int act,
                                                  float* __restrict__ aux, int64_t ld_aux) {
  __shared__ __align__(16) float As[BK][LDS];
  __shared__ __align__(16) float Bs[BK][LDS];
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int ty = threadIdx.x / 16, tx = threadIdx.x % 16;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  float ra[8], rb[8];
  load_slice(A, a_mn, lda, M, K, m0, 0, ra);
  load_slice(B, b_mn, ldb, N, K, n0, 0, rb);
  for (int k0 = 0; k0 < K; k0 += BK) {
    store_slice(As, a_mn, ra);
    store_slice(Bs, b_mn, rb);
    __syncthreads();
    if (k0 + BK < K) {
      load_slice(A, a_mn, lda, M, K, m0, k0 + BK, ra);
      load_slice(B, b_mn, ldb, N, K, n0, k0 + BK, rb);
    }
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[kk][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (n >= N) continue;
      float v = acc[i][j];
      if (bias) v += bias[n];
      if (act == 1) {
        aux[(int64_t)m * ld_aux + n] = v;
        v = gelu_tanh(v);
      } else if (act == 2) {
        v *= gelu_tanh_grad(aux[(int64_t)m * ld_aux + n]);
      }
      float* c = C + (int64_t)m * ldc + n;
      *c = accumulate ? *c + v : v;
    }
  }
}

// ------------------------------------------------------------------ attention
// Causal softmax(Q K^T / sqrt(dh)) V over the fused [B*T, (Hq+2Hkv)*dh] fp32
// projection (q heads | k heads | v heads; q head h reads kv head h / (Hq/Hkv)).
// Forward: CTA = 32 query rows of one (b, h); 8 warps x 4 rows; lanes split
// the 64 keys of a shared-memory K/V tile for the scores and the head
// dimension for the output (online softmax, exact expf/logf).
constexpr int QT = 32, KT = 64;

template <int DH>
__global__ void __launch_bounds__(256) attn_fwd_kernel(const float* __restrict__ qkv, float* __restrict__ o,
                                                       float* __restrict__ lse, int T, int Hq, int Hkv,
                                                       float scale) {
  constexpr int DPL = DH / 32;  // output dims per lane
  extern __shared__ float smem[];
  float(*Qs)[DH] = reinterpret_cast<float(*)[DH]>(smem);
  float(*Ks)[DH + 1] = reinterpret_cast<float(*)[DH + 1]>(smem + QT * DH);
  float(*Vs)[DH] = reinterpret_cast<float(*)[DH]>(smem + QT * DH + KT * (DH + 1));
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int hk = h / (Hq / Hkv);
  const int64_t ld = (int64_t)(Hq + 2 * Hkv) * DH;
  const float* base = qkv + (int64_t)b * T * ld;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int q0 = qt * QT;
  for (int e = threadIdx.x; e < QT * DH; e += 256) {
    const int r = e / DH, c = e % DH;
    Qs[r][c] = (q0 + r < T) ? base[(int64_t)(q0 + r) * ld + h * DH + c] : 0.f;
  }
  float mrow[4], lrow[4], acc[4][DPL];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    mrow[r] = -INFINITY; lrow[r] = 0.f;
#pragma unroll
    for (int c = 0; c < DPL; ++c) acc[r][c] = 0.f;
  }
  const int qlast = min(T, q0 + QT) - 1;
  for (int k0 = 0; k0 <= qlast; k0 += KT) {
    __syncthreads();
    for (int e = threadIdx.x; e < KT * DH; e += 256) {
      const int r = e / DH, c = e % DH;
      const bool ok = k0 + r < T;
      Ks[r][c] = ok ? base[(int64_t)(k0 + r) * ld + (Hq + hk) * DH + c] : 0.f;
      Vs[r][c] = ok ? base[(int64_t)(k0 + r) * ld + (Hq + Hkv + hk) * DH + c] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int qi = q0 + w * 4 + r;
      if (qi >= T) continue;
      float s[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int kj = k0 + lane + 32 * u;
        float d = 0.f;
#pragma unroll 8
        for (int c = 0; c < DH; ++c) d = fmaf(Qs[w * 4 + r][c], Ks[lane + 32 * u][c], d);
        s[u] = (kj <= qi) ? d * scale : -INFINITY;
      }
      const float mt = warp_max(fmaxf(s[0], s[1]));
      const float mn = fmaxf(mrow[r], mt);
      const float alpha = (mrow[r] == -INFINITY) ? 0.f : expf(mrow[r] - mn);
      const float p0 = (s[0] == -INFINITY) ? 0.f : expf(s[0] - mn);
      const float p1 = (s[1] == -INFINITY) ? 0.f : expf(s[1] - mn);
      lrow[r] = lrow[r] * alpha + warp_sum(p0 + p1);
      mrow[r] = mn;
#pragma unroll
      for (int c = 0; c < DPL; ++c) acc[r][c] *= alpha;
      for (int j = 0; j < 32; ++j) {
        const float pa = __shfl_sync(0xffffffffu, p0, j), pb = __shfl_sync(0xffffffffu, p1, j);
#pragma unroll
        for (int c = 0; c < DPL; ++c)
          acc[r][c] = fmaf(pa, Vs[j][lane + 32 * c], fmaf(pb, Vs[j + 32][lane + 32 * c], acc[r][c]));
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int qi = q0 + w * 4 + r;
    if (qi >= T) continue;
    const float inv = 1.f / lrow[r];
    float* orow = o + ((int64_t)b * T + qi) * Hq * DH + h * DH;
#pragma unroll
    for (int c = 0; c < DPL; ++c) orow[lane + 32 * c] = acc[r][c] * inv;
    if (lane == 0) lse[((int64_t)b * Hq + h) * T + qi] = mrow[r] + logf(lrow[r]);
  }
}

// D[b,h,i] = sum_d dO[i,d] * O[i,d]  (one warp per row)
template <int DH>
__global__ void attn_bwd_dsum_kernel(const float* __restrict__ o, const float* __restrict__ dout,
                                     float* __restrict__ dsum, int B, int T, int Hq) {
  const int64_t rows = (int64_t)B * T * Hq;
  const int lane = threadIdx.x & 31;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < rows;
       r += ((int64_t)gridDim.x * blockDim.x) / 32) {
    const int64_t m = r / Hq;  // token row b*T + t
    const int h = (int)(r % Hq);
    float s = 0.f;
    for (int c = lane; c < DH; c += 32) s = fmaf(o[m * Hq * DH + h * DH + c], dout[m * Hq * DH + h * DH + c], s);
    s = warp_sum(s);
    if (lane == 0) {
      const int64_t b = m / T, t = m % T;
      dsum[(b * Hq + h) * T + t] = s;
    }
  }
}

// dK, dV: CTA = 32 keys of one (b, kv head); warp w owns keys 4w..4w+3 (lanes
// hold dK/dV dims). Loops over the group's q heads and the causal query tiles;
// lanes split the 32 queries of a tile for the scores. Deterministic.
template <int DH>
__global__ void __launch_bounds__(256) attn_bwd_dkv_kernel(const float* __restrict__ qkv,
                                                           const float* __restrict__ dout,
                                                           const float* __restrict__ lse,
                                                           const float* __restrict__ dsum,
                                                           float* __restrict__ dqkv, int T, int Hq, int Hkv,
                                                           float scale) {
  constexpr int DPL = DH / 32;
  extern __shared__ float smem[];
  float(*Ks)[DH + 1] = reinterpret_cast<float(*)[DH + 1]>(smem);
  float(*Vs)[DH + 1] = Ks + 32;
  float(*Qs)[DH + 1] = Ks + 64;
  float(*Ds)[DH + 1] = Ks + 96;  // dO tile
  float* Ls = smem + 128 * (DH + 1);
  float* Dd = Ls + 32;
  const int kt = blockIdx.x, hk = blockIdx.y, b = blockIdx.z;
  const int grp = Hq / Hkv;
  const int64_t ld = (int64_t)(Hq + 2 * Hkv) * DH;
  const float* base = qkv + (int64_t)b * T * ld;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int k0 = kt * 32;
  for (int e = threadIdx.x; e < 32 * DH; e += 256) {
    const int r = e / DH, c = e % DH;
    const bool ok = k0 + r < T;
    Ks[r][c] = ok ? base[(int64_t)(k0 + r) * ld + (Hq + hk) * DH + c] : 0.f;
    Vs[r][c] = ok ? base[(int64_t)(k0 + r) * ld + (Hq + Hkv + hk) * DH + c] : 0.f;
  }
  float dk[4][DPL], dv[4][DPL];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < DPL; ++c) { dk[r][c] = 0.f; dv[r][c] = 0.f; }
  for (int hh = 0; hh < grp; ++hh) {
    const int h = hk * grp + hh;
    for (int q0 = k0; q0 < T; q0 += 32) {
      __syncthreads();
      for (int e = threadIdx.x; e < 32 * DH; e += 256) {
        const int r = e / DH, c = e % DH;
        const bool ok = q0 + r < T;
        Qs[r][c] = ok ? base[(int64_t)(q0 + r) * ld + h * DH + c] : 0.f;
        Ds[r][c] = ok ? dout[((int64_t)b * T + q0 + r) * Hq * DH + h * DH + c] : 0.f;
      }
      if (threadIdx.x < 32) {
        const bool ok = q0 + threadIdx.x < T;
        Ls[threadIdx.x] = ok ? lse[((int64_t)b * Hq + h) * T + q0 + threadIdx.x] : 0.f;
        Dd[threadIdx.x] = ok ? dsum[((int64_t)b * Hq + h) * T + q0 + threadIdx.x] : 0.f;
      }
      __syncthreads();
      const int qi = q0 + lane;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int kr = w * 4 + r, kj = k0 + kr;
        float s = 0.f, dp = 0.f;
#pragma unroll 8
        for (int c = 0; c < DH; ++c) {
          s = fmaf(Qs[lane][c], Ks[kr][c], s);
          dp = fmaf(Ds[lane][c], Vs[kr][c], dp);
        }
        const bool live = qi < T && kj < T && kj <= qi;
        const float p = live ? expf(s * scale - Ls[lane]) : 0.f;
        const float ds = live ? p * (dp - Dd[lane]) : 0.f;
        for (int i = 0; i < 32; ++i) {
          const float pi = __shfl_sync(0xffffffffu, p, i), dsi = __shfl_sync(0xffffffffu, ds, i);
#pragma unroll
          for (int c = 0; c < DPL; ++c) {
            dv[r][c] = fmaf(pi, Ds[i][lane + 32 * c], dv[r][c]);
            dk[r][c] = fmaf(dsi, Qs[i][lane + 32 * c], dk[r][c]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int kj = k0 + w * 4 + r;
    if (kj >= T) continue;
    float* row = dqkv + ((int64_t)b * T + kj) * ld;
#pragma unroll
    for (int c = 0; c < DPL; ++c) {
      row[(Hq + hk) * DH + lane + 32 * c] = dk[r][c] * scale;
      row[(Hq + Hkv + hk) * DH + lane + 32 * c] = dv[r][c];
    }
  }
}

// dQ: CTA = 32 query rows of one (b, h); warp w owns rows 4w..4w+3; lanes
// split the 32 keys of a K/V tile for the scores and the dims for dQ.
template <int DH>
__global__ void __launch_bounds__(256) attn_bwd_dq_kernel(const float* __restrict__ qkv,
                                                          const float* __restrict__ dout,
                                                          const float* __restrict__ lse,
                                                          const float* __restrict__ dsum,
                                                          float* __restrict__ dqkv, int T, int Hq, int Hkv,
                                                          float scale) {
  constexpr int DPL = DH / 32;
  extern __shared__ float smem[];
  float(*Qs)[DH] = reinterpret_cast<float(*)[DH]>(smem);
  float(*Ds)[DH] = Qs + 32;
  float(*Ks)[DH + 1] = reinterpret_cast<float(*)[DH + 1]>(smem + 64 * DH);
  float(*Vs)[DH + 1] = Ks + 32;
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int hk = h / (Hq / Hkv);
  const int64_t ld = (int64_t)(Hq + 2 * Hkv) * DH;
  const float* base = qkv + (int64_t)b * T * ld;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int q0 = qt * 32;
  for (int e = threadIdx.x; e < 32 * DH; e += 256) {
    const int r = e / DH, c = e % DH;
    const bool ok = q0 + r < T;
    Qs[r][c] = ok ? base[(int64_t)(q0 + r) * ld + h * DH + c] : 0.f;
    Ds[r][c] = ok ? dout[((int64_t)b * T + q0 + r) * Hq * DH + h * DH + c] : 0.f;
  }
  float lrow[4], drow[4], dq[4][DPL];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int qi = q0 + w * 4 + r;
    lrow[r] = qi < T ? lse[((int64_t)b * Hq + h) * T + qi] : 0.f;
    drow[r] = qi < T ? dsum[((int64_t)b * Hq + h) * T + qi] : 0.f;
#pragma unroll
    for (int c = 0; c < DPL; ++c) dq[r][c] = 0.f;
  }
  const int qlast = min(T, q0 + 32) - 1;
  for (int k0 = 0; k0 <= qlast; k0 += 32) {
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * DH; e += 256) {
      const int r = e / DH, c = e % DH;
      const bool ok = k0 + r < T;
      Ks[r][c] = ok ? base[(int64_t)(k0 + r) * ld + (Hq + hk) * DH + c] : 0.f;
      Vs[r][c] = ok ? base[(int64_t)(k0 + r) * ld + (Hq + Hkv + hk) * DH + c] : 0.f;
    }
    __syncthreads();
    const int kj = k0 + lane;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int qr = w * 4 + r, qi = q0 + qr;
      float s = 0.f, dp = 0.f;
#pragma unroll 8
      for (int c = 0; c < DH; ++c) {
        s = fmaf(Qs[qr][c], Ks[lane][c], s);
        dp = fmaf(Ds[qr][c], Vs[lane][c], dp);
      }
      const bool live = qi < T && kj < T && kj <= qi;
      const float p = live ? expf(s * scale - lrow[r]) : 0.f;
      const float ds = live ? p * (dp - drow[r]) : 0.f;
      for (int j = 0; j < 32; ++j) {
        const float dsj = __shfl_sync(0xffffffffu, ds, j);
#pragma unroll
        for (int c = 0; c < DPL; ++c) dq[r][c] = fmaf(dsj, Ks[j][lane + 32 * c], dq[r][c]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int qi = q0 + w * 4 + r;
    if (qi >= T) continue;
    float* row = dqkv + ((int64_t)b * T + qi) * ld + h * DH;
#pragma unroll
    for (int c = 0; c < DPL; ++c) row[lane + 32 * c] = dq[r][c] * scale;
  }
}

template <int DH>
static int attn_fwd(const float* qkv, float* o, float* lse, int B, int T, int Hq, int Hkv, cudaStream_t st) {
  dim3 grid((T + QT - 1) / QT, Hq, B);
  constexpr int smem = (QT * DH + KT * (DH + 1) + KT * DH) * 4;
  cudaFuncSetAttribute(attn_fwd_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  attn_fwd_kernel<DH><<<grid, 256, smem, st>>>(qkv, o, lse, T, Hq, Hkv, 1.f / sqrtf((float)DH));
  return check_launch("attn_fwd_f32");
}

template <int DH>
static int attn_bwd(const float* qkv, const float* o, const float* dout, const float* lse, float* dqkv,
                    float* dsum, int B, int T, int Hq, int Hkv, cudaStream_t st) {
  const float scale = 1.f / sqrtf((float)DH);
  attn_bwd_dsum_kernel<DH><<<kNumSMs * 8, 256, 0, st>>>(o, dout, dsum, B, T, Hq);
  constexpr int smem_kv = (128 * (DH + 1) + 64) * 4, smem_q = (64 * DH + 64 * (DH + 1)) * 4;
  cudaFuncSetAttribute(attn_bwd_dkv_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv);
  cudaFuncSetAttribute(attn_bwd_dq_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_q);
  attn_bwd_dkv_kernel<DH><<<dim3((T + 31) / 32, Hkv, B), 256, smem_kv, st>>>(qkv, dout, lse, dsum, dqkv, T, Hq, Hkv,
                                                                        scale);
  attn_bwd_dq_kernel<DH><<<dim3((T + 31) / 32, Hq, B), 256, smem_q, st>>>(qkv, dout, lse, dsum, dqkv, T, Hq, Hkv,
                                                                      scale);
  return check_launch("attn_bwd_f32", 3);
}

}  // namespace f32
}  // namespace b2s

using namespace b2s;

extern "C" {

int b2s_gemm_f32(const float* d_A, int a_mn_major, int64_t lda, const float* d_B, int b_mn_major, int64_t ldb,
                 float* d_C, int64_t ldc, int M, int N, int K, int accumulate, const float* d_bias, int act,
                 float* d_aux, int64_t ld_aux, b2s_stream_t stream) {
  B2S_REQUIRE(M >= 0 && N >= 0 && K >= 0, B2S_EINVAL, "gemm_f32: negative size");
  B2S_REQUIRE(act == 0 || ((act == 1 || act == 2) && d_aux), B2S_EINVAL, "gemm_f32: activation needs d_aux");
  B2S_REQUIRE(!(accumulate && act == 1), B2S_EINVAL, "gemm_f32: accumulate with GELU is not supported");
  if (M == 0 || N == 0) return B2S_OK;
  dim3 grid((N + f32::BN - 1) / f32::BN, (M + f32::BM - 1) / f32::BM);
  f32::gemm_kernel<<<grid, f32::NT, 0, (cudaStream_t)stream>>>(d_A, a_mn_major, lda, d_B, b_mn_major, ldb, d_C, ldc,
                                                               M, N, K, accumulate, d_bias, act, d_aux, ld_aux);
  return check_launch("gemm_f32");
}

int b2s_attn_fwd_f32(const float* d_qkv, float* d_o, float* d_lse, int B, int T, int Hq, int Hkv, int dh,
                     b2s_stream_t stream) {
  B2S_REQUIRE(Hkv > 0 && Hq % Hkv == 0 && T > 0 && B > 0, B2S_EINVAL, "attention_f32: bad shape");
  cudaStream_t st = (cudaStream_t)stream;
  switch (dh) {
    case 32: return f32::attn_fwd<32>(d_qkv, d_o, d_lse, B, T, Hq, Hkv, st);
    case 64: return f32::attn_fwd<64>(d_qkv, d_o, d_lse, B, T, Hq, Hkv, st);
    case 128: return f32::attn_fwd<128>(d_qkv, d_o, d_lse, B, T, Hq, Hkv, st);
  }
  set_error("attention_f32: head dim %d not implemented (32, 64, 128)", dh);
  return B2S_EUNSUPPORTED;
}

int b2s_attn_bwd_f32(const float* d_qkv, const float* d_o, const float* d_do, const float* d_lse, float* d_dqkv,
                     float* d_work, int B, int T, int Hq, int Hkv, int dh, b2s_stream_t stream) {
  B2S_REQUIRE(Hkv > 0 && Hq % Hkv == 0 && T > 0 && B > 0, B2S_EINVAL, "attention_f32: bad shape");
  cudaStream_t st = (cudaStream_t)stream;
  switch (dh) {
    case 32: return f32::attn_bwd<32>(d_qkv, d_o, d_do, d_lse, d_dqkv, d_work, B, T, Hq, Hkv, st);
    case 64: return f32::attn_bwd<64>(d_qkv, d_o, d_do, d_lse, d_dqkv, d_work, B, T, Hq, Hkv, st);
    case 128: return f32::attn_bwd<128>(d_qkv, d_o, d_do, d_lse, d_dqkv, d_work, B, T, Hq, Hkv, st);
  }
  set_error("attention_f32: head dim %d not implemented (32, 64, 128)", dh);
  return B2S_EUNSUPPORTED;
}

}  // extern "C"
