// Causal multi-head / grouped-query attention on tcgen05 (K7), head dims 64 and 128.
//
// Layout: q/k/v are read straight out of the fused QKV projection output
// [B*T, (Hq + 2*Hkv) * dh] (bf16, head h of q at column h*dh, kv head j of k
// at (Hq + j)*dh and of v at (Hq + Hkv + j)*dh) by 2-D TMA boxes of
// 64 (dh) x 128 (tokens) -- no transpose/copy kernel (two boxes per tile at
// dh = 128: a tile is then two 128B-swizzle atoms, 16 KB apart). Output o is
// [B*T, Hq*dh] bf16 (the O-projection GEMM's A operand) and the per-row
// log-sum-exp lse[B, Hq, T] (fp32, natural log) is kept for the backward.
//
// Forward CTA = (batch, q head, 128-query tile); roles: warp0 TMA, warp1 MMA,
// warps 2..5 softmax (one query row per thread, the row is a TMEM lane).
//   S_j = Q K_j^T  -> TMEM (double-buffered, M=128 N=128 K=64)
//   P_j = exp2(S_j * scale*log2e - m_j) -> bf16 -> swizzled smem
//   PV_j = P_j V_j -> TMEM (M=128 N=64 K=128, V as an MN-major operand)
//   O   = O * 2^(m_{j-1} - m_j) + PV_j   (fp32, registers)
// S_{j+1} is issued before PV_j, so QK^T of the next block overlaps softmax.
//
// Backward CTA = (batch, kv head, 128-key tile), looping over the q heads of
// its group and the causal query tiles: S^T = K Q^T, dP^T = V dO^T (TMEM),
// P^T and dS^T = P^T (dP^T - D) to smem (thread = key row), then
// dV += P^T dO, dK += dS^T Q (TMEM accumulators across the loop) and
// dQ_i = dS K (TMEM) -> fp32 smem -> TMA add-reduce into a dQ accumulator.
#include "common.cuh"
#include "sm100.cuh"

namespace b2s {
using namespace sm100;
namespace attn {

constexpr int BQ = 128, BKV = 128;

constexpr int kTile = BQ * 64 * 2;  // 16 KB: one 128-row x 64-column bf16 swizzle atom
constexpr int kPBuf = BQ * BKV * 2; // 32 KB: a 128 x 128 bf16 P tile (two atoms)
constexpr int kStages = 2;
constexpr float kLog2e = 1.4426950408889634f;

// byte offset of 16-B chunk c of row r in a 128B-swizzled tile of 128-B rows
__device__ __forceinline__ uint32_t swz(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

// Round a dynamic-smem pointer up to 1024 B by offsetting it (not via an
// integer round trip), so the compiler keeps the shared address space and
// emits STS/LDS instead of generic stores.
__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  return p + ((1024u - (a & 1023u)) & 1023u);
}
__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct Params {
  int B, T, Hq, Hkv, nqt;
  float scale_log2;  // log2(e) / sqrt(dh)
  float scale;       // 1 / sqrt(dh)
  float* lse;        // [B, Hq, T]
  const float* dsum; // bwd: D = rowsum(dO * O), [B, Hq, T]
  float* dq_acc;     // bwd (dh 64): fp32 dQ accumulator [B*T, Hq*dh]
};

// =====================================================================================
// forward
// =====================================================================================
// CTA = (batch, q head, pair of 128-query tiles A = 2p, B = 2p+1). Two softmax
// warpgroups (warps 2-5 -> tile A, warps 6-9 -> tile B) share each K/V block
// and the MMA warp ping-pongs between them:
//   S_A(0) S_B(0) | PV_A(j) S_A(j+1) PV_B(j) S_B(j+1) | ...
// O accumulates in TMEM (PV MMAs chain with accumulate=1). A softmax thread
// only rescales its O row (tcgen05.ld / st) when its running max grows by
// more than 2^8 -- otherwise P is formed against the stale max and stays
// <= 256 -- so the softmax loop never waits for the PV MMA it just enabled.
// P is double-buffered in smem per tile so P(j+1) can be written while
// PV(j) still reads P(j).
// dh = 128 runs one query tile per CTA (TILES = 1, warps 6-9 absent): the
// 32 KB Q / K / V tiles leave room for 2 K/V stages and a double-buffered P
// only for one tile in 227 KB of shared memory.
#ifndef B2S_ATTN_FWD64_MODE
#define B2S_ATTN_FWD64_MODE 0  // dh 64: 0 two ping-pong tiles per CTA (default, fastest measured);
                               // 1 one tile per CTA, two CTAs per SM (2 K/V stages, 1 P buffer): 25% slower
#endif
#ifndef B2S_ATTN_FWD64_KVS
#define B2S_ATTN_FWD64_KVS 2  // dh 64 K / V stages (2..4)
#endif
#ifndef B2S_ATTN_FWD128_TILES
#define B2S_ATTN_FWD128_TILES 2  // dh 128: 2 = two query tiles per CTA with P aliasing S; 1 = one tile
#endif
#ifndef B2S_ATTN_FWD_PT
#define B2S_ATTN_FWD_PT 1  // P in TMEM (PV by the TMEM-A MMA form) instead of shared memory
#endif
template <int DH>
struct Fwd {
  static constexpr int MODE = DH == 64 ? B2S_ATTN_FWD64_MODE : 0;
  static constexpr bool PT = B2S_ATTN_FWD_PT && MODE == 0;
  // dh 128 with P in TMEM: two ping-pong query tiles, P aliasing the tile's S columns
  // (S / O of two tiles fill all 512 columns); S_t(j+1) is issued behind PV_t(j)
  static constexpr bool ALIAS = DH == 128 && PT && B2S_ATTN_FWD128_TILES == 2;
  static constexpr int TILES = ((DH == 64 && MODE == 0) || ALIAS) ? 2 : 1;
  // K / V smem stages (dh 64 with P in TMEM has room for more)
  static constexpr int KVS = MODE == 2 ? 1 : ((DH == 64 && PT) ? B2S_ATTN_FWD64_KVS : 2);
  static constexpr int PB = (MODE == 1 || PT) ? 1 : 2;  // P buffers per tile (smem, or one TMEM block)
  static constexpr int MINB = MODE == 0 ? 1 : 2;      // CTAs per SM
  static constexpr int TCOLS = MODE == 0 ? 512 : 256; // TMEM columns allocated
  static constexpr int OCOL = MODE == 0 ? 256 : 128;  // first O column
  static constexpr int kThreads = 64 + 128 * TILES;
  static constexpr int kTileQ = BQ * DH * 2;  // Q / K / V tile bytes (DH/64 atoms)
  static constexpr int PCOL = OCOL + TILES * DH;      // PT: P (bf16 pairs, 64 columns per tile)
  static constexpr int pcol(int t) { return ALIAS ? t * BKV : PCOL + t * 64; }
  static constexpr int kSmem = 1024 + TILES * kTileQ + 2 * KVS * kTileQ + (PT ? 0 : TILES * PB * kPBuf) + 256;
  static_assert(kSmem * MINB <= 232448, "forward tiles exceed shared memory");
  static_assert(KVS >= 2 && KVS <= 4, "S(j+1) is issued before PV(j): one K/V stage would deadlock");
};
constexpr float kRescaleThresh = 8.0f;  // log2 units

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA / ALU pipes (no MUFU): x = n + f, n = rint(x) by the 1.5*2^23
// magic add, f in [-0.5, 0.5], 2^f by a degree-3 minimax polynomial (max
// relative error 1.0e-4, well below the bf16 rounding P is stored with), the
// exponent added as integer n << 23. x is clamped to >= -127 (2^-127 ~ 0).
// Offloads part of the softmax exponentials from the 16/clk/SM MUFU unit.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -127.f);
  const float j = x + 12582912.f;
  const float f = x - (j - 12582912.f);
  float p = fmaf(fmaf(fmaf(0.05500891f, f, 0.242211f), f, 0.69328293f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(j) << 23));
}
#ifndef B2S_EXP_POLY_MASK
#define B2S_EXP_POLY_MASK 0x00  // 8-column groups (bitmask) using ex2_poly; 0: measured fastest (the softmax is latency-, not MUFU-bound)
#endif

// P = 2^(s*sl2 - m) for 64 columns of one row -> bf16 -> swizzled smem; returns
// the row sum. The causal mask is a template branch so off-diagonal blocks run
// the mask-free instruction stream.
template <bool DIAG>
__device__ __forceinline__ float exp_pack(const uint32_t* v, int col0, int r, float sl2, float m,
                                          uint8_t* dst) {
  // row sum as 4 independent partial sums combined by a tree: a single serial
  // FADD chain over 64 elements would be longer than the MUFU work it follows
  float rs4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int k8 = 0; k8 < 8; ++k8) {
    float e[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float a = fmaf(__uint_as_float(v[k8 * 8 + i]), sl2, -m);
      const float x = ((B2S_EXP_POLY_MASK >> k8) & 1) ? ex2_poly(a) : ex2(a);
      e[i] = (DIAG && col0 + k8 * 8 + i > r) ? 0.f : x;
    }
    rs4[k8 & 3] += ((e[0] + e[1]) + (e[2] + e[3])) + ((e[4] + e[5]) + (e[6] + e[7]));
    uint4 w;
    w.x = pack_bf16x2(e[0], e[1]);
    w.y = pack_bf16x2(e[2], e[3]);
    w.z = pack_bf16x2(e[4], e[5]);
    w.w = pack_bf16x2(e[6], e[7]);
    *reinterpret_cast<uint4*>(dst + swz(r, k8)) = w;
  }
  return (rs4[0] + rs4[1]) + (rs4[2] + rs4[3]);
}

// Same, for all BKV columns of the row, packed as bf16 pairs into out[0 .. BKV/2)
// (out may alias v: pair k is written after v[2k], v[2k+1] are read).
template <bool DIAG>
__device__ __forceinline__ float exp_pack_regs(const uint32_t* v, int r, float sl2, float m, uint32_t* out) {
  float rs4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int k8 = 0; k8 < BKV / 8; ++k8) {
    float e[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float a = fmaf(__uint_as_float(v[k8 * 8 + i]), sl2, -m);
      const float x = ((B2S_EXP_POLY_MASK >> (k8 & 7)) & 1) ? ex2_poly(a) : ex2(a);
      e[i] = (DIAG && k8 * 8 + i > r) ? 0.f : x;
    }
    rs4[k8 & 3] += ((e[0] + e[1]) + (e[2] + e[3])) + ((e[4] + e[5]) + (e[6] + e[7]));
#pragma unroll
    for (int i = 0; i < 4; ++i) out[k8 * 4 + i] = pack_bf16x2(e[2 * i], e[2 * i + 1]);
  }
  return (rs4[0] + rs4[1]) + (rs4[2] + rs4[3]);
}

template <int DH>
__global__ void __launch_bounds__(Fwd<DH>::kThreads, Fwd<DH>::MINB)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_o,
                    Params p) {
  using C = Fwd<DH>;
  constexpr int TILES = C::TILES, kTQ = C::kTileQ, NA = DH / 64;  // NA: 64-column atoms per tile
  constexpr int KVS = C::KVS, PB = C::PB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sQ = align1024(smem_raw);          // [TILES] tiles A, B
  uint8_t* sK = sQ + TILES * kTQ;             // [KVS]
  uint8_t* sV = sK + KVS * kTQ;               // [KVS]
  uint8_t* sP = sV + KVS * kTQ;               // [tile][buf] x 32 KB (two 64-key atoms each)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + (C::PT ? 0 : TILES * PB * kPBuf));
  uint64_t* q_full = bars;                    // 1
  constexpr int kKV = 4;                      // barrier slots per K / V array (>= KVS)
  uint64_t* k_full = bars + 1;                // [KVS]
  uint64_t* v_full = k_full + kKV;            // [KVS]
  uint64_t* kv_empty = v_full + kKV;          // [KVS]
  uint64_t* s_full = kv_empty + kKV;          // [2] per tile
  uint64_t* s_empty = s_full + 2;             // [2]
  uint64_t* p_full = s_empty + 2;             // [tile][buf]: per buffer, so a group running a block
                                              // ahead of the MMA warp cannot alias a barrier phase
  uint64_t* p_empty = p_full + 4;             // [tile][buf]
  uint64_t* o_done = p_empty + 4;             // [2] last PV of the tile retired
  uint64_t* pv_done = o_done + 2;             // [2] each PV retired (rescale fence)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(pv_done + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int npair = (p.nqt + TILES - 1) / TILES;
  const int nbh = p.B * p.Hq;
  const int pr = npair - 1 - (int)(blockIdx.x / nbh);  // heaviest pairs first
  const int bh = blockIdx.x % nbh;
  const int b = bh / p.Hq, h = bh % p.Hq;
  const int kvh = h / (p.Hq / p.Hkv);
  const int qtA = TILES * pr, qtB = TILES * pr + 1;
  const bool hasB = TILES == 2 && qtB < p.nqt;
  const int nA = qtA + 1, nB = hasB ? qtB + 1 : 0;
  const int nkv = hasB ? nB : nA;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    mbar_init(q_full, 1);
    for (int s = 0; s < KVS; ++s) { mbar_init(&k_full[s], 1); mbar_init(&v_full[s], 1); mbar_init(&kv_empty[s], 1); }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1); mbar_init(&s_empty[t], 4);
      mbar_init(&p_full[2 * t], 4); mbar_init(&p_full[2 * t + 1], 4);
      mbar_init(&o_done[t], 1); mbar_init(&pv_done[t], 1);
      mbar_init(&p_empty[2 * t], 1); mbar_init(&p_empty[2 * t + 1], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::TCOLS>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  // TMEM: S_A [0,128) S_B [128,256) O_A [OCOL,OCOL+DH) O_B [OCOL+DH,OCOL+2DH)

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, hasB ? 2 * kTQ : kTQ);
      for (int a = 0; a < NA; ++a) {
        tma_load_2d(sQ + a * kTile, &tm_qkv, q_full, h * DH + a * 64, b * p.T + qtA * BQ);
        if (hasB) tma_load_2d(sQ + kTQ + a * kTile, &tm_qkv, q_full, h * DH + a * 64, b * p.T + qtB * BQ);
      }
      for (int j = 0; j < nkv; ++j) {
        const int s = j % KVS;
        mbar_wait(&kv_empty[s], ((j / KVS) & 1) ^ 1);
        const int r = b * p.T + j * BKV;
        mbar_arrive_expect_tx(&k_full[s], kTQ);
        for (int a = 0; a < NA; ++a)
          tma_load_2d(sK + s * kTQ + a * kTile, &tm_qkv, &k_full[s], (p.Hq + kvh) * DH + a * 64, r);
        mbar_arrive_expect_tx(&v_full[s], kTQ);
        for (int a = 0; a < NA; ++a)
          tma_load_2d(sV + s * kTQ + a * kTile, &tm_qkv, &v_full[s], (p.Hq + p.Hkv + kvh) * DH + a * 64, r);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    {  // whole warp, converged; one lane elected per tcgen05 instruction
      constexpr uint32_t idS = make_idesc_bf16(BQ, BKV, false, false);
      constexpr uint32_t idO = make_idesc_bf16(BQ, DH, false, true);
      const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aV = smem_u32(sV), aP = smem_u32(sP);
      auto issue_S = [&](int t, int j) {
        const int s = j % KVS;
        mbar_wait(&k_full[s], (j / KVS) & 1);
        mbar_wait(&s_empty[t], (j & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t ko = (kk >> 2) * kTile + (kk & 3) * 32;  // atom, then 16-element K step
          mma_bf16_ss_w(tbase + t * BKV, make_sdesc(aQ + t * kTQ + ko, 16, 1024),
                        make_sdesc(aK + s * kTQ + ko, 16, 1024), idS, kk > 0);
        }
        mma_commit_w(&s_full[t]);
      };
      auto issue_PV = [&](int t, int j, bool last) {
        const int s = j % KVS;
        mbar_wait(&v_full[s], (j / KVS) & 1);
        mbar_wait(&p_full[2 * t + (j % PB)], (j / PB) & 1);
        tc_fence_after();
        const uint32_t pbase = aP + (PB * t + (j % PB)) * kPBuf;
        // V as an MN-major operand: 16 keys per K step (2 KB of 128-B rows), dh atoms LBO = 16 KB apart
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk) {
          if constexpr (C::PT)  // P from TMEM: 16 keys = 8 columns of bf16 pairs per K step
            mma_bf16_ts_w(tbase + C::OCOL + t * DH, tbase + C::pcol(t) + kk * 8,
                          make_sdesc(aV + s * kTQ + kk * 2048, kTile, 1024), idO, (j > 0 || kk > 0) ? 1u : 0u);
          else
            mma_bf16_ss_w(tbase + C::OCOL + t * DH, make_sdesc(pbase + (kk >> 2) * kTile + (kk & 3) * 32, 16, 1024),
                          make_sdesc(aV + s * kTQ + kk * 2048, kTile, 1024), idO, (j > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit_w(&p_empty[2 * t + (j % PB)]);
        mma_commit_w(&pv_done[t]);
        if (last) mma_commit_w(&o_done[t]);
      };
      mbar_wait(q_full, 0);
      issue_S(0, 0);
      if (nB > 0) issue_S(1, 0);
      for (int j = 0; j < nkv; ++j) {
        if constexpr (C::ALIAS) {
          // P_t(j) lives in S_t's columns: S_t(j+1) goes in behind PV_t(j) (the tensor
          // pipe runs one CTA's MMAs in order), while the other tile's softmax runs
          if (j < nA) issue_PV(0, j, j + 1 == nA);
          if (j + 1 < nA) issue_S(0, j + 1);
          if (j < nB) issue_PV(1, j, j + 1 == nB);
          if (j + 1 < nB) issue_S(1, j + 1);
        } else {
          // QK^T of block j+1 goes in as soon as each softmax group holds S(j) in
          // registers, so it is ready when the group finishes block j
          if (j + 1 < nA) issue_S(0, j + 1);
          if (j + 1 < nB) issue_S(1, j + 1);
          if (j < nA) issue_PV(0, j, j + 1 == nA);
          if (j < nB) issue_PV(1, j, j + 1 == nB);
        }
        mma_commit_w(&kv_empty[j % KVS]);  // K_j / V_j no longer read once these retire
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ softmax warpgroups
    const int t = (warp - 2) >> 2;  // 0: tile A, 1: tile B
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const int qt = t == 0 ? qtA : qtB;
    const int nj = t == 0 ? nA : nB;
    const uint32_t lrow = (uint32_t)(q4 * 32) << 16;
    const uint32_t tS = tbase + lrow + t * BKV;
    const uint32_t tO = tbase + lrow + C::OCOL + t * DH;
    const float sl2 = p.scale_log2;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nj; ++j) {
      mbar_wait(&s_full[t], j & 1);
      tc_fence_after();
      const bool diag = (j == qt);
      // the whole 128-column S row in registers: one TMEM round trip per block
      uint32_t v[BKV];
#pragma unroll
      for (int c = 0; c < BKV / 32; ++c) tmem_ld32(tS + c * 32, v + c * 32);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[t]);  // S(j) is in registers: QK^T(j+1) may overwrite it
      // row max over 8 independent partial maxima (short dependency chains)
      float mx8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = -INFINITY;
      if (diag) {
#pragma unroll
        for (int i = 0; i < BKV; ++i)
          if (i <= r) mx8[i & 7] = fmaxf(mx8[i & 7], __uint_as_float(v[i]));
      } else {  // three-input max (FMNMX3): two new elements per instruction
#pragma unroll
        for (int i = 0; i < BKV / 2; ++i)
          mx8[i & 7] = fmax3(mx8[i & 7], __uint_as_float(v[2 * i]), __uint_as_float(v[2 * i + 1]));
      }
      const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                             fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      const float m_cand = mx * sl2;
      // lazy rescale: keep the old max unless the new one exceeds it by > 2^8
      float m_use = m;
      bool resc = false;
      if (m_cand > m + kRescaleThresh) { m_use = m_cand; resc = (j > 0); }
      const float alpha = ex2(m - m_use);  // 0 on the first block (m = -inf)
      if (__any_sync(0xffffffffu, resc)) {
        // O must not be in flight: wait for the previous PV of this tile, then O *= alpha
        mbar_wait(&pv_done[t], (j - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < DH / 16; ++c) {
          uint32_t o[16];
          tmem_ld16(tO + c * 16, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * (resc ? alpha : 1.f));
          tmem_st16(tO + c * 16, o);
        }
        tmem_wait_st();
      }
      // P = 2^(s*sl2 - m_use) -> bf16 -> smem buffer (j & 1) or TMEM; row sum
      const int pb = j % PB;
      float rs = 0.f;
      if constexpr (C::PT) {
        // exponentials first (bf16 pairs packed over the S registers), then wait for
        // PV(j-1) to release this tile's TMEM P block, then one TMEM store round
        uint32_t* pk = v;
        rs = diag ? exp_pack_regs<true>(v, r, sl2, m_use, pk) : exp_pack_regs<false>(v, r, sl2, m_use, pk);
        if (j >= 1) mbar_wait(&p_empty[2 * t], (j - 1) & 1);
        tc_fence_after();
        tmem_st32(tbase + lrow + C::pcol(t), pk);
        tmem_st32(tbase + lrow + C::pcol(t) + 32, pk + 32);
        tmem_wait_st();
      } else {
        if (j >= PB) mbar_wait(&p_empty[2 * t + pb], ((j / PB) - 1) & 1);
        uint8_t* myP = sP + (PB * t + pb) * kPBuf;
        if (diag) {
          rs += exp_pack<true>(v, 0, r, sl2, m_use, myP);
          rs += exp_pack<true>(v + 64, 64, r, sl2, m_use, myP + kTile);
        } else {
          rs += exp_pack<false>(v, 0, r, sl2, m_use, myP);
          rs += exp_pack<false>(v + 64, 64, r, sl2, m_use, myP + kTile);
        }
        fence_proxy_async_smem();
      }
      l = l * alpha + rs;
      m = m_use;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[2 * t + pb]);
    }
    if (nj > 0) {
      // epilogue: O (TMEM) / l -> bf16 -> this tile's Q buffer (all MMAs retired) -> TMA store
      mbar_wait(&o_done[t], 0);
      tc_fence_after();
      uint8_t* sO = sQ + t * kTQ;
      const float inv = 1.f / l;
#pragma unroll
      for (int c = 0; c < DH / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + c * 32, o);
        tmem_wait_ld();
#pragma unroll
        for (int k8 = 0; k8 < 4; ++k8) {
          uint4 w;
          w.x = pack_bf16x2(__uint_as_float(o[8 * k8 + 0]) * inv, __uint_as_float(o[8 * k8 + 1]) * inv);
          w.y = pack_bf16x2(__uint_as_float(o[8 * k8 + 2]) * inv, __uint_as_float(o[8 * k8 + 3]) * inv);
          w.z = pack_bf16x2(__uint_as_float(o[8 * k8 + 4]) * inv, __uint_as_float(o[8 * k8 + 5]) * inv);
          w.w = pack_bf16x2(__uint_as_float(o[8 * k8 + 6]) * inv, __uint_as_float(o[8 * k8 + 7]) * inv);
          *reinterpret_cast<uint4*>(sO + (c >> 1) * kTile + swz(r, (c & 1) * 4 + k8)) = w;
        }
      }
      p.lse[((size_t)b * p.Hq + h) * p.T + qt * BQ + r] = (m + log2f(l)) * (1.f / kLog2e);
      fence_proxy_async_smem();
      named_sync(1 + t, 128);
      if (q4 == 0 && lane == 0) {
        for (int a = 0; a < NA; ++a) tma_store_2d(&tm_o, sO + a * kTile, h * DH + a * 64, b * p.T + qt * BQ);
        bulk_commit();
        bulk_wait_read<0>();
      }
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::TCOLS>(tbase);
  }
}

// =====================================================================================
// backward
// =====================================================================================
// D'[b, h, q] = scale * sum_d dO * O (row-wise), lse2 = lse * log2(e), and zero
// the fp32 dQ accumulator (if any). The backward then forms the already-scaled
// dS' = scale * P (dP - D) = P * (scale * dP - D') with one FFMA, and
// P = 2^(s * scale * log2(e) - lse2) with one FFMA, per element.
template <int DH>
__global__ void attn_bwd_prep_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                                     const float* __restrict__ lse, float* __restrict__ dsum,
                                     float* __restrict__ lse2, float* __restrict__ dq_acc, int B, int T, int Hq,
                                     float scale) {
  // DH/8 lanes per (row, head): each lane a 16-byte vector of o and dO
  constexpr int LPR = DH / 8;
  const int sub = threadIdx.x & (LPR - 1);
  const int64_t nrows = (int64_t)B * T * Hq;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPR; w < nrows;
       w += ((int64_t)gridDim.x * blockDim.x) / LPR) {
    const int64_t row = (int64_t)((uint32_t)w / (uint32_t)Hq);  // B*T*Hq < 2^32 (host-checked)
    const int h = (int)(w - row * Hq);
    const int64_t off = row * Hq * DH + h * DH + sub * 8;
    float a[8], g[8];
    unpack8(*reinterpret_cast<const bf16x8*>(o + off), a);
    unpack8(*reinterpret_cast<const bf16x8*>(dout + off), g);
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += a[i] * g[i];
#pragma unroll
    for (int x = 1; x < LPR; x <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, x);
    if (dq_acc) {
      *reinterpret_cast<float4*>(dq_acc + off) = make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(dq_acc + off + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (sub == 0) {
      const int64_t b = (int64_t)((uint32_t)row / (uint32_t)T), t = row - b * T;
      const int64_t i = (b * Hq + h) * T + t;
      dsum[i] = acc * scale;
      lse2[i] = lse[i] * kLog2e;
    }
  }
}

// dqkv[:, q heads] = bf16(dq_acc)  (dh = 64 path). Blocks stride over rows (a row
// is Hq*64 floats), so no 64-bit division per element.
__global__ void __launch_bounds__(256) attn_bwd_dq_kernel(const float* __restrict__ dq_acc,
                                                          __nv_bfloat16* __restrict__ dqkv, int64_t M, int Hq,
                                                          int64_t ldq) {
  constexpr int DH = 64;
  const int nv = Hq * DH / 4;  // float4 vectors per row
  for (int64_t row = blockIdx.x; row < M; row += gridDim.x) {
    const float* src = dq_acc + row * (int64_t)(Hq * DH);
    __nv_bfloat16* dst = dqkv + row * ldq;
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
      const float4 a = __ldcs(reinterpret_cast<const float4*>(src) + v);
      uint2 u;
      u.x = pack_bf16x2(a.x, a.y);
      u.y = pack_bf16x2(a.z, a.w);
      *reinterpret_cast<uint2*>(dst + 4 * v) = u;
    }
  }
}

// Backward CTA = (batch, kv head, 128-key tile); 8 compute warps: warp w owns
// key rows 32*(w&3).. (its TMEM lane quarter) and query columns
// 64*((w-2)>>2).. of each 128x128 S^T / dP^T block. MMA order per step t:
//   S(t+1), dP(t+1)  [as soon as the compute warps hold S(t), dP(t) in registers]
//   dV += P^T dO, dK += dS^T Q, dQ[t&1] = dS K     [after P^T, dS^T(t) reach smem]
// so the next step's QK^T / V dO^T overlap this step's exponentials, and dQ is
// double-buffered in TMEM: the compute warps drain dQ(t-1) (TMA add-reduce
// into the fp32 accumulator) after publishing P/dS(t).
constexpr int kBwdThreads = 320;

// P^T = 2^(s*sl2 - lse2[q]) and the scaled dS^T = P^T (scale dP^T - D'[q]) for
// 32 query columns of one key row, in place in sv / dv (bit patterns of fp32).
// Mask = template branch.
template <bool DIAG>
__device__ __forceinline__ void p_ds(uint32_t* sv, uint32_t* dv, int q0, int r, float sl2, float scale,
                                     const float* lse2, const float* dd) {
  // the 32 columns' LSE / D values are the same for every thread: 16-byte
  // broadcast loads (8 + 8 LDS.128 instead of 64 scalar LDS)
  float ls[32], ds[32];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float4 l4 = *reinterpret_cast<const float4*>(lse2 + q0 + 4 * k);
    const float4 d4 = *reinterpret_cast<const float4*>(dd + q0 + 4 * k);
    ls[4 * k] = l4.x; ls[4 * k + 1] = l4.y; ls[4 * k + 2] = l4.z; ls[4 * k + 3] = l4.w;
    ds[4 * k] = d4.x; ds[4 * k + 1] = d4.y; ds[4 * k + 2] = d4.z; ds[4 * k + 3] = d4.w;
  }
#pragma unroll
  for (int e = 0; e < 32; ++e) {
    const int q = q0 + e;
#ifdef B2S_EXP_NOEXP
    float pv = __uint_as_float(sv[e]);
#else
    float pv = ex2(fmaf(__uint_as_float(sv[e]), sl2, -ls[e]));
#endif
    if (DIAG && q < r) pv = 0.f;  // query index below key index: masked
    sv[e] = __float_as_uint(pv);
    dv[e] = __float_as_uint(pv * fmaf(__uint_as_float(dv[e]), scale, -ds[e]));
  }
}
// dh = 64: dQ fused (TMEM S^T 128 + dP^T 128 + dV 64 + dK 64 + dQ 2x64 = 512
// columns) and Q / dO double-buffered. dh = 128: dV + dK take 256 columns, so
// this kernel computes dK / dV only (single-buffered Q / dO to fit 227 KB of
// smem) and attn_bwd_q_kernel produces dQ per query tile.
#ifndef B2S_ATTN_BWD_SPLIT_DQ
#define B2S_ATTN_BWD_SPLIT_DQ 0  // 1: dh = 64 also takes the separate query-tile dQ kernel
#endif
#ifndef B2S_ATTN_BWD_DQ_RED
#define B2S_ATTN_BWD_DQ_RED 0  // 1: dQ drained by red.global.add.v4.f32 from registers (no smem staging)
#endif
#ifndef B2S_ATTN_BWD_PT
#define B2S_ATTN_BWD_PT 1  // dh 64: P^T goes to TMEM (dV by the TMEM-A MMA form), single-buffered dQ
#endif
template <int DH>
struct Bwd {
  static constexpr bool DQ = DH == 64 && !B2S_ATTN_BWD_SPLIT_DQ;  // dQ fused into the key-tile kernel
  // P^T in TMEM columns [448, 512) (freed by a single dQ buffer): no P^T shared-memory
  // stores and no A-operand smem reads for dV -- the kernel is smem-bandwidth bound
  static constexpr bool PT = DQ && B2S_ATTN_BWD_PT;
  static constexpr int QS = DH == 64 ? 2 : 1; // Q / dO stages
  static constexpr int kTileQ = BQ * DH * 2;
  static constexpr int kSmem = 1024 + 2 * kTileQ /*K,V*/ + 2 * QS * kTileQ /*Q,dO*/ + (PT ? 1 : 2) * kPBuf /*P^T,dS^T*/ +
                               (DQ ? 2 * kTile : 0) /*dQ fp32 staging: 8 warps x 4 KB*/ + 4 * BQ * 4 /*LSE, D x2*/ +
                               256;
  static_assert(kSmem <= 232448, "backward tiles exceed shared memory");
};

template <int DH>
__global__ void __launch_bounds__(320, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dkv, Params p) {
  using C = Bwd<DH>;
  constexpr int kTQ = C::kTileQ, QS = C::QS, NA = DH / 64;
  constexpr bool DQ = C::DQ, PT = C::PT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sK = align1024(smem_raw);
  uint8_t* sV = sK + kTQ;
  uint8_t* sQ = sV + kTQ;            // [QS]
  uint8_t* sdO = sQ + QS * kTQ;      // [QS]
  uint8_t* sP = sdO + QS * kTQ;      // P^T  [128 keys][128 q] as two 64-column atoms (smem P only)
  uint8_t* sdS = sP + (PT ? 0 : kPBuf);  // dS^T
  uint8_t* sdQ = sdS + kPBuf;        // fp32 128 x 64 as two 32-column boxes (16 KB each), dh 64 only
  float* sLse = reinterpret_cast<float*>(sdQ + (DQ ? 2 * kTile : 0));  // [2][128] natural-log LSE (TMA bulk)
  float* sD = sLse + 2 * BQ;                                 // [2][128] rowsum(dO*O)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + 2 * BQ);
  uint64_t* kv_full = bars;
  uint64_t* qd_full = bars + 1;   // [2]
  uint64_t* qd_empty = bars + 3;  // [2]
  uint64_t* st_full = bars + 5;
  uint64_t* st_empty = bars + 6;
  uint64_t* pds_full = bars + 7;
  uint64_t* pds_empty = bars + 8;
  uint64_t* dq_full = bars + 9;   // [2]
  uint64_t* dq_empty = bars + 11; // [2]
  uint64_t* done = bars + 13;
  uint64_t* st_ld_full = bars + 14;   // [2] lse / D of a step landed
  uint64_t* st_ld_empty = bars + 16;  // [2] all compute warps done with them
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 18);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbk = p.B * p.Hkv;
  const int kt = (int)(blockIdx.x / nbk);  // kt = 0 has the most query tiles: launched first
  const int bk = blockIdx.x % nbk;
  const int b = bk / p.Hkv, kvh = bk % p.Hkv;
  const int G = p.Hq / p.Hkv;
  const int nq = p.nqt - kt;  // query tiles i = kt .. nqt-1
  const int nsteps = G * nq;
  const int krow0 = b * p.T + kt * BKV;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    mbar_init(kv_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&qd_full[s], 1); mbar_init(&qd_empty[s], 1); mbar_init(&dq_full[s], 1); mbar_init(&dq_empty[s], 8);
    }
    mbar_init(st_full, 1);
    mbar_init(st_empty, 8);
    mbar_init(pds_full, 8);
    mbar_init(pds_empty, 1);
    mbar_init(done, 1);
    for (int s = 0; s < 2; ++s) { mbar_init(&st_ld_full[s], 1); mbar_init(&st_ld_empty[s], 8); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  // dQ: [2] x 64 (dh 64 only), or [1] x 64 + P^T (bf16 pairs) in [448, 512) with PT
  const uint32_t tS = tbase, tdP = tbase + 128, tdV = tbase + 256, tdK = tbase + 256 + DH, tdQ = tbase + 384;
  const uint32_t tPT = tbase + 448;
  // dQ buffer / barrier of step t, and how many times that buffer was used before
  auto dq_buf = [&](int t) { return PT ? 0 : (t & 1); };
  auto dq_use = [&](int t) { return PT ? t : (t >> 1); };

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * kTQ);
      for (int a = 0; a < NA; ++a) {
        tma_load_2d(sK + a * kTile, &tm_qkv, kv_full, (p.Hq + kvh) * DH + a * 64, krow0);
        tma_load_2d(sV + a * kTile, &tm_qkv, kv_full, (p.Hq + p.Hkv + kvh) * DH + a * 64, krow0);
      }
      for (int t = 0; t < nsteps; ++t) {
        const int h = kvh * G + t / nq, i = kt + t % nq;
        const int s = t & 1;
        mbar_wait(&st_ld_empty[s], ((t >> 1) & 1) ^ 1);
        const size_t off = ((size_t)b * p.Hq + h) * p.T + (size_t)i * BQ;
        mbar_arrive_expect_tx(&st_ld_full[s], 2 * BQ * 4);
        bulk_load_1d(sLse + s * BQ, p.lse + off, BQ * 4, &st_ld_full[s]);
        bulk_load_1d(sD + s * BQ, p.dsum + off, BQ * 4, &st_ld_full[s]);
        const int qs = t % QS;
        mbar_wait(&qd_empty[qs], ((t / QS) & 1) ^ 1);
        mbar_arrive_expect_tx(&qd_full[qs], 2 * kTQ);
        for (int a = 0; a < NA; ++a) {
          tma_load_2d(sQ + qs * kTQ + a * kTile, &tm_qkv, &qd_full[qs], h * DH + a * 64, b * p.T + i * BQ);
          tma_load_2d(sdO + qs * kTQ + a * kTile, &tm_do, &qd_full[qs], h * DH + a * 64, b * p.T + i * BQ);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    {  // whole warp, converged; one lane elected per tcgen05 instruction
      constexpr uint32_t idSS = make_idesc_bf16(128, 128, false, false);  // S^T, dP^T
      constexpr uint32_t idKM = make_idesc_bf16(128, DH, false, true);    // dV, dK
      constexpr uint32_t idMM = make_idesc_bf16(128, DH, true, true);     // dQ
      const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aQ = smem_u32(sQ), adO = smem_u32(sdO);
      const uint32_t aP = smem_u32(sP), adS = smem_u32(sdS);
      auto issue_S = [&](int t) {
        const int qs = t % QS;
        mbar_wait(&qd_full[qs], (t / QS) & 1);
        if (t > 0) mbar_wait(st_empty, (t - 1) & 1);
        tc_fence_after();
        const uint32_t q_ = aQ + qs * kTQ, do_ = adO + qs * kTQ;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t ko = (kk >> 2) * kTile + (kk & 3) * 32;
          mma_bf16_ss_w(tS, make_sdesc(aK + ko, 16, 1024), make_sdesc(q_ + ko, 16, 1024), idSS, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t ko = (kk >> 2) * kTile + (kk & 3) * 32;
          mma_bf16_ss_w(tdP, make_sdesc(aV + ko, 16, 1024), make_sdesc(do_ + ko, 16, 1024), idSS, kk > 0);
        }
        mma_commit_w(st_full);
      };
      mbar_wait(kv_full, 0);
      issue_S(0);
      for (int t = 0; t < nsteps; ++t) {
        const int s = t & 1, qs = t % QS;
        const uint32_t q_ = aQ + qs * kTQ, do_ = adO + qs * kTQ;
        // with a single Q / dO stage, S(t+1) needs this step's dV / dK MMAs to have read Q(t) / dO(t)
        if (QS == 2 && t + 1 < nsteps) issue_S(t + 1);
        mbar_wait(pds_full, t & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BQ / 16; ++kk) {
          const uint64_t a_p = make_sdesc(aP + (kk >> 2) * kTile + (kk & 3) * 32, 16, 1024);
          const uint64_t a_ds = make_sdesc(adS + (kk >> 2) * kTile + (kk & 3) * 32, 16, 1024);
          if constexpr (PT)
            mma_bf16_ts_w(tdV, tPT + kk * 8, make_sdesc(do_ + kk * 2048, kTile, 1024), idKM, (t > 0 || kk > 0));
          else
            mma_bf16_ss_w(tdV, a_p, make_sdesc(do_ + kk * 2048, kTile, 1024), idKM, (t > 0 || kk > 0));
          mma_bf16_ss_w(tdK, a_ds, make_sdesc(q_ + kk * 2048, kTile, 1024), idKM, (t > 0 || kk > 0));
        }
        if constexpr (DQ) {
          mbar_wait(&dq_empty[dq_buf(t)], (dq_use(t) & 1) ^ 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk)
            mma_bf16_ss_w(tdQ + dq_buf(t) * DH, make_sdesc(adS + kk * 2048, kTile, 1024),
                          make_sdesc(aK + kk * 2048, kTile, 1024), idMM, kk > 0);
        }
        mma_commit_w(&qd_empty[qs]);
        mma_commit_w(pds_empty);
        if constexpr (DQ) mma_commit_w(&dq_full[dq_buf(t)]);
        if (QS == 1 && t + 1 < nsteps) issue_S(t + 1);
      }
      mma_commit_w(done);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ compute warps
    const int ct = threadIdx.x - 64;  // 0..255
    const int q4 = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = q4 * 32 + lane;  // key row (S^T / dP^T / dV / dK lanes) and query row (dQ lanes)
    const uint32_t lrow = (uint32_t)(q4 * 32) << 16;
    // dQ(t) (TMEM buffer t&1): each warp drains its own 32 query rows x 32 columns
    // through a private 4 KB staging tile and its own TMA add-reduce (no CTA-wide sync)
    uint8_t* mystage = sdQ + (warp - 2) * 4096;
    auto drain_dq = [&](int t) {
      if constexpr (!DQ) return;
      const int h = kvh * G + t / nq, i = kt + t % nq;
      mbar_wait(&dq_full[dq_buf(t)], dq_use(t) & 1);
      tc_fence_after();
      uint32_t qv[32];
      tmem_ld32(tdQ + lrow + dq_buf(t) * DH + half * 32, qv);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
#if B2S_ATTN_BWD_DQ_RED
      if (lane == 0) mbar_arrive(&dq_empty[dq_buf(t)]);
      // straight from registers: 8 x 16-byte fp32 add-reductions into this thread's query row
      float* dst = p.dq_acc + ((size_t)b * p.T + (size_t)i * BQ + r) * (p.Hq * DH) + h * DH + half * 32;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * c), "r"(qv[4 * c]),
                     "r"(qv[4 * c + 1]), "r"(qv[4 * c + 2]), "r"(qv[4 * c + 3])
                     : "memory");
      return;
#endif
      if (lane == 0) {
        mbar_arrive(&dq_empty[dq_buf(t)]);
        bulk_wait_read<0>();  // this warp's previous add-reduce has read its staging tile
      }
      __syncwarp();
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<float4*>(mystage + swz(lane, c)) =
            make_float4(__uint_as_float(qv[4 * c]), __uint_as_float(qv[4 * c + 1]), __uint_as_float(qv[4 * c + 2]),
                        __uint_as_float(qv[4 * c + 3]));  // dS is pre-scaled
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
#ifndef B2S_EXP_NO_DQ_REDUCE  // timing experiment only: dQ not accumulated
        tma_reduce_add_2d(&tm_dq, mystage, h * DH + half * 32, b * p.T + i * BQ + q4 * 32);
#endif
        bulk_commit();
      }
    };
    for (int t = 0; t < nsteps; ++t) {
      const int i = kt + t % nq;
      const bool diag = (i == kt);
      mbar_wait(&st_ld_full[t & 1], (t >> 1) & 1);
      const float* lse2 = sLse + (t & 1) * BQ;  // natural log; p_ds folds in log2(e)
      const float* dd = sD + (t & 1) * BQ;
      mbar_wait(st_full, t & 1);
      tc_fence_after();
      // 168 registers per thread (3 warps on some SMSPs): two 32-column passes
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        uint32_t sv[32], dv[32], pt[16];
        tmem_ld32(tS + lrow + half * 64 + qq * 32, sv);
        tmem_ld32(tdP + lrow + half * 64 + qq * 32, dv);
        tmem_wait_ld();
        if (qq == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(st_empty);  // the next step's S^T / dP^T may overwrite TMEM
        }
#ifndef B2S_EXP_NOCOMPUTE  // timing experiment only: protocol without the softmax math / P, dS stores
        if (diag) p_ds<true>(sv, dv, half * 64 + qq * 32, r, p.scale_log2, p.scale, lse2, dd);
        else p_ds<false>(sv, dv, half * 64 + qq * 32, r, p.scale_log2, p.scale, lse2, dd);
#endif
#ifndef B2S_EXP_NO_PDS_WAIT  // timing experiment only: races on sP / sdS
        if (qq == 0 && t > 0) mbar_wait(pds_empty, (t - 1) & 1);  // step t-1's MMAs released sP / sdS
#endif
#ifndef B2S_EXP_NOCOMPUTE
#pragma unroll
        for (int k8 = 0; k8 < 4; ++k8) {
          uint4 w, z;
          w.x = pack_bf16x2(__uint_as_float(sv[8 * k8 + 0]), __uint_as_float(sv[8 * k8 + 1]));
          w.y = pack_bf16x2(__uint_as_float(sv[8 * k8 + 2]), __uint_as_float(sv[8 * k8 + 3]));
          w.z = pack_bf16x2(__uint_as_float(sv[8 * k8 + 4]), __uint_as_float(sv[8 * k8 + 5]));
          w.w = pack_bf16x2(__uint_as_float(sv[8 * k8 + 6]), __uint_as_float(sv[8 * k8 + 7]));
          z.x = pack_bf16x2(__uint_as_float(dv[8 * k8 + 0]), __uint_as_float(dv[8 * k8 + 1]));
          z.y = pack_bf16x2(__uint_as_float(dv[8 * k8 + 2]), __uint_as_float(dv[8 * k8 + 3]));
          z.z = pack_bf16x2(__uint_as_float(dv[8 * k8 + 4]), __uint_as_float(dv[8 * k8 + 5]));
          z.w = pack_bf16x2(__uint_as_float(dv[8 * k8 + 6]), __uint_as_float(dv[8 * k8 + 7]));
          const uint32_t off = half * kTile + swz(r, qq * 4 + k8);
          if constexpr (PT) {
            pt[4 * k8 + 0] = w.x; pt[4 * k8 + 1] = w.y; pt[4 * k8 + 2] = w.z; pt[4 * k8 + 3] = w.w;
          } else {
            *reinterpret_cast<uint4*>(sP + off) = w;
          }
          *reinterpret_cast<uint4*>(sdS + off) = z;
        }
        if constexpr (PT) tmem_st16(tPT + lrow + half * 32 + qq * 16, pt);
#else
        if (lane == 99) *reinterpret_cast<uint32_t*>(sP) = sv[0] + dv[7];
#endif
      }
      if constexpr (PT) {
        tmem_wait_st();  // P^T is in TMEM before the MMA warp is told
        tc_fence_before();
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(pds_full);
        mbar_arrive(&st_ld_empty[t & 1]);
      }
#ifndef B2S_EXP_NODQ
      if (t > 0) drain_dq(t - 1);
#else
      if (t > 0) { mbar_wait(&dq_full[(t - 1) & 1], ((t - 1) >> 1) & 1); tc_fence_after(); __syncwarp(); if (lane == 0) mbar_arrive(&dq_empty[(t - 1) & 1]); }
#endif
    }
#ifndef B2S_EXP_NODQ
    if (nsteps > 0) drain_dq(nsteps - 1);
#else
    if (nsteps > 0) { mbar_wait(&dq_full[(nsteps - 1) & 1], ((nsteps - 1) >> 1) & 1); if (lane == 0) mbar_arrive(&dq_empty[(nsteps - 1) & 1]); }
#endif
    if (DQ && lane == 0) bulk_wait_read<0>();  // this warp's add-reduces have read their staging smem (kernel exit orders their writes)
    __syncwarp();
    // dK (from the pre-scaled dS) and dV -> bf16 -> smem (Q / dO stages are free) -> TMA store into dqkv
    mbar_wait(done, 0);
    tc_fence_after();
    uint8_t* sdK_out = sQ;
    uint8_t* sdV_out = DQ ? sQ + kTile : sdO;
#pragma unroll
    for (int cc = 0; cc < DH / 64; ++cc) {  // this warp's half of the DH columns, 32 at a time
      const int col0 = half * (DH / 2) + cc * 32;
      uint32_t kv[32], vv[32];
      tmem_ld32(tdK + lrow + col0, kv);
      tmem_ld32(tdV + lrow + col0, vv);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint4 w, z;
        w.x = pack_bf16x2(__uint_as_float(kv[8 * c + 0]), __uint_as_float(kv[8 * c + 1]));
        w.y = pack_bf16x2(__uint_as_float(kv[8 * c + 2]), __uint_as_float(kv[8 * c + 3]));
        w.z = pack_bf16x2(__uint_as_float(kv[8 * c + 4]), __uint_as_float(kv[8 * c + 5]));
        w.w = pack_bf16x2(__uint_as_float(kv[8 * c + 6]), __uint_as_float(kv[8 * c + 7]));
        z.x = pack_bf16x2(__uint_as_float(vv[8 * c + 0]), __uint_as_float(vv[8 * c + 1]));
        z.y = pack_bf16x2(__uint_as_float(vv[8 * c + 2]), __uint_as_float(vv[8 * c + 3]));
        z.z = pack_bf16x2(__uint_as_float(vv[8 * c + 4]), __uint_as_float(vv[8 * c + 5]));
        z.w = pack_bf16x2(__uint_as_float(vv[8 * c + 6]), __uint_as_float(vv[8 * c + 7]));
        const int chunk = col0 / 8 + c;  // 16-byte chunk of the row: atom chunk / 8, position chunk % 8
        *reinterpret_cast<uint4*>(sdK_out + (chunk >> 3) * kTile + swz(r, chunk & 7)) = w;
        *reinterpret_cast<uint4*>(sdV_out + (chunk >> 3) * kTile + swz(r, chunk & 7)) = z;
      }
    }
    fence_proxy_async_smem();
    named_sync(1, 256);
    if (ct == 0) {
      for (int a = 0; a < NA; ++a) {
        tma_store_2d(&tm_dkv, sdK_out + a * kTile, (p.Hq + kvh) * DH + a * 64, krow0);
        tma_store_2d(&tm_dkv, sdV_out + a * kTile, (p.Hq + p.Hkv + kvh) * DH + a * 64, krow0);
      }
      bulk_commit();
      bulk_wait_read<0>();
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

// -------------------------------------------------------------------------------------
// dQ for dh = 128: CTA = (batch, q head, 128-query tile), looping over the causal key
// tiles j <= i. S = Q K_j^T and dP = dO V_j^T into TMEM, thread = query row:
// dS = P (dP - D) -> bf16 -> smem, dQ += dS K_j (TMEM accumulator across the loop,
// K_j as an MN-major operand) -> x scale -> bf16 -> TMA store into dqkv.
// smem 224 KB: Q, dO (32 KB each), K / V 2 stages (128 KB), dS (32 KB).
template <int DH>
struct BwdQ {
  static constexpr int kTileQ = BQ * DH * 2;
  static constexpr int kSmem = 1024 + 2 * kTileQ + 2 * kStages * kTileQ + kPBuf + 256;
  static_assert(kSmem <= 232448, "dQ tiles exceed shared memory");
};

template <int DH>
__global__ void __launch_bounds__(320, 1)
    attn_bwd_q_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                      const __grid_constant__ CUtensorMap tm_dqkv, Params p) {
  constexpr int kTQ = BwdQ<DH>::kTileQ, NA = DH / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sQ = align1024(smem_raw);
  uint8_t* sdO = sQ + kTQ;
  uint8_t* sK = sdO + kTQ;              // [kStages]
  uint8_t* sV = sK + kStages * kTQ;     // [kStages]
  uint8_t* sdS = sV + kStages * kTQ;    // dS [128 q][128 keys], two 64-key atoms
  uint64_t* bars = reinterpret_cast<uint64_t*>(sdS + kPBuf);
  uint64_t* qd_full = bars;
  uint64_t* k_full = bars + 1;          // [kStages]
  uint64_t* v_full = k_full + kStages;  // [kStages]
  uint64_t* kv_empty = v_full + kStages;
  uint64_t* st_full = kv_empty + kStages;
  uint64_t* st_empty = st_full + 1;
  uint64_t* pds_full = st_empty + 1;
  uint64_t* pds_empty = pds_full + 1;
  uint64_t* done = pds_empty + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbh = p.B * p.Hq;
  const int i = p.nqt - 1 - (int)(blockIdx.x / nbh);  // heaviest query tiles first
  const int bh = blockIdx.x % nbh;
  const int b = bh / p.Hq, h = bh % p.Hq;
  const int kvh = h / (p.Hq / p.Hkv);
  const int nkv = i + 1;
  const int qrow0 = b * p.T + i * BQ;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    mbar_init(qd_full, 1);
    for (int s = 0; s < kStages; ++s) { mbar_init(&k_full[s], 1); mbar_init(&v_full[s], 1); mbar_init(&kv_empty[s], 1); }
    mbar_init(st_full, 1);
    mbar_init(st_empty, 8);
    mbar_init(pds_full, 8);
    mbar_init(pds_empty, 1);
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t tS = tbase, tdP = tbase + 128, tdQ = tbase + 256;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(qd_full, 2 * kTQ);
      for (int a = 0; a < NA; ++a) {
        tma_load_2d(sQ + a * kTile, &tm_qkv, qd_full, h * DH + a * 64, qrow0);
        tma_load_2d(sdO + a * kTile, &tm_do, qd_full, h * DH + a * 64, qrow0);
      }
      for (int j = 0; j < nkv; ++j) {
        const int s = j % kStages;
        mbar_wait(&kv_empty[s], ((j / kStages) & 1) ^ 1);
        const int r = b * p.T + j * BKV;
        mbar_arrive_expect_tx(&k_full[s], kTQ);
        for (int a = 0; a < NA; ++a)
          tma_load_2d(sK + s * kTQ + a * kTile, &tm_qkv, &k_full[s], (p.Hq + kvh) * DH + a * 64, r);
        mbar_arrive_expect_tx(&v_full[s], kTQ);
        for (int a = 0; a < NA; ++a)
          tma_load_2d(sV + s * kTQ + a * kTile, &tm_qkv, &v_full[s], (p.Hq + p.Hkv + kvh) * DH + a * 64, r);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    {
      constexpr uint32_t idSS = make_idesc_bf16(BQ, BKV, false, false);  // S, dP
      constexpr uint32_t idQ = make_idesc_bf16(BQ, DH, false, true);     // dQ += dS K (K MN-major)
      const uint32_t aQ = smem_u32(sQ), adO = smem_u32(sdO), aK = smem_u32(sK), aV = smem_u32(sV);
      const uint32_t adS = smem_u32(sdS);
      auto issue_S = [&](int j) {
        const int s = j % kStages;
        mbar_wait(&k_full[s], (j / kStages) & 1);
        mbar_wait(&v_full[s], (j / kStages) & 1);
        if (j > 0) mbar_wait(st_empty, (j - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t ko = (kk >> 2) * kTile + (kk & 3) * 32;
          mma_bf16_ss_w(tS, make_sdesc(aQ + ko, 16, 1024), make_sdesc(aK + s * kTQ + ko, 16, 1024), idSS, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t ko = (kk >> 2) * kTile + (kk & 3) * 32;
          mma_bf16_ss_w(tdP, make_sdesc(adO + ko, 16, 1024), make_sdesc(aV + s * kTQ + ko, 16, 1024), idSS,
                        kk > 0);
        }
        mma_commit_w(st_full);
      };
      mbar_wait(qd_full, 0);
      issue_S(0);
      for (int j = 0; j < nkv; ++j) {
        const int s = j % kStages;
        if (j + 1 < nkv) issue_S(j + 1);
        mbar_wait(pds_full, j & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)
          mma_bf16_ss_w(tdQ, make_sdesc(adS + (kk >> 2) * kTile + (kk & 3) * 32, 16, 1024),
                        make_sdesc(aK + s * kTQ + kk * 2048, kTile, 1024), idQ, (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit_w(pds_empty);
        mma_commit_w(&kv_empty[s]);
      }
      mma_commit_w(done);
    }
    __syncwarp();
  } else {
    const int ct = threadIdx.x - 64;
    const int q4 = warp & 3;
    const int half = (warp - 2) >> 2;  // key columns half*64 .. +63
    const int r = q4 * 32 + lane;      // query row
    const uint32_t lrow = (uint32_t)(q4 * 32) << 16;
    const size_t roff = ((size_t)b * p.Hq + h) * p.T + (size_t)i * BQ + r;
    const float lse2 = p.lse[roff];  // log2 units (prep kernel)
    const float dd = p.dsum[roff];
    const float sl2 = p.scale_log2;
    for (int j = 0; j < nkv; ++j) {
      const bool diag = (j == i);
      mbar_wait(st_full, j & 1);
      tc_fence_after();
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        uint32_t sv[32], dv[32];
        tmem_ld32(tS + lrow + half * 64 + qq * 32, sv);
        tmem_ld32(tdP + lrow + half * 64 + qq * 32, dv);
        tmem_wait_ld();
        if (qq == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(st_empty);
        }
        const int k0 = half * 64 + qq * 32;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          float pv = ex2(fmaf(__uint_as_float(sv[e]), sl2, -lse2));
          if (diag && k0 + e > r) pv = 0.f;  // key after query: masked
          dv[e] = __float_as_uint(pv * fmaf(__uint_as_float(dv[e]), p.scale, -dd));  // scaled dS
        }
        if (qq == 0 && j > 0) mbar_wait(pds_empty, (j - 1) & 1);
#pragma unroll
        for (int k8 = 0; k8 < 4; ++k8) {
          uint4 z;
          z.x = pack_bf16x2(__uint_as_float(dv[8 * k8 + 0]), __uint_as_float(dv[8 * k8 + 1]));
          z.y = pack_bf16x2(__uint_as_float(dv[8 * k8 + 2]), __uint_as_float(dv[8 * k8 + 3]));
          z.z = pack_bf16x2(__uint_as_float(dv[8 * k8 + 4]), __uint_as_float(dv[8 * k8 + 5]));
          z.w = pack_bf16x2(__uint_as_float(dv[8 * k8 + 6]), __uint_as_float(dv[8 * k8 + 7]));
          *reinterpret_cast<uint4*>(sdS + half * kTile + swz(r, qq * 4 + k8)) = z;
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(pds_full);
    }
    // dQ (TMEM) * scale -> bf16 -> smem (Q / dO are free once every MMA retired) -> TMA store
    mbar_wait(done, 0);
    tc_fence_after();
#pragma unroll
    for (int cc = 0; cc < DH / 64; ++cc) {
      const int col0 = half * (DH / 2) + cc * 32;
      uint32_t qv[32];
      tmem_ld32(tdQ + lrow + col0, qv);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint4 w;
        w.x = pack_bf16x2(__uint_as_float(qv[8 * c + 0]), __uint_as_float(qv[8 * c + 1]));
        w.y = pack_bf16x2(__uint_as_float(qv[8 * c + 2]), __uint_as_float(qv[8 * c + 3]));
        w.z = pack_bf16x2(__uint_as_float(qv[8 * c + 4]), __uint_as_float(qv[8 * c + 5]));
        w.w = pack_bf16x2(__uint_as_float(qv[8 * c + 6]), __uint_as_float(qv[8 * c + 7]));
        const int chunk = col0 / 8 + c;
        *reinterpret_cast<uint4*>(sQ + (chunk >> 3) * kTile + swz(r, chunk & 7)) = w;
      }
    }
    fence_proxy_async_smem();
    named_sync(1, 256);
    if (ct == 0) {
      for (int a = 0; a < NA; ++a) tma_store_2d(&tm_dqkv, sQ + a * kTile, h * DH + a * 64, qrow0);
      bulk_commit();
      bulk_wait_read<0>();
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

}  // namespace attn
}  // namespace b2s

using namespace b2s;

namespace {
template <int DH>
int attn_fwd_dh(const void* d_qkv, void* d_o, float* d_lse, int B, int T, int Hq, int Hkv, cudaStream_t st) {
  using C = attn::Fwd<DH>;
  const int ldq = (Hq + 2 * Hkv) * DH;
  CUtensorMap tq, to;
  int rc = encode_tma_2d(&tq, d_qkv, 2, (uint64_t)ldq, (uint64_t)B * T, (uint64_t)ldq * 2, 64, 128, 128);
  if (rc) return rc;
  rc = encode_tma_2d(&to, d_o, 2, (uint64_t)Hq * DH, (uint64_t)B * T, (uint64_t)Hq * DH * 2, 64, 128, 128);
  if (rc) return rc;
  attn::Params p{B, T, Hq, Hkv, T / attn::BQ, attn::kLog2e / sqrtf((float)DH), 1.f / sqrtf((float)DH), d_lse,
                 nullptr, nullptr};
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn::attn_fwd_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    attr = true;
  }
  const unsigned grid = (unsigned)(B * Hq * ((T / attn::BQ + C::TILES - 1) / C::TILES));
  attn::attn_fwd_kernel<DH><<<grid, C::kThreads, C::kSmem, st>>>(tq, to, p);
  return check_launch("attn_fwd");
}

template <int DH>
int attn_bwd_dh(const void* d_qkv, const void* d_o, const void* d_do, const float* d_lse, void* d_dqkv,
                float* d_work, int B, int T, int Hq, int Hkv, cudaStream_t st) {
  using C = attn::Bwd<DH>;
  const int ldq = (Hq + 2 * Hkv) * DH;
  const int64_t M = (int64_t)B * T;
  float* dq_acc = C::DQ ? d_work : nullptr;
  float* dsum = d_work + M * Hq * DH;
  float* lse2 = dsum + M * Hq;
  attn::attn_bwd_prep_kernel<DH><<<kNumSMs * 8, 256, 0, st>>>(
      (const __nv_bfloat16*)d_o, (const __nv_bfloat16*)d_do, d_lse, dsum, lse2, dq_acc, B, T, Hq,
      1.f / sqrtf((float)DH));
  int rc = check_launch("attn_bwd_prep");
  if (rc) return rc;
  CUtensorMap tq, tdo, tdq, tdkv;
  rc = encode_tma_2d(&tq, d_qkv, 2, (uint64_t)ldq, (uint64_t)M, (uint64_t)ldq * 2, 64, 128, 128);
  if (rc) return rc;
  rc = encode_tma_2d(&tdo, d_do, 2, (uint64_t)Hq * DH, (uint64_t)M, (uint64_t)Hq * DH * 2, 64, 128, 128);
  if (rc) return rc;
  rc = encode_tma_2d(&tdq, d_work, 4, (uint64_t)Hq * DH, (uint64_t)M, (uint64_t)Hq * DH * 4, 32, 32, 128);
  if (rc) return rc;
  rc = encode_tma_2d(&tdkv, d_dqkv, 2, (uint64_t)ldq, (uint64_t)M, (uint64_t)ldq * 2, 64, 128, 128);
  if (rc) return rc;
  attn::Params p{B, T, Hq, Hkv, T / attn::BQ, attn::kLog2e / sqrtf((float)DH), 1.f / sqrtf((float)DH), lse2,
                 dsum, dq_acc};
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn::attn_bwd_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if constexpr (!C::DQ)
      cudaFuncSetAttribute(attn::attn_bwd_q_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           attn::BwdQ<DH>::kSmem);
    attr = true;
  }
  const unsigned grid = (unsigned)(B * Hkv * (T / attn::BQ));
  attn::attn_bwd_kernel<DH><<<grid, attn::kBwdThreads, C::kSmem, st>>>(tq, tdo, tdq, tdkv, p);
  rc = check_launch("attn_bwd");
  if (rc) return rc;
  if constexpr (C::DQ) {
    attn::attn_bwd_dq_kernel<<<(unsigned)(M < kNumSMs * 16 ? M : kNumSMs * 16), 256, 0, st>>>(
        dq_acc, (__nv_bfloat16*)d_dqkv, M, Hq, ldq);
    return check_launch("attn_bwd_dq");
  } else {
    attn::attn_bwd_q_kernel<DH><<<(unsigned)(B * Hq * (T / attn::BQ)), 320, attn::BwdQ<DH>::kSmem, st>>>(tq, tdo,
                                                                                                       tdkv, p);
    return check_launch("attn_bwd_q");
  }
}
}  // namespace

extern "C" int b2s_attn_fwd(const void* d_qkv, void* d_o, float* d_lse, int B, int T, int Hq, int Hkv, int dh,
                            b2s_stream_t stream) {
  B2S_REQUIRE(dh == 64 || dh == 128, B2S_EUNSUPPORTED, "attention: head dim %d not implemented (64, 128)", dh);
  B2S_REQUIRE(T % attn::BQ == 0 && T > 0, B2S_EUNSUPPORTED, "attention: T must be a multiple of 128");
  B2S_REQUIRE(Hkv > 0 && Hq % Hkv == 0, B2S_EINVAL, "attention: Hq must be a multiple of Hkv");
  cudaStream_t st = (cudaStream_t)stream;
  return dh == 64 ? attn_fwd_dh<64>(d_qkv, d_o, d_lse, B, T, Hq, Hkv, st)
                  : attn_fwd_dh<128>(d_qkv, d_o, d_lse, B, T, Hq, Hkv, st);
}

extern "C" int64_t b2s_attn_bwd_work_floats(int B, int T, int Hq, int dh) {
  return (int64_t)B * T * Hq * dh + 2 * (int64_t)B * Hq * T;  // dQ acc | D' | lse2
}

extern "C" int b2s_attn_bwd(const void* d_qkv, const void* d_o, const void* d_do, const float* d_lse, void* d_dqkv,
                            float* d_work, int B, int T, int Hq, int Hkv, int dh, b2s_stream_t stream) {
  B2S_REQUIRE(dh == 64 || dh == 128, B2S_EUNSUPPORTED, "attention: head dim %d not implemented (64, 128)", dh);
  B2S_REQUIRE(T % attn::BQ == 0 && T > 0, B2S_EUNSUPPORTED, "attention: T must be a multiple of 128");
  B2S_REQUIRE(Hkv > 0 && Hq % Hkv == 0, B2S_EINVAL, "attention: Hq must be a multiple of Hkv");
  B2S_REQUIRE((int64_t)B * T * Hq < (1LL << 32), B2S_EUNSUPPORTED, "attention: B*T*Hq must be < 2^32");
  cudaStream_t st = (cudaStream_t)stream;
  return dh == 64 ? attn_bwd_dh<64>(d_qkv, d_o, d_do, d_lse, d_dqkv, d_work, B, T, Hq, Hkv, st)
                  : attn_bwd_dh<128>(d_qkv, d_o, d_do, d_lse, d_dqkv, d_work, B, T, Hq, Hkv, st);
}
