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
// Forward: persistent, one CTA per SM working through (batch, q head, pair of 128-query
// tiles) items heaviest first (see "forward (persistent)" below): S = QK^T and O = PV in TMEM,
// P = 2^(S*scale*log2e - m) in TMEM (TMEM-A MMA form), lazy O rescale, one MMA issuer per
// query tile and the two tiles' softmax warpgroups alternating on the MUFU.
//
// Backward CTA = (batch, kv head, 128-key tile), looping over the q heads of
// its group and the causal query tiles: S^T = K Q^T, dP^T = V dO^T (TMEM),
// P^T and dS^T = P^T (dP^T - D) (thread = key row), then dV += P^T dO, dK += dS^T Q
// (TMEM accumulators across the loop).
//   dh 64 (attn_bwd_kernel): P^T to TMEM (TMEM-A dV), dS^T to smem, and dQ_i = dS K fused
//   (TMEM) -> fp32 smem -> TMA add-reduce into a dQ accumulator.
//   dh 128 (attn_bwd128_kernel + attn_bwd_q_kernel): the key-tile kernel writes P^T / dS^T back
//   over the S^T / dP^T columns (TMEM-A dV and dK), and a query-tile kernel recomputes S / dP
//   and accumulates dQ in TMEM (dS in TMEM, TMEM-A dQ MMA).
#include <mutex>
#include "common.cuh"
#include "sm100.cuh"

namespace b2s {
using namespace sm100;
namespace attn {

constexpr int BQ = 128, BKV = 128;

constexpr int kTile = BQ * 64 * 2;  // 16 KB: one 128-row x 64-column bf16 swizzle atom
constexpr int kPBuf = BQ * BKV * 2; // 32 KB: a 128 x 128 bf16 P tile (two atoms)
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
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct Params {
  int B, T, Hq, Hkv, nqt;
  float scale_log2;  // log2(e) / sqrt(dh)
  float scale;       // 1 / sqrt(dh)
  float* lse;        // [B, Hq, T]
  const float* dsum; // bwd: D = rowsum(dO * O), [B, Hq, T]
  float* dq_acc;     // bwd (dh 64): fp32 dQ accumulator [B*T, Hq*dh]
  int* sched;        // persistent kernels: {next work item, CTAs done} (zero between launches)
};

// Timeline tracing of the forward's roles (experiment builds: -DB2S_ATTN_TRACE; see
// tools/attn_trace.py): lane 0 of each warp of CTAs 0..kTraceCtas-1 records (clock64, event).
#ifdef B2S_ATTN_TRACE
constexpr int kTraceCtas = 4, kTraceRecs = 8192;
__device__ unsigned long long g_trace[kTraceCtas][18][kTraceRecs][2];
#define TRACE(ev, aux)                                                                              \
  do {                                                                                              \
    if (blockIdx.x < kTraceCtas && lane == 0 && tr_n < kTraceRecs) {                                \
      g_trace[blockIdx.x][warp][tr_n][0] = clock64();                                               \
      g_trace[blockIdx.x][warp][tr_n][1] = ((unsigned long long)(ev) << 32) | (unsigned)(aux);     \
      ++tr_n;                                                                                       \
    }                                                                                               \
  } while (0)
#else
#define TRACE(ev, aux) \
  do {                 \
  } while (0)
#endif

// =====================================================================================
// forward (persistent)
// =====================================================================================
// Grid = one CTA per SM. A work item is (batch, q head, pair of 128-query tiles A = 2p,
// B = 2p+1); items are numbered heaviest pair first and handed out by a global atomic
// counter (longest-processing-time order: the tail is one light item, and CTAs that start
// late -- SMs held by NCCL kernels on the comm stream -- take fewer items). The producer
// warp fetches the next item index one item ahead and publishes it through a smem ring to
// the MMA and softmax warps, so the next item's Q / K / V loads and its first QK^T run
// while the current item's last blocks and epilogue finish (a non-persistent grid exposes
// that prologue once per item: ~10% of the dh-64 forward).
// Roles: warp0 TMA, warp1 MMA, warps 2-5 softmax of tile A, warps 6-9 of tile B (one
// query row per thread, the row is a TMEM lane). Per KV block j of an item:
//   S_t(j) = Q_t K_j^T -> TMEM;  P_t = 2^(S_t*scale*log2e - m) -> bf16 -> TMEM;
//   O_t += P_t V_j (TMEM-A MMA form, V as an MN-major operand).
// O accumulates in TMEM; a softmax thread rescales its O row (tcgen05.ld / st) only when
// its running max grows by more than 2^8 -- otherwise P is formed against the stale max and
// stays <= 256 -- so the softmax loop rarely waits on the PV MMA it just enabled.
// TMEM columns: dh 64: S_A [0,128) S_B [128,256) O_A [256,320) O_B [320,384) P_A [384,448)
//   P_B [448,512); MMA order S_A(j+1) S_B(j+1) PV_A(j) PV_B(j).
// dh 128: S_A [0,128) S_B [128,256) O_A [256,384) O_B [384,512), P_t written over S_t's
//   columns; MMA order PV_A(j) S_A(j+1) PV_B(j) S_B(j+1) (the tensor pipe runs one CTA's
//   MMAs in issue order, so S_t(j+1) overwrites P_t(j) only after PV_t(j) read it).
// The item's O is normalised by the softmax warps, staged through that item's Q buffer
// (Q is double-buffered across items) and written by TMA.
template <int DH>
struct Fwd {
  static constexpr bool ALIAS = DH == 128;      // P over S (dh 128: O takes 2 x 128 columns)
  static constexpr bool kFusedMax = DH == 128;  // block max inside the exponential loop (see below)
  // K / V stages: the K load of block j + KVS waits for both tiles' PV(j); two stages leave it
  // about one softmax period of TMA latency, which is not enough at dh 64 (dh 128 has no room)
  static constexpr int KVS = DH == 64 ? 4 : 2;
  static constexpr int kThreads = 352;          // TMA, MMA(A), 8 softmax warps, MMA(B)
  static constexpr int kTileQ = BQ * DH * 2;    // Q / K / V tile bytes (DH/64 swizzle atoms)
  static constexpr int OCOL = 256;              // first O column
  static constexpr int pcol(int t) { return ALIAS ? t * BKV : OCOL + 2 * DH + t * 64; }
  static constexpr int kRing = 4;               // item-index ring depth
  // Q buffers (item-level double buffering; dh 128 has room for one: the next item's Q then
  // loads once the current item's O stores have read their staging)
  static constexpr int QB = DH == 64 ? 2 : 1;
  static constexpr int kSmem = 1024 + QB * 2 * kTileQ /*Q: QB items x 2 tiles*/ + 2 * KVS * kTileQ + 512;
  static_assert(kSmem <= 232448, "forward tiles exceed shared memory");
  static_assert(KVS >= 2 && KVS <= 4, "K / V stages: 2..4 barrier slots");
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

// P = 2^(s*sl2 - m) for all BKV columns of one row, packed as bf16 pairs into out[0 .. BKV/2)
// (out may alias v: pair k is written after v[2k], v[2k+1] are read); returns the row sum.
// The causal mask is a template branch so off-diagonal blocks run the mask-free stream.
// Packed fp32 pairs (FFMA2 / FADD2, sm_100): two elements per issue slot in the forward's
// exponential stream, whose non-MUFU instructions compete for issue with the other tile's group
// (Llama-8B forward 272 -> 269 us, 1B unchanged; the same packing in the backward's P / dS
// streams measured slower: 1B 836 -> 842 us, dh 128 824 -> 852 us).
__device__ __forceinline__ float2 f2(uint32_t a, uint32_t b) { return make_float2(__uint_as_float(a), __uint_as_float(b)); }
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

template <bool DIAG>
__device__ __forceinline__ float exp_pack_regs(const uint32_t* v, int r, float sl2, float m, uint32_t* out) {
  // row sum as 2 x 2 independent partial sums combined by a tree: a single serial FADD chain
  // over 128 elements would be longer than the MUFU work it follows
  const float2 sc2 = f2(sl2), nm2 = f2(-m);
  float2 rs2[2] = {f2(0.f), f2(0.f)};
#pragma unroll
  for (int k8 = 0; k8 < BKV / 8; ++k8) {
    float2 e[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 x = __ffma2_rn(f2(v[k8 * 8 + 2 * i], v[k8 * 8 + 2 * i + 1]), sc2, nm2);
      e[i] = make_float2(ex2(x.x), ex2(x.y));
      if (DIAG && k8 * 8 + 2 * i > r) e[i].x = 0.f;
      if (DIAG && k8 * 8 + 2 * i + 1 > r) e[i].y = 0.f;
    }
    rs2[k8 & 1] = __fadd2_rn(rs2[k8 & 1], __fadd2_rn(__fadd2_rn(e[0], e[1]), __fadd2_rn(e[2], e[3])));
#pragma unroll
    for (int i = 0; i < 4; ++i) out[k8 * 4 + i] = pack_bf16x2(e[i].x, e[i].y);
  }
  const float2 t = __fadd2_rn(rs2[0], rs2[1]);
  return t.x + t.y;
}

// Same, against the running max m of the previous blocks, without a separate row-max pass:
// xmax returns max(s*sl2 - m) over the row's unmasked columns. When it is <= kRescaleThresh the
// P values are <= 2^8 exactly as if the row max had been taken first (lazy rescale); otherwise
// the caller shifts m by an integer k >= xmax and scales P, the sum and O by 2^-k (exact in
// bf16 / fp32). P <= 2^xmax meanwhile: finite for xmax < 128 (log2 units).
template <bool DIAG>
__device__ __forceinline__ float exp_pack_regs_mx(const uint32_t* v, int r, float sl2, float m, uint32_t* out,
                                                  float& xmax) {
  const float2 sc2 = f2(sl2), nm2 = f2(-m);
  float2 rs2[2] = {f2(0.f), f2(0.f)};
  float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
  for (int k8 = 0; k8 < BKV / 8; ++k8) {
    float2 x[4], e[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      x[i] = __ffma2_rn(f2(v[k8 * 8 + 2 * i], v[k8 * 8 + 2 * i + 1]), sc2, nm2);
      if (DIAG && k8 * 8 + 2 * i > r) x[i].x = -INFINITY;  // masked: exp 0, not in the max
      if (DIAG && k8 * 8 + 2 * i + 1 > r) x[i].y = -INFINITY;
      e[i] = make_float2(ex2(x[i].x), ex2(x[i].y));
    }
    mx4[k8 & 3] = fmax3(mx4[k8 & 3], fmax3(x[0].x, x[0].y, x[1].x), fmax3(x[1].y, x[2].x, x[2].y));
    mx4[k8 & 3] = fmax3(mx4[k8 & 3], x[3].x, x[3].y);
    rs2[k8 & 1] = __fadd2_rn(rs2[k8 & 1], __fadd2_rn(__fadd2_rn(e[0], e[1]), __fadd2_rn(e[2], e[3])));
#pragma unroll
    for (int i = 0; i < 4; ++i) out[k8 * 4 + i] = pack_bf16x2(e[i].x, e[i].y);
  }
  xmax = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
  const float2 t = __fadd2_rn(rs2[0], rs2[1]);
  return t.x + t.y;
}

template <int DH>
__global__ void __launch_bounds__(Fwd<DH>::kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_o,
                    Params p) {
  using C = Fwd<DH>;
  constexpr int kTQ = C::kTileQ, NA = DH / 64, KVS = C::KVS, R = C::kRing, QB = C::QB;  // NA: atoms per tile
  constexpr int kThreadsMMA2 = C::kThreads - 32;  // first thread of the tile-B MMA warp
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sQ = align1024(smem_raw);  // [item buffer][tile]
  uint8_t* sK = sQ + QB * 2 * kTQ;    // [KVS]
  uint8_t* sV = sK + KVS * kTQ;       // [KVS]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + KVS * kTQ);
  uint64_t* q_full = bars;             // [2] item buffer loaded
  uint64_t* q_empty = bars + 2;        // [2] item buffer's O staging read by the stores (2 tiles)
  uint64_t* k_full = bars + 4;         // [KVS]
  uint64_t* v_full = k_full + 4;       // [KVS]
  uint64_t* kv_empty = v_full + 4;     // [KVS]
  uint64_t* s_full = kv_empty + 4;     // [tile]
  uint64_t* s_empty = s_full + 2;      // [tile]
  uint64_t* p_full = s_empty + 2;      // [tile]
  uint64_t* p_empty = p_full + 2;      // [tile] PV retired: P may be rewritten
  uint64_t* pv_done = p_empty + 2;     // [tile] each PV retired (rescale fence)
  uint64_t* o_done = pv_done + 2;      // [tile] the item's last PV retired
  uint64_t* r_full = o_done + 2;       // [R] item index published
  uint64_t* r_empty = r_full + R;      // [R] read by the MMA warp and the 8 softmax warps
  int* ring = reinterpret_cast<int*>(r_empty + R);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(ring + R);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef B2S_ATTN_TRACE
  int tr_n = 0;
#endif
  const int npair = (p.nqt + 1) / 2;
  const int nbh = p.B * p.Hq;
  const int nitems = npair * nbh;
  // item w -> (query tiles, batch, head); heaviest pairs first
  auto decode = [&](int w, int& qtA, int& nA, int& nB, int& b, int& h) {
    const int pr = npair - 1 - w / nbh, bh = w % nbh;
    b = bh / p.Hq;
    h = bh % p.Hq;
    qtA = 2 * pr;
    nA = qtA + 1;
    nB = qtA + 1 < p.nqt ? qtA + 2 : 0;
  };
  auto ring_get = [&](int it) -> int {
    mbar_wait(&r_full[it % R], (it / R) & 1);
    return *reinterpret_cast<volatile int*>(&ring[it % R]);
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_o);
    for (int i = 0; i < 2; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], 2); }
    for (int s = 0; s < KVS; ++s) { mbar_init(&k_full[s], 1); mbar_init(&v_full[s], 1); mbar_init(&kv_empty[s], 2); }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1); mbar_init(&s_empty[t], 4);
      mbar_init(&p_full[t], 4); mbar_init(&p_empty[t], 1);
      mbar_init(&pv_done[t], 1); mbar_init(&o_done[t], 1);
    }
    for (int i = 0; i < R; ++i) { mbar_init(&r_full[i], 1); mbar_init(&r_empty[i], 10); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    // ------------------------------------------------ producer: item ring + TMA loads
    if (lane == 0) {
      int next = blockIdx.x;  // first item static, later ones from the counter
      uint32_t kv = 0;        // K / V blocks loaded by this CTA
      for (int it = 0;; ++it) {
        const int slot = it % R;
        mbar_wait(&r_empty[slot], ((it / R) & 1) ^ 1);
        const int w = next < nitems ? next : nitems;
        ring[slot] = w;
        mbar_arrive(&r_full[slot]);
        if (w >= nitems) break;
        next = gridDim.x + atomicAdd(p.sched, 1);  // latency hidden behind this item's loads
        int qtA, nA, nB, b, h;
        decode(w, qtA, nA, nB, b, h);
        const int kvh = h / (p.Hq / p.Hkv);
        const int qb = it % QB;
        mbar_wait(&q_empty[qb], ((it / QB) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qb], (nB ? 2 : 1) * kTQ);
        for (int a = 0; a < NA; ++a) {
          tma_load_2d(sQ + (2 * qb) * kTQ + a * kTile, &tm_qkv, &q_full[qb], h * DH + a * 64, b * p.T + qtA * BQ);
          if (nB)
            tma_load_2d(sQ + (2 * qb + 1) * kTQ + a * kTile, &tm_qkv, &q_full[qb], h * DH + a * 64,
                        b * p.T + (qtA + 1) * BQ);
        }
        const int nkv = nB ? nB : nA;
        for (int j = 0; j < nkv; ++j, ++kv) {
          const int s = kv % KVS;
          mbar_wait(&kv_empty[s], ((kv / KVS) & 1) ^ 1);
          const int r = b * p.T + j * BKV;
          mbar_arrive_expect_tx(&k_full[s], kTQ);
          for (int a = 0; a < NA; ++a)
            tma_load_2d(sK + s * kTQ + a * kTile, &tm_qkv, &k_full[s], (p.Hq + kvh) * DH + a * 64, r);
          mbar_arrive_expect_tx(&v_full[s], kTQ);
          for (int a = 0; a < NA; ++a)
            tma_load_2d(sV + s * kTQ + a * kTile, &tm_qkv, &v_full[s], (p.Hq + p.Hkv + kvh) * DH + a * 64, r);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1 || warp == kThreadsMMA2 / 32) {
    // ------------------------------------------------ MMA issuers: warp 1 tile A, the last warp tile B
    // (whole warp, one lane elected per op). One issuer per tile: a single in-order issuer
    // for both tiles stalls one tile's QK^T / PV behind the other tile's softmax.
    const int tt = warp == 1 ? 0 : 1;
    constexpr uint32_t idS = make_idesc_bf16(BQ, BKV, false, false);
    constexpr uint32_t idO = make_idesc_bf16(BQ, DH, false, true);
    const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aV = smem_u32(sV);
    const uint32_t tSt = tbase + tt * BKV, tOt = tbase + C::OCOL + tt * DH, tPt = tbase + C::pcol(tt);
    uint32_t kv = 0;   // K / V blocks consumed (the producer's order)
    uint32_t ns = 0;   // S MMAs issued for this tile (s_empty phases)
    uint32_t np = 0;   // PV MMAs issued for this tile (p_full phases)
    for (int it = 0;; ++it) {
      const int w = ring_get(it);
      __syncwarp();
      if (lane == 0) mbar_arrive(&r_empty[it % R]);
      if (w >= nitems) break;
      int qtA, nA, nB, b, h;
      decode(w, qtA, nA, nB, b, h);
      const int qb = it % QB;
      const int nkv = nB ? nB : nA;
      const int nt = tt == 0 ? nA : nB;
      const uint32_t kv0 = kv;
      auto issue_S = [&](int j) {
        const uint32_t g = kv0 + j, s = g % KVS;
        TRACE(10, g);
        mbar_wait(&k_full[s], (g / KVS) & 1);
        TRACE(12, g);
        mbar_wait(&s_empty[tt], (ns & 1) ^ 1);
        TRACE(14, g);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t ko = (kk >> 2) * kTile + (kk & 3) * 32;  // atom, then 16-element K step
          mma_bf16_ss_w(tSt, make_sdesc(aQ + (2 * qb + tt) * kTQ + ko, 16, 1024),
                        make_sdesc(aK + s * kTQ + ko, 16, 1024), idS, kk > 0);
        }
        mma_commit_w(&s_full[tt]);
        ++ns;
      };
      auto issue_PV = [&](int j, bool last) {
        const uint32_t g = kv0 + j, s = g % KVS;
        TRACE(20, g);
        mbar_wait(&v_full[s], (g / KVS) & 1);
        TRACE(22, g);
        mbar_wait(&p_full[tt], np & 1);
        TRACE(24, g);
        tc_fence_after();
        // V as an MN-major operand: 16 keys per K step (2 KB of 128-B rows), dh atoms 16 KB apart;
        // P from TMEM: 16 keys = 8 columns of bf16 pairs per K step
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)
          mma_bf16_ts_w(tOt, tPt + kk * 8, make_sdesc(aV + s * kTQ + kk * 2048, kTile, 1024), idO,
                        (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit_w(&p_empty[tt]);
        mma_commit_w(&pv_done[tt]);
        if (last) mma_commit_w(&o_done[tt]);
        mma_commit_w(&kv_empty[s]);  // this tile's reads of K_j / V_j retired
        ++np;
      };
      if (nt > 0) {
        mbar_wait(&q_full[qb], (it / QB) & 1);
        issue_S(0);
        for (int j = 0; j < nt; ++j) {
          if constexpr (C::ALIAS) {  // P_t(j) lives in S_t's columns: S_t(j+1) goes in behind PV_t(j)
            issue_PV(j, j + 1 == nt);
            if (j + 1 < nt) issue_S(j + 1);
          } else {  // QK^T(j+1) as soon as the softmax holds S(j) in registers
            if (j + 1 < nt) issue_S(j + 1);
            issue_PV(j, j + 1 == nt);
          }
        }
      }
      // blocks of the item this tile does not use: release their K / V stage once it has been
      // loaded (so this arrival cannot count toward the stage's previous use)
      for (int j = nt; j < nkv; ++j) {
        const uint32_t g = kv0 + j, s = g % KVS;
        mbar_wait(&k_full[s], (g / KVS) & 1);
        mbar_wait(&v_full[s], (g / KVS) & 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&kv_empty[s]);
      }
      kv += nkv;
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ softmax warpgroups (tile t = 0: A, 1: B)
    const int t = (warp - 2) >> 2;
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const uint32_t lrow = (uint32_t)(q4 * 32) << 16;
    const uint32_t tS = tbase + lrow + t * BKV;
    const uint32_t tO = tbase + lrow + C::OCOL + t * DH;
    const float sl2 = p.scale_log2;
    uint32_t ns = 0;    // S blocks consumed by this tile (s_full / p phases)
    uint32_t nitm = 0;  // items with blocks for this tile (o_done phase)
    const int my_turn = 3 + t, other_turn = 4 - t;
    if (t == 1) named_arrive(3, 256);  // tile A goes first
    for (int it = 0;; ++it) {
      const int w = ring_get(it);
      __syncwarp();
      if (lane == 0) mbar_arrive(&r_empty[it % R]);
      if (w >= nitems) break;
      int qtA, nA, nB, b, h;
      decode(w, qtA, nA, nB, b, h);
      const int qb = it % QB;
      const int qt = qtA + t;
      const int nj = t == 0 ? nA : nB;
      const int nturns = nB ? nB : nA;
      float m = -INFINITY, l = 0.f;
      for (int j = nj; j < nturns; ++j) {  // turns without a block of this tile: pass them on
        named_sync(my_turn, 256);
        named_arrive(other_turn, 256);
      }
      for (int j = 0; j < nj; ++j, ++ns) {
        TRACE(30, ns);
        mbar_wait(&s_full[t], ns & 1);
        TRACE(31, ns);
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
        TRACE(32, ns);
        // P = 2^(S*scale*log2e - m) as bf16 pairs over the S registers
        uint32_t* pk = v;
        float m_use, alpha, rs;
        // dh 128: after the first block, no separate row-max pass (its max is tracked inside the
        // exponential loop; 282 -> 273 us at the Llama-8B shape). dh 64 keeps the max pass:
        // there the fused loop lengthened the MUFU turn (443 -> 453 us at the 1B shape).
        if (j == 0 || !C::kFusedMax) {
          // the row max first (8 independent partial maxima)
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
          m_use = m;
          bool resc = false;
          if (m_cand > m + kRescaleThresh) { m_use = m_cand; resc = (j > 0); }
          alpha = ex2(m - m_use);  // 0 on the first block (m = -inf)
          if (__any_sync(0xffffffffu, resc)) {
            // O must not be in flight: wait for the previous PV of this tile, then O *= alpha
            mbar_wait(&pv_done[t], (ns - 1) & 1);
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
          TRACE(33, ns);
          named_sync(my_turn, 256);
          TRACE(37, ns);
          rs = diag ? exp_pack_regs<true>(v, r, sl2, m_use, pk) : exp_pack_regs<false>(v, r, sl2, m_use, pk);
          named_arrive(other_turn, 256);
          TRACE(34, ns);
        } else {
          // later blocks: exponentials against the running max straight away, the block max
          // tracked inside the same loop (no separate max pass ahead of the MUFU turn)
          TRACE(33, ns);
          named_sync(my_turn, 256);
          TRACE(37, ns);
          float xmax;
          rs = diag ? exp_pack_regs_mx<true>(v, r, sl2, m, pk, xmax) : exp_pack_regs_mx<false>(v, r, sl2, m, pk, xmax);
          named_arrive(other_turn, 256);
          TRACE(34, ns);
          m_use = m;
          alpha = 1.f;
          // lazy rescale: only when the block max exceeds the running one by > 2^8
          const bool resc = xmax > kRescaleThresh;
          if (__any_sync(0xffffffffu, resc)) {
            if (resc) {  // shift the max by an integer k: P, the sum and O scale by 2^-k exactly
              const float k = ceilf(xmax);
              alpha = ex2(-k);
              m_use = m + k;
              rs *= alpha;
#pragma unroll
              for (int i = 0; i < BKV / 2; ++i) {
                const float lo = __uint_as_float(pk[i] << 16), hi = __uint_as_float(pk[i] & 0xffff0000u);
                pk[i] = pack_bf16x2(lo * alpha, hi * alpha);
              }
            }
            // O must not be in flight: wait for the previous PV of this tile, then O *= alpha
            mbar_wait(&pv_done[t], (ns - 1) & 1);
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
        }
        if (ns > 0) mbar_wait(&p_empty[t], (ns - 1) & 1);
        TRACE(35, ns);
        tc_fence_after();
        if constexpr (DH == 64) {  // x16 stores (TMEM writes ~35% faster than x32): 439 -> 431 us at 1B
#pragma unroll
          for (int c = 0; c < BKV / 32; ++c) tmem_st16(tbase + lrow + C::pcol(t) + c * 16, pk + c * 16);
        } else {  // P over S at dh 128: x16 measured slower there (272 -> 280 us)
          tmem_st32(tbase + lrow + C::pcol(t), pk);
          tmem_st32(tbase + lrow + C::pcol(t) + 32, pk + 32);
        }
        tmem_wait_st();
        l = l * alpha + rs;
        m = m_use;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[t]);
        TRACE(36, ns);
      }
      if (nj > 0) {
        // epilogue: O (TMEM) / l -> bf16 -> this tile's Q buffer (all its MMAs retired) -> TMA store
        mbar_wait(&o_done[t], nitm & 1);
        ++nitm;
        tc_fence_after();
        uint8_t* sO = sQ + (2 * qb + t) * kTQ;
        const float inv = 1.f / l;
#pragma unroll
        for (int c = 0; c < DH / 32; ++c) {
          uint32_t o[32];
          tmem_ld32(tO + c * 32, o);
          tmem_wait_ld();
#pragma unroll
          for (int k8 = 0; k8 < 4; ++k8) {
            uint4 w4;
            w4.x = pack_bf16x2(__uint_as_float(o[8 * k8 + 0]) * inv, __uint_as_float(o[8 * k8 + 1]) * inv);
            w4.y = pack_bf16x2(__uint_as_float(o[8 * k8 + 2]) * inv, __uint_as_float(o[8 * k8 + 3]) * inv);
            w4.z = pack_bf16x2(__uint_as_float(o[8 * k8 + 4]) * inv, __uint_as_float(o[8 * k8 + 5]) * inv);
            w4.w = pack_bf16x2(__uint_as_float(o[8 * k8 + 6]) * inv, __uint_as_float(o[8 * k8 + 7]) * inv);
            *reinterpret_cast<uint4*>(sO + (c >> 1) * kTile + swz(r, (c & 1) * 4 + k8)) = w4;
          }
        }
        tc_fence_before();  // O read out: the next item's first PV may overwrite it
        p.lse[((size_t)b * p.Hq + h) * p.T + qt * BQ + r] = (m + log2f(l)) * (1.f / kLog2e);
        fence_proxy_async_smem();
        named_sync(1 + t, 128);
        if (q4 == 0 && lane == 0) {
          for (int a = 0; a < NA; ++a) tma_store_2d(&tm_o, sO + a * kTile, h * DH + a * 64, b * p.T + qt * BQ);
          bulk_commit();
          bulk_wait_read<0>();  // the staging (this item's Q buffer) may be reloaded
          mbar_arrive(&q_empty[qb]);
        }
      } else if (q4 == 0 && lane == 0) {
        mbar_arrive(&q_empty[qb]);  // no tile B in this item: nothing staged
      }
      __syncwarp();
    }
    if (t == 0) named_sync(3, 256);  // consume tile B's last hand-over: no barrier left pending
    if (q4 == 0 && lane == 0) bulk_wait<0>();  // the last item's O stores complete
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
  // every CTA has fetched its sentinel: the last one out re-arms the counter for the next launch
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(p.sched + 1, 1) == (int)gridDim.x - 1) {
      p.sched[0] = 0;
      p.sched[1] = 0;
      __threadfence();
    }
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
  // DH/8 lanes per (row, head): each lane a 16-byte vector of o and dO. Work items run in the
  // [b, h, t] order of lse / D' (t fastest), so those 4-byte reads and writes coalesce across
  // consecutive items; each item's o / dO / dQ slices are whole 128 / 256-byte lines either way.
  constexpr int LPR = DH / 8;
  const int sub = threadIdx.x & (LPR - 1);
  const int64_t nrows = (int64_t)B * T * Hq;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPR; w < nrows;
       w += ((int64_t)gridDim.x * blockDim.x) / LPR) {
    const uint32_t bh = (uint32_t)w / (uint32_t)T;  // B*T*Hq < 2^32 (host-checked)
    const int64_t t = (int64_t)((uint32_t)w - bh * (uint32_t)T);
    const uint32_t b = bh / (uint32_t)Hq, h = bh - b * (uint32_t)Hq;
    const int64_t row = (int64_t)b * T + t;
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
      dsum[w] = acc * scale;  // w = (b * Hq + h) * T + t
      lse2[w] = lse[w] * kLog2e;
    }
  }
}

// dqkv[:, q heads] = bf16(dq_acc)  (dh = 64 path), with ROPE the inverse rotary embedding
// applied on the way (the forward rotated q after the QKV projection, so dq w.r.t. the
// projection output is dq rotated back: pairs (j, j + 32), position row % T). Blocks stride
// over rows (a row is Hq*64 floats), so no 64-bit division per element.
template <bool ROPE>
__global__ void __launch_bounds__(256) attn_bwd_dq_kernel(const float* __restrict__ dq_acc,
                                                          __nv_bfloat16* __restrict__ dqkv, int64_t M, int Hq,
                                                          int64_t ldq, int T, const float* __restrict__ cos_t,
                                                          const float* __restrict__ sin_t) {
  constexpr int DH = 64;
  if constexpr (!ROPE) {
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
  } else {
    const int nv = Hq * 8;  // 4 rotation pairs per thread-step: head v / 8, pairs 4 (v % 8) .. + 3
    for (int64_t row = blockIdx.x; row < M; row += gridDim.x) {
      const float* src = dq_acc + row * (int64_t)(Hq * DH);
      __nv_bfloat16* dst = dqkv + row * ldq;
      const int t = (int)(row % T);
      for (int v = threadIdx.x; v < nv; v += blockDim.x) {
        const int h = v >> 3, j0 = (v & 7) * 4;
        const float4 a = __ldcs(reinterpret_cast<const float4*>(src + h * DH + j0));
        const float4 b = __ldcs(reinterpret_cast<const float4*>(src + h * DH + j0 + 32));
        const float4 c = __ldg(reinterpret_cast<const float4*>(cos_t + (int64_t)t * 32 + j0));
        const float4 sn = __ldg(reinterpret_cast<const float4*>(sin_t + (int64_t)t * 32 + j0));
        // inverse rotation: s -> -s (the rope kernel's inverse form)
        const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
        const float cv[4] = {c.x, c.y, c.z, c.w}, sv[4] = {-sn.x, -sn.y, -sn.z, -sn.w};
        float oa[4], ob[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          oa[k] = av[k] * cv[k] - bv[k] * sv[k];
          ob[k] = bv[k] * cv[k] + av[k] * sv[k];
        }
        uint2 ua, ub;
        ua.x = pack_bf16x2(oa[0], oa[1]);
        ua.y = pack_bf16x2(oa[2], oa[3]);
        ub.x = pack_bf16x2(ob[0], ob[1]);
        ub.y = pack_bf16x2(ob[2], ob[3]);
        *reinterpret_cast<uint2*>(dst + h * DH + j0) = ua;
        *reinterpret_cast<uint2*>(dst + h * DH + j0 + 32) = ub;
      }
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
constexpr int kBwdGroups = 8;  // (batch, kv head) groups per chunk of the backward grid

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
    float pv = ex2(fmaf(__uint_as_float(sv[e]), sl2, -ls[e]));
    if (DIAG && q < r) pv = 0.f;  // query index below key index: masked
    sv[e] = __float_as_uint(pv);
    dv[e] = __float_as_uint(pv * fmaf(__uint_as_float(dv[e]), scale, -ds[e]));
  }
}
// dh = 64: dQ fused (TMEM S^T 128 + dP^T 128 + dV 64 + dK 64 + dQ 64 + P^T 64 = 512
// columns). dh = 128 launches attn_bwd128_kernel (dK / dV, P^T and dS^T in TMEM) and
// attn_bwd_q_kernel (dQ per query tile) instead; this template's non-DQ branches are the
// round-1 dh-128 form (P^T / dS^T in shared memory, one Q / dO stage), kept compilable.
template <int DH>
struct Bwd {
  static constexpr bool DQ = DH == 64;  // dQ fused into the key-tile kernel
  // P^T in TMEM columns [448, 512) (freed by a single dQ buffer): no P^T shared-memory
  // stores and no A-operand smem reads for dV -- the kernel is smem-bandwidth bound
  static constexpr bool PT = DQ;
  // Q / dO stages. A stage is freed when step t's dV / dK / dQ MMAs retire and its next
  // TMA load takes ~1700 clk (L2 / DRAM) -- longer than a step -- so dh 64 keeps two loads in
  // flight ahead of the step being computed (three stages; two left S(t+1) waiting on its Q).
  static constexpr int QS = DH == 64 ? 3 : 1;
  static constexpr int LS = 4;  // lse / D stages (512 B each, loaded LS - 1 steps ahead)
  static constexpr int kTileQ = BQ * DH * 2;
  static constexpr int kSmem = 1024 + 2 * kTileQ /*K,V*/ + 2 * QS * kTileQ /*Q,dO*/ + (PT ? 1 : 2) * kPBuf /*P^T,dS^T*/ +
                               (DQ ? 2 * kTile : 0) /*dQ fp32 staging: 8 warps x 4 KB*/ + 2 * LS * BQ * 4 /*LSE, D*/ +
                               256;
  static_assert(kSmem <= 232448, "backward tiles exceed shared memory");
};

template <int DH>
__global__ void __launch_bounds__(320, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dkv, Params p) {
  using C = Bwd<DH>;
  constexpr int kTQ = C::kTileQ, QS = C::QS, LS = C::LS, NA = DH / 64;
  constexpr bool DQ = C::DQ, PT = C::PT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sK = align1024(smem_raw);
  uint8_t* sV = sK + kTQ;
  uint8_t* sQ = sV + kTQ;            // [QS]
  uint8_t* sdO = sQ + QS * kTQ;      // [QS]
  uint8_t* sP = sdO + QS * kTQ;      // P^T  [128 keys][128 q] as two 64-column atoms (smem P only)
  uint8_t* sdS = sP + (PT ? 0 : kPBuf);  // dS^T
  uint8_t* sdQ = sdS + kPBuf;        // fp32 128 x 64 as two 32-column boxes (16 KB each), dh 64 only
  float* sLse = reinterpret_cast<float*>(sdQ + (DQ ? 2 * kTile : 0));  // [LS][128] natural-log LSE (TMA bulk)
  float* sD = sLse + LS * BQ;                                // [LS][128] rowsum(dO*O)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + LS * BQ);
  uint64_t* kv_full = bars;
  uint64_t* qd_full = bars + 1;        // [QS]
  uint64_t* qd_empty = qd_full + QS;   // [QS]
  uint64_t* st_full = qd_empty + QS;
  uint64_t* st_empty = st_full + 1;
  uint64_t* pds_full = st_full + 2;
  uint64_t* pds_empty = st_full + 3;
  uint64_t* dq_full = st_full + 4;     // [2]
  uint64_t* dq_empty = dq_full + 2;    // [2]
  uint64_t* done = dq_empty + 2;
  uint64_t* st_ld_full = done + 1;         // [LS] lse / D of a step landed
  uint64_t* st_ld_empty = st_ld_full + LS; // [LS] all compute warps done with them
  uint32_t* tslot = reinterpret_cast<uint32_t*>(st_ld_empty + LS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef B2S_ATTN_TRACE
  int tr_n = 0;
#endif
  // Block order: the (batch, kv head) groups in chunks of kBwdGroups; inside a chunk,
  // heaviest key tile first (kt = 0 has the most query tiles). A chunk's dQ accumulator rows
  // (kBwdGroups x T x G heads x dh fp32, 32 MB at the Llama-1B shape) stay in L2 while its
  // key tiles add into them; all groups at once (134 MB) made every add-reduce a DRAM
  // read-modify-write (1.6 GB of DRAM traffic per launch).
  const int nbk = p.B * p.Hkv;
  const int gc = nbk < kBwdGroups ? nbk : kBwdGroups;  // groups per chunk (the last may be smaller)
  const int chunk = (int)(blockIdx.x / (gc * p.nqt));
  const int in_chunk = (int)(blockIdx.x - chunk * gc * p.nqt);
  const int gcur = min(gc, nbk - chunk * gc);  // groups in this chunk
  const int kt = in_chunk / gcur;
  const int bk = chunk * gc + in_chunk % gcur;
  const int b = bk / p.Hkv, kvh = bk % p.Hkv;
  const int G = p.Hq / p.Hkv;
  const int nq = p.nqt - kt;  // query tiles i = kt .. nqt-1
  const int nsteps = G * nq;
  const int krow0 = b * p.T + kt * BKV;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    mbar_init(kv_full, 1);
    for (int s = 0; s < QS; ++s) { mbar_init(&qd_full[s], 1); mbar_init(&qd_empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&dq_full[s], 1); mbar_init(&dq_empty[s], 8); }
    mbar_init(st_full, 1);
    mbar_init(st_empty, 8);
    mbar_init(pds_full, 8);
    mbar_init(pds_empty, 1);
    mbar_init(done, 1);
    for (int s = 0; s < LS; ++s) { mbar_init(&st_ld_full[s], 1); mbar_init(&st_ld_empty[s], 8); }
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
        const int s = t % LS;
        mbar_wait(&st_ld_empty[s], ((t / LS) & 1) ^ 1);
        const size_t off = ((size_t)b * p.Hq + h) * p.T + (size_t)i * BQ;
        mbar_arrive_expect_tx(&st_ld_full[s], 2 * BQ * 4);
        bulk_load_1d(sLse + s * BQ, p.lse + off, BQ * 4, &st_ld_full[s]);
        bulk_load_1d(sD + s * BQ, p.dsum + off, BQ * 4, &st_ld_full[s]);
        const int qs = t % QS;
        mbar_wait(&qd_empty[qs], ((t / QS) & 1) ^ 1);
        TRACE(70, t);
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
        TRACE(71, t);
        if (t > 0) mbar_wait(st_empty, (t - 1) & 1);
        TRACE(72, t);
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
        TRACE(50, t);
      };
      mbar_wait(kv_full, 0);
      issue_S(0);
      for (int t = 0; t < nsteps; ++t) {
        const int qs = t % QS;
        const uint32_t q_ = aQ + qs * kTQ, do_ = adO + qs * kTQ;
        // with a single Q / dO stage, S(t+1) needs this step's dV / dK MMAs to have read Q(t) / dO(t)
        if (QS >= 2 && t + 1 < nsteps) issue_S(t + 1);
        mbar_wait(pds_full, t & 1);
        TRACE(51, t);
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
        TRACE(52, t);
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
      TRACE(67, t);
      tc_fence_after();
      uint32_t qv[32];
      tmem_ld32(tdQ + lrow + dq_buf(t) * DH + half * 32, qv);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
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
        tma_reduce_add_2d(&tm_dq, mystage, h * DH + half * 32, b * p.T + i * BQ + q4 * 32);
        bulk_commit();
      }
    };
    for (int t = 0; t < nsteps; ++t) {
      const int i = kt + t % nq;
      const bool diag = (i == kt);
      mbar_wait(&st_ld_full[t % LS], (t / LS) & 1);
      const float* lse2 = sLse + (t % LS) * BQ;  // natural log; p_ds folds in log2(e)
      const float* dd = sD + (t % LS) * BQ;
      mbar_wait(st_full, t & 1);
      TRACE(60, t);
      tc_fence_after();
      // Two 32-column passes. Both passes' S^T / dP^T are read from TMEM (and st_empty released,
      // so S(t+1) / dP(t+1) can start) before waiting for step t-1's MMAs to free P^T / dS^T:
      // the packed bf16 results wait in registers.
      uint32_t pw[2][16], zw[2][16];
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        uint32_t sv[32], dv[32];
        tmem_ld32(tS + lrow + half * 64 + qq * 32, sv);
        tmem_ld32(tdP + lrow + half * 64 + qq * 32, dv);
        tmem_wait_ld();
        TRACE(61 + 3 * qq, t);
        if (qq == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(st_empty);  // the next step's S^T / dP^T may overwrite TMEM
        }
        if (diag) p_ds<true>(sv, dv, half * 64 + qq * 32, r, p.scale_log2, p.scale, lse2, dd);
        else p_ds<false>(sv, dv, half * 64 + qq * 32, r, p.scale_log2, p.scale, lse2, dd);
        TRACE(62 + 3 * qq, t);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          pw[qq][k] = pack_bf16x2(__uint_as_float(sv[2 * k]), __uint_as_float(sv[2 * k + 1]));
          zw[qq][k] = pack_bf16x2(__uint_as_float(dv[2 * k]), __uint_as_float(dv[2 * k + 1]));
        }
      }
      if (t > 0) mbar_wait(pds_empty, (t - 1) & 1);  // step t-1's MMAs released P^T / dS^T
      TRACE(63, t);
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
#pragma unroll
        for (int k8 = 0; k8 < 4; ++k8) {
          const uint32_t off = half * kTile + swz(r, qq * 4 + k8);
          if constexpr (!PT)
            *reinterpret_cast<uint4*>(sP + off) =
                make_uint4(pw[qq][4 * k8], pw[qq][4 * k8 + 1], pw[qq][4 * k8 + 2], pw[qq][4 * k8 + 3]);
          *reinterpret_cast<uint4*>(sdS + off) =
              make_uint4(zw[qq][4 * k8], zw[qq][4 * k8 + 1], zw[qq][4 * k8 + 2], zw[qq][4 * k8 + 3]);
        }
        if constexpr (PT) tmem_st16(tPT + lrow + half * 32 + qq * 16, pw[qq]);
      }
      if constexpr (PT) {
        tmem_wait_st();  // P^T is in TMEM before the MMA warp is told
        tc_fence_before();
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(pds_full);
        mbar_arrive(&st_ld_empty[t % LS]);
      }
      TRACE(66, t);
      if (t > 0) drain_dq(t - 1);
      TRACE(68, t);
    }
    if (nsteps > 0) drain_dq(nsteps - 1);
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
// dK / dV at dh 128 (attn_bwd128_kernel; dQ comes from attn_bwd_q_kernel). CTA = (batch, kv
// head, 128-key tile) in the block order of attn_bwd_kernel. TMEM holds S^T, dP^T, dV and dK
// (4 x 128 columns), so P^T and dS^T go back into TMEM over the S^T / dP^T columns their warp
// just read (pass qq of warp half h: columns 64h + 32qq + [0, 16) of each block, bf16 pairs):
// no P^T / dS^T shared-memory tiles, which leaves room for two Q / dO stages -- with one, every
// step waited for its Q / dO reload (~3000 clk) behind the previous step's MMAs -- and dV / dK
// run in the TMEM-A MMA form. MMA order per step t: dV(t) S(t+1) dK(t) dP(t+1), dV(t) as soon as
// P^T(t) is stored (p_full), so dV(t) and S(t+1) run while dS(t) is formed: the tensor pipe
// runs one thread's MMAs in order, so S(t+1) overwrites P^T(t) after dV(t) read it and dP(t+1)
// overwrites dS^T(t) after dK(t), while the compute warps start P(t+1) as soon as S(t+1) lands.
struct Bwd128 {
  static constexpr int DH = 128, kTileQ = BQ * DH * 2, QS = 2, LS = 4;
  static constexpr int kSmem = 1024 + 2 * kTileQ /*K, V*/ + 2 * QS * kTileQ /*Q, dO*/ + 2 * LS * BQ * 4 + 256;
  static_assert(kSmem <= 232448, "backward tiles exceed shared memory");
};

__global__ void __launch_bounds__(320, 1)
    attn_bwd128_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                       const __grid_constant__ CUtensorMap tm_dkv, Params p) {
  constexpr int DH = Bwd128::DH, kTQ = Bwd128::kTileQ, QS = Bwd128::QS, LS = Bwd128::LS, NA = DH / 64;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sK = align1024(smem_raw);
  uint8_t* sV = sK + kTQ;
  uint8_t* sQ = sV + kTQ;        // [QS]
  uint8_t* sdO = sQ + QS * kTQ;  // [QS]
  float* sLse = reinterpret_cast<float*>(sdO + QS * kTQ);  // [LS][128]
  float* sD = sLse + LS * BQ;                              // [LS][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + LS * BQ);
  uint64_t* kv_full = bars;
  uint64_t* qd_full = bars + 1;           // [QS]
  uint64_t* qd_empty = qd_full + QS;      // [QS]
  uint64_t* s_full = qd_empty + QS;
  uint64_t* dp_full = s_full + 1;
  uint64_t* p_full = s_full + 2;   // P^T(t) written over the S^T columns (dV(t), then S(t+1) may go)
  uint64_t* ds_full = s_full + 3;  // dS^T(t) written over the dP^T columns (dK(t), then dP(t+1))
  uint64_t* done = s_full + 4;
  uint64_t* st_ld_full = s_full + 5;        // [LS]
  uint64_t* st_ld_empty = st_ld_full + LS;  // [LS]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(st_ld_empty + LS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef B2S_ATTN_TRACE
  int tr_n = 0;
#endif
  // block order: see attn_bwd_kernel
  const int nbk = p.B * p.Hkv;
  const int gc = nbk < kBwdGroups ? nbk : kBwdGroups;
  const int chunk = (int)(blockIdx.x / (gc * p.nqt));
  const int in_chunk = (int)(blockIdx.x - chunk * gc * p.nqt);
  const int gcur = min(gc, nbk - chunk * gc);
  const int kt = in_chunk / gcur;
  const int bk = chunk * gc + in_chunk % gcur;
  const int b = bk / p.Hkv, kvh = bk % p.Hkv;
  const int G = p.Hq / p.Hkv;
  const int nq = p.nqt - kt;
  const int nsteps = G * nq;
  const int krow0 = b * p.T + kt * BKV;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    mbar_init(kv_full, 1);
    for (int s = 0; s < QS; ++s) { mbar_init(&qd_full[s], 1); mbar_init(&qd_empty[s], 1); }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(p_full, 8);
    mbar_init(ds_full, 8);
    mbar_init(done, 1);
    for (int s = 0; s < LS; ++s) { mbar_init(&st_ld_full[s], 1); mbar_init(&st_ld_empty[s], 8); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t tS = tbase, tdP = tbase + 128, tdV = tbase + 256, tdK = tbase + 384;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * kTQ);
      for (int a = 0; a < NA; ++a) {
        tma_load_2d(sK + a * kTile, &tm_qkv, kv_full, (p.Hq + kvh) * DH + a * 64, krow0);
        tma_load_2d(sV + a * kTile, &tm_qkv, kv_full, (p.Hq + p.Hkv + kvh) * DH + a * 64, krow0);
      }
      for (int t = 0; t < nsteps; ++t) {
        const int h = kvh * G + t / nq, i = kt + t % nq;
        const int s = t % LS;
        mbar_wait(&st_ld_empty[s], ((t / LS) & 1) ^ 1);
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
    // ------------------------------------------------ MMA issuer (whole warp, one lane elected per op)
    constexpr uint32_t idSS = make_idesc_bf16(128, 128, false, false);  // S^T, dP^T
    constexpr uint32_t idKM = make_idesc_bf16(128, DH, false, true);    // dV, dK (B = dO / Q, MN-major)
    const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aQ = smem_u32(sQ), adO = smem_u32(sdO);
    auto issue_S = [&](int t) {  // S^T(t) = K Q(t)^T
      const int qs = t % QS;
      mbar_wait(&qd_full[qs], (t / QS) & 1);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk) {
        const uint32_t ko = (kk >> 2) * kTile + (kk & 3) * 32;
        mma_bf16_ss_w(tS, make_sdesc(aK + ko, 16, 1024), make_sdesc(aQ + qs * kTQ + ko, 16, 1024), idSS, kk > 0);
      }
      mma_commit_w(s_full);
    };
    auto issue_dP = [&](int t) {  // dP^T(t) = V dO(t)^T
      const int qs = t % QS;
      mbar_wait(&qd_full[qs], (t / QS) & 1);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk) {
        const uint32_t ko = (kk >> 2) * kTile + (kk & 3) * 32;
        mma_bf16_ss_w(tdP, make_sdesc(aV + ko, 16, 1024), make_sdesc(adO + qs * kTQ + ko, 16, 1024), idSS, kk > 0);
      }
      mma_commit_w(dp_full);
    };
    mbar_wait(kv_full, 0);
    issue_S(0);
    issue_dP(0);
    for (int t = 0; t < nsteps; ++t) {
      const int qs = t % QS;
      const uint32_t q_ = aQ + qs * kTQ, do_ = adO + qs * kTQ;
      mbar_wait(p_full, t & 1);  // dV(t) and S(t+1) overlap the dS phase of step t
      TRACE(51, t);
      tc_fence_after();
      // K step kk = queries 16kk.. : warp half kk >> 2, pass (kk >> 1) & 1, 8 packed columns
#pragma unroll
      for (int kk = 0; kk < BQ / 16; ++kk) {
        const uint32_t col = 64 * (kk >> 2) + 32 * ((kk >> 1) & 1) + (kk & 1) * 8;
        mma_bf16_ts_w(tdV, tS + col, make_sdesc(do_ + kk * 2048, kTile, 1024), idKM, (t > 0 || kk > 0));
      }
      if (t + 1 < nsteps) issue_S(t + 1);  // after dV(t) read P^T(t) from these columns
      TRACE(50, t + 1);
      mbar_wait(ds_full, t & 1);
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < BQ / 16; ++kk) {
        const uint32_t col = 64 * (kk >> 2) + 32 * ((kk >> 1) & 1) + (kk & 1) * 8;
        mma_bf16_ts_w(tdK, tdP + col, make_sdesc(q_ + kk * 2048, kTile, 1024), idKM, (t > 0 || kk > 0));
      }
      mma_commit_w(&qd_empty[qs]);
      if (t + 1 < nsteps) issue_dP(t + 1);  // after dK(t) read dS^T(t)
      TRACE(52, t);
    }
    mma_commit_w(done);
    __syncwarp();
  } else {
    // ------------------------------------------------ compute warps
    const int q4 = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = q4 * 32 + lane;  // key row
    const uint32_t lrow = (uint32_t)(q4 * 32) << 16;
    for (int t = 0; t < nsteps; ++t) {
      const int i = kt + t % nq;
      const bool diag = (i == kt);
      mbar_wait(&st_ld_full[t % LS], (t / LS) & 1);
      const float* lse2 = sLse + (t % LS) * BQ;
      const float* dd = sD + (t % LS) * BQ;
      mbar_wait(s_full, t & 1);
      TRACE(60, t);
      tc_fence_after();
      // P^T = 2^(s scale log2e - lse2[q]) for this warp's 64 query columns: fp32 kept for dS,
      // bf16 pairs stored over the S^T columns just read
      float pf[2][32];
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        uint32_t sv[32], pw[16];
        tmem_ld32(tS + lrow + half * 64 + qq * 32, sv);
        tmem_wait_ld();
        const int q0 = half * 64 + qq * 32;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float4 l4 = *reinterpret_cast<const float4*>(lse2 + q0 + 4 * k);
          const float ls[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int j = 4 * k + e;
            float pv = ex2(fmaf(__uint_as_float(sv[j]), p.scale_log2, -ls[e]));
            if (diag && q0 + j < r) pv = 0.f;  // query index below key index: masked
            pf[qq][j] = pv;
          }
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) pw[k] = pack_bf16x2(pf[qq][2 * k], pf[qq][2 * k + 1]);
        tmem_st16(tS + lrow + half * 64 + qq * 32, pw);
      }
      // dS^T = P^T (scale dP^T - D') once dP(t) lands, bf16 pairs over the dP^T columns just read
      tmem_wait_st();  // P^T is in TMEM before the MMA warp is told
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      TRACE(62, t);
      mbar_wait(dp_full, t & 1);
      TRACE(63, t);
      tc_fence_after();
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        uint32_t dv[32], zw[16];
        tmem_ld32(tdP + lrow + half * 64 + qq * 32, dv);
        tmem_wait_ld();
        const int q0 = half * 64 + qq * 32;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float4 d4 = *reinterpret_cast<const float4*>(dd + q0 + 4 * k);
          const float ds[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int j = 4 * k + e;
            dv[j] = __float_as_uint(pf[qq][j] * fmaf(__uint_as_float(dv[j]), p.scale, -ds[e]));
          }
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) zw[k] = pack_bf16x2(__uint_as_float(dv[2 * k]), __uint_as_float(dv[2 * k + 1]));
        tmem_st16(tdP + lrow + half * 64 + qq * 32, zw);
      }
      tmem_wait_st();  // dS^T is in TMEM before the MMA warp is told
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(ds_full);
        mbar_arrive(&st_ld_empty[t % LS]);
      }
      TRACE(66, t);
    }
    // dK (from the pre-scaled dS) and dV -> bf16 -> smem (the Q / dO stages are free) -> TMA store
    mbar_wait(done, 0);
    tc_fence_after();
    uint8_t* sdK_out = sQ;
    uint8_t* sdV_out = sdO;
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {  // this warp's 64 of the 128 columns, 32 at a time
      const int col0 = half * 64 + cc * 32;
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
        const int chunk16 = col0 / 8 + c;  // 16-byte chunk of the row: atom chunk16 / 8, position % 8
        *reinterpret_cast<uint4*>(sdK_out + (chunk16 >> 3) * kTile + swz(r, chunk16 & 7)) = w;
        *reinterpret_cast<uint4*>(sdV_out + (chunk16 >> 3) * kTile + swz(r, chunk16 & 7)) = z;
      }
    }
    fence_proxy_async_smem();
    named_sync(1, 256);
    if (threadIdx.x == 64) {
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
// dS = P (dP - D) -> bf16 -> TMEM (columns 384..447), dQ += dS K_j (TMEM-A MMA form, TMEM accumulator across the loop,
// K_j as an MN-major operand) -> x scale -> bf16 -> TMA store into dqkv.
// smem 192 KB: Q, dO (32 KB each), K / V 2 stages (128 KB).
template <int DH>
struct BwdQ {
  static constexpr int kTileQ = BQ * DH * 2;
  // K / V stages: a K stage is freed when dQ(j) retires, a V stage as soon as dP(j) does; the
  // reload takes ~3000 clk under load, so with two K stages S(j+2) waited on it every block
  static constexpr int KS = 3, VS = 2;
  static constexpr int kSmem = 1024 + 2 * kTileQ + (KS + VS) * kTileQ + 256;
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
  constexpr int KS = BwdQ<DH>::KS, VS = BwdQ<DH>::VS;
  uint8_t* sK = sdO + kTQ;              // [KS]
  uint8_t* sV = sK + KS * kTQ;          // [VS]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + VS * kTQ);
  uint64_t* qd_full = bars;
  uint64_t* k_full = bars + 1;          // [KS]
  uint64_t* k_empty = k_full + KS;      // [KS]
  uint64_t* v_full = k_empty + KS;      // [VS]
  uint64_t* v_empty = v_full + VS;      // [VS]
  uint64_t* s_full = v_empty + VS;
  uint64_t* s_empty = s_full + 1;
  uint64_t* dp_full = s_full + 2;
  uint64_t* dp_empty = s_full + 3;
  uint64_t* pds_full = s_full + 4;
  uint64_t* pds_empty = s_full + 5;
  uint64_t* done = pds_empty + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#if defined(B2S_ATTN_TRACE) && !defined(B2S_TRACE_KV)
  int tr_n = 0;
#else
#undef TRACE
#define TRACE(ev, aux) \
  do {                 \
  } while (0)
#endif
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
    for (int s = 0; s < KS; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
    for (int s = 0; s < VS; ++s) { mbar_init(&v_full[s], 1); mbar_init(&v_empty[s], 1); }
    mbar_init(s_full, 1);
    mbar_init(s_empty, 8);
    mbar_init(dp_full, 1);
    mbar_init(dp_empty, 8);
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
  // dS (bf16 pairs, 64 columns) in TMEM [384, 448): the dQ MMA takes it in the TMEM-A form
  const uint32_t tS = tbase, tdP = tbase + 128, tdQ = tbase + 256, tDS = tbase + 384;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(qd_full, 2 * kTQ);
      for (int a = 0; a < NA; ++a) {
        tma_load_2d(sQ + a * kTile, &tm_qkv, qd_full, h * DH + a * 64, qrow0);
        tma_load_2d(sdO + a * kTile, &tm_do, qd_full, h * DH + a * 64, qrow0);
      }
      for (int j = 0; j < nkv; ++j) {
        const int r = b * p.T + j * BKV;
        const int sk = j % KS, sv = j % VS;
        mbar_wait(&k_empty[sk], ((j / KS) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[sk], kTQ);
        for (int a = 0; a < NA; ++a)
          tma_load_2d(sK + sk * kTQ + a * kTile, &tm_qkv, &k_full[sk], (p.Hq + kvh) * DH + a * 64, r);
        mbar_wait(&v_empty[sv], ((j / VS) & 1) ^ 1);
        mbar_arrive_expect_tx(&v_full[sv], kTQ);
        for (int a = 0; a < NA; ++a)
          tma_load_2d(sV + sv * kTQ + a * kTile, &tm_qkv, &v_full[sv], (p.Hq + p.Hkv + kvh) * DH + a * 64, r);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    {
      constexpr uint32_t idSS = make_idesc_bf16(BQ, BKV, false, false);  // S, dP
      constexpr uint32_t idQ = make_idesc_bf16(BQ, DH, false, true);     // dQ += dS K (K MN-major)
      const uint32_t aQ = smem_u32(sQ), adO = smem_u32(sdO), aK = smem_u32(sK), aV = smem_u32(sV);
      // S(j) and dP(j) are released separately (the compute warps read all of S first), so S(j+1)
      // runs while block j's dS is still being formed
      auto issue_S = [&](int j) {
        const int sk = j % KS;
        mbar_wait(&k_full[sk], (j / KS) & 1);
        if (j > 0) mbar_wait(s_empty, (j - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t ko = (kk >> 2) * kTile + (kk & 3) * 32;
          mma_bf16_ss_w(tS, make_sdesc(aQ + ko, 16, 1024), make_sdesc(aK + sk * kTQ + ko, 16, 1024), idSS, kk > 0);
        }
        mma_commit_w(s_full);
        TRACE(50, j);
      };
      auto issue_dP = [&](int j) {
        const int sv = j % VS;
        mbar_wait(&v_full[sv], (j / VS) & 1);
        if (j > 0) mbar_wait(dp_empty, (j - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t ko = (kk >> 2) * kTile + (kk & 3) * 32;
          mma_bf16_ss_w(tdP, make_sdesc(adO + ko, 16, 1024), make_sdesc(aV + sv * kTQ + ko, 16, 1024), idSS,
                        kk > 0);
        }
        mma_commit_w(dp_full);
        mma_commit_w(&v_empty[sv]);  // V(j) is read by dP(j) only
      };
      mbar_wait(qd_full, 0);
      issue_S(0);
      issue_dP(0);
      for (int j = 0; j < nkv; ++j) {
        const int s = j % KS;
        if (j + 1 < nkv) {
          issue_S(j + 1);
          issue_dP(j + 1);
        }
        mbar_wait(pds_full, j & 1);
        TRACE(51, j);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)  // K step kk = keys 16kk.. = packed dS columns 8kk..
          mma_bf16_ts_w(tdQ, tDS + kk * 8, make_sdesc(aK + s * kTQ + kk * 2048, kTile, 1024), idQ,
                        (j > 0 || kk > 0) ? 1u : 0u);
        mma_commit_w(pds_empty);
        mma_commit_w(&k_empty[s]);
        TRACE(52, j);
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
      mbar_wait(s_full, j & 1);
      TRACE(60, j);
      tc_fence_after();
      // all of this warp's S columns first, then S(j+1) may overwrite them
      uint32_t sv[2][32];
      tmem_ld32(tS + lrow + half * 64, sv[0]);
      tmem_ld32(tS + lrow + half * 64 + 32, sv[1]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_empty);
      TRACE(61, j);
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        const int k0 = half * 64 + qq * 32;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          float pv = ex2(fmaf(__uint_as_float(sv[qq][e]), sl2, -lse2));
          if (diag && k0 + e > r) pv = 0.f;  // key after query: masked
          sv[qq][e] = __float_as_uint(pv);
        }
      }
      mbar_wait(dp_full, j & 1);
      tc_fence_after();
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        uint32_t dv[32];
        tmem_ld32(tdP + lrow + half * 64 + qq * 32, dv);
        tmem_wait_ld();
        TRACE(61 + 3 * qq, j);
        if (qq == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(dp_empty);
        }
#pragma unroll
        for (int e = 0; e < 32; ++e)  // scaled dS
          dv[e] = __float_as_uint(__uint_as_float(sv[qq][e]) * fmaf(__uint_as_float(dv[e]), p.scale, -dd));
        TRACE(62 + 3 * qq, j);
        if (qq == 0 && j > 0) mbar_wait(pds_empty, (j - 1) & 1);  // dQ(j-1) has read dS(j-1)
        if (qq == 0) TRACE(63, j);
        uint32_t zw[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) zw[e] = pack_bf16x2(__uint_as_float(dv[2 * e]), __uint_as_float(dv[2 * e + 1]));
        tmem_st16(tDS + lrow + half * 32 + qq * 16, zw);
      }
      tmem_wait_st();  // dS is in TMEM before the MMA warp is told
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(pds_full);
      TRACE(66, j);
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
// Per-device pool of zeroed work-item counters {next, ctas_done} for the persistent kernels;
// launches rotate through it so kernels in flight on different streams never share one.
static int* sched_slot() {
  constexpr int kSlots = 64;
  static int* pool[64] = {};
  static int next[64] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (!pool[dev]) {
    if (cudaMalloc(&pool[dev], kSlots * 2 * sizeof(int)) != cudaSuccess) return nullptr;
    cudaMemset(pool[dev], 0, kSlots * 2 * sizeof(int));
    cudaDeviceSynchronize();
  }
  int* p = pool[dev] + 2 * next[dev];
  next[dev] = (next[dev] + 1) % kSlots;
  return p;
}

template <int DH>
int attn_fwd_dh(const void* d_qkv, void* d_o, float* d_lse, int B, int T, int Hq, int Hkv, cudaStream_t st) {
  using C = attn::Fwd<DH>;
  const int ldq = (Hq + 2 * Hkv) * DH;
  CUtensorMap tq, to;
  int rc = encode_tma_2d(&tq, d_qkv, 2, (uint64_t)ldq, (uint64_t)B * T, (uint64_t)ldq * 2, 64, 128, 128);
  if (rc) return rc;
  rc = encode_tma_2d(&to, d_o, 2, (uint64_t)Hq * DH, (uint64_t)B * T, (uint64_t)Hq * DH * 2, 64, 128, 128);
  if (rc) return rc;
  int* sched = sched_slot();
  B2S_REQUIRE(sched, B2S_ECUDA, "attention: work-item counter allocation failed");
  attn::Params p{B, T, Hq, Hkv, T / attn::BQ, attn::kLog2e / sqrtf((float)DH), 1.f / sqrtf((float)DH), d_lse,
                 nullptr, nullptr, sched};
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn::attn_fwd_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    attr = true;
  }
  const int items = B * Hq * ((T / attn::BQ + 1) / 2);
  const unsigned grid = (unsigned)(items < kNumSMs ? items : kNumSMs);
  attn::attn_fwd_kernel<DH><<<grid, C::kThreads, C::kSmem, st>>>(tq, to, p);
  return check_launch("attn_fwd");
}

template <int DH>
int attn_bwd_dh(const void* d_qkv, const void* d_o, const void* d_do, const float* d_lse, void* d_dqkv,
                float* d_work, int B, int T, int Hq, int Hkv, cudaStream_t st, const float* rope_cos = nullptr,
                const float* rope_sin = nullptr) {
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
                 dsum, dq_acc, nullptr};
  static bool attr = false;
  if (!attr) {
    if constexpr (DH == 128)
      cudaFuncSetAttribute(attn::attn_bwd128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, attn::Bwd128::kSmem);
    else
      cudaFuncSetAttribute(attn::attn_bwd_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if constexpr (!C::DQ)
      cudaFuncSetAttribute(attn::attn_bwd_q_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           attn::BwdQ<DH>::kSmem);
    attr = true;
  }
  const unsigned grid = (unsigned)(B * Hkv * (T / attn::BQ));
  if constexpr (DH == 128)
    attn::attn_bwd128_kernel<<<grid, attn::kBwdThreads, attn::Bwd128::kSmem, st>>>(tq, tdo, tdkv, p);
  else
    attn::attn_bwd_kernel<DH><<<grid, attn::kBwdThreads, C::kSmem, st>>>(tq, tdo, tdq, tdkv, p);
  rc = check_launch("attn_bwd");
  if (rc) return rc;
  if constexpr (C::DQ) {
    const unsigned g = (unsigned)(M < kNumSMs * 16 ? M : kNumSMs * 16);
    if (rope_cos)
      attn::attn_bwd_dq_kernel<true><<<g, 256, 0, st>>>(dq_acc, (__nv_bfloat16*)d_dqkv, M, Hq, ldq, T, rope_cos,
                                                        rope_sin);
    else
      attn::attn_bwd_dq_kernel<false><<<g, 256, 0, st>>>(dq_acc, (__nv_bfloat16*)d_dqkv, M, Hq, ldq, T, nullptr,
                                                         nullptr);
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

#ifdef B2S_ATTN_TRACE
// experiment builds only (not declared in b2s.h): copy the forward's timeline records to host
extern "C" int b2s_attn_trace_read(void* host, int64_t bytes) {
  return cudaMemcpyFromSymbol(host, attn::g_trace, (size_t)bytes) == cudaSuccess ? 0 : -3;
}
#endif

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

// Backward of attention applied to rotary-embedded q / k (Llama): dq, dk w.r.t. the projection
// output, i.e. b2s_attn_bwd followed by the inverse rotation of the q and k heads of d_dqkv.
// dh 64: dq is rotated back inside the dq conversion pass (no extra pass over the q heads) and
// one b2s_rope launch covers the k heads only; dh 128: b2s_rope over q and k heads.
extern "C" int b2s_rope(void* d_qkv, int64_t M, int T, int64_t ld, int nheads, int dh, const float* d_cos,
                        const float* d_sin, int inverse, b2s_stream_t stream);
extern "C" int b2s_attn_bwd_rope(const void* d_qkv, const void* d_o, const void* d_do, const float* d_lse,
                                 void* d_dqkv, float* d_work, int B, int T, int Hq, int Hkv, int dh, const float* d_cos,
                                 const float* d_sin, b2s_stream_t stream) {
  B2S_REQUIRE(dh == 64 || dh == 128, B2S_EUNSUPPORTED, "attention: head dim %d not implemented (64, 128)", dh);
  B2S_REQUIRE(T % attn::BQ == 0 && T > 0, B2S_EUNSUPPORTED, "attention: T must be a multiple of 128");
  B2S_REQUIRE(Hkv > 0 && Hq % Hkv == 0, B2S_EINVAL, "attention: Hq must be a multiple of Hkv");
  B2S_REQUIRE((int64_t)B * T * Hq < (1LL << 32), B2S_EUNSUPPORTED, "attention: B*T*Hq must be < 2^32");
  B2S_REQUIRE(d_cos && d_sin && ((uintptr_t)d_cos % 16) == 0 && ((uintptr_t)d_sin % 16) == 0, B2S_EINVAL,
              "attn_bwd_rope: null / misaligned rotary tables");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t M = (int64_t)B * T, ld = (int64_t)(Hq + 2 * Hkv) * dh;
  int rc;
  if (dh == 64) {
    rc = attn_bwd_dh<64>(d_qkv, d_o, d_do, d_lse, d_dqkv, d_work, B, T, Hq, Hkv, st, d_cos, d_sin);
    if (rc) return rc;
    return b2s_rope((__nv_bfloat16*)d_dqkv + (int64_t)Hq * dh, M, T, ld, Hkv, dh, d_cos, d_sin, 1, stream);
  }
  rc = attn_bwd_dh<128>(d_qkv, d_o, d_do, d_lse, d_dqkv, d_work, B, T, Hq, Hkv, st);
  if (rc) return rc;
  return b2s_rope(d_dqkv, M, T, ld, Hq + Hkv, dh, d_cos, d_sin, 1, stream);
}
