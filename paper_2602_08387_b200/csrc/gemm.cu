// Persistent warp-specialised tcgen05 GEMM for sm_100a (K5).
//
//   C[M,N] = epilogue( sum_k A(m,k) * B(n,k) )
//
// A and B are bf16 and each may be K-major (row-major [M][K] / [N][K]) or
// MN-major ([K][M] / [K][N]); that covers forward (X W^T), dgrad (dY W) and
// wgrad (dY^T X) of a row-major nn.Linear without any transpose kernel.
//
// Roles (320 threads): warp0 = TMA producer, warp1 = TMEM owner + MMA issuer,
// warps 2..9 = epilogue. Operand tiles are staged by TMA into 128B-swizzled
// shared memory (kStages-deep ring of full/empty mbarriers); the fp32
// accumulator lives in TMEM, double-buffered so the epilogue of tile i
// overlaps the MMAs of tile i+1. The epilogue moves 32x32 sub-tiles
// TMEM -> registers (bias / GELU / dGELU applied there) -> swizzled smem ->
// TMA store (or TMA add-reduce when accumulating), so global writes are
// full-line and asynchronous. Grid = #SMs; tiles are handed out dynamically
// from a global atomic counter (the producer warp of the CTA / CTA-pair
// leader fetches the next tile index and publishes it through an smem ring to
// the MMA and epilogue warps -- and to the peer CTA of a pair), so CTAs that
// start late (SMs busy with NCCL kernels on the comm stream) take fewer tiles
// instead of stretching the kernel.
#include <algorithm>
#include <map>
#include <mutex>
#include <string.h>
#include <tuple>
#include <vector>
#include <stdio.h>
#include <stdlib.h>
#include <cuda_fp16.h>
#include "common.cuh"
#include "sm100.cuh"

namespace b2s {
using namespace sm100;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// 2-D tensor map over a row-major [outer][inner] array (row stride in bytes).
// Resolved through the runtime so the library needs no -lcuda at link time.
int encode_tma_2d(CUtensorMap* map, const void* base, int elem_bytes, uint64_t inner,
                  uint64_t outer, uint64_t row_stride_bytes, uint32_t box_inner,
                  uint32_t box_outer, int swizzle_bytes) {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) { set_error("cuTensorMapEncodeTiled unavailable"); return B2S_ECUDA; }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                        : swizzle_bytes == 64  ? CU_TENSOR_MAP_SWIZZLE_64B
                        : swizzle_bytes == 32  ? CU_TENSOR_MAP_SWIZZLE_32B
                                               : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUtensorMapDataType dt = elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  CUresult r = fn(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { set_error("cuTensorMapEncodeTiled failed (%d)", (int)r); return B2S_ECUDA; }
  return B2S_OK;
}

namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle row
constexpr int UMMA_K = 16;
// Epilogue warps per CTA (EW, a multiple of 4: one group per TMEM lane quarter,
// splitting the tile's 32-column chunks): 12 for CTA-pair GEMMs with an
// activation epilogue (GELU / dGELU: epilogue-latency bound at K = 768), which
// costs one smem pipeline stage; 8 otherwise.
constexpr int kStageSlot = 4096;  // one 32x32 fp32 (or bf16) staging sub-tile

// Wait accounting of one launch (experiment builds, -DB2S_GEMM_PROF; tools/gemm_prof.py): per CTA,
// role 0 = the MMA issuer [total, waits for a free accumulator, for a loaded stage, for the first
// stage of a tile], role 1 = epilogue warp 2 [total, waits for a finished accumulator, -, tiles],
// role 2 = the TMA producer [total, tile-index step, waits for a free stage, tiles, of which the
// leader's wait for a free tile-ring slot]; [4] of role 0 is the first-stage wait.
#ifdef B2S_GEMM_PROF
__device__ unsigned long long g_gprof[148][3][5];
#define GPROF_DECL long long gp_start = clock64(), gp_t0 = 0, gp_w[3] = {0, 0, 0}; int gp_tiles = 0;
#define GPROF_T0 gp_t0 = clock64();
#define GPROF_ACC(i) gp_w[i] += clock64() - gp_t0;
#define GPROF_TILE ++gp_tiles;
#define GPROF_END(role)                                                                              \
  if ((threadIdx.x & 31) == 0 && (role != 1 || warp == 2) && blockIdx.x < 148) {                     \
    g_gprof[blockIdx.x][role][0] = clock64() - gp_start;                                             \
    g_gprof[blockIdx.x][role][1] = gp_w[1];                                                          \
    g_gprof[blockIdx.x][role][2] = gp_w[2];                                                          \
    g_gprof[blockIdx.x][role][3] = gp_tiles;                                                         \
    g_gprof[blockIdx.x][role][4] = gp_w[0];                                                          \
  }
#else
#define GPROF_DECL
#define GPROF_T0
#define GPROF_ACC(i)
#define GPROF_TILE
#define GPROF_END(role)
#endif

constexpr int kRing = 8;  // tile-index ring depth (producer runs ahead of MMA + 2 epilogue buffers)

struct Epi {
  int out_f32;                // 1: fp32 output, 0: bf16
  int accumulate;             // C += result (TMA add-reduce)
  const __nv_bfloat16* bias;  // [N] or null
  int act;                    // 0 none, 1 gelu-tanh (aux <- pre-activation), 2 x gelu'(aux),
                              // 3 SwiGLU forward, 4 SwiGLU backward (see b2s_gemm_swiglu_*),
                              // 5 gelu-tanh (aux <- gelu'(pre-activation)), 6 x aux
  const __nv_bfloat16* aux_in;  // act=2/6: [M, ld_aux]; act=4: gu [M, ld_aux = 2F]
  int64_t ld_aux;
  int glu_F;                  // act 3 / 4: the gate / up split F
  float* colsum_part;         // bf16 generic epilogue: per-32-row column sums of the stored C,
                              // [ceil(M/32)][N] fp32 (the bias gradient of a dgrad), or null
  // act 7 (RoPE on the fused QKV projection, see b2s_gemm_rope): columns [0, rope_cols) are
  // heads of width rope_dh rotated (rotate-half pairs j, j + dh/2) by the fp32 tables
  // cos / sin [T, dh/2] at position row % T; the rest (the V heads) is stored as is
  const float* rope_cos;
  const float* rope_sin;
  int rope_T, rope_dh, rope_cols;
};

// sigmoid as MUFU.EX2 + MUFU.RCP (approximate reciprocal, ~1 ulp): the IEEE __frcp_rn adds
// Newton steps and a special-case subroutine call per element to the SwiGLU epilogues
__device__ __forceinline__ float silu_sig(float g, float& sg) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(1.f + __expf(-g)));
  sg = y;
  return g * sg;
}

__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float u = k0 * (x + k1 * x * x * x);
  return 0.5f * x * (1.f + tanh_fast(u));
}
// Packed half2 forms for the epilogue (two elements per instruction; the
// epilogue of the K = 768 GPT-2 GEMMs is instruction-issue bound). fp16 keeps
// 11 mantissa bits (error ~1e-3 relative on the activation / its derivative,
// below the bf16 rounding of the stored result) and the range of |x| < 64 the
// tanh argument needs; tanh.approx.f16x2 runs two elements per MUFU op.
__device__ __forceinline__ __half2 tanh_h2(__half2 x) {
  uint32_t y, xi = *reinterpret_cast<uint32_t*>(&x);
  asm("tanh.approx.f16x2 %0, %1;" : "=r"(y) : "r"(xi));
  return *reinterpret_cast<__half2*>(&y);
}
// gelu(x) for the pair (a, b) -> float2
__device__ __forceinline__ float2 gelu_tanh2(float a, float b) {
  const __half2 x = __floats2half2_rn(a, b);
  const __half2 x2 = __hmul2(x, x);
  const __half2 u = __hmul2(x, __hfma2(x2, __float2half2_rn(0.7978845608f * 0.044715f), __float2half2_rn(0.7978845608f)));
  const __half2 hx = __hmul2(x, __float2half2_rn(0.5f));
  const __half2 g = __hfma2(hx, tanh_h2(u), hx);  // 0.5 x (1 + tanh u)
  return __half22float2(g);
}
// gelu'(x) for the pair (a, b) -> float2
__device__ __forceinline__ float2 gelu_tanh_grad2(float a, float b) {
  const float k0 = 0.7978845608f, k1 = 0.044715f;
  const __half2 x = __floats2half2_rn(a, b);
  const __half2 x2 = __hmul2(x, x);
  const __half2 t = tanh_h2(__hmul2(x, __hfma2(x2, __float2half2_rn(k0 * k1), __float2half2_rn(k0))));
  const __half2 half_ = __float2half2_rn(0.5f);
  const __half2 a_ = __hfma2(half_, t, half_);                        // 0.5 (1 + t)
  const __half2 b_ = __hfma2(__hneg2(t), t, __float2half2_rn(1.f));    // 1 - t^2
  const __half2 c_ = __hmul2(x, __hfma2(x2, __float2half2_rn(1.5f * k0 * k1), __float2half2_rn(0.5f * k0)));
  return __half22float2(__hfma2(c_, b_, a_));
}
// gelu(x) and gelu'(x) for the pair (a, b), sharing tanh(u): the forward stores
// gelu' as the aux output so the backward epilogue is a single multiply (act 5 / 6).
__device__ __forceinline__ void gelu_and_grad2(float a, float b, float2& g, uint32_t& dpacked) {
  const float k0 = 0.7978845608f, k1 = 0.044715f;
  const __half2 x = __floats2half2_rn(a, b);
  const __half2 x2 = __hmul2(x, x);
  const __half2 t = tanh_h2(__hmul2(x, __hfma2(x2, __float2half2_rn(k0 * k1), __float2half2_rn(k0))));
  const __half2 half_ = __float2half2_rn(0.5f);
  const __half2 hx = __hmul2(x, half_);
  g = __half22float2(__hfma2(hx, t, hx));                                 // 0.5 x (1 + t)
  const __half2 a_ = __hfma2(half_, t, half_);                           // 0.5 (1 + t)
  const __half2 b_ = __hfma2(__hneg2(t), t, __float2half2_rn(1.f));       // 1 - t^2
  const __half2 c_ = __hmul2(x, __hfma2(x2, __float2half2_rn(1.5f * k0 * k1), __float2half2_rn(0.5f * k0)));
  const float2 d = __half22float2(__hfma2(c_, b_, a_));
  dpacked = pack_bf16x2(d.x, d.y);
}
__device__ __forceinline__ float gelu_tanh_grad(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float x2 = x * x;
  float u = k0 * (x + k1 * x2 * x);
  float t = tanh_fast(u);
  return 0.5f * (1.f + t) + 0.5f * x * (1.f - t * t) * k0 * (1.f + 3.f * k1 * x2);
}

template <int BN, int CG, int EW = 8>
struct Cfg {
  static constexpr int kEpiWarps = EW;
  static constexpr int kThreads = 64 + 32 * EW;
  static constexpr int kRing = 2 * kStageSlot;  // per-warp staging ring
  static constexpr int kEpiSmem = kEpiWarps * kRing;
  static constexpr int kABytes = BM * BK * 2;          // this CTA's 128 rows of A
  static constexpr int kBBytes = (BN / CG) * BK * 2;   // this CTA's share of B's BN rows
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (CG == 2) ? (EW == 8 ? 5 : 4) : (BN == 256 ? 3 : 4);
  static constexpr int kTmemCols = 2 * BN;  // double-buffered accumulator
  static constexpr int kSmem = kStages * kStageBytes + kEpiSmem + 1024 /*align*/ + 512 /*barriers, tile ring*/;
  static_assert((2 * kStages + 4 + 2 * 8) * 8 + 8 * 4 + 8 + 2 * kEpiWarps * 8 <= 512, "barrier region");
  static_assert(kSmem <= 227 * 1024, "smem budget");
};

// Stage one 32x32 sub-tile (row `lane` of this warp) into swizzled smem.
// bf16 rows are 64 B (TMA SWIZZLE_64B), fp32 rows 128 B (SWIZZLE_128B); the
// XOR below is the same address permutation the tensor map applies.
__device__ __forceinline__ void stage_bf16(uint8_t* buf, int lane, const float* v) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint4 w;
    w.x = pack_bf16x2(v[8 * c + 0], v[8 * c + 1]);
    w.y = pack_bf16x2(v[8 * c + 2], v[8 * c + 3]);
    w.z = pack_bf16x2(v[8 * c + 4], v[8 * c + 5]);
    w.w = pack_bf16x2(v[8 * c + 6], v[8 * c + 7]);
    const int pc = c ^ ((lane >> 1) & 3);
    *reinterpret_cast<uint4*>(buf + lane * 64 + pc * 16) = w;
  }
}
// Same swizzled slot layout for 32 values already packed as 16 bf16 pairs.
__device__ __forceinline__ void stage_bf16_packed(uint8_t* buf, int lane, const uint32_t* w16) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int pc = c ^ ((lane >> 1) & 3);
    *reinterpret_cast<uint4*>(buf + lane * 64 + pc * 16) =
        make_uint4(w16[4 * c], w16[4 * c + 1], w16[4 * c + 2], w16[4 * c + 3]);
  }
}
__device__ __forceinline__ void stage_f32(uint8_t* buf, int lane, const float* v) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int pc = c ^ (lane & 7);
    *reinterpret_cast<float4*>(buf + lane * 128 + pc * 16) =
        make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  }
}

// Tile raster (host-chosen, see choose_raster): tile index mn -> (m block, n block).
// raster > 0: groups of `raster` M blocks; inside a group the M block varies fastest and the
//   group sweeps every N block before the next group starts.
// raster < 0: the same with the roles of M and N swapped (groups of -raster N blocks).
// Tiles are handed out in index order, so the ~74 tiles in flight at once (one per CTA pair)
// form a (group x span) rectangle: the operand blocks they share are loaded from DRAM once and
// hit in L2 for the rest of the wave. raster = num_m is the plain M-fastest order.
__device__ __forceinline__ void tile_mn(int mn, int num_m, int num_n, int raster, int& mi, int& ni) {
  if (raster > 0) {
    const int gt = raster * num_n, g = mn / gt, local = mn - g * gt;
    const int gm = min(raster, num_m - g * raster);
    mi = g * raster + local % gm;
    ni = local / gm;
  } else {
    const int G = -raster, gt = G * num_m, g = mn / gt, local = mn - g * gt;
    const int gn = min(G, num_n - g * G);
    ni = g * G + local % gn;
    mi = local / gn;
  }
}

// CG = 1: one CTA computes a 128 x BN tile.
// CG = 2: a CTA pair (cluster of 2) computes a 256 x BN tile with
//   tcgen05.mma.cta_group::2 (M = 256): each CTA stages its 128 rows of A and
//   BN/2 rows of B, TMA completion bytes of both land on the leader's barrier,
//   the leader alone issues the MMAs, and commits multicast to both CTAs.
//   Each CTA's TMEM holds its own 128 x BN half of the accumulator, which its
//   own epilogue warps drain. Per-SM operand traffic drops by 1/3.
// SPEC selects a specialised epilogue at compile time (0: the generic bias / GELU / aux-product
// / column-sum epilogue, 3: SwiGLU forward, 4: SwiGLU backward, 7: RoPE), so each instantiation
// carries only its own epilogue's registers.
template <int BN, int CG, bool A_MN, bool B_MN, int EW, int SPEC>
__global__ void __launch_bounds__(Cfg<BN, CG, EW>::kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmAux,
                int M, int N, int K, int splits, int raster, int l2hints, Epi epi, int* __restrict__ sched) {
  using C_ = Cfg<BN, CG, EW>;
  constexpr int kEpiWarps = C_::kEpiWarps, kEpiSmem = C_::kEpiSmem;
  constexpr int kEG = kEpiWarps / 4;  // epilogue warps per TMEM lane quarter
  constexpr uint32_t kIdesc = make_idesc_bf16(BM * CG, BN, A_MN, B_MN);
  constexpr int BNc = BN / CG;  // B rows (N) staged by this CTA
  extern __shared__ uint8_t smem_raw[];
  // align by offsetting (keeps the shared address space: STS, not generic stores)
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  uint8_t* epi_smem = smem + C_::kStages * C_::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_smem + kEpiSmem);
  uint64_t* empty = full + C_::kStages;
  uint64_t* tfull = empty + C_::kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* rfull = tempty + 2;       // [kRing] tile index published
  uint64_t* rempty = rfull + kRing;   // [kRing] every reader done with the slot (leader CTA's count)
  int* ring = reinterpret_cast<int*>(rempty + kRing);
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(ring + kRing);
  uint64_t* abar_all = reinterpret_cast<uint64_t*>(tmem_base_slot + 2);  // [epilogue warp][2] aux tile landed

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0;
  const bool leader = rank == 0;
  const int num_m = (M + BM * CG - 1) / (BM * CG), num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n * splits;  // split-K tiles add-reduce into C
  const int num_kb_all = (K + BK - 1) / BK;
  const int kb_per = (num_kb_all + splits - 1) / splits;
  // readers of a ring slot: MMA warp + 8 epilogue warps (+ the peer's producer and 8 epilogue warps)
  constexpr uint32_t kRingReaders = (CG == 2) ? 2 + 2 * kEpiWarps : 1 + kEpiWarps;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmC);
    for (int s = 0; s < C_::kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], CG * kEpiWarps); }
    for (int i = 0; i < kRing; ++i) { mbar_init(&rfull[i], 1); mbar_init(&rempty[i], kRingReaders); }
    for (int i = 0; i < 2 * kEpiWarps; ++i) mbar_init(&abar_all[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (CG == 2) tmem_alloc_pair<C_::kTmemCols>(tmem_base_slot);
    else tmem_alloc<C_::kTmemCols>(tmem_base_slot);
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();  // peer barriers initialised before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  // tile-index ring: get the i-th tile of this CTA (blocking), then release the slot
  auto ring_get = [&](int i) -> int {
    if (CG == 2 && !leader) mbar_wait_cluster(&rfull[i % kRing], (i / kRing) & 1);  // published by the leader
    else mbar_wait(&rfull[i % kRing], (i / kRing) & 1);
    return *reinterpret_cast<volatile int*>(&ring[i % kRing]);
  };
  // release slot i after reading `tile` from it (relaxed, data-dependent on the read)
  auto ring_release = [&](int i, int tile) {
    const uint32_t rank_of_leader = 0;
    mbar_arrive_cluster_relaxed_after(CG == 2 ? mapa_shared(smem_u32(&rempty[i % kRing]), rank_of_leader)
                                              : smem_u32(&rempty[i % kRing]),
                                      tile);
  };

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // L2 policies of the A / B loads (l2hints: 2 bits per operand, see launch())
      const uint64_t polA = l2_policy(l2hints & 3), polB = l2_policy((l2hints >> 2) & 3);
      // first tile static (blockIdx), later ones from the counter; the atomic for
      // tile i+1 is issued when tile i starts loading, so its latency is hidden
      const int tstride = gridDim.x / CG;
      int next = blockIdx.x / CG;
      GPROF_DECL
      // leader: tile i -> ring slot i (local readers: rfull arrive; the peer: see below)
      auto publish = [&](int i, int t) {
        const int slot = i % kRing;
#ifdef B2S_GEMM_PROF
        const long long gp_r0 = clock64();
#endif
        mbar_wait(&rempty[slot], ((i / kRing) & 1) ^ 1);
#ifdef B2S_GEMM_PROF
        gp_w[0] += clock64() - gp_r0;
#endif
        ring[slot] = t;
        mbar_arrive(&rfull[slot]);
        if constexpr (CG == 2) {
          // to the peer: an asynchronous remote store that completes the transaction count of the
          // peer's rfull[slot] (whose one arrival is the peer producer's expect_tx) -- no release
          // fence, so the producer goes straight on to the next tile's loads (a st.shared::cluster
          // + release-arrive cost ~1000 clk here, in front of every tile's first load)
          const uint32_t peer_slot = mapa_shared(smem_u32(&ring[slot]), 1);
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(peer_slot),
                       "r"(t), "r"(mapa_shared(smem_u32(&rfull[slot]), 1))
                       : "memory");
        }
      };
      for (int it = 0;; ++it) {
        int tile;
        GPROF_T0
        if (leader) {
          tile = next < num_tiles ? next : num_tiles;  // num_tiles = sentinel: no more work
          publish(it, tile);
        } else {
          mbar_arrive_expect_tx(&rfull[it % kRing], 4);  // the peer's one arrival; the leader's st.async the bytes
          tile = ring_get(it);
          ring_release(it, tile);
        }
        GPROF_ACC(1)
        if (tile >= num_tiles) {
          GPROF_END(2)
          break;
        }
        GPROF_TILE
        if (leader) next = sched ? tstride + atomicAdd(sched, 1) : tile + tstride;
        const int mn = tile % (num_m * num_n), ks = tile / (num_m * num_n);
        int mi, ni;
        tile_mn(mn, num_m, num_n, raster, mi, ni);
        const int m0 = mi * BM * CG + rank * BM;
        // act 3 (SwiGLU forward, CTA pairs): tile n covers gate rows [128n, 128n+128) (leader)
        // and the matching up rows [F + 128n, ...) (peer), so each accumulator holds both
        const int n0 = SPEC == 3 ? (rank ? epi.glu_F : 0) + ni * (BN / 2) : ni * BN + rank * BNc;
        const int kb0 = ks * kb_per, kb1 = min(num_kb_all, kb0 + kb_per);
        for (int kb = kb0; kb < kb1; ++kb) {
          GPROF_T0
          mbar_wait(&empty[stage], phase ^ 1);
          GPROF_ACC(2)
          uint8_t* sa = smem + stage * C_::kStageBytes;
          uint8_t* sb = sa + C_::kABytes;
          const int k0 = kb * BK;
          if constexpr (CG == 1) {
            if constexpr (A_MN) {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j) tma_load_2d_hint(sa + j * (64 * BK * 2), &tmA, &full[stage], m0 + 64 * j, k0, polA);
            } else {
              tma_load_2d_hint(sa, &tmA, &full[stage], k0, m0, polA);
            }
            if constexpr (B_MN) {
#pragma unroll
              for (int j = 0; j < BNc / 64; ++j) tma_load_2d_hint(sb + j * (64 * BK * 2), &tmB, &full[stage], n0 + 64 * j, k0, polB);
            } else {
              tma_load_2d_hint(sb, &tmB, &full[stage], k0, n0, polB);
            }
            mbar_arrive_expect_tx(&full[stage], C_::kStageBytes);
          } else {
            const uint32_t bar = mapa_shared(smem_u32(&full[stage]), 0);  // the leader's barrier
            if (leader) mbar_arrive_expect_tx(&full[stage], 2 * C_::kStageBytes);
            if constexpr (A_MN) {
#pragma unroll
              for (int j = 0; j < BM / 64; ++j) tma_load_2d_pair_hint(sa + j * (64 * BK * 2), &tmA, bar, m0 + 64 * j, k0, polA);
            } else {
              tma_load_2d_pair_hint(sa, &tmA, bar, k0, m0, polA);
            }
            if constexpr (B_MN) {
#pragma unroll
              for (int j = 0; j < BNc / 64; ++j) tma_load_2d_pair_hint(sb + j * (64 * BK * 2), &tmB, bar, n0 + 64 * j, k0, polB);
            } else {
              tma_load_2d_pair_hint(sb, &tmB, bar, k0, n0, polB);
            }
          }
          if (++stage == C_::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer (leader CTA)
    if (lane == 0 && leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      GPROF_DECL
      for (int it = 0;; ++it) {
        const int tile = ring_get(it);
        ring_release(it, tile);
        if (tile >= num_tiles) break;
        GPROF_T0
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        GPROF_ACC(1)
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        const int ks = tile / (num_m * num_n);
        const int kb0 = ks * kb_per, kb1 = min(num_kb_all, kb0 + kb_per);
        for (int kb = kb0; kb < kb1; ++kb) {
          GPROF_T0
          mbar_wait(&full[stage], phase);
          GPROF_ACC(2)
#ifdef B2S_GEMM_PROF
          if (kb == kb0) gp_w[0] += clock64() - gp_t0;
#endif
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C_::kStageBytes);
          const uint32_t sb = sa + C_::kABytes;
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; ++kk) {
            uint64_t ad, bd;
            if constexpr (A_MN) ad = make_sdesc(sa + kk * (UMMA_K * 128), 64 * BK * 2, 1024);
            else ad = make_sdesc(sa + kk * (UMMA_K * 2), 16, 1024);
            if constexpr (B_MN) bd = make_sdesc(sb + kk * (UMMA_K * 128), 64 * BK * 2, 1024);
            else bd = make_sdesc(sb + kk * (UMMA_K * 2), 16, 1024);
            if constexpr (CG == 2) mma_bf16_ss_pair(d_tmem, ad, bd, kIdesc, (kb > kb0 || kk) ? 1u : 0u);
            else mma_bf16_ss(d_tmem, ad, bd, kIdesc, (kb > kb0 || kk) ? 1u : 0u);
          }
          // frees the smem slot (in both CTAs) once these MMAs retire
          if constexpr (CG == 2) mma_commit_pair(&empty[stage], 0x3);
          else mma_commit(&empty[stage]);
          if (++stage == C_::kStages) { stage = 0; phase ^= 1; }
        }
        // accumulator ready for the epilogue(s)
        if constexpr (CG == 2) mma_commit_pair(&tfull[acc], 0x3);
        else mma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        GPROF_TILE
      }
      GPROF_END(0)
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ epilogue warps 2..9
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;  // this warp owns chunks half, half + kEG, ... of each tile
    uint8_t* ring = epi_smem + (warp - 2) * C_::kRing;
    // L2 policies of the C stores and the aux loads / stores (l2hints bits 4-5, 6-7; see launch())
    const uint64_t polC = l2_policy((l2hints >> 4) & 3), polX = l2_policy((l2hints >> 6) & 3);
    int slot = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    // Hand the next staging slot to this warp: the bulk store issued from it
    // two jobs ago must have finished reading smem.
    // fp32 outputs: two 4 KB slots (wait until <= 1 store group still reads smem);
    // bf16 outputs: four 2 KB slots (<= 3 pending) -- the GELU / SwiGLU epilogues
    // issue 2-3 stores per chunk and would otherwise wait on their own stores.
    // act 2 / 6 read their aux tiles through slots 2, 3 (TMA loads, one 32 x 32 bf16
    // box per chunk, 64-byte swizzle like the stores); their outputs use slots 0, 1
    const bool aux_tma = (epi.act == 2 || epi.act == 6);
    const bool two_slots = aux_tma || epi.act == 4;  // outputs staged through slots 0, 1 only
    uint64_t* abar = abar_all + 2 * (warp - 2);
    uint32_t aux_issued = 0, aux_used = 0;
    auto next_slot = [&]() -> uint8_t* {
      uint8_t* b;
      if (epi.out_f32) {
        if (lane == 0) bulk_wait_read<1>();
        b = ring + (slot & 1) * kStageSlot;
      } else if (two_slots) {
        if (lane == 0) bulk_wait_read<1>();
        b = ring + (slot & 1) * (kStageSlot / 2);
      } else {
        if (lane == 0) bulk_wait_read<3>();
        b = ring + (slot & 3) * (kStageSlot / 2);
      }
      __syncwarp();
      ++slot;
      return b;
    };
    // dGELU epilogue: this lane's 32 pre-activation values of the chunk, loaded
    // into registers one chunk ahead (the next chunk's loads are in flight while
    // the current one is processed), so the aux read latency is off the path.
    uint4 aux[4];
    auto load_aux = [&](int tile, int c) {
      if (!aux_tma) return;
      int mi_, ni_;
      tile_mn(tile % (num_m * num_n), num_m, num_n, raster, mi_, ni_);
      const int row0 = mi_ * BM * CG + rank * BM + q * 32;
      const int col = ni_ * BN + c * 32;
      const int s_ = aux_issued & 1;
      if (lane == 0) {  // out-of-range rows / columns are zero-filled and still counted
        mbar_arrive_expect_tx(&abar[s_], 32 * 32 * 2);
        tma_load_2d_hint(ring + (2 + s_) * (kStageSlot / 2), &tmAux, &abar[s_], col, row0, polX);
      }
      ++aux_issued;
    };
    // this chunk's aux tile -> registers (each lane its row's 64 bytes)
    auto take_aux = [&](bool read) {
      const int s_ = aux_used & 1;
      mbar_wait(&abar[s_], (aux_used >> 1) & 1);
      if (read) {
        const uint8_t* b = ring + (2 + s_) * (kStageSlot / 2);
#pragma unroll
        for (int k = 0; k < 4; ++k) aux[k] = *reinterpret_cast<const uint4*>(b + lane * 64 + ((k ^ ((lane >> 1) & 3)) * 16));
      }
      ++aux_used;
      __syncwarp();  // every lane has read the slot before its next TMA load is issued
    };
    GPROF_DECL
    for (int it = 0;; ++it) {
      const int tile = ring_get(it);
      __syncwarp();
      if (lane == 0) ring_release(it, tile);
      if (tile >= num_tiles) {
        GPROF_END(1)
        break;
      }
      GPROF_TILE
      load_aux(tile, half);  // first two chunks' aux tiles: in flight while the MMAs finish
      if (half + kEG < BN / 32) load_aux(tile, half + kEG);
      int mi, ni;
      tile_mn(tile % (num_m * num_n), num_m, num_n, raster, mi, ni);
      const int m0 = mi * BM * CG + rank * BM, n0 = ni * BN;
      GPROF_T0
      mbar_wait(&tfull[acc], acc_phase);
      GPROF_ACC(1)
      tc_fence_after();
      const int rbase = m0 + q * 32;
      if constexpr (SPEC == 3) {  // SwiGLU forward: gate chunk c with up chunk c + BN/64 of the same rows
        const int F = epi.glu_F, h0 = ni * (BN / 2);
#pragma unroll 1
        for (int c = half; c < BN / 64; c += kEG) {
          uint32_t rg[32], ru[32];
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, rg);
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + (c + BN / 64) * 32, ru);
          tmem_wait_ld();
          if (c + kEG >= BN / 64) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if constexpr (CG == 2) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&tempty[acc]), 0));
              else mbar_arrive(&tempty[acc]);
            }
          }
          const int hc = h0 + c * 32;
          if (rbase >= M || hc >= F) continue;
          float g[32], u[32], hv[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {  // what the unfused path stores and re-reads: bf16 gate / up
            g[i] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(rg[i])));
            u[i] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(ru[i])));
            float sg;
            hv[i] = silu_sig(g[i], sg) * u[i];
          }
          const float* outs[3] = {g, u, hv};
          const int cols[3] = {hc, F + hc, hc};
#pragma unroll
          for (int o = 0; o < 3; ++o) {
            uint8_t* b = next_slot();
            stage_bf16(b, lane, outs[o]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (o == 2) tma_store_2d_hint(&tmAux, b, cols[o], rbase, polX);
              else tma_store_2d_hint(&tmC, b, cols[o], rbase, polC);
              bulk_commit();
            }
          }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        continue;
      }
      if constexpr (SPEC == 7) {  // RoPE: a head's two halves (chunks k and k + dh/64) rotated together
        const int dh = epi.rope_dh, hc = dh / 64;  // chunk pairs per head
        const int units = BN / dh;
        const int tpos = rbase % epi.rope_T, rlane = (rbase + lane) % epi.rope_T;
        (void)tpos;
#pragma unroll 1
        for (int u = half; u < units; u += kEG) {
#pragma unroll 1
          for (int k = 0; k < hc; ++k) {
            const int ca = u * (dh / 32) + k, cb = ca + hc;  // TMEM chunks of the pair halves
            const int col_a = n0 + ca * 32, col_b = n0 + cb * 32;
            uint32_t ra[32], rb[32];
            tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + ca * 32, ra);
            tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + cb * 32, rb);
            tmem_wait_ld();
            if (u + kEG >= units && k + 1 == hc) {  // this warp's last chunks read: release the accumulator
              tc_fence_before();
              __syncwarp();
              if (lane == 0) {
                if constexpr (CG == 2) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&tempty[acc]), 0));
                else mbar_arrive(&tempty[acc]);
              }
            }
            if (rbase >= M || col_a >= N) continue;
            float va[32], vb[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {  // what the unfused path stores and the rope kernel re-reads
              va[i] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(ra[i])));
              vb[i] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(rb[i])));
            }
            if (col_a < epi.rope_cols) {
              const float* cp = epi.rope_cos + (int64_t)rlane * (dh / 2) + k * 32;
              const float* sp = epi.rope_sin + (int64_t)rlane * (dh / 2) + k * 32;
#pragma unroll
              for (int i4 = 0; i4 < 8; ++i4) {
                const float4 c4 = __ldg(reinterpret_cast<const float4*>(cp) + i4);
                const float4 s4 = __ldg(reinterpret_cast<const float4*>(sp) + i4);
                const float cc[4] = {c4.x, c4.y, c4.z, c4.w}, ss[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int i = 4 * i4 + e;
                  const float a = va[i], b = vb[i];
                  va[i] = a * cc[e] - b * ss[e];
                  vb[i] = b * cc[e] + a * ss[e];
                }
              }
            }
            const float* outs[2] = {va, vb};
            const int cols[2] = {col_a, col_b};
#pragma unroll
            for (int o = 0; o < 2; ++o) {
              uint8_t* b = next_slot();
              stage_bf16(b, lane, outs[o]);
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d_hint(&tmC, b, cols[o], rbase, polC);
                bulk_commit();
              }
            }
          }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        continue;
      }
      if constexpr (SPEC == 4) {  // SwiGLU backward: dh chunk (accumulator) -> [dgate | dup] using gu
        const int F = epi.glu_F;
        uint4 gq[4], uq[4];  // this chunk's gate / up rows (64 bytes each per lane)
        // gate and up 32 x 32 tiles of a chunk land in slots 2, 3 by TMA (zero-filled out of range)
        auto load_gu = [&](int col) {
          if (lane == 0) {
            mbar_arrive_expect_tx(&abar[0], 2 * 32 * 32 * 2);
            tma_load_2d_hint(ring + 2 * (kStageSlot / 2), &tmAux, &abar[0], col, rbase, polX);
            tma_load_2d_hint(ring + 3 * (kStageSlot / 2), &tmAux, &abar[0], col + F, rbase, polX);
          }
        };
        load_gu(n0 + half * 32);
#pragma unroll 1
        for (int c = half; c < BN / 32; c += kEG) {
          const int col0 = n0 + c * 32;
          const bool live = rbase < M && col0 < N;
          mbar_wait(&abar[0], aux_used & 1);
          ++aux_used;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int off = lane * 64 + ((k ^ ((lane >> 1) & 3)) * 16);
            gq[k] = *reinterpret_cast<const uint4*>(ring + 2 * (kStageSlot / 2) + off);
            uq[k] = *reinterpret_cast<const uint4*>(ring + 3 * (kStageSlot / 2) + off);
          }
          __syncwarp();  // slots 2, 3 read by every lane: the next chunk's tiles may land
          if (c + kEG < BN / 32) load_gu(col0 + kEG * 32);
          uint32_t r[32];
          tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, r);
          tmem_wait_ld();
          if (c + kEG >= BN / 32) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if constexpr (CG == 2) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&tempty[acc]), 0));
              else mbar_arrive(&tempty[acc]);
            }
          }
          if (!live) continue;
          float dg[32], du[32];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            float g8[8], u8[8];
            unpack8(*reinterpret_cast<const bf16x8*>(&gq[k]), g8);
            unpack8(*reinterpret_cast<const bf16x8*>(&uq[k]), u8);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float d = __bfloat162float(__float2bfloat16_rn(__uint_as_float(r[8 * k + j])));  // bf16 dh
              float sg;
              const float silu = silu_sig(g8[j], sg);
              du[8 * k + j] = d * silu;
              dg[8 * k + j] = d * u8[j] * sg * (1.f + g8[j] * (1.f - sg));
            }
          }
          const float* outs[2] = {dg, du};
#pragma unroll
          for (int o = 0; o < 2; ++o) {
            uint8_t* b = next_slot();
            stage_bf16(b, lane, outs[o]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d_hint(&tmC, b, col0 + o * F, rbase, polC);
              bulk_commit();
            }
          }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        continue;
      }
if constexpr (SPEC == 0) {
#pragma unroll 1
      for (int c = half; c < BN / 32; c += kEG) {
        const int col0 = n0 + c * 32;
        const bool live = rbase < M && col0 < N;  // warp-uniform
        // the chunk's bias (same 32 values for every lane): loads issued before the
        // TMEM wait so their latency overlaps it
        uint4 bias4[4];
        if (epi.bias && live) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (col0 + 8 * k < N) bias4[k] = __ldg(reinterpret_cast<const uint4*>(epi.bias + col0 + 8 * k));
        }
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, r);
        tmem_wait_ld();
        if (c + kEG >= BN / 32) {  // this warp's last chunk read: release the accumulator
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            // relaxed: the accumulator hand-off is a TMEM hazard, ordered by the tcgen05 fences
            if constexpr (CG == 2) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&tempty[acc]), 0));
            else mbar_arrive(&tempty[acc]);
          }
        }
        if (!live) {
          if (aux_tma) {
            take_aux(false);
            if (c + 2 * kEG < BN / 32) load_aux(tile, c + 2 * kEG);  // keep the chain going
          }
          continue;
        }
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        if (epi.bias) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (col0 + 8 * k < N) {
              float bb[8];
              unpack8(*reinterpret_cast<const bf16x8*>(&bias4[k]), bb);
#pragma unroll
              for (int j = 0; j < 8; ++j) v[8 * k + j] += bb[j];
            }
          }
        }
        if (epi.act == 1) {
          uint8_t* b = next_slot();
          stage_bf16(b, lane, v);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) { tma_store_2d_hint(&tmAux, b, col0, rbase, polX); bulk_commit(); }
#pragma unroll
          for (int i = 0; i < 32; i += 2) {  // GELU of the bf16-rounded pre-activation (what the backward sees)
            const float2 g = gelu_tanh2(__bfloat162float(__float2bfloat16_rn(v[i])),
                                        __bfloat162float(__float2bfloat16_rn(v[i + 1])));
            v[i] = g.x;
            v[i + 1] = g.y;
          }
        } else if (epi.act == 5) {  // GELU, aux <- gelu'(z) (bf16) for the backward's plain multiply
          uint32_t dg[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            float2 g;
            gelu_and_grad2(v[i], v[i + 1], g, dg[i / 2]);
            v[i] = g.x;
            v[i + 1] = g.y;
          }
          uint8_t* b = next_slot();
          stage_bf16_packed(b, lane, dg);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) { tma_store_2d_hint(&tmAux, b, col0, rbase, polX); bulk_commit(); }
        } else if (epi.act == 6) {  // x aux (gelu' stored by the act-5 forward)
          take_aux(true);
          if (c + 2 * kEG < BN / 32) load_aux(tile, c + 2 * kEG);  // two chunks ahead (both slots busy)
#pragma unroll
          for (int c8 = 0; c8 < 4; ++c8) {
            float h[8];
            unpack8(*reinterpret_cast<const bf16x8*>(&aux[c8]), h);
#pragma unroll
            for (int j = 0; j < 8; ++j) v[c8 * 8 + j] *= h[j];
          }
        } else if (epi.act == 2) {
          take_aux(true);
          if (c + 2 * kEG < BN / 32) load_aux(tile, c + 2 * kEG);  // two chunks ahead (both slots busy)
#pragma unroll
          for (int c8 = 0; c8 < 4; ++c8) {
            float h[8];
            unpack8(*reinterpret_cast<const bf16x8*>(&aux[c8]), h);
#pragma unroll
            for (int j = 0; j < 8; j += 2) {
              const float2 g = gelu_tanh_grad2(h[j], h[j + 1]);
              v[c8 * 8 + j] *= g.x;
              v[c8 * 8 + j + 1] *= g.y;
            }
          }
        }
        uint8_t* b = next_slot();
        if (epi.out_f32) stage_f32(b, lane, v);
        else stage_bf16(b, lane, v);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (epi.accumulate) tma_reduce_add_2d(&tmC, b, col0, rbase);
          else tma_store_2d_hint(&tmC, b, col0, rbase, polC);
          bulk_commit();
        }
        if (epi.colsum_part && !epi.out_f32) {
          // column sums of the staged (bf16-rounded) 32 x 32 tile: lane l sums columns
          // 2(l & 15), +1 over rows 16 (l >> 4) .. +15, then the two row halves combine
          const int cw = lane & 15, rh = lane >> 4;
          float s0 = 0.f, s1 = 0.f;
#pragma unroll
          for (int r = 0; r < 16; ++r) {
            const int row = rh * 16 + r;
            const uint32_t w = *reinterpret_cast<const uint32_t*>(
                b + row * 64 + (((cw >> 2) ^ ((row >> 1) & 3)) * 16) + (cw & 3) * 4);
            s0 += __uint_as_float(w << 16);
            s1 += __uint_as_float(w & 0xffff0000u);
          }
          s0 += __shfl_xor_sync(0xffffffffu, s0, 16);
          s1 += __shfl_xor_sync(0xffffffffu, s1, 16);
          const int col = col0 + 2 * cw;
          if (lane < 16 && col < N)
            *reinterpret_cast<float2*>(epi.colsum_part + (int64_t)(rbase >> 5) * N + col) = make_float2(s0, s1);
        }
      }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
  }

  tc_fence_before();
  if constexpr (CG == 2) cluster_sync();  // no CTA leaves while its peer may still signal it
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc_pair<C_::kTmemCols>(tmem_base);
    else tmem_dealloc<C_::kTmemCols>(tmem_base);
  }
  // every CTA has fetched its sentinel: the last one out re-arms the counter for the next launch
  if (sched && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(sched + 1, 1) == (int)gridDim.x - 1) {
      sched[0] = 0;
      sched[1] = 0;
      __threadfence();
    }
  }
}

// SMs the persistent GEMM grid occupies: all of them (reserving some for NCCL's CTAs at W > 1
// was measured slower; the dynamic tile counter already lets late CTAs take fewer).
static int gemm_sms() { return kNumSMs; }

// Per-device pool of zeroed scheduler counters {next_tile, ctas_done}; launches
// rotate through the pool so GEMMs in flight on different streams never share one.
constexpr int kSchedSlots = 64;
static int* sched_slot() {
  static int* pool[64] = {};
  static int next[64] = {};
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (!pool[dev]) {
    if (cudaMalloc(&pool[dev], kSchedSlots * 2 * sizeof(int)) != cudaSuccess) return nullptr;
    cudaMemset(pool[dev], 0, kSchedSlots * 2 * sizeof(int));
    cudaDeviceSynchronize();
  }
  int* p = pool[dev] + 2 * next[dev];
  next[dev] = (next[dev] + 1) % kSchedSlots;
  return p;
}

// Raster choice by a wave model of L2 reuse. Tiles run in index order, `slots` at a time
// (one per CTA / CTA pair). A wave loads every distinct A block (BM*CG rows x K) and B block
// (BN rows x K) its tiles touch once -- concurrent tiles stream the same K slices in near
// lockstep -- and a block the previous wave also touched is still in L2 with probability
// min(1, budget / bytes of that wave's blocks). The candidate with the fewest modelled DRAM
// bytes wins: M-grouped or N-grouped, group sizes 1, 2, 4, ... (the full extent is the plain
// M- / N-fastest order). Cached per shape.
static int choose_raster(int num_m, int num_n, double a_blk, double b_blk, int slots) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, long long, long long, int>, int> cache;
  const auto key = std::make_tuple(num_m, num_n, (long long)a_blk, (long long)b_blk, slots);
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  const double budget = 48e6;  // of the 126 MB L2: two dies, outputs stream through it too
  const int total = num_m * num_n;
  auto cost = [&](int raster) {
    std::vector<int> seenA(num_m, -2), seenB(num_n, -2);  // last wave that touched the block
    double bytes = 0.0, prev_bytes = 0.0;
    for (int w0 = 0, w = 0; w0 < total; w0 += slots, ++w) {
      double wave_bytes = 0.0, load = 0.0;
      const double f = prev_bytes > 0 ? std::min(1.0, budget / prev_bytes) : 0.0;
      for (int t = w0; t < std::min(total, w0 + slots); ++t) {
        int mi, ni;
        if (raster > 0) {
          const int gt = raster * num_n, g = t / gt, l = t - g * gt, gm = std::min(raster, num_m - g * raster);
          mi = g * raster + l % gm;
          ni = l / gm;
        } else {
          const int G = -raster, gt = G * num_m, g = t / gt, l = t - g * gt, gn = std::min(G, num_n - g * G);
          ni = g * G + l % gn;
          mi = l / gn;
        }
        if (seenA[mi] != w) {
          load += a_blk * (seenA[mi] == w - 1 ? 1.0 - f : 1.0);
          seenA[mi] = w;
          wave_bytes += a_blk;
        }
        if (seenB[ni] != w) {
          load += b_blk * (seenB[ni] == w - 1 ? 1.0 - f : 1.0);
          seenB[ni] = w;
          wave_bytes += b_blk;
        }
      }
      bytes += load;
      prev_bytes = wave_bytes;
    }
    return bytes;
  };
  int best = num_m;  // M-fastest
  double best_cost = cost(best);
  for (int g = 1;; g *= 2) {
    const bool more_m = g < num_m, more_n = g < num_n;
    if (!more_m && !more_n) break;
    if (more_m) {
      const double c = cost(g);
      if (c < best_cost * 0.98) { best_cost = c; best = g; }
    }
    const double c = cost(-std::min(g, num_n));
    if (c < best_cost * 0.98) { best_cost = c; best = -std::min(g, num_n); }
  }
  std::lock_guard<std::mutex> lock(mu);
  cache[key] = best;
  return best;
}

template <int BN, int CG, bool A_MN, bool B_MN, int EW, int SPEC>
static int launch(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                  const CUtensorMap& tx, int M, int N, int K, int splits, const Epi& e, cudaStream_t st) {
  using C_ = Cfg<BN, CG, EW>;
  auto kern = gemm_kernel<BN, CG, A_MN, B_MN, EW, SPEC>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::kSmem);
    if (CG == 2) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    attr_set = true;
  }
  const int tiles = ((M + BM * CG - 1) / (BM * CG)) * ((N + BN - 1) / BN) * splits;
  const int slots = gemm_sms() / CG;
  const int grid = (tiles < slots ? tiles : slots) * CG;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(C_::kThreads);
  cfg.dynamicSmemBytes = C_::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int* sched = sched_slot();
  if (!sched) { set_error("gemm: scheduler counter allocation failed"); return B2S_ECUDA; }
  const int num_m = (M + BM * CG - 1) / (BM * CG), num_n = (N + BN - 1) / BN;
  // B2S_GEMM_RASTER (tests / A-B runs): "mfast" = plain M-fastest order, an integer = that raster
  // (clamped to the tile grid); read per launch like B2S_GEMM_FORCE
  const char* rs = getenv("B2S_GEMM_RASTER");
  const double kbytes = 2.0 * ((K + splits - 1) / splits);
  int raster;
  if (rs && strcmp(rs, "mfast") == 0) raster = num_m;
  else if (rs && atoi(rs) != 0) raster = atoi(rs) > 0 ? std::min(atoi(rs), num_m) : -std::min(-atoi(rs), num_n);
  else raster = choose_raster(num_m, num_n, BM * CG * kbytes, BN * kbytes, slots);
  // L2 hints for the rasters where one operand is streamed through exactly once and the other
  // is re-read by every wave: raster 1 (each M block meets all N blocks back to back) streams A
  // and re-reads B, raster -1 the reverse. The streamed operand is loaded evict_first when the
  // re-read one is at most 40 MB, so the streamed bytes stop pushing it out (e.g. the long-K
  // down-projection, whose W2 otherwise returns from DRAM once per wave). (evict_last on the
  // re-read operand was measured worse: the sticky lines outlive the kernel.)
  // B2S_GEMM_L2HINT=0 disables them (A/B runs).
  int l2hints = 0;
  static const bool hints_on = !(getenv("B2S_GEMM_L2HINT") && atoi(getenv("B2S_GEMM_L2HINT")) == 0);
  if (hints_on && (long long)num_m * num_n > slots && splits == 1) {
    const double a_tot = (double)M * K * 2, b_tot = (double)N * K * 2;
    if (raster == 1 && num_n <= slots && b_tot <= 40e6) l2hints = 1;
    else if (raster == -1 && num_m <= slots && a_tot <= 40e6) l2hints = 1 << 2;
  }
  // Epilogue streams written or read exactly once, evict_first so they stop displacing the
  // mainloop's re-read operand blocks: the saved activations (SwiGLU gate|up, GELU
  // pre-activation / gelu'), the aux inputs of the backward epilogues, dgu, and C when it is
  // far larger than L2 (the LM-head logits). Measured on the Llama-1B SwiGLU backward:
  // 521 -> 483 us. B2S_GEMM_EPI_HINT=0 disables them (A/B runs).
  static const bool epi_hints_on = !(getenv("B2S_GEMM_EPI_HINT") && atoi(getenv("B2S_GEMM_EPI_HINT")) == 0);
  if (epi_hints_on) {
    const double c_bytes = (double)M * N * (e.out_f32 ? 4 : 2);
    const bool c_stream = e.act == 3 || e.act == 4 || (!e.accumulate && c_bytes >= 512e6);
    const bool x_stream = e.act == 1 || e.act == 2 || e.act == 4 || e.act == 5 || e.act == 6;
    l2hints |= (c_stream ? 1 << 4 : 0) | (x_stream ? 1 << 6 : 0);
  }
  cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, tx, M, N, K, splits, raster, l2hints, e, sched);
  return check_launch("gemm");
}

template <int BN, int CG, int EW = 8, int SPEC = 0>
static int dispatch(bool amn, bool bmn, const CUtensorMap& ta, const CUtensorMap& tb,
                    const CUtensorMap& tc, const CUtensorMap& tx, int M, int N, int K,
                    int splits, const Epi& e, cudaStream_t st) {
  if (!amn && !bmn) return launch<BN, CG, false, false, EW, SPEC>(ta, tb, tc, tx, M, N, K, splits, e, st);
  if (!amn && bmn) return launch<BN, CG, false, true, EW, SPEC>(ta, tb, tc, tx, M, N, K, splits, e, st);
  if (amn && !bmn) return launch<BN, CG, true, false, EW, SPEC>(ta, tb, tc, tx, M, N, K, splits, e, st);
  return launch<BN, CG, true, true, EW, SPEC>(ta, tb, tc, tx, M, N, K, splits, e, st);
}

// Tile choice: (BN, CTA group, split-K) maximising filled SM slots in the last
// wave, weighted by the measured per-tile speed of each configuration.
struct Choice {
  int bn, cg, splits;
};
static Choice choose(int M, int N, int K, bool can_split) {
  const int nkb = (K + BK - 1) / BK;
  if (const char* f = getenv("B2S_GEMM_FORCE")) {  // "bn,cg,splits" (tests / tuning)
    Choice c{256, 1, 1};
    if (sscanf(f, "%d,%d,%d", &c.bn, &c.cg, &c.splits) == 3 && (c.bn == 128 || c.bn == 256) &&
        (c.cg == 1 || (c.cg == 2 && c.bn == 256)) && c.splits >= 1) {
      if (!can_split) c.splits = 1;
      return c;
    }
  }
  const Choice cands[3] = {{256, 2, 1}, {256, 1, 1}, {128, 1, 1}};
  const double speed[3] = {1.2, 1.05, 1.0};
  Choice best = cands[2];
  double best_score = -1.0;
  for (int i = 0; i < 3; ++i) {
    for (int sp = 1; sp <= (can_split ? 16 : 1); sp *= 2) {
      if (sp > 1 && nkb / sp < 8) break;
      const Choice c{cands[i].bn, cands[i].cg, sp};
      const long mt = (M + BM * c.cg - 1) / (BM * c.cg), nt = (N + c.bn - 1) / c.bn;
      const long tiles = mt * nt * sp, slots = gemm_sms() / c.cg;
      const long waves = (tiles + slots - 1) / slots;
      const double fill = (double)tiles / (double)(waves * slots);
      const double pad = ((double)M / (mt * BM * c.cg)) * ((double)N / (nt * c.bn));
      const double split_cost = 1.0 - 0.02 * (sp - 1);  // extra fp32 add-reduce traffic
      const double score = fill * pad * speed[i] * split_cost;
      if (score > best_score * 1.001) { best_score = score; best = c; }
    }
  }
  return best;
}

}  // namespace gemm
}  // namespace b2s

#ifdef B2S_GEMM_PROF
extern "C" int b2s_gemm_prof_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, b2s::gemm::g_gprof, sizeof(b2s::gemm::g_gprof)) == cudaSuccess ? 0 : -1;
}
#endif

namespace {
// Shared host path. glu_F / c_width: SwiGLU epilogues (act 3: N = 2F, aux = h [M, F];
// act 4: N = F, C = dgu [M, 2F] of width c_width, aux = gu).
int gemm_run(const void* d_A, int a_mn_major, int64_t lda, const void* d_B, int b_mn_major, int64_t ldb, void* d_C,
             int64_t ldc, int c_f32, int M, int N, int K, int accumulate, const void* d_bias, int act, void* d_aux,
             int64_t ld_aux, int glu_F, int64_t c_width, int64_t aux_width, cudaStream_t st,
             float* d_colsum_part = nullptr, const float* rope_cos = nullptr, const float* rope_sin = nullptr,
             int rope_T = 0, int rope_dh = 0, int rope_cols = 0) {
  using namespace b2s;
  B2S_REQUIRE(M > 0 && N > 0 && K > 0, B2S_EINVAL, "gemm: empty shape %d x %d x %d", M, N, K);
  B2S_REQUIRE(d_A && d_B && d_C, B2S_EINVAL, "gemm: null operand");
  B2S_REQUIRE((lda * 2) % 16 == 0 && (ldb * 2) % 16 == 0, B2S_EUNSUPPORTED,
              "gemm: operand row strides must be multiples of 8 elements");
  B2S_REQUIRE(((uintptr_t)d_A % 16) == 0 && ((uintptr_t)d_B % 16) == 0 && ((uintptr_t)d_C % 16) == 0,
              B2S_EUNSUPPORTED, "gemm: operands must be 16-byte aligned");
  B2S_REQUIRE((ldc * (c_f32 ? 4 : 2)) % 16 == 0 && N % 8 == 0, B2S_EUNSUPPORTED,
              "gemm: N and ldc must keep output rows 16B aligned");
  B2S_REQUIRE(act == 0 || act == 7 ||
                  (act >= 1 && act <= 6 && d_aux && !c_f32 && (ld_aux * 2) % 16 == 0 && ((uintptr_t)d_aux % 16) == 0),
              B2S_EINVAL, "gemm: activation epilogue needs an aligned bf16 aux buffer and bf16 output");
  B2S_REQUIRE(!(accumulate && (act == 1 || act == 3 || act == 4 || act == 5 || act == 7)), B2S_EINVAL,
              "gemm: accumulate with a GELU / SwiGLU epilogue is not supported");
  B2S_REQUIRE(accumulate != 2 || (c_f32 && act == 0 && !d_bias), B2S_EINVAL,
              "gemm: overwrite mode (accumulate=2) needs an fp32 C without bias / activation");
  gemm::Choice ch = gemm::choose(M, N, K, accumulate && !d_bias && act == 0);
  if (accumulate == 2) {  // overwrite: a store when K is not split, else zero C and add-reduce the splits
    if (ch.splits == 1) {
      accumulate = 0;
    } else {
      if (cudaMemset2DAsync(d_C, (size_t)ldc * 4, 0, (size_t)N * 4, (size_t)M, st) != cudaSuccess)
        return check_launch("gemm overwrite memset");
      accumulate = 1;
    }
  }
  if (act == 3) ch = gemm::Choice{256, 2, 1};  // the gate / up interleave needs CTA-pair 256-wide tiles
  if (act == 4) ch = gemm::Choice{256, 2, 1};
  if (act == 7) ch = gemm::Choice{256, 2, 1};  // a 256-wide tile holds whole heads (dh 64 / 128)
  const int bn = ch.bn, bnc = ch.bn / ch.cg;
  CUtensorMap ta, tb, tc, tx;
  int rc;
  if (a_mn_major) rc = encode_tma_2d(&ta, d_A, 2, (uint64_t)M, (uint64_t)K, (uint64_t)lda * 2, 64, gemm::BK, 128);
  else rc = encode_tma_2d(&ta, d_A, 2, (uint64_t)K, (uint64_t)M, (uint64_t)lda * 2, gemm::BK, gemm::BM, 128);
  if (rc) return rc;
  if (b_mn_major) rc = encode_tma_2d(&tb, d_B, 2, (uint64_t)N, (uint64_t)K, (uint64_t)ldb * 2, 64, gemm::BK, 128);
  else rc = encode_tma_2d(&tb, d_B, 2, (uint64_t)K, (uint64_t)N, (uint64_t)ldb * 2, gemm::BK, (uint32_t)bnc, 128);
  if (rc) return rc;
  if (c_f32) rc = encode_tma_2d(&tc, d_C, 4, (uint64_t)c_width, (uint64_t)M, (uint64_t)ldc * 4, 32, 32, 128);
  else rc = encode_tma_2d(&tc, d_C, 2, (uint64_t)c_width, (uint64_t)M, (uint64_t)ldc * 2, 32, 32, 64);
  if (rc) return rc;
  if (act >= 1 && act <= 6)
    rc = encode_tma_2d(&tx, d_aux, 2, (uint64_t)aux_width, (uint64_t)M, (uint64_t)ld_aux * 2, 32, 32, 64);
  else tx = tc;
  if (rc) return rc;
  gemm::Epi e{c_f32, accumulate, (const __nv_bfloat16*)d_bias, act, (const __nv_bfloat16*)d_aux, ld_aux, glu_F,
              d_colsum_part, rope_cos, rope_sin, rope_T, rope_dh, rope_cols};
  const int splits = ch.splits;
  // specialised epilogues: SwiGLU forward (x, W13 both K-major), SwiGLU backward (W2 MN-major),
  // RoPE (K-major); all on 256-wide CTA-pair tiles
  // (SwiGLU forward: 8 epilogue warps and the 5-stage mainloop, 766 vs 803 us with 12 at the
  // Llama-1B gate|up shape; the backward keeps 12: 509 vs 525 us)
  if (act == 3) return gemm::launch<256, 2, false, false, 8, 3>(ta, tb, tc, tx, M, N, K, splits, e, st);
  if (act == 4) return gemm::launch<256, 2, false, true, 12, 4>(ta, tb, tc, tx, M, N, K, splits, e, st);
  if (act == 7) return gemm::launch<256, 2, false, false, 8, 7>(ta, tb, tc, tx, M, N, K, splits, e, st);
  if (ch.cg == 2 && act != 0 && act != 6)  // activation epilogue: 12 epilogue warps (see EW above);
    // the x aux product (act 6) is light enough for 8 warps and the deeper 5-stage mainloop
    return gemm::dispatch<256, 2, 12>(a_mn_major, b_mn_major, ta, tb, tc, tx, M, N, K, splits, e, st);
  if (ch.cg == 2) return gemm::dispatch<256, 2>(a_mn_major, b_mn_major, ta, tb, tc, tx, M, N, K, splits, e, st);
  if (bn == 256) return gemm::dispatch<256, 1>(a_mn_major, b_mn_major, ta, tb, tc, tx, M, N, K, splits, e, st);
  return gemm::dispatch<128, 1>(a_mn_major, b_mn_major, ta, tb, tc, tx, M, N, K, splits, e, st);
}
}  // namespace

extern "C" int b2s_gemm(const void* d_A, int a_mn_major, int64_t lda, const void* d_B,
                        int b_mn_major, int64_t ldb, void* d_C, int64_t ldc, int c_f32, int M,
                        int N, int K, int accumulate, const void* d_bias, int act, void* d_aux,
                        int64_t ld_aux, b2s_stream_t stream) {
  B2S_REQUIRE(act == 0 || act == 1 || act == 2 || act == 5 || act == 6, B2S_EINVAL,
              "gemm: act must be 0, 1, 2, 5 or 6 (SwiGLU: b2s_gemm_swiglu_*)");
  B2S_REQUIRE(!(accumulate && (act == 1 || act == 5)), B2S_EINVAL, "gemm: accumulate with GELU is not supported");
  return gemm_run(d_A, a_mn_major, lda, d_B, b_mn_major, ldb, d_C, ldc, c_f32, M, N, K, accumulate, d_bias, act,
                  d_aux, ld_aux, 0, N, N, (cudaStream_t)stream);
}

extern "C" int b2s_gemm_colsum(const void* d_A, int a_mn_major, int64_t lda, const void* d_B, int b_mn_major,
                               int64_t ldb, void* d_C, int64_t ldc, int M, int N, int K, int act, void* d_aux,
                               int64_t ld_aux, float* d_colsum_part, b2s_stream_t stream) {
  B2S_REQUIRE(act == 0 || act == 2 || act == 6, B2S_EINVAL, "gemm_colsum: act must be 0, 2 or 6");
  B2S_REQUIRE(d_colsum_part && ((uintptr_t)d_colsum_part % 8) == 0, B2S_EINVAL, "gemm_colsum: null / misaligned partials");
  return gemm_run(d_A, a_mn_major, lda, d_B, b_mn_major, ldb, d_C, ldc, 0, M, N, K, 0, nullptr, act, d_aux, ld_aux, 0, N,
                  N, (cudaStream_t)stream, d_colsum_part);
}

extern "C" int b2s_gemm_swiglu_fwd(const void* d_x, int64_t ldx, const void* d_w13, int64_t ldw, void* d_gu,
                                   int64_t ld_gu, void* d_h, int64_t ld_h, int M, int F, int K,
                                   b2s_stream_t stream) {
  B2S_REQUIRE(F > 0 && F % 128 == 0, B2S_EUNSUPPORTED, "gemm_swiglu_fwd: F must be a multiple of 128, got %d", F);
  return gemm_run(d_x, 0, ldx, d_w13, 0, ldw, d_gu, ld_gu, 0, M, 2 * F, K, 0, nullptr, 3, d_h, ld_h, F, 2 * F, F,
                  (cudaStream_t)stream);
}

extern "C" int b2s_gemm_swiglu_bwd(const void* d_dy, int64_t ld_dy, const void* d_w2, int64_t ldw, const void* d_gu,
                                   int64_t ld_gu, void* d_dgu, int64_t ld_dgu, int M, int F, int K,
                                   b2s_stream_t stream) {
  B2S_REQUIRE(F > 0 && F % 8 == 0, B2S_EUNSUPPORTED, "gemm_swiglu_bwd: F must be a multiple of 8");
  return gemm_run(d_dy, 0, ld_dy, d_w2, 1, ldw, d_dgu, ld_dgu, 0, M, F, K, 0, nullptr, 4, const_cast<void*>(d_gu),
                  ld_gu, F, 2 * F, 2 * F, (cudaStream_t)stream);
}

extern "C" int b2s_gemm_rope(const void* d_x, int64_t ldx, const void* d_w, int64_t ldw, void* d_out, int64_t ldo,
                             int M, int N, int K, const float* d_cos, const float* d_sin, int T, int dh, int rope_cols,
                             b2s_stream_t stream) {
  B2S_REQUIRE(dh == 64 || dh == 128, B2S_EUNSUPPORTED, "gemm_rope: head dim must be 64 or 128, got %d", dh);
  B2S_REQUIRE(N % 256 == 0 && rope_cols % dh == 0 && rope_cols <= N, B2S_EUNSUPPORTED,
              "gemm_rope: N (%d) must be a multiple of 256 and rope_cols (%d) of dh", N, rope_cols);
  B2S_REQUIRE(d_cos && d_sin && T > 0 && ((uintptr_t)d_cos % 16) == 0 && ((uintptr_t)d_sin % 16) == 0, B2S_EINVAL,
              "gemm_rope: null / misaligned tables");
  return gemm_run(d_x, 0, ldx, d_w, 0, ldw, d_out, ldo, 0, M, N, K, 0, nullptr, 7, nullptr, 0, 0, N, N,
                  (cudaStream_t)stream, nullptr, d_cos, d_sin, T, dh, rope_cols);
}
