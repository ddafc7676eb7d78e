// Tensor-pipe time of the attention backward's per-step MMA mix (dh 64), issued back to back
// by one thread with nothing else running: S^T = K Q^T and dP^T = V dO^T (M128 N128 K64, SS),
// dV += P^T dO (TMEM-A, M128 N64 K128), dK += dS^T Q (SS, B MN-major), dQ = dS K (SS, both
// MN-major). Floor per step = 1280 clk (tcgen05: 128*N/256 clk per K=16 MMA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2602_08387_b200/csrc \
//        -o bwd_mma bwd_mma.cu -lcuda && ./bwd_mma
#include <cstdio>
#include "sm100.cuh"
using namespace b2s::sm100;

constexpr int kTile = 128 * 64 * 2;

template <int MIX>
__global__ void __launch_bounds__(128, 1) k(long long* cyc, int steps) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  uint8_t *sK = sm, *sV = sm + kTile, *sQ = sm + 2 * kTile, *sdO = sm + 3 * kTile, *sdS = sm + 4 * kTile;
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 6 * kTile / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot;
  const uint32_t tS = tb, tdP = tb + 128, tdV = tb + 256, tdK = tb + 320, tdQ = tb + 384, tPT = tb + 448;
  if (warp == 1) {
    constexpr uint32_t idSS = make_idesc_bf16(128, 128, false, false);
    constexpr uint32_t idKM = make_idesc_bf16(128, 64, false, true);
    constexpr uint32_t idMM = make_idesc_bf16(128, 64, true, true);
    const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aQ = smem_u32(sQ), adO = smem_u32(sdO), adS = smem_u32(sdS);
    long long t0 = clock64();
    for (int t = 0; t < steps; ++t) {
      if (MIX == 0 || MIX == 1) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16_ss_w(tS, make_sdesc(aK + kk * 32, 16, 1024), make_sdesc(aQ + kk * 32, 16, 1024), idSS, kk > 0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16_ss_w(tdP, make_sdesc(aV + kk * 32, 16, 1024), make_sdesc(adO + kk * 32, 16, 1024), idSS, kk > 0);
      }
      if (MIX == 0 || MIX == 2 || MIX == 3) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t a_ds = make_sdesc(adS + (kk >> 2) * kTile + (kk & 3) * 32, 16, 1024);
          if (MIX == 3)
            mma_bf16_ss_w(tdV, a_ds, make_sdesc(adO + kk * 2048, kTile, 1024), idKM, 1);
          else
            mma_bf16_ts_w(tdV, tPT + kk * 8, make_sdesc(adO + kk * 2048, kTile, 1024), idKM, 1);
          mma_bf16_ss_w(tdK, a_ds, make_sdesc(aQ + kk * 2048, kTile, 1024), idKM, 1);
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_bf16_ss_w(tdQ, make_sdesc(adS + kk * 2048, kTile, 1024), make_sdesc(aK + kk * 2048, kTile, 1024), idMM,
                        kk > 0);
      }
      if (MIX == 4) {  // dQ only
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_bf16_ss_w(tdQ, make_sdesc(adS + kk * 2048, kTile, 1024), make_sdesc(aK + kk * 2048, kTile, 1024), idMM,
                        kk > 0);
      }
      if (MIX == 5) {  // dK only
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t a_ds = make_sdesc(adS + (kk >> 2) * kTile + (kk & 3) * 32, 16, 1024);
          mma_bf16_ss_w(tdK, a_ds, make_sdesc(aQ + kk * 2048, kTile, 1024), idKM, 1);
        }
      }
      if (MIX == 6) {  // dV (TMEM A) only
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_bf16_ts_w(tdV, tPT + kk * 8, make_sdesc(adO + kk * 2048, kTile, 1024), idKM, 1);
      }
      mma_commit_w(&bar);
    }
    mbar_wait(&bar, (steps - 1) & 1);
    long long t1 = clock64();
    if (threadIdx.x == 32) cyc[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

template <int MIX>
void run(const char* name, double floor_clk) {
  long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  const int smem = 6 * kTile + 1024;
  cudaFuncSetAttribute(k<MIX>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int steps = 2000;
  k<MIX><<<148, 128, smem>>>(cyc, 10);
  k<MIX><<<148, 128, smem>>>(cyc, steps);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 148; ++i) m += h[i];
  m /= 148.0 * steps;
  printf("%-34s %7.1f clk/step  floor %6.0f  (%.0f%%)  %s\n", name, m, floor_clk, 100 * floor_clk / m,
         cudaGetErrorString(e));
  cudaFree(cyc);
}

int main() {
  run<0>("full step mix (S dP dV dK dQ)", 1280);
  run<1>("S^T + dP^T (N128 SS)", 512);
  run<2>("dV(ts) dK dQ", 768);
  run<3>("dV(ss) dK dQ", 768);
  run<4>("dQ only (MN/MN)", 256);
  run<5>("dK only (K/MN)", 256);
  run<6>("dV only (TMEM A)", 256);
  return 0;
}
