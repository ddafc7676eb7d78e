// TMEM load throughput by tcgen05.ld shape: each warp reads 128 columns of its lane quarter
// (16 KB) as 8 x 32x32b.x16, 4 x .x32, 2 x .x64 or 1 x .x128, then one tcgen05.wait::ld.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ld tmem_ld.cu && ./tmem_ld
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#define R4(i) "=r"(r[i]), "=r"(r[i + 1]), "=r"(r[i + 2]), "=r"(r[i + 3])
template <int X>
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t* r) {
  if constexpr (X == 16)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : R4(0), R4(4), R4(8), R4(12) : "r"(taddr));
  if constexpr (X == 32)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : R4(0), R4(4), R4(8), R4(12), R4(16), R4(20), R4(24), R4(28) : "r"(taddr));
  if constexpr (X == 64)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,"
                 "%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
                 : R4(0), R4(4), R4(8), R4(12), R4(16), R4(20), R4(24), R4(28), R4(32), R4(36), R4(40), R4(44), R4(48),
                   R4(52), R4(56), R4(60)
                 : "r"(taddr));
}

template <int X>
__global__ void k(uint32_t* out, long long* cyc, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[128];
#pragma unroll
    for (int c = 0; c < 128 / X; ++c) ld<X>(base + c * X, r + c * X);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 128; ++i) acc ^= r[i];
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int X>
void run(int warps) {
  const int blocks = 148, iters = 1024;
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, blocks * 1024 * 4);
  cudaMalloc(&cyc, blocks * 8);
  k<X><<<blocks, warps * 32>>>(out, cyc, 16);
  k<X><<<blocks, warps * 32>>>(out, cyc, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < blocks; ++i) m += h[i];
  m /= blocks;
  printf("32x32b.x%-3d x%d per wait  warps %d: %6.1f clk/iter  %6.1f B/clk/SM (%s)\n", X, 128 / X, warps, m / iters,
         (double)warps * 16384 * iters / m, cudaGetErrorString(e));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 8}) { run<16>(w); run<32>(w); run<64>(w); }
  return 0;
}
