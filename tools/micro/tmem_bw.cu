// TMEM read / write throughput on one SM (sm_100a): W warps each issue tcgen05.ld (32x32b) of
// X columns from their lane quarter, then tcgen05.wait::ld, in a loop; clock64 per CTA.
// Prints bytes per clock per SM -- the bound on how fast softmax / epilogue warps can drain
// accumulators (the attention backward reads 160 KB of TMEM per 128x128 step).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu && ./tmem_bw
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#define LD32(taddr, r)                                                                                      \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 "                                                   \
               "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"                                   \
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                 \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),      \
                 "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),   \
                 "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),             \
                 "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),             \
                 "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])              \
               : "r"(taddr))
#define ST32(taddr, r)                                                                                      \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "                                             \
               "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"                                  \
               "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"                         \
               ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),  \
                 "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),          \
                 "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]),       \
                 "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),       \
                 "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory")

// OP 0: ld x32 + wait per iteration; OP 1: four ld x32 (128 columns) then one wait;
// OP 2: st x32 + wait::st; OP 3: ld x32 + wait then 32 dependent FFMA (a softmax-like body)
template <int OP>
__global__ void k(uint32_t* out, long long* cyc, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  const int colw = (warp >> 2) * 128;  // warps of the same quarter take different column ranges
  uint32_t acc = 0, r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = lane + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if constexpr (OP == 0 || OP == 3) {
      LD32(base + ((colw + (it & 3) * 32) & 511), r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if constexpr (OP == 3) {
        float f = 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) f = fmaf(__uint_as_float(r[i]), 1.0001f, f);
        acc += __float_as_uint(f);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) acc ^= r[i];
      }
    } else if constexpr (OP == 1) {
      uint32_t q0[32], q1[32], q2[32], q3[32];
      LD32(base + colw, q0);
      LD32(base + colw + 32, q1);
      LD32(base + colw + 64, q2);
      LD32(base + colw + 96, q3);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) acc ^= q0[i] ^ q1[i] ^ q2[i] ^ q3[i];
    } else if constexpr (OP == 2) {
      r[it & 31] += it;
      ST32(base + ((colw + (it & 3) * 32) & 511), r);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + r[0];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int OP>
void run(const char* name, int warps) {
  const int blocks = 148, iters = 4096;
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, blocks * 1024 * 4);
  cudaMalloc(&cyc, blocks * 8);
  k<OP><<<blocks, warps * 32>>>(out, cyc, 16);
  k<OP><<<blocks, warps * 32>>>(out, cyc, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < blocks; ++i) mean += h[i];
  mean /= blocks;
  const double bytes = (OP == 1 ? 4.0 : 1.0) * warps * 32.0 * 32 * 4 * iters;
  printf("%-28s warps %2d: %7.1f clk/iter  %7.1f B/clk/SM  (%s)\n", name, warps, mean / iters, bytes / mean,
         cudaGetErrorString(e));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16}) run<0>("ld32x32b.x32 + wait", w);
  for (int w : {4, 8, 16}) run<1>("4 x ld.x32 then wait", w);
  for (int w : {4, 8, 16}) run<2>("st32x32b.x32 + wait", w);
  for (int w : {4, 8, 16}) run<3>("ld.x32 + wait + 32 FFMA", w);
  return 0;
}
