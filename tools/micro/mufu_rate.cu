// MUFU.EX2 throughput per SM (sm_100a): W warps per CTA, one CTA per SM, each thread runs
// `iters` x 8 independent ex2.approx.ftz; optionally with the attention forward's per-element
// companions (FFMA scale-subtract, FADD row sum, F2FP pack). Prints ex2 per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_rate mufu_rate.cu && ./mufu_rate
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int MIX>
__global__ void k(float* out, long long* cyc, int iters, float sl2, float m) {
  float x[8], acc = 0.f;
  uint32_t pk = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = (threadIdx.x + i) * 1e-3f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float e[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) e[i] = ex2(MIX ? fmaf(x[i], sl2, -m) : x[i]);
    if (MIX) {
      acc += ((e[0] + e[1]) + (e[2] + e[3])) + ((e[4] + e[5]) + (e[6] + e[7]));
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 b = __floats2bfloat162_rn(e[2 * i], e[2 * i + 1]);
        pk ^= *reinterpret_cast<uint32_t*>(&b);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = __uint_as_float(__float_as_uint(x[i]) ^ (pk & 1));
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = e[i];
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float s = acc + __uint_as_float(pk);
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MIX>
void run(int warps) {
  const int blocks = 148, iters = 4096;
  float* out;
  long long* cyc;
  cudaMalloc(&out, blocks * 1024 * 4);
  cudaMalloc(&cyc, blocks * 8);
  k<MIX><<<blocks, warps * 32>>>(out, cyc, 16, 1.4427f, 0.5f);
  k<MIX><<<blocks, warps * 32>>>(out, cyc, iters, 1.4427f, 0.5f);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < blocks; ++i) mean += h[i];
  mean /= blocks;
  printf("%-26s warps %2d: %6.2f ex2/clk/SM  (%s)\n", MIX ? "ex2 + ffma/fadd/f2fp mix" : "ex2 chains x8", warps,
         8.0 * iters * warps * 32 / mean, cudaGetErrorString(e));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {1, 2, 4, 8, 16}) run<0>(w);
  for (int w : {4, 8, 16}) run<1>(w);
  return 0;
}
