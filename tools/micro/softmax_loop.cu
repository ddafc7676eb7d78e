// Clocks per 128-element softmax row block for the attention forward's exponential loop
// (exp_pack_regs shape: FFMA + ex2 + row-sum tree + bf16 pack), one row per thread, run with
// 1 or 2 warps per SMSP and no TMEM / barrier traffic: is the loop MUFU-bound by itself?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o softmax_loop softmax_loop.cu && ./softmax_loop
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}

template <int NCOL>
__global__ void k(const float* in, uint32_t* out, float* rs_out, long long* cyc, int iters, float sl2) {
  uint32_t v[NCOL];
#pragma unroll
  for (int i = 0; i < NCOL; ++i) v[i] = __float_as_uint(in[(threadIdx.x * 7 + i) & 1023]);
  float m = 1.5f, acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float rs4[4] = {0.f, 0.f, 0.f, 0.f};
    uint32_t pk[NCOL / 2];
#pragma unroll
    for (int k8 = 0; k8 < NCOL / 8; ++k8) {
      float e[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) e[i] = ex2(fmaf(__uint_as_float(v[k8 * 8 + i]), sl2, -m));
      rs4[k8 & 3] += ((e[0] + e[1]) + (e[2] + e[3])) + ((e[4] + e[5]) + (e[6] + e[7]));
#pragma unroll
      for (int i = 0; i < 4; ++i) pk[k8 * 4 + i] = pack_bf16x2(e[2 * i], e[2 * i + 1]);
    }
    acc += (rs4[0] + rs4[1]) + (rs4[2] + rs4[3]);
    // feed the packed values back so nothing is dead code (one XOR per pair)
#pragma unroll
    for (int i = 0; i < NCOL / 2; ++i) v[2 * i] ^= (pk[i] & 1u);
    m += 1e-7f;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  rs_out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  out[blockIdx.x * blockDim.x + threadIdx.x] = v[0];
}

int main() {
  float* in;
  uint32_t* out;
  float* rs;
  long long* cyc;
  cudaMalloc(&in, 4096 * 4);
  cudaMemset(in, 0, 4096 * 4);
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&rs, 1 << 20);
  cudaMalloc(&cyc, 1024);
  for (int warps : {4, 8, 16}) {
    const int iters = 64;
    for (int rep = 0; rep < 2; ++rep) k<128><<<1, 32 * warps>>>(in, out, rs, cyc, iters, 0.18f);
    cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("warps %2d (per SMSP %d): %.0f clk per 128-col block per warp; MUFU-bound ideal %d\n", warps, warps / 4,
           (double)c / iters, 1024 * (warps / 4));
  }
  return 0;
}
