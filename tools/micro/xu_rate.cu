// Throughput of the softmax instruction classes on one SM (sm_100a): ex2.approx, cvt.rn.bf16x2.f32
// (F2FP pack), 3-input max, FFMA; warps x independent chains, clock64 per CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xu_rate xu_rate.cu && ./xu_rate
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, long long* cyc, int iters) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 0.001f * (threadIdx.x + i);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1) {
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        acc += r;
      }
      if (OP == 2) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 3) & 7]), "f"(a[(i + 5) & 7]));
      if (OP == 3) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 3) & 7]), "f"(a[(i + 5) & 7]));
      if (OP == 4) {  // ex2 on packed f16x2 (two elements per lane per instruction)
        uint32_t x = __float_as_uint(a[i]);
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(x));
        a[i] = __uint_as_float(x);
      }
      if (OP == 5) {  // ex2 on packed bf16x2
        uint32_t x = __float_as_uint(a[i]);
        asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(x));
        a[i] = __uint_as_float(x);
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1024);
  const char* names[6] = {"ex2.approx.f32", "cvt.rn.bf16x2.f32", "max.f32 (3-input)", "fma.rn.f32",
                          "ex2.approx.f16x2 (x2)", "ex2.approx.ftz.bf16x2 (x2)"};
  for (int op = 0; op < 6; ++op) {
    for (int warps : {4, 8, 16, 32}) {
      const int iters = 256;
      for (int rep = 0; rep < 2; ++rep) {
        if (op == 0) k<0><<<1, 32 * warps>>>(out, cyc, iters);
        if (op == 1) k<1><<<1, 32 * warps>>>(out, cyc, iters);
        if (op == 2) k<2><<<1, 32 * warps>>>(out, cyc, iters);
        if (op == 3) k<3><<<1, 32 * warps>>>(out, cyc, iters);
        if (op == 4) k<4><<<1, 32 * warps>>>(out, cyc, iters);
        if (op == 5) k<5><<<1, 32 * warps>>>(out, cyc, iters);
      }
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double ops = (double)iters * 8 * 32 * warps * (op >= 4 ? 2 : 1);  // elements
      printf("%-20s warps %2d : %.2f thread-ops / clk / SM\n", names[op], warps, ops / c);
    }
  }
  return 0;
}
