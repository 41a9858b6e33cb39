// Throughput of MUFU exp2 variants on one B200 SM-set (diagnostics):
//   ex2.approx.ftz.f32  vs  ex2.approx.ftz.bf16x2  vs  ex2.approx.f16x2
// results per clock per SM (each packed op yields two results).
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

template <int V>
__global__ void k(float* out, int iters, long long* clk) {
  float a[8];
  uint32_t b[8];
  for (int i = 0; i < 8; ++i) { a[i] = -0.001f * (threadIdx.x + i); b[i] = 0xbc00bc00u + i; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (V == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (V == 1) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(b[i]));
      if (V == 2) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(b[i]));
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(b[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

int main() {
  float* out; long long* clk; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&clk, 8);
  const int iters = 4096;
  const char* names[3] = {"ex2.f32", "ex2.bf16x2", "ex2.f16x2"};
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      if (v == 0) k<0><<<148, 1024>>>(out, iters, clk);
      if (v == 1) k<1><<<148, 1024>>>(out, iters, clk);
      if (v == 2) k<2><<<148, 1024>>>(out, iters, clk);
      cudaDeviceSynchronize();
    }
    long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    const double ops = 1024.0 * iters * 8;  // instructions (per SM: one CTA of 1024 threads)
    const double res = ops * (v == 0 ? 1 : 2);
    printf("%-12s %6.2f instr/clk/SM  %6.2f results/clk/SM\n", names[v], ops / c, res / c);
  }
  return 0;
}
