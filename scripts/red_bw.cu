// Throughput of fp32 reductions into global memory on B200 (diagnostics):
//   st    : plain st.global.v4 (write bandwidth reference)
//   red4  : red.global.add.v4.f32, fully coalesced (each warp instruction = 512 contiguous B)
//   red1  : red.global.add.f32 scalar, coalesced
//   bulk  : cp.reduce.async.bulk.global.shared::cta.add.f32 of CH-byte chunks staged in smem
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_bw red_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_st(float4* p, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_float4(1.f, 1.f, 1.f, 1.f);
}
__global__ void k_red4(float* p, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p + 4 * i), "f"(1.f), "f"(1.f), "f"(1.f), "f"(1.f) : "memory");
}
__global__ void k_red1(float* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p + i), "f"(1.f) : "memory");
}
template <int CH>
__global__ void k_bulk(float* p, size_t nbytes) {
  __shared__ __align__(128) float buf[8][CH / 4];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int i = l; i < CH / 4; i += 32) buf[w][i] = 1.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const size_t nch = nbytes / CH;
  for (size_t c = (blockIdx.x * 8 + w) * 32 + l; c < nch; c += (size_t)gridDim.x * 8 * 32) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"((char*)p + c * CH),
                 "r"((unsigned)__cvta_generic_to_shared(buf[w])), "n"(CH) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t bytes = 100ull << 20;  // 100 MiB (cfg2 dQ fp32)
  float* p;
  cudaMalloc(&p, bytes);
  cudaMemset(p, 0, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 148;
  auto run = [&](const char* name, auto fn) {
    fn();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) fn();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-10s %8.1f us  %7.0f GB/s (bytes updated / time)\n", name, ms * 200, 5 * bytes / (ms * 1e-3) / 1e9);
  };
  run("st", [&] { k_st<<<sms * 8, 256>>>((float4*)p, bytes / 16); });
  run("red4", [&] { k_red4<<<sms * 8, 256>>>(p, bytes / 16); });
  run("red1", [&] { k_red1<<<sms * 8, 256>>>(p, bytes / 4); });
  run("bulk256", [&] { k_bulk<256><<<sms * 4, 256>>>(p, bytes); });
  run("bulk1024", [&] { k_bulk<1024><<<sms * 4, 256>>>(p, bytes); });
  run("bulk4096", [&] { k_bulk<4096><<<sms * 4, 256>>>(p, bytes); });
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
