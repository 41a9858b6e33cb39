// mma_issue.cu — tcgen05.mma issue cost from one thread (warp-uniform loop, elected issue).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2306_01160_b200/csrc -o mi scripts/mma_issue.cu
//
// Per CTA (one per SM): operands in shared memory (contents irrelevant), D in TMEM.
// Measures clocks to issue N MMAs (M=128, K=16, N in {64, 128}) and then to their completion
// (tcgen05.commit -> mbarrier), for dependent (same D, accumulate) and independent chains.
#include <stdio.h>

#include "scfa_common.cuh"

using namespace scfa;

template <int N, bool DEP, bool TS = false>
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1) {
    constexpr uint32_t idesc = make_idesc_bf16(128, N, false, TS);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 16384);
    long long t0 = clock64(), t1 = 0, t2 = 0;
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const uint32_t d = DEP ? tmem : tmem + (k % 4) * N;
          if (TS)  // A from TMEM columns [384, 448): 16 bf16 per K step = 8 columns
            umma_ts(DEP ? tmem : tmem + (k % 2) * N, tmem + 384 + (k & 7) * 8,
                    make_sdesc_sw128(b + (k & 3) * 2048, N * 128, 1024), idesc, k > 0 || it > 0);
          else
            umma_ss(d, make_sdesc_sw128(a + (k & 3) * 32, 16, 1024), make_sdesc_sw128(b + (k & 3) * 32, 16, 1024),
                    idesc, k > 0 || it > 0);
        }
      }
      __syncwarp();
    }
    t1 = clock64();
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    t2 = clock64();
    if ((threadIdx.x & 31) == 0) {
      out[blockIdx.x * 2] = t1 - t0;
      out[blockIdx.x * 2 + 1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int N, bool DEP, bool TS = false>
static void run(unsigned long long* d) {
  const int iters = 64;
  cudaFuncSetAttribute(mma_kernel<N, DEP, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  mma_kernel<N, DEP, TS><<<148, 128, 64 * 1024>>>(iters, d);
  cudaDeviceSynchronize();
  mma_kernel<N, DEP, TS><<<148, 128, 64 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double n = iters * 16.0;
  printf("%s N=%3d %s: issue %.1f clk/mma, complete %.1f clk/mma (ideal pipe %d)  %s\n", TS ? "TS" : "SS", N, DEP ? "dependent  " : "independent",
         h[0] / n, h[1] / n, 128 * N / 256, cudaGetErrorString(e));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 16);
  run<64, true>(d);
  run<64, false>(d);
  run<128, true>(d);
  run<128, false>(d);
  run<64, true, true>(d);
  run<64, false, true>(d);
  run<128, false, true>(d);
  return 0;
}
