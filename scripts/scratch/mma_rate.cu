// mma_contention.cu — does row-thread TMEM traffic (tcgen05.ld / st) slow tcgen05.mma?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2306_01160_b200/csrc -o mc scripts/mma_contention.cu
//
// One CTA per SM, 384 threads: warp 1 issues TS-mode MMAs (M=128, N=64, K=16; A from TMEM,
// B MN-major or K-major from smem, accumulating into TMEM like dV / dK or S / dP); when
// `load` is set, warps 4..11 (two "row" warpgroups) meanwhile stream TMEM loads of 32
// columns (and stores of 16) as the dK/dV row threads do.  Reports clk per MMA.
#include <stdio.h>

#include "scfa_common.cuh"

using namespace scfa;

template <bool BMN, int N>
__global__ void __launch_bounds__(384, 1) k(int iters, int load, unsigned long long* out, int* stop) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    done = 0;
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1) {
    constexpr uint32_t idesc = make_idesc_bf16(128, N, false, BMN);
    const uint32_t b = smem_u32(smem);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)
          umma_ts(tmem + 256 + (kk & 1) * 64, tmem + 384 + (kk & 7) * 8,
                  BMN ? make_sdesc_sw128(b + (kk & 3) * 2048, 64 * 128, 1024) : make_sdesc_sw128(b + (kk & 3) * 32, 16, 1024),
                  idesc, kk > 1 || it > 0);
      }
      __syncwarp();
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[blockIdx.x] = t1 - t0;
    done = 1;
  } else if (warp >= 4 && load) {
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    uint32_t acc = 0;
    while (!done) {
      uint32_t v[32];
      tmem_ld32(tmem + lane_off + ((warp >> 2) - 1) * 64, v);
      tmem_wait_ld();
      uint32_t w[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) { acc += v[2 * i] ^ v[2 * i + 1]; w[i] = v[i] + acc; }
      tmem_st16(tmem + lane_off + 128 + ((warp >> 2) - 1) * 32, w);
      tmem_wait_st();
    }
    if (acc == 12345) stop[0] = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <bool BMN, int N>
static void run(unsigned long long* d, int* s, int load) {
  const int iters = 256;
  cudaFuncSetAttribute(k<BMN, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k<BMN, N><<<148, 384, 64 * 1024>>>(iters, load, d, s);
  cudaDeviceSynchronize();
  k<BMN, N><<<148, 384, 64 * 1024>>>(iters, load, d, s);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("TS N=%d B %s, row TMEM traffic %s: %.1f clk/mma  %s\n", N, BMN ? "MN-major" : "K-major ", load ? "on " : "off",
         h / (iters * 16.0), cudaGetErrorString(e));
}

int main() {
  unsigned long long* d;
  int* s;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&s, 4);
  run<false, 16>(d, s, 0);
  run<false, 32>(d, s, 0);
  run<false, 64>(d, s, 0);
  run<false, 128>(d, s, 0);
  run<false, 256>(d, s, 0);
  return 0;
}
