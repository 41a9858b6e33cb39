// softmax_loop.cu — the forward row loop in isolation (no MMA, no barriers): how close
// does the per-chunk instruction sequence get to the MUFU bound (16 ex2/clk/SM,
// 1024 clk per 128x128 tile per SM) with two row warpgroups per SM (one per stream)?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2306_01160_b200/csrc -o sl scripts/softmax_loop.cu
//
// Variants (per thread = one TMEM lane; S in TMEM columns [0,128) of the warpgroup's half,
// P written as bf16 to [192,256)):
//   0 full    : ld32 -> wait -> max chain -> vote -> 32 x (ffma2, 2 ex2, add2, f2fp) -> st16
//   1 pipe    : as 0, the next chunk's ld issued before this chunk's exponentials
//   2 nomax   : as 0 without the max chain / vote (exponent base fixed)
//   3 mufu    : exponentials only on register data (no TMEM traffic)
//   4 full+mma: as 0 while a ninth warp issues back-to-back M=128 N=64 K=16 MMAs into the
//               unused TMEM columns [128,192) of both halves (TMEM / tensor-pipe contention)
//   5 full+ts : as 4 with TS-mode MMAs (A = the P columns in TMEM, as the PV MMA)
#include <stdio.h>

#include "scfa_common.cuh"

using namespace scfa;

template <int V>
__device__ __forceinline__ void tile(uint32_t t_s, uint32_t t_p, float sl, float& m_run, float& l_run,
                                     float (&xr)[32]) {
  float la[4] = {0.f, 0.f, 0.f, 0.f};
  float xn[32];
  if (V == 1) {
    tmem_ld32(t_s, *reinterpret_cast<uint32_t(*)[32]>(xn));
    tmem_wait_ld();
  }
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
    float x[32];
    if (V == 3) {
#pragma unroll
      for (int c = 0; c < 32; ++c) x[c] = xr[c] + ch;
    } else if (V == 1) {
#pragma unroll
      for (int c = 0; c < 32; ++c) x[c] = xn[c];
      if (ch + 1 < 4) tmem_ld32(t_s + 32 * (ch + 1), *reinterpret_cast<uint32_t(*)[32]>(xn));
    } else {
      tmem_ld32(t_s + 32 * ch, *reinterpret_cast<uint32_t(*)[32]>(x));
      tmem_wait_ld();
    }
    if (V == 0 || V == 1) {
      float e0 = -INFINITY, e1 = -INFINITY;
#pragma unroll
      for (int c = 0; c < 32; c += 4) {
        e0 = max3(e0, x[c], x[c + 1]);
        e1 = max3(e1, x[c + 2], x[c + 3]);
      }
      const float ms = fmaxf(e0, e1) * sl;
      const bool raise = ms > m_run + 64.f;
      if (__any_sync(0xffffffffu, raise)) {
        const float alpha = (raise && m_run != -INFINITY) ? ex2(m_run - ms) : (raise ? 0.f : 1.f);
        if (raise) m_run = ms;
        l_run *= alpha;
#pragma unroll
        for (int i = 0; i < 4; ++i) la[i] *= alpha;
      }
    }
    const float nm = -m_run;
    uint32_t pk[16];
#pragma unroll
    for (int c = 0; c < 32; c += 2) {
      float a0, a1;
      fma2(a0, a1, x[c], x[c + 1], sl, sl, nm, nm);
      a0 = ex2(a0);
      a1 = ex2(a1);
      const int q = (c >> 1) & 1;
      add2(la[2 * q], la[2 * q + 1], la[2 * q], la[2 * q + 1], a0, a1);
      pk[c >> 1] = pack_bf16(a0, a1);
    }
    if (V == 3) {
#pragma unroll
      for (int i = 0; i < 16; ++i) xr[i] += __uint_as_float(pk[i]) * 1e-30f;
    } else {
      tmem_st16(t_p + 16 * ch, pk);
    }
    if (V == 1 && ch + 1 < 4) tmem_wait_ld();
  }
  l_run += (la[0] + la[1]) + (la[2] + la[3]);
  if (V != 3) tmem_wait_st();
}

template <int V>
__global__ void __launch_bounds__(288, 1) loop_kernel(int tiles, unsigned long long* out, float* sink) {
  __shared__ uint32_t slot;
  __shared__ int done;
  extern __shared__ __align__(1024) uint8_t dsm[];
  const int warp = threadIdx.x >> 5, wg = warp >> 2;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) done = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 8) {
    __syncthreads();
    if (V == 4 || V == 5) {
      constexpr uint32_t idesc = make_idesc_bf16(128, 64, false, false);
      constexpr uint32_t idesc_ts = make_idesc_bf16(128, 64, false, true);
      const uint32_t a = smem_u32(dsm), b = smem_u32(dsm + 16384);
      for (int it = 0; *reinterpret_cast<volatile int*>(&done) < 256 && it < 1000000; ++it) {
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (V == 4)
              umma_ss(slot + 128 + (k & 1) * 256, make_sdesc_sw128(a + (k & 3) * 32, 16, 1024),
                      make_sdesc_sw128(b + (k & 3) * 32, 16, 1024), idesc, 1);
            else
              umma_ts(slot + 128 + (k & 1) * 256, slot + 192 + (k & 1) * 256 + (k >> 1) * 8,
                      make_sdesc_sw128(b + (k & 3) * 2048, 128 * 128, 1024), idesc_ts, 1);
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();
    tc_fence_before();
    __syncthreads();
    return;
  }
  const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
  const uint32_t t_s = slot + lane_base + wg * 256, t_p = t_s + 192;
  // fill S with something finite
  {
    uint32_t v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(0.01f * ((threadIdx.x + i) & 63));
#pragma unroll
    for (int c = 0; c < 128; c += 32) tmem_st32(t_s + c, v);
    tmem_wait_st();
  }
  float xr[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) xr[i] = 0.01f * i;
  float m_run = -INFINITY, l_run = 0.f;
  const float sl = 0.18f;
  __syncthreads();
  const long long t0 = clock64();
  for (int t = 0; t < tiles; ++t) tile<(V >= 4) ? 0 : V>(t_s, t_p, sl, m_run, l_run, xr);
  const long long t1 = clock64();
  atomicAdd(&done, 1);
  __syncthreads();
  sink[blockIdx.x * 256 + threadIdx.x] = l_run + m_run + xr[3];
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(slot);
}

template <int V>
static void run(const char* name, unsigned long long* d, float* sink) {
  const int tiles = 512;
  cudaFuncSetAttribute(loop_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int rep = 0; rep < 2; ++rep) {
    loop_kernel<V><<<148, 288, 65536>>>(tiles, d, sink);
    cudaDeviceSynchronize();
  }
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  s /= 148;
  // two warpgroups each ran `tiles` tiles of 128x128: per-SM clk per tile = s / (2*tiles)
  printf("%-6s: %.0f clk per tile-pair per warp (%.0f clk per tile per SM; MUFU bound 1024) %s\n", name, s / tiles,
         s / (2.0 * tiles), cudaGetErrorString(e));
}

int main() {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 148 * 256 * 4);
  run<0>("full", d, sink);
  run<1>("pipe", d, sink);
  run<2>("nomax", d, sink);
  run<3>("mufu", d, sink);
  run<4>("full+mma", d, sink);
  run<5>("full+ts", d, sink);
  return 0;
}
