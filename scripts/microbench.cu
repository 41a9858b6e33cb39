// microbench.cu — measured per-SM rates that bound the SCFA softmax loop on B200.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/microbench scripts/microbench.cu
//
// tmem_ld : tcgen05.ld 32x32b.xN throughput (bytes/clk/SM) with W warps
// ex2     : ex2.approx.ftz.f32 lanes/clk/SM
// f2fp    : cvt.rn.bf16x2.f32 lanes/clk/SM (pairs)
// ffma2   : fma.rn.f32x2 lanes/clk/SM (element pairs)
// fsel    : predicated select lanes/clk/SM
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int NCOL>
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t* r);

template <>
__device__ __forceinline__ void ld<32>(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

template <>
__device__ __forceinline__ void ld<16>(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

template <int NCOL, int PER_WAIT>
__global__ void tmem_ld_kernel(int iters, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
  const uint32_t col_base = (warp >> 2) * 128;  // warps 4-7 read other columns
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[PER_WAIT][NCOL];
#pragma unroll
    for (int j = 0; j < PER_WAIT; ++j) ld<NCOL>(tmem + lane_off + col_base + ((i * PER_WAIT + j) * NCOL) % 128, r[j]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < PER_WAIT; ++j)
#pragma unroll
      for (int c = 0; c < NCOL; ++c) acc ^= r[j][c];
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int OP>
__global__ void alu_kernel(int iters, unsigned long long* cyc, float* sink, float seed) {
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = seed * (threadIdx.x + i);
  uint32_t u[8] = {0};
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (OP == 0) {
        v[i] = ex2(v[i]);
        v[i + 1] = ex2(v[i + 1]);
      } else if (OP == 1) {
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v[i]), "f"(v[i + 1]));
        u[i >> 1] += r;
        v[i] += 1.0f;
      } else if (OP == 2) {
        asm volatile(
            "{\n\t.reg .b64 ra, rb;\n\tmov.b64 ra, {%0, %1};\n\tmov.b64 rb, {%2, %3};\n\t"
            "fma.rn.f32x2 ra, ra, rb, rb;\n\tmov.b64 {%0, %1}, ra;\n\t}"
            : "+f"(v[i]), "+f"(v[i + 1])
            : "f"(seed), "f"(seed));
      } else {
        const bool p = (__float_as_uint(v[i]) >> (it & 31)) & 1;
        v[i] = p ? v[i + 1] : -v[i];
        v[i + 1] = p ? v[i] : v[i + 1] * 0.5f;
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += __uint_as_float(u[i]);
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static double median_cycles(unsigned long long* d, int n) {
  unsigned long long h[1024];
  cudaMemcpy(h, d, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  // insertion sort
  for (int i = 1; i < n; ++i)
    for (int j = i; j > 0 && h[j] < h[j - 1]; --j) {
      unsigned long long t = h[j];
      h[j] = h[j - 1];
      h[j - 1] = t;
    }
  return static_cast<double>(h[n / 2]);
}

template <int NCOL, int PW>
static int run_tmem(int warps, unsigned long long* cyc, uint32_t* sink) {
  const int iters = 4096;
  tmem_ld_kernel<NCOL, PW><<<148, warps * 32>>>(iters, cyc, sink);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  tmem_ld_kernel<NCOL, PW><<<148, warps * 32>>>(iters, cyc, sink);
  CK(cudaDeviceSynchronize());
  const double c = median_cycles(cyc, 148);
  const double bytes = static_cast<double>(iters) * PW * warps * 32 * NCOL * 4;
  printf("tmem_ld x%-3d per_wait %d warps %d : %7.1f B/clk/SM  (%.1f clk per 32-lane x32 load per warp)\n", NCOL, PW,
         warps, bytes / c, c / (iters * PW * (NCOL / 32.0)));
  return 0;
}

template <int OP>
static int run_alu(const char* name, int warps, unsigned long long* cyc, float* sink) {
  const int iters = 4096;
  alu_kernel<OP><<<148, warps * 32>>>(iters, cyc, sink, 1e-3f);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  alu_kernel<OP><<<148, warps * 32>>>(iters, cyc, sink, 1e-3f);
  CK(cudaDeviceSynchronize());
  const double c = median_cycles(cyc, 148);
  const double ops = static_cast<double>(iters) * 16 * warps * 32;  // elements
  printf("%-6s warps %2d : %7.2f elements/clk/SM\n", name, warps, ops / c);
  return 0;
}

int main() {
  unsigned long long* cyc;
  uint32_t* sink;
  float* fsink;
  CK(cudaMalloc(&cyc, 148 * sizeof(unsigned long long)));
  CK(cudaMalloc(&sink, 148 * 1024 * 4));
  CK(cudaMalloc(&fsink, 148 * 1024 * 4));
  for (int w : {4, 8}) {
    run_tmem<32, 1>(w, cyc, sink);
    run_tmem<32, 2>(w, cyc, sink);
    run_tmem<32, 4>(w, cyc, sink);
    run_tmem<16, 4>(w, cyc, sink);
  }
  for (int w : {4, 8, 16}) {
    run_alu<0>("ex2", w, cyc, fsink);
    run_alu<1>("f2fp", w, cyc, fsink);
    run_alu<2>("ffma2", w, cyc, fsink);
    run_alu<3>("fsel", w, cyc, fsink);
  }
  return 0;
}
