// gather_bw.cu — TMA load throughput: tiled 128-row boxes vs tile::gather4 (sequential
// and random rows), 148 CTAs x STAGES tiles in flight.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gb scripts/gather_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

constexpr int STAGES = 8;
constexpr int TILE = 128 * 128;  // 128 rows x 128 B

__global__ void __launch_bounds__(32) load_kernel(const __grid_constant__ CUtensorMap tiled,
                                                  const __grid_constant__ CUtensorMap g4, const int* rows, int nrows,
                                                  int tiles_per_cta, int mode, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[STAGES];
  const int lane = threadIdx.x;
  if (lane == 0) {
    for (int i = 0; i < STAGES; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  const long long t0 = clock64();
  for (int t = 0; t < tiles_per_cta; ++t) {
    const int st = t % STAGES;
    if (t >= STAGES) {
      const uint32_t par = ((t / STAGES) - 1) & 1;
      asm volatile(
          "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W;\n\t}" ::"r"(
              smem_u32(&bar[st])),
          "r"(par)
          : "memory");
    }
    uint8_t* dst = buf + st * TILE;
    const int tile_id = blockIdx.x * tiles_per_cta + t;
    const int row0 = (tile_id * 128) % (nrows - 128);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[st])), "r"(TILE));
    __syncwarp();
    if (mode == 0) {
      if (lane == 0)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                smem_u32(dst)),
            "l"(reinterpret_cast<uint64_t>(&tiled)), "r"(0), "r"(row0), "r"(smem_u32(&bar[st]))
            : "memory");
    } else {
      int4 r4;
      if (mode == 1) r4 = make_int4(row0 + 4 * lane, row0 + 4 * lane + 1, row0 + 4 * lane + 2, row0 + 4 * lane + 3);
      else r4 = __ldg(reinterpret_cast<const int4*>(rows + (static_cast<size_t>(tile_id) * 128) % (nrows - 128)) + lane);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst + lane * 512)),
          "l"(reinterpret_cast<uint64_t>(&g4)), "r"(0), "r"(r4.x), "r"(r4.y), "r"(r4.z), "r"(r4.w),
          "r"(smem_u32(&bar[st]))
          : "memory");
    }
  }
  for (int t = tiles_per_cta - STAGES; t < tiles_per_cta; ++t) {
    if (t < 0) continue;
    const int st = t % STAGES;
    const uint32_t par = (t / STAGES) & 1;
    asm volatile(
        "{\n\t.reg .pred P1;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W2;\n\t}" ::"r"(
            smem_u32(&bar[st])),
        "r"(par)
        : "memory");
  }
  const long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x] = t1 - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const long long R = 4LL * 8192 * 12;  // rows of a cfg2 (B, T, H, D=64) bf16 tensor: 48 MiB
  uint16_t* d;
  cudaMalloc(&d, R * 128);
  cudaMemset(d, 0, R * 128);
  int* h = (int*)malloc(R * 4);
  srand(1);
  for (long long i = 0; i < R; ++i) h[i] = (int)(((long long)rand() * 2654435761LL) % R);
  int* rows;
  cudaMalloc(&rows, R * 4);
  cudaMemcpy(rows, h, R * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  CUtensorMap tiled, g4;
  cuuint64_t dims[2] = {64, (cuuint64_t)R};
  cuuint64_t strides[1] = {128};
  cuuint32_t box_t[2] = {64, 128}, box_g[2] = {64, 1}, es[2] = {1, 1};
  enc(&tiled, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box_t, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&g4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box_g, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 1024 * 8);
  const size_t smem = STAGES * TILE + 1024;
  cudaFuncSetAttribute(load_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const char* names[3] = {"tiled 128-row box", "gather4 sequential rows", "gather4 random rows"};
  for (int grid : {148, 296}) {
    const int tiles = (int)(R / 128 / grid);  // one pass over the 48 MiB tensor
    for (int mode = 0; mode < 3; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        load_kernel<<<grid, 32, smem>>>(tiled, g4, rows, (int)R, tiles, mode, cyc);
        cudaEventRecord(b);
        cudaError_t e = cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (rep == 1)
          printf("grid %d %-26s: %.1f us, %.0f GB/s (%s)\n", grid, names[mode], ms * 1e3,
                 (double)grid * tiles * TILE / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
      }
    }
  }
  return 0;
}
