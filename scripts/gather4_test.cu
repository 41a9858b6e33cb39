// gather4_test.cu — does TMA tile::gather4 with SWIZZLE_128B reproduce the tiled
// SWIZZLE_128B shared-memory layout when 4-row groups land at 512-byte offsets?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o g4 scripts/gather4_test.cu -lcuda
//
// A (R x 64) bf16 matrix holds value (row * 64 + col) & 0xffff.  Kernel 1 loads a
// 128-row tiled box (rows 0..127); kernel 2 gathers rows perm[0..127] = 0..127 with
// 32 gather4 calls.  Identical smem images => address-based swizzle (usable).
// Kernel 3 gathers a real permutation and is checked against the tiled image of the
// permuted matrix.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void load_kernel(const __grid_constant__ CUtensorMap tiled, const __grid_constant__ CUtensorMap g4,
                            const int* perm, int mode, uint16_t* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* buf = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(128 * 128));
    if (mode == 0) {
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              smem_u32(buf)),
          "l"(reinterpret_cast<uint64_t>(&tiled)), "r"(0), "r"(0), "r"(smem_u32(&bar))
          : "memory");
    } else {
      for (int g = 0; g < 32; ++g) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(buf + g * 512)),
            "l"(reinterpret_cast<uint64_t>(&g4)), "r"(0), "r"(perm[4 * g]), "r"(perm[4 * g + 1]), "r"(perm[4 * g + 2]),
            "r"(perm[4 * g + 3]), "r"(smem_u32(&bar))
            : "memory");
      }
    }
  }
  asm volatile(
      "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
          smem_u32(&bar))
      : "memory");
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(buf)[i];
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int R = 1024;
  uint16_t* h = (uint16_t*)malloc(R * 64 * 2);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < 64; ++c) h[r * 64 + c] = (uint16_t)((r * 64 + c) & 0xffff);
  uint16_t* d;
  cudaMalloc(&d, R * 64 * 2);
  cudaMemcpy(d, h, R * 64 * 2, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  CUtensorMap tiled, g4;
  cuuint64_t dims[2] = {64, (cuuint64_t)R};
  cuuint64_t strides[1] = {128};
  cuuint32_t box_t[2] = {64, 128}, box_g[2] = {64, 1}, es[2] = {1, 1};
  CUresult r1 = enc(&tiled, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box_t, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&g4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box_g, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode tiled %d gather4(box 64x1) %d\n", (int)r1, (int)r2);
  int hp[128];
  int* dp;
  cudaMalloc(&dp, 128 * 4);
  uint16_t *o1, *o2;
  cudaMalloc(&o1, 128 * 64 * 2);
  cudaMalloc(&o2, 128 * 64 * 2);
  uint16_t a[128 * 64], b[128 * 64];
  cudaFuncSetAttribute(load_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
  // identity
  for (int i = 0; i < 128; ++i) hp[i] = i;
  cudaMemcpy(dp, hp, 512, cudaMemcpyHostToDevice);
  load_kernel<<<1, 128, 20000>>>(tiled, g4, dp, 0, o1);
  load_kernel<<<1, 128, 20000>>>(tiled, g4, dp, 1, o2);
  cudaError_t e = cudaDeviceSynchronize();
  printf("identity run: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  cudaMemcpy(a, o1, sizeof(a), cudaMemcpyDeviceToHost);
  cudaMemcpy(b, o2, sizeof(b), cudaMemcpyDeviceToHost);
  printf("identity gather4 == tiled: %s\n", memcmp(a, b, sizeof(a)) == 0 ? "YES" : "NO");
  int diffs = 0;
  for (int i = 0; i < 128 * 64 && diffs < 8; ++i)
    if (a[i] != b[i]) { printf("  diff at %d (row %d chunk %d): tiled %d gather %d\n", i, i / 64, (i % 64) / 8, a[i], b[i]); ++diffs; }
  // permutation: gathered rows perm[i] should equal tiled load of a matrix whose row i is row perm[i]
  for (int i = 0; i < 128; ++i) hp[i] = (i * 37 + 11) % R;
  cudaMemcpy(dp, hp, 512, cudaMemcpyHostToDevice);
  load_kernel<<<1, 128, 20000>>>(tiled, g4, dp, 1, o2);
  e = cudaDeviceSynchronize();
  cudaMemcpy(b, o2, sizeof(b), cudaMemcpyDeviceToHost);
  // expected: tiled image a (rows 0..127 of the identity) with row i's values replaced by row perm[i]'s
  int bad = 0;
  for (int r = 0; r < 128; ++r)
    for (int k = 0; k < 64; ++k) {
      // tiled image position of (r, col c): chunk (c/8) stored at chunk ((c/8) ^ (r & 7))
      int c = k;
      int pos = r * 64 + (((c / 8) ^ (r & 7)) * 8) + (c % 8);
      uint16_t want = (uint16_t)((hp[r] * 64 + c) & 0xffff);
      if (b[pos] != want) ++bad;
    }
  printf("permuted gather4 matches address-swizzled layout: %s (%d bad)\n", bad == 0 ? "YES" : "NO", bad);
  // also check the tiled image itself follows the assumed formula
  bad = 0;
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < 64; ++c) {
      int pos = r * 64 + (((c / 8) ^ (r & 7)) * 8) + (c % 8);
      if (a[pos] != (uint16_t)((r * 64 + c) & 0xffff)) ++bad;
    }
  printf("tiled image follows chunk ^ (row & 7): %s\n", bad == 0 ? "YES" : "NO");
  return 0;
}
