// scfa_lsh.cu — angular LSH bucket ids on the device (the bucket producer feeding the
// hash path).
//
// Reference: lsh_buckets (pkg/src/scfa/hash_sparse.py:34-52): per (b, h) a D x nb/2
// standard-normal projection R (drawn on the host from the reference's Philox stream,
// tensors.py:86-93, so the ids agree with the reference), rot = x[b, :, h, :] @ R, and
// the id is the argmax of the 2*(nb/2)-vector [rot, -rot] (first maximum, np.argmax).
//
// HBM-bound: each (b, t, h) row of x is read once (D elements), the projection of the
// (b, h) slice (D * nb/2 doubles, <= 192 x 32 x 8 B = 48 KB) sits in shared memory, and
// one id (8 B) is written.  Arithmetic in float64 like the reference (x is upcast, as
// numpy does for `float32 @ float64`); the dot products run in d order with FMA.
#include "scfa_common.cuh"
#include "scfa_internal.h"

namespace scfa {

namespace {

constexpr int kLshThreads = 256;
constexpr int kLshMaxD = 192;  // 192 x 32 doubles = 48 KB of static shared memory
constexpr int kLshMaxHalf = 32;  // nb <= 64

SCFA_DEVICE double load_x(const void* p, int dt, int64_t i) {
  switch (dt) {
    case SCFA_DT_F32: return static_cast<double>(static_cast<const float*>(p)[i]);
    case SCFA_DT_F64: return static_cast<const double*>(p)[i];
    default: return static_cast<double>(__bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]));
  }
}

// One CTA per ((b, h) slice, chunk of kLshThreads positions); one thread per position.
// HALF: nb/2 rounded up to a power of two (projection columns >= half are zero and
// never win the argmax).
template <int HALF>
__global__ void __launch_bounds__(kLshThreads) lsh_kernel(const void* __restrict__ x, int dt, int64_t T, int64_t H,
                                                          int64_t D, int64_t sb, int64_t st, int64_t sh, int64_t sd,
                                                          const double* __restrict__ R, int half,
                                                          int64_t* __restrict__ out, int64_t ob, int64_t ot,
                                                          int64_t oh) {
  __shared__ double Rs[kLshMaxD * HALF];
  const int64_t bh = blockIdx.y;
  const int64_t b = bh / H, h = bh - b * H;
  const double* Rg = R + bh * D * half;
  for (int64_t i = threadIdx.x; i < D * HALF; i += blockDim.x) {
    const int64_t d = i / HALF, j = i - d * HALF;
    Rs[i] = j < half ? Rg[d * half + j] : 0.0;
  }
  __syncthreads();
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kLshThreads + threadIdx.x;
  if (t >= T) return;
  const int64_t base = b * sb + t * st + h * sh;
  double rot[HALF];
#pragma unroll
  for (int j = 0; j < HALF; ++j) rot[j] = 0.0;
  for (int64_t d = 0; d < D; ++d) {
    const double xv = load_x(x, dt, base + d * sd);
    const double* rr = Rs + d * HALF;
#pragma unroll
    for (int j = 0; j < HALF; ++j) rot[j] = fma(xv, rr[j], rot[j]);
  }
  // argmax over [rot, -rot], first maximum
  int best = 0;
  double bv = rot[0];
#pragma unroll
  for (int j = 1; j < HALF; ++j)
    if (j < half && rot[j] > bv) { bv = rot[j]; best = j; }
#pragma unroll
  for (int j = 0; j < HALF; ++j)
    if (j < half && -rot[j] > bv) { bv = -rot[j]; best = half + j; }
  out[b * ob + t * ot + h * oh] = best;
}

template <int HALF>
int launch_lsh(const void* x, int dt, int64_t B, int64_t T, int64_t H, int64_t D, int64_t sb, int64_t st, int64_t sh,
               int64_t sd, const double* R, int half, int64_t* out, int64_t ob, int64_t ot, int64_t oh,
               cudaStream_t stream) {
  dim3 grid(static_cast<unsigned>((T + kLshThreads - 1) / kLshThreads), static_cast<unsigned>(B * H));
  lsh_kernel<HALF><<<grid, kLshThreads, 0, stream>>>(x, dt, T, H, D, sb, st, sh, sd, R, half, out, ob, ot, oh);
  return cudaGetLastError() == cudaSuccess ? SCFA_OK : SCFA_ERR_CUDA;
}

}  // namespace

}  // namespace scfa

using namespace scfa;

extern "C" int scfa_lsh_buckets(const void* x, int x_dtype, int64_t B, int64_t T, int64_t H, int64_t D, int64_t sb,
                                int64_t st, int64_t sh, int64_t sd, const double* R, int nb, int64_t* out,
                                int64_t ob, int64_t ot, int64_t oh, void* stream) {
  if (nb < 2 || nb % 2 != 0 || nb / 2 > kLshMaxHalf) {
    set_error("lsh_buckets: number of buckets must be even, in [2, %d], got %d", 2 * kLshMaxHalf, nb);
    return SCFA_ERR_PARAM;
  }
  if (x_dtype != SCFA_DT_F32 && x_dtype != SCFA_DT_F64 && x_dtype != SCFA_DT_BF16) {
    set_error("lsh_buckets: x must be f32, f64 or bf16");
    return SCFA_ERR_PARAM;
  }
  if (D < 1 || D > kLshMaxD || B < 0 || T < 0 || H < 0) {
    set_error("lsh_buckets: bad shape (B=%lld T=%lld H=%lld D=%lld, D <= %d)", (long long)B, (long long)T,
              (long long)H, (long long)D, kLshMaxD);
    return SCFA_ERR_SHAPE;
  }
  if (B * T * H == 0) return SCFA_OK;
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc;
  const int half = nb / 2;
#define SCFA_LSH(P) launch_lsh<P>(x, x_dtype, B, T, H, D, sb, st, sh, sd, R, half, out, ob, ot, oh, s)
  if (half <= 1) rc = SCFA_LSH(1);
  else if (half <= 2) rc = SCFA_LSH(2);
  else if (half <= 4) rc = SCFA_LSH(4);
  else if (half <= 8) rc = SCFA_LSH(8);
  else if (half <= 16) rc = SCFA_LSH(16);
  else rc = SCFA_LSH(32);
#undef SCFA_LSH
  if (rc) set_error("lsh_buckets launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  return rc;
}
