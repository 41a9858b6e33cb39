#include <cstdio>
#include <cmath>
#include "../paper_2306_01160_b200/csrc/scfa_common.cuh"
using namespace scfa;
__global__ void k(float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float x0 = -130.f + 200.f * (float)i / n, x1 = x0 + 0.37f;
  float y0, y1; ex2_poly2(y0, y1, x0, x1);
  out[2*i] = y0; out[2*i+1] = y1;
}
int main() {
  const int n = 1 << 20; float* d; cudaMalloc(&d, 8 * n); k<<<n/256, 256>>>(d, n);
  float* h = (float*)malloc(8 * n); cudaMemcpy(h, d, 8 * n, cudaMemcpyDeviceToHost);
  double worst = 0; int bad = 0;
  for (int i = 0; i < n; ++i) for (int e = 0; e < 2; ++e) {
    double x = -130.0 + 200.0 * (double)((float)i / n); float xf = (float)(-130.f + 200.f * (float)i / n); if (e) xf += 0.37f;
    double xc = fmin(fmax((double)xf, -126.0), 127.0);
    double ref = exp2(xc), got = h[2*i+e];
    double rel = fabs(got - ref) / ref; if (rel > worst) worst = rel; if (rel > 1e-3) ++bad;
  }
  printf("poly exp2 worst rel err %.3e, bad %d\n", worst, bad);
}
