// Error of the hardware tanh approximations against tanh in double (K7 epilogue sizing,
// DESIGN.md §6b): tanh.approx.f32 on fp32 inputs, tanh.approx.f16x2 on fp16 inputs (every
// finite fp16), and the current ex2 + Newton tanh_fast.  Prints max abs / rel errors.
#include <cstdio>
#include <cmath>
#include <cuda_fp16.h>
__global__ void k32(const float* x, float* y, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { float r; asm("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(x[i])); y[i] = r; }
}
__global__ void k16(const unsigned* x, unsigned* y, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { unsigned r; asm("tanh.approx.f16x2 %0, %1;" : "=r"(r) : "r"(x[i])); y[i] = r; }
}
int main() {
  const int n = 1 << 22;
  float *x, *y; cudaMallocManaged(&x, n * 4); cudaMallocManaged(&y, n * 4);
  for (int i = 0; i < n; ++i) x[i] = -12.f + 24.f * (float)i / n;
  k32<<<(n + 255) / 256, 256>>>(x, y, n); cudaDeviceSynchronize();
  double ma = 0, mr = 0, ma_small = 0;
  for (int i = 0; i < n; ++i) {
    double t = tanh((double)x[i]), e = fabs(y[i] - t);
    ma = fmax(ma, e); if (fabs(t) > 1e-3) mr = fmax(mr, e / fabs(t));
  }
  printf("tanh.approx.f32: max abs %.3g max rel (|t|>1e-3) %.3g\n", ma, mr);
  const int m = 65536 / 2;
  unsigned *hx, *hy; cudaMallocManaged(&hx, m * 4); cudaMallocManaged(&hy, m * 4);
  for (int i = 0; i < m; ++i) hx[i] = (unsigned)(2 * i) | ((unsigned)(2 * i + 1) << 16);
  k16<<<(m + 255) / 256, 256>>>(hx, hy, m); cudaDeviceSynchronize();
  double ha = 0, hr = 0, hulp = 0;
  for (int i = 0; i < m; ++i) for (int h = 0; h < 2; ++h) {
    __half_raw a; a.x = (unsigned short)(hx[i] >> (16 * h)); __half_raw b; b.x = (unsigned short)(hy[i] >> (16 * h));
    float xv = __half2float(__half(a)), yv = __half2float(__half(b));
    if (!std::isfinite(xv)) continue;
    double t = tanh((double)xv), e = fabs(yv - t);
    ha = fmax(ha, e); if (fabs(t) > 1e-3) hr = fmax(hr, e / fabs(t));
    double ulp = ldexp(1.0, (int)floor(log2(fmax(fabs(t), 6.1e-5))) - 10);
    hulp = fmax(hulp, e / ulp);
  }
  printf("tanh.approx.f16x2: max abs %.3g max rel (|t|>1e-3) %.3g max err in fp16 ulps of tanh %.3g\n", ha, hr, hulp);
  return 0;
}
