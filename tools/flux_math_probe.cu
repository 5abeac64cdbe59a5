#include <cstdio>
#include <cmath>
#include "/root/repo/paper_1601_07613_b200/csrc/dg_kernels.cuh"
__global__ void k(double* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = 0.05 + 3.0 * (i / double(n)) + 1e-3 * sin(double(i));
  out[4 * i] = mcdg::flux_rcp(x) * x - 1.0;
  out[4 * i + 1] = (mcdg::flux_rcp(x) - 1.0 / x) / (1.0 / x);
  out[4 * i + 2] = (mcdg::flux_sqrt(x) - sqrt(x)) / sqrt(x);
  out[4 * i + 3] = (mcdg::flux_sqrt(x * 1e-3) - sqrt(x * 1e-3)) / sqrt(x * 1e-3);
}
int main() {
  const int n = 1 << 20;
  double* d; cudaMalloc(&d, sizeof(double) * 4 * n);
  k<<<n / 256, 256>>>(d, n);
  double* h = new double[4 * n];
  cudaMemcpy(h, d, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost);
  double m[4] = {0, 0, 0, 0};
  for (int i = 0; i < n; ++i) for (int j = 0; j < 4; ++j) m[j] = fmax(m[j], fabs(h[4 * i + j]));
  printf("max rel err: rcp*x-1 %.3e  rcp %.3e  sqrt %.3e  sqrt(small) %.3e\n", m[0], m[1], m[2], m[3]);
}
