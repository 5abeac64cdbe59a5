// Probe: achievable HBM bandwidth of the colored sweep's access pattern
// without any arithmetic.  Elements are 24-double (192 B) blocks; one
// "color" pairs every element once (left ascending, right random), and each
// element side is read (U), read (R) and written (R) -- the TPE kernel's
// traffic for a middle color pass.  Also a streaming copy for reference.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
constexpr int W = 24;
__device__ __forceinline__ void ld4(const double* p, double& a, double& b, double& c, double& d) {
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p)); }
__device__ __forceinline__ void ld4c(const double* p, double& a, double& b, double& c, double& d) {
  asm("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p)); }
__device__ __forceinline__ void st4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory"); }
__global__ void __launch_bounds__(128, 3) side_pass(const int2* lr, const double* U, double* R, int n) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < 2 * n; k += gridDim.x * blockDim.x) {
    int2 e2 = lr[k >> 1]; int e = (k & 1) ? e2.y : e2.x;
    double u[W], r[W];
    #pragma unroll
    for (int j = 0; j < W / 4; ++j) ld4(U + (size_t)e * W + 4 * j, u[4*j], u[4*j+1], u[4*j+2], u[4*j+3]);
    #pragma unroll
    for (int j = 0; j < W / 4; ++j) ld4c(R + (size_t)e * W + 4 * j, r[4*j], r[4*j+1], r[4*j+2], r[4*j+3]);
    #pragma unroll
    for (int j = 0; j < W; ++j) r[j] += 1e-3 * u[j];
    #pragma unroll
    for (int j = 0; j < W / 4; ++j) st4(R + (size_t)e * W + 4 * j, r[4*j], r[4*j+1], r[4*j+2], r[4*j+3]);
  }
}
__global__ void copy_k(const double4* a, double4* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  const int ne = 1 << 20, ns = ne / 2;
  std::vector<int> perm(ne); for (int i = 0; i < ne; ++i) perm[i] = i;
  std::mt19937 g(1); std::shuffle(perm.begin(), perm.end(), g);
  std::vector<int2> lr(ns), lr_seq(ns);
  for (int k = 0; k < ns; ++k) { int a = perm[2*k], b = perm[2*k+1]; lr[k] = make_int2(std::min(a,b), std::max(a,b)); lr_seq[k] = make_int2(k, ns + k); }
  std::sort(lr.begin(), lr.end(), [](int2 x, int2 y){ return x.x < y.x; });
  double *U, *R; int2 *dlr, *dseq;
  cudaMalloc(&U, (size_t)ne * W * 8); cudaMalloc(&R, (size_t)ne * W * 8);
  cudaMemset(U, 0, (size_t)ne * W * 8); cudaMemset(R, 0, (size_t)ne * W * 8);
  cudaMalloc(&dlr, ns * 8); cudaMalloc(&dseq, ns * 8);
  cudaMemcpy(dlr, lr.data(), ns * 8, cudaMemcpyHostToDevice); cudaMemcpy(dseq, lr_seq.data(), ns * 8, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int pass = 0; pass < 2; ++pass) {
    const int2* idx = pass ? dseq : dlr;
    for (int grid : {sms * 3, sms * 6, 2 * ns / 128}) {
      side_pass<<<grid, 128>>>(idx, U, R, ns); cudaEventRecord(a);
      for (int it = 0; it < 10; ++it) side_pass<<<grid, 128>>>(idx, U, R, ns);
      cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
      double bytes = 10.0 * 2 * ns * (3.0 * W * 8 + 4);
      printf("%s grid %6d: %.3f ms/pass  %.0f GB/s\n", pass ? "coalesced" : "random-right", grid, ms / 10, bytes / (ms / 10 * 1e-3) / 1e9 / 10);
    }
  }
  size_t n4 = (size_t)ne * W / 4;
  copy_k<<<sms * 8, 256>>>((double4*)U, (double4*)R, n4); cudaEventRecord(a);
  for (int it = 0; it < 10; ++it) copy_k<<<sms * 8, 256>>>((double4*)U, (double4*)R, n4);
  cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
  printf("copy: %.0f GB/s (%s)\n", 10.0 * 2 * n4 * 32 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}
