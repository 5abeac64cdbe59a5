// Probe: fragment layout of mma.sync.m8n8k4 f64 on sm_100a.
#include <cstdio>
#include <cmath>
__global__ void k(const double* A, const double* B, double* D) {
  int l = threadIdx.x;
  double a = A[(l >> 2) * 4 + (l & 3)];        // A 8x4 row-major, A[l>>2][l&3]
  double b = B[(l & 3) * 8 + (l >> 2)];        // B 4x8 row-major, B[l&3][l>>2]
  double d0, d1, c0 = 0, c1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
  D[(l >> 2) * 8 + 2 * (l & 3)] = d0;          // D[l>>2][2(l&3)+i]
  D[(l >> 2) * 8 + 2 * (l & 3) + 1] = d1;
}
int main() {
  double hA[32], hB[32], hD[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = 1.0 + i * 0.37; hB[i] = 2.0 - i * 0.11; }
  for (int r = 0; r < 8; ++r) for (int c = 0; c < 8; ++c) { double s = 0; for (int k = 0; k < 4; ++k) s += hA[r*4+k] * hB[k*8+c]; ref[r*8+c] = s; }
  double *dA, *dB, *dD; cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dD, 512);
  cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(dA, dB, dD); cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost);
  double err = 0; for (int i = 0; i < 64; ++i) err = fmax(err, fabs(hD[i] - ref[i]));
  printf("dmma layout max err %g (%s)\n", err, cudaGetErrorString(cudaGetLastError()));
  return err < 1e-12 ? 0 : 1;
}
