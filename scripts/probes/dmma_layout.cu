#include <cstdio>
#include <cuda_runtime.h>
// probe: D = A(8x4) * B(4x8) with mma.sync.m8n8k4.row.col.f64; print which layout matches
__global__ void k(const double *A, const double *B, double *D) {
  int lane = threadIdx.x, gid = lane >> 2, tig = lane & 3;
  double a = A[gid * 4 + tig];          // A[row=gid][col=tig]
  double b = B[tig * 8 + gid];          // B[row=tig][col=gid]
  double c0 = 0, c1 = 0;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  D[gid * 8 + 2 * tig] = c0;             // D[row=gid][col=2tig], [2tig+1]
  D[gid * 8 + 2 * tig + 1] = c1;
}
int main() {
  double hA[32], hB[32], hD[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = i + 1; hB[i] = (i * 7) % 11 - 5; }
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 8; ++j) { double s = 0; for (int k = 0; k < 4; ++k) s += hA[i*4+k] * hB[k*8+j]; ref[i*8+j] = s; }
  double *A, *B, *D; cudaMalloc(&A, 256); cudaMalloc(&B, 256); cudaMalloc(&D, 512);
  cudaMemcpy(A, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(A, B, D); cudaMemcpy(hD, D, 512, cudaMemcpyDeviceToHost);
  double err = 0; for (int i = 0; i < 64; ++i) err += fabs(hD[i] - ref[i]);
  printf("dmma layout err %g (%s)\n", err, cudaGetErrorString(cudaGetLastError()));
}
