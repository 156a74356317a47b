// Probe: latency of fp64 ops and of the r x r factorizations (kernels.cuh) in
// one block, clock64-timed inside the kernel (no launch overhead).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//      -I../../paper_2006_16438_b200/csrc smallla_probe.cu -o smallla_probe
#include <cstdio>
#include <vector>
#include "kernels.cuh"
using namespace cparls;

__global__ void k_ops(double *out, long long *cyc, double x0) {
  double x = x0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < 1000; ++i) x = fma(x, 0.999999, 1e-7);
  long long t1 = clock64();
  double y = x;
  for (int i = 0; i < 100; ++i) y = sqrt(y + 1.0);
  long long t2 = clock64();
  double z = y;
  for (int i = 0; i < 100; ++i) z = 1.5 / (z + 1.0);
  long long t3 = clock64();
  double w = z;
  for (int i = 0; i < 100; ++i) w = __shfl_sync(0xffffffffu, w, (threadIdx.x + 1) & 31) + 1.0;
  long long t4 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
  out[threadIdx.x] = x + y + z + w;
}

__global__ void k_chol(const double *Gg, int r, long long *cyc, double *outLi) {
  extern __shared__ double sm[];
  double *G = sm, *L = sm + r * r, *Li = sm + 2 * r * r;
  __shared__ int ok;
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) G[i] = Gg[i];
  __syncthreads();
  long long t0 = clock64();
  int g1 = 0;
  g1 = block_chol_inv32(r, G, L, Li);
  __syncthreads();
  long long t1 = clock64();
  int g2 = block_cholesky(r, G, L, &ok);
  if (g2) block_tri_inverse(r, L, Li);
  __syncthreads();
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = g1; cyc[3] = g2; }
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) outLi[i] = Li[i];
}

int main() {
  double *d; long long *c;
  cudaMalloc(&d, 1 << 20); cudaMalloc(&c, 64 * 8);
  k_ops<<<1, 32>>>(d, c, 1.0);
  long long h[8];
  cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("dfma chain %.2f clk/op, sqrt %.1f clk/op, div %.1f clk/op, shfl+add %.1f clk/op\n", h[0] / 1000.0, h[1] / 100.0, h[2] / 100.0, h[3] / 100.0);
  const int r = 25;
  std::vector<double> A(r * r), G(r * r, 0.0);
  for (int i = 0; i < r * r; ++i) A[i] = ((i * 7919) % 1000) / 1000.0 + (i % (r + 1) == 0 ? 3.0 : 0.0);
  for (int i = 0; i < r; ++i) for (int j = 0; j < r; ++j) for (int k = 0; k < r; ++k) G[i * r + j] += A[k * r + i] * A[k * r + j];
  double *dG; cudaMalloc(&dG, r * r * 8);
  cudaMemcpy(dG, G.data(), r * r * 8, cudaMemcpyHostToDevice);
  for (int threads : {128, 256}) {
    k_chol<<<1, threads, 3 * r * r * 8>>>(dG, r, c, d);
    cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("threads %d: block_chol_inv32 %lld clk (ok %lld), block_cholesky+tri_inverse %lld clk (ok %lld)\n", threads, h[0], h[2], h[1], h[3]);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
