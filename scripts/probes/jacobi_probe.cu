// Probe: sweeps and cycles of block_jacobi (kernels.cuh) on the Grams of
// jacobi_G_C2.txt (C2 normalized factors; mode 1 has 24 < r rows: rank 24).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//      -I../../paper_2006_16438_b200/csrc jacobi_probe.cu -o jacobi_probe
#include <cstdio>
#include <vector>
#include "kernels.cuh"
using namespace cparls;

__global__ void k_probe(const double *Gs, int n, int r, int *sweeps, long long *cyc, double *w) {
  extern __shared__ double sm[];
  double *a = sm, *V = sm + r * r;
  for (int m = 0; m < n; ++m) {
    for (int i = threadIdx.x; i < r * r; i += blockDim.x) a[i] = Gs[(size_t)m * r * r + i];
    __syncthreads();
    long long t0 = clock64();
    int sw = block_jacobi(r, a, V);
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) { sweeps[m] = sw; cyc[m] = t1 - t0; }
    for (int i = threadIdx.x; i < r; i += blockDim.x) w[m * r + i] = a[i * r + i];
    __syncthreads();
  }
}

int main(int argc, char **argv) {
  const char *path = argc > 1 ? argv[1] : "jacobi_G_C2.txt";
  FILE *f = fopen(path, "r");
  if (!f) { printf("no %s\n", path); return 1; }
  std::vector<double> g;
  char line[65536];
  while (fgets(line, sizeof line, f)) {
    if (line[0] == '#') continue;
    char *p = line, *e;
    for (double v = strtod(p, &e); p != e; v = strtod(p, &e)) { g.push_back(v); p = e; }
  }
  const int r = 25, n = (int)(g.size() / (r * r));
  double *dG, *dw; int *ds; long long *dc;
  cudaMalloc(&dG, g.size() * 8); cudaMalloc(&dw, n * r * 8); cudaMalloc(&ds, n * 4); cudaMalloc(&dc, n * 8);
  cudaMemcpy(dG, g.data(), g.size() * 8, cudaMemcpyHostToDevice);
  for (int threads : {128, 256}) {
    k_probe<<<1, threads, 2 * r * r * 8>>>(dG, n, r, ds, dc, dw);
    cudaDeviceSynchronize();
    std::vector<int> s(n); std::vector<long long> c(n);
    cudaMemcpy(s.data(), ds, n * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(c.data(), dc, n * 8, cudaMemcpyDeviceToHost);
    for (int m = 0; m < n; ++m) printf("threads %d G%d sweeps %d cycles %lld (%.1f us at 1.9 GHz)\n", threads, m, s[m], c[m], c[m] / 1900.0);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
