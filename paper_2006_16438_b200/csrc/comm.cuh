// comm.cuh -- collectives of the row-sharded CP-ARLS-LEV path.
//
// Two backends behind one interface:
//  * NcclComm: one process per GPU, NCCL over NVLink/NVSwitch (ncclAllReduce,
//    grouped ncclBroadcast for the variable-size factor allgather, grouped
//    ncclSend/ncclRecv for the build-time all-to-all).
//  * LocalComm: P shards driven by P host threads of ONE process on one GPU
//    (the shard simulator used by tests on a single B200).  Every collective
//    is a host rendezvous: each shard drains its own stream, deposits its
//    pointers, and the last arriving shard performs the exchange with device
//    copies / a sum kernel on its stream before releasing the others.  No
//    kernel ever waits on another shard's kernel.
// Reductions are summed in rank order (deterministic for both backends only
// up to NCCL's own ordering).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace cparls {

#define NCK(x)                                                                                         \
  do {                                                                                                 \
    ncclResult_t r_ = (x);                                                                             \
    if (r_ != ncclSuccess)                                                                             \
      throw ::cparls::ApiError(4, std::string(#x) + ": " + ncclGetErrorString(r_) + " @" + __FILE__ + \
                                      ":" + std::to_string(__LINE__));                                \
  } while (0)

struct Comm {
  int world = 1, rank = 0;
  virtual ~Comm() {}
  virtual void allreduce_f64(double *buf, size_t n, cudaStream_t st) = 0;
  virtual void allreduce_u64(unsigned long long *buf, size_t n, cudaStream_t st) = 0;
  // block q = [off[q], off[q+1]) doubles of buf lives on rank q; afterwards
  // every rank has every block (variable-size allgather, in place)
  virtual void allgatherv_f64(double *buf, const std::vector<int64_t> &off, cudaStream_t st) = 0;
  // send[soff[q], soff[q+1]) bytes go to rank q; receive rank q's block into
  // recv[roff[q], roff[q+1])
  virtual void alltoallv(const char *send, const std::vector<int64_t> &soff, char *recv,
                         const std::vector<int64_t> &roff, cudaStream_t st) = 0;
  // host allgather of one int64 per rank
  virtual std::vector<int64_t> allgather_host(const std::vector<int64_t> &mine, cudaStream_t st) = 0;
};

__global__ void k_sum_into(double *__restrict__ dst, const double *__restrict__ src, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}
__global__ void k_sum_into_u64(unsigned long long *__restrict__ dst, const unsigned long long *__restrict__ src,
                               size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

// ------------------------------------------------------------------ NCCL
struct NcclComm : Comm {
  ncclComm_t c = nullptr;
  bool owns = false;
  ~NcclComm() override {
    if (c && owns) ncclCommDestroy(c);
  }
  void allreduce_f64(double *buf, size_t n, cudaStream_t st) override {
    NCK(ncclAllReduce(buf, buf, n, ncclDouble, ncclSum, c, st));
  }
  void allreduce_u64(unsigned long long *buf, size_t n, cudaStream_t st) override {
    NCK(ncclAllReduce(buf, buf, n, ncclUint64, ncclSum, c, st));
  }
  void allgatherv_f64(double *buf, const std::vector<int64_t> &off, cudaStream_t st) override {
    NCK(ncclGroupStart());
    for (int q = 0; q < world; ++q) {
      const size_t cnt = (size_t)(off[q + 1] - off[q]);
      if (cnt) NCK(ncclBroadcast(buf + off[q], buf + off[q], cnt, ncclDouble, q, c, st));
    }
    NCK(ncclGroupEnd());
  }
  void alltoallv(const char *send, const std::vector<int64_t> &soff, char *recv, const std::vector<int64_t> &roff,
                 cudaStream_t st) override {
    NCK(ncclGroupStart());
    for (int q = 0; q < world; ++q) {
      const size_t sb = (size_t)(soff[q + 1] - soff[q]), rb = (size_t)(roff[q + 1] - roff[q]);
      if (sb) NCK(ncclSend(send + soff[q], sb, ncclChar, q, c, st));
      if (rb) NCK(ncclRecv(recv + roff[q], rb, ncclChar, q, c, st));
    }
    NCK(ncclGroupEnd());
  }
  std::vector<int64_t> allgather_host(const std::vector<int64_t> &mine, cudaStream_t st) override {
    const size_t m = mine.size();
    int64_t *d = nullptr;
    CK(cudaMalloc(&d, sizeof(int64_t) * m * world));
    CK(cudaMemcpyAsync(d + m * rank, mine.data(), sizeof(int64_t) * m, cudaMemcpyHostToDevice, st));
    NCK(ncclAllGather(d + m * rank, d, m, ncclInt64, c, st));
    std::vector<int64_t> all(m * world);
    CK(cudaMemcpyAsync(all.data(), d, sizeof(int64_t) * m * world, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    cudaFree(d);
    return all;
  }
};

// ------------------------------------------------------------------ local group
struct LocalGroup {
  int P;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<void *> a, b;                       // per-rank pointers
  std::vector<const std::vector<int64_t> *> va, vb;
  std::vector<std::vector<int64_t>> host_in;
  std::vector<int64_t> host_out;
  cudaStream_t st = nullptr;                      // stream of the exchanging shard
  explicit LocalGroup(int p) : P(p), a(p), b(p), va(p), vb(p), host_in(p) {}

  // every shard calls with its own deposit; `op` runs once (by the last) while
  // all shards wait; afterwards all return
  void rendezvous(int rank, const std::function<void()> &deposit, const std::function<void()> &op) {
    std::unique_lock<std::mutex> lk(mu);
    deposit();
    const uint64_t g = gen;
    if (++arrived == P) {
      op();
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct LocalComm : Comm {
  LocalGroup *g = nullptr;
  void allreduce_f64(double *buf, size_t n, cudaStream_t st) override {
    CK(cudaStreamSynchronize(st));
    g->rendezvous(rank, [&] { g->a[rank] = buf; }, [&] {
      double *acc = nullptr;
      CK(cudaMalloc(&acc, sizeof(double) * std::max<size_t>(n, 1)));
      CK(cudaMemcpyAsync(acc, g->a[0], sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
      for (int q = 1; q < g->P; ++q) k_sum_into<<<128, 256, 0, st>>>(acc, (const double *)g->a[q], n);
      for (int q = 0; q < g->P; ++q)
        CK(cudaMemcpyAsync(g->a[q], acc, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
      CK(cudaStreamSynchronize(st));
      cudaFree(acc);
    });
  }
  void allreduce_u64(unsigned long long *buf, size_t n, cudaStream_t st) override {
    CK(cudaStreamSynchronize(st));
    g->rendezvous(rank, [&] { g->a[rank] = buf; }, [&] {
      unsigned long long *acc = nullptr;
      CK(cudaMalloc(&acc, sizeof(unsigned long long) * std::max<size_t>(n, 1)));
      CK(cudaMemcpyAsync(acc, g->a[0], sizeof(unsigned long long) * n, cudaMemcpyDeviceToDevice, st));
      for (int q = 1; q < g->P; ++q)
        k_sum_into_u64<<<128, 256, 0, st>>>(acc, (const unsigned long long *)g->a[q], n);
      for (int q = 0; q < g->P; ++q)
        CK(cudaMemcpyAsync(g->a[q], acc, sizeof(unsigned long long) * n, cudaMemcpyDeviceToDevice, st));
      CK(cudaStreamSynchronize(st));
      cudaFree(acc);
    });
  }
  void allgatherv_f64(double *buf, const std::vector<int64_t> &off, cudaStream_t st) override {
    CK(cudaStreamSynchronize(st));
    g->rendezvous(rank, [&] { g->a[rank] = buf; }, [&] {
      for (int src = 0; src < g->P; ++src) {
        const size_t cnt = (size_t)(off[src + 1] - off[src]);
        if (!cnt) continue;
        for (int dst = 0; dst < g->P; ++dst)
          if (dst != src)
            CK(cudaMemcpyAsync((double *)g->a[dst] + off[src], (double *)g->a[src] + off[src],
                               sizeof(double) * cnt, cudaMemcpyDeviceToDevice, st));
      }
      CK(cudaStreamSynchronize(st));
    });
  }
  void alltoallv(const char *send, const std::vector<int64_t> &soff, char *recv, const std::vector<int64_t> &roff,
                 cudaStream_t st) override {
    CK(cudaStreamSynchronize(st));
    g->rendezvous(rank, [&] {
      g->a[rank] = (void *)send; g->b[rank] = recv; g->va[rank] = &soff; g->vb[rank] = &roff;
    }, [&] {
      for (int p = 0; p < g->P; ++p)
        for (int q = 0; q < g->P; ++q) {
          const std::vector<int64_t> &so = *g->va[p], &ro = *g->vb[q];
          const size_t bytes = (size_t)(so[q + 1] - so[q]);
          if (bytes)
            CK(cudaMemcpyAsync((char *)g->b[q] + ro[p], (const char *)g->a[p] + so[q], bytes,
                               cudaMemcpyDeviceToDevice, st));
        }
      CK(cudaStreamSynchronize(st));
    });
  }
  std::vector<int64_t> allgather_host(const std::vector<int64_t> &mine, cudaStream_t st) override {
    std::vector<int64_t> out;
    g->rendezvous(rank, [&] { g->host_in[rank] = mine; }, [&] {
      g->host_out.clear();
      for (int q = 0; q < g->P; ++q) g->host_out.insert(g->host_out.end(), g->host_in[q].begin(), g->host_in[q].end());
    });
    {
      std::lock_guard<std::mutex> lk(g->mu);
      out = g->host_out;
    }
    // second rendezvous so nobody overwrites host_out before everyone copied it
    g->rendezvous(rank, [] {}, [] {});
    return out;
  }
};

}  // namespace cparls
