// prims.cuh -- scan, ordered compaction and stable LSD radix sort used on the
// per-iteration path (sizes up to a few million).  Hand-written for sm_100a:
// 256-thread blocks, 8 items per thread, warp-shuffle scans, __match_any_sync
// stable ranking.
#pragma once
#include <algorithm>

#include "common.cuh"

namespace cparls {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048

// inclusive warp scan
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// Block-wide exclusive scan of one value per thread (blockDim == kScanThreads).
// Returns exclusive prefix; *total receives the block sum (all threads).
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T *total) {
  constexpr int kW = kScanThreads / 32;
  __shared__ T wsum[kW + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  if (w == 0) {
    T x = (lane < kW) ? wsum[lane] : T(0);
    T xi = warp_incl_scan(x);
    if (lane < kW) wsum[lane] = xi - x;
    if (lane == kW - 1) wsum[kW] = xi;
  }
  __syncthreads();
  T excl = wsum[w] + inc - v;
  *total = wsum[kW];
  __syncthreads();
  return excl;
}

// ---- generic 3-phase exclusive scan of int64 counts ---------------------------
// n_dev: the count lives on the device (grid sized for an upper bound, blocks
// past the count write zero partials); ctl: asynchronous-step guard.
__global__ void k_scan_partials(const int64_t *__restrict__ in, int64_t n, int64_t *__restrict__ part,
                                const int64_t *n_dev = nullptr, const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  n = dcount(n, n_dev);
  int64_t base = (int64_t)blockIdx.x * kScanTile;
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t idx = base + (int64_t)i * kScanThreads + threadIdx.x;
    if (idx < n) s += in[idx];
  }
  int64_t tot;
  block_excl_scan<int64_t>(s, &tot);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// single block: exclusive scan of part[0..nb) in place; total -> *total
__global__ void k_scan_part(int64_t *part, int64_t nb, int64_t *total, const int64_t *n_dev = nullptr,
                            const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  if (n_dev) nb = ceil_div(*n_dev, kScanTile);
  int64_t carry = 0;
  for (int64_t base = 0; base < nb; base += kScanThreads) {
    int64_t idx = base + threadIdx.x;
    int64_t v = idx < nb ? part[idx] : 0;
    int64_t tot;
    int64_t ex = block_excl_scan<int64_t>(v, &tot);
    if (idx < nb) part[idx] = carry + ex;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

__global__ void k_scan_final(const int64_t *__restrict__ in, int64_t n, const int64_t *__restrict__ part,
                             int64_t *__restrict__ out, const int64_t *n_dev = nullptr,
                             const StepCtl *ctl = nullptr) {
  CPARLS_GUARD(ctl);
  n = dcount(n, n_dev);
  if ((int64_t)blockIdx.x * kScanTile >= n) return;
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t v[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t idx = base + i;
    v[i] = idx < n ? in[idx] : 0;
    s += v[i];
  }
  int64_t tot;
  int64_t ex = block_excl_scan<int64_t>(s, &tot) + part[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t idx = base + i;
    if (idx < n) out[idx] = ex;
    ex += v[i];
  }
}

// exclusive scan of n int64 values; part must hold ceil(n/2048) entries;
// total (device pointer) may be null.  in and out may alias.
inline int exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t n, int64_t *part, int64_t *total,
                              cudaStream_t st) {
  if (n <= 0) {
    if (total) CK(cudaMemsetAsync(total, 0, sizeof(int64_t), st));
    return 1;
  }
  int64_t nb = ceil_div(n, kScanTile);
  k_scan_partials<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, part);
  CK_LAUNCH();
  k_scan_part<<<1, kScanThreads, 0, st>>>(part, nb, total);
  CK_LAUNCH();
  k_scan_final<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, part, out);
  CK_LAUNCH();
  return 3;
}

// The same scan with the count on the device (n_dev, at most n_max) inside an
// asynchronous step: grids sized for n_max, no host synchronisation.
inline int exclusive_scan_i64_dev(const int64_t *in, int64_t *out, int64_t n_max, const int64_t *n_dev,
                                  int64_t *part, int64_t *total, cudaStream_t st, const StepCtl *ctl) {
  const int64_t nb = ceil_div(std::max<int64_t>(n_max, 1), kScanTile);
  k_scan_partials<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n_max, part, n_dev, ctl);
  CK_LAUNCH();
  k_scan_part<<<1, kScanThreads, 0, st>>>(part, nb, total, n_dev, ctl);
  CK_LAUNCH();
  k_scan_final<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n_max, part, out, n_dev, ctl);
  CK_LAUNCH();
  return 3;
}

// ---- single-pass exclusive scan (decoupled look-back) ---------------------------
// One launch instead of partials + part + final.  Tiles (kScanTile entries) are
// taken in block start order from a monotonic ticket (a block waits only on
// tiles of blocks that started before it); each publishes its aggregate, finds
// its exclusive prefix by looking back over 32 predecessors at a time and
// publishes its inclusive prefix.  Tile flags carry the call's epoch, so stale
// flags of earlier calls read as "not yet published" and nothing is cleared
// between calls; the value words are written before the flag (release) and
// read after it (acquire).
struct ScanState {
  unsigned long long *flag = nullptr;   // (epoch << 2) | 1 aggregate, | 2 inclusive prefix
  int64_t *agg = nullptr;
  int64_t *inc = nullptr;
  unsigned long long *ticket = nullptr;
  int64_t cap = 0;                      // tiles
  unsigned long long epoch = 0;         // host: calls so far
  unsigned long long base = 0;          // host: tickets handed out so far
};

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(kScanThreads) k_scan_1pass(const int64_t *in, int64_t *out, int64_t n_max,
                                                             const int64_t *n_dev, int64_t *total,
                                                             unsigned long long *flag, int64_t *agg,
                                                             int64_t *inc, unsigned long long *ticket,
                                                             unsigned long long epoch, unsigned long long base,
                                                             const StepCtl *ctl) {
  __shared__ int64_t s_tile, s_prefix;
  if (threadIdx.x == 0) s_tile = (int64_t)(atomicAdd(ticket, 1ull) - base);
  __syncthreads();
  CPARLS_GUARD(ctl);   // after the ticket: the host counts one per block
  const int64_t t = s_tile;
  const int64_t n = n_dev ? min(*n_dev, n_max) : n_max;
  const int64_t nt = ceil_div(n, kScanTile);
  if (n <= 0) {
    if (t == 0 && threadIdx.x == 0 && total) *total = 0;
    return;
  }
  if (t >= nt) return;
  const int64_t b0 = t * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t v[kScanItems];
  int64_t sum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = b0 + i < n ? in[b0 + i] : 0;
    sum += v[i];
  }
  int64_t tot;
  const int64_t excl = block_excl_scan<int64_t>(sum, &tot);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int64_t prefix = 0;
    if (t == 0) {
      if (lane == 0) { inc[0] = tot; st_release_u64(flag, (epoch << 2) | 2ull); }
    } else {
      if (lane == 0) { agg[t] = tot; st_release_u64(flag + t, (epoch << 2) | 1ull); }
      int64_t j = t - 1;   // window [j - 31, j], lane l reads tile j - l
      while (true) {
        const int64_t jt = j - lane;
        unsigned f = 2u;
        int64_t val = 0;   // past tile 0: an empty inclusive prefix
        if (jt >= 0) {
          const unsigned long long w = ld_acquire_u64(flag + jt);
          f = (w >> 2) == epoch ? (unsigned)(w & 3ull) : 0u;
          if (f == 2u) val = *(volatile int64_t *)(inc + jt);
          else if (f == 1u) val = *(volatile int64_t *)(agg + jt);
        }
        const unsigned incl = __ballot_sync(0xffffffffu, f == 2u);
        const int stop = incl ? __ffs(incl) - 1 : 31;   // nearest inclusive predecessor
        const unsigned unpub = __ballot_sync(0xffffffffu, f == 0u) & (0xffffffffu >> (31 - stop));
        if (unpub) continue;
        prefix += warp_sum<int64_t>(lane <= stop ? val : 0);
        if (incl) break;
        j -= 32;
      }
      if (lane == 0) { inc[t] = prefix + tot; st_release_u64(flag + t, (epoch << 2) | 2ull); }
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  int64_t ex = s_prefix + excl;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (b0 + i < n) out[b0 + i] = ex;
    ex += v[i];
  }
  if (t == nt - 1 && threadIdx.x == kScanThreads - 1 && total) *total = ex;
}

// The single-pass scan of n_dev (at most n_max) values; ss must hold
// ceil(n_max / kScanTile) tiles.  in and out may alias.
inline int exclusive_scan_i64_1p(const int64_t *in, int64_t *out, int64_t n_max, const int64_t *n_dev,
                                 int64_t *total, ScanState &ss, cudaStream_t st, const StepCtl *ctl) {
  const int64_t nb = std::max<int64_t>(1, ceil_div(n_max, kScanTile));
  ++ss.epoch;
  k_scan_1pass<<<(unsigned)nb, kScanThreads, 0, st>>>(in, out, n_max, n_dev, total, ss.flag, ss.agg, ss.inc,
                                                       ss.ticket, ss.epoch, ss.base, ctl);
  CK_LAUNCH();
  ss.base += (unsigned long long)nb;
  return 1;
}

// ---- stable LSD radix sort of (u64 key, u32 value) pairs ------------------------
constexpr int kRadixBits = 8;
constexpr int kRadixBins = 1 << kRadixBits;

__global__ void k_radix_hist(const uint64_t *__restrict__ keys, int64_t n, int shift,
                             uint32_t *__restrict__ hist /* [bins][nblocks] */) {
  __shared__ uint32_t h[kRadixBins];
  for (int i = threadIdx.x; i < kRadixBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kScanTile;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t idx = base + (int64_t)i * kScanThreads + threadIdx.x;
    if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & (kRadixBins - 1)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kRadixBins; i += blockDim.x) hist[(int64_t)i * gridDim.x + blockIdx.x] = h[i];
}

// single block: exclusive scan over hist (bins-major) in place; each thread
// scans kScanItems consecutive entries serially, one block scan per 2048
__global__ void k_radix_scan(uint32_t *hist, int64_t len) {
  uint32_t carry = 0;
  for (int64_t base = 0; base < len; base += kScanTile) {
    const int64_t b0 = base + (int64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t sum = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      v[i] = b0 + i < len ? hist[b0 + i] : 0u;
      sum += v[i];
    }
    uint32_t tot;
    uint32_t ex = carry + block_excl_scan<uint32_t>(sum, &tot);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
      if (b0 + i < len) hist[b0 + i] = ex;
      ex += v[i];
    }
    carry += tot;
    __syncthreads();
  }
}

// Stable scatter: warp w owns items [w*256, (w+1)*256) of the block tile,
// processed as 8 coalesced chunks of 32; ranks via __match_any_sync.
__global__ void k_radix_scatter(const uint64_t *__restrict__ kin, const uint32_t *__restrict__ vin, int64_t n,
                                int shift, const uint32_t *__restrict__ hist, uint64_t *__restrict__ kout,
                                uint32_t *__restrict__ vout) {
  constexpr int kWarps = kScanThreads / 32;
  __shared__ uint32_t wh[kWarps][kRadixBins];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kWarps * kRadixBins; i += blockDim.x) (&wh[0][0])[i] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)w * (32 * kScanItems);
  uint32_t rank[kScanItems];
  uint32_t dig[kScanItems];
#pragma unroll
  for (int c = 0; c < kScanItems; ++c) {
    int64_t idx = base + c * 32 + lane;
    bool valid = idx < n;
    uint32_t d = valid ? (uint32_t)((kin[idx] >> shift) & (kRadixBins - 1)) : 0u;
    unsigned vmask = __ballot_sync(0xffffffffu, valid);
    dig[c] = d;
    if (valid) {
      unsigned peers = __match_any_sync(vmask, d);
      uint32_t before = wh[w][d];
      rank[c] = before + __popc(peers & lanemask_lt());
      __syncwarp(vmask);
      int leader = __ffs(peers) - 1;
      if (lane == leader) wh[w][d] = before + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  // exclusive prefix across warps per digit
  for (int d = threadIdx.x; d < kRadixBins; d += blockDim.x) {
    uint32_t run = 0;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) {
      uint32_t t = wh[ww][d];
      wh[ww][d] = run;
      run += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < kScanItems; ++c) {
    int64_t idx = base + c * 32 + lane;
    if (idx < n) {
      uint32_t d = dig[c];
      uint64_t pos = (uint64_t)hist[(int64_t)d * gridDim.x + blockIdx.x] + wh[w][d] + rank[c];
      kout[pos] = kin[idx];
      vout[pos] = vin[idx];
    }
  }
}

// Sorts (keys, vals) by key bits [0, end_bit) stably.  Ping-pongs between the
// given buffers; returns the index (0 = keys/vals, 1 = ktmp/vtmp) holding the
// result.  hist needs 256*ceil(n/2048) entries.  n must be < 2^32.
// Small lists: one CTA sorts (key, val) pairs in shared memory by the
// composite (key, val) -- a bitonic network over the next power of two, padded
// with (max, max).  With distinct vals (row indices, sample positions) the
// order equals the stable radix order by key.
constexpr int kSmallSortMax = 4096;   // 48 KB of static shared memory
constexpr int kSmallSortThreads = 1024;

__global__ void __launch_bounds__(kSmallSortThreads) k_small_sort_pairs(uint64_t *__restrict__ keys,
                                                                        uint32_t *__restrict__ vals, int n) {
  __shared__ uint64_t sk[kSmallSortMax];
  __shared__ uint32_t sv[kSmallSortMax];
  int np = 1;
  while (np < n) np <<= 1;
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    sk[i] = i < n ? keys[i] : ~0ull;
    sv[i] = i < n ? vals[i] : 0xFFFFFFFFu;
  }
  __syncthreads();
  for (int size = 2; size <= np; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (np >> 1); t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint64_t a = sk[lo], b = sk[hi];
        const uint32_t va = sv[lo], vb = sv[hi];
        const bool gt = (a > b) || (a == b && va > vb);
        if (gt == up) {
          sk[lo] = b; sk[hi] = a;
          sv[lo] = vb; sv[hi] = va;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    keys[i] = sk[i];
    vals[i] = sv[i];
  }
}

// One-CTA sort with the count on the device: n > kSmallSortMax raises abort
// (the step then goes to the host-driven path, which has the multi-CTA sort).
__global__ void __launch_bounds__(kSmallSortThreads) k_small_sort_pairs_dev(uint64_t *__restrict__ keys,
                                                                            uint32_t *__restrict__ vals,
                                                                            const int64_t *n_dev, StepCtl *ctl,
                                                                            int64_t step) {
  CPARLS_GUARD(ctl);
  const int64_t n64 = *n_dev;
  if (n64 > kSmallSortMax) {
    if (threadIdx.x == 0) step_abort(ctl, step);
    return;
  }
  const int n = (int)n64;
  if (n <= 1) return;
  __shared__ uint64_t sk[kSmallSortMax];
  __shared__ uint32_t sv[kSmallSortMax];
  int np = 1;
  while (np < n) np <<= 1;
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    sk[i] = i < n ? keys[i] : ~0ull;
    sv[i] = i < n ? vals[i] : 0xFFFFFFFFu;
  }
  __syncthreads();
  for (int size = 2; size <= np; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (np >> 1); t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint64_t a = sk[lo], b = sk[hi];
        const uint32_t va = sv[lo], vb = sv[hi];
        const bool gt = (a > b) || (a == b && va > vb);
        if (gt == up) {
          sk[lo] = b; sk[hi] = a;
          sv[lo] = vb; sv[hi] = va;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    keys[i] = sk[i];
    vals[i] = sv[i];
  }
}

inline int radix_sort_pairs(uint64_t *keys, uint32_t *vals, uint64_t *ktmp, uint32_t *vtmp, int64_t n,
                            int end_bit, uint32_t *hist, cudaStream_t st, int64_t *launches) {
  if (n <= 1) return 0;
  if (n <= kSmallSortMax) {   // in place, one launch (requires distinct vals; callers pass indices)
    k_small_sort_pairs<<<1, kSmallSortThreads, 0, st>>>(keys, vals, (int)n);
    CK_LAUNCH();
    if (launches) *launches += 1;
    return 0;
  }
  int64_t nb = ceil_div(n, kScanTile);
  uint64_t *kb[2] = {keys, ktmp};
  uint32_t *vb[2] = {vals, vtmp};
  int cur = 0;
  for (int shift = 0; shift < end_bit; shift += kRadixBits) {
    k_radix_hist<<<(unsigned)nb, kScanThreads, 0, st>>>(kb[cur], n, shift, hist);
    CK_LAUNCH();
    k_radix_scan<<<1, kScanThreads, 0, st>>>(hist, nb * kRadixBins);
    CK_LAUNCH();
    k_radix_scatter<<<(unsigned)nb, kScanThreads, 0, st>>>(kb[cur], vb[cur], n, shift, hist, kb[cur ^ 1],
                                                           vb[cur ^ 1]);
    CK_LAUNCH();
    cur ^= 1;
    if (launches) *launches += 3;
  }
  return cur;
}

}  // namespace cparls
