// sampler.cuh -- the asynchronous (host-synchronisation-free) parts of SkrpLev
// (Alg. 1): the control kernels that carry the sample sizes on the
// device between the DIDX / SIDX / CIDX kernels of kernels.cuh, and SIDX
// (Alg. 2) as ONE persistent kernel that draws attempts until
// s_rnd are accepted ("samples and rejects indices in bulk, oversampling",
// P:819-820), keeping the first s_rnd accepted attempts in attempt order
// (AMB-8) with a decoupled look-back prefix over attempt tiles.
#pragma once
#include "kernels.cuh"

namespace cparls {

// ---- DIDX candidates of every other mode in two launches:
// k_cand_append marks the rows with prod_with(p~_i) > tau of all d modes in
// one grid and appends them with a counter per mode (any order); k_cand_sort
// (one CTA per mode) sorts each list by the composite (~bits(p~), row) --
// p~ descending, ties by row -- which fixes the order whatever the append
// order was.  A list longer than kSmallSortMax raises abort (host path).
struct CandBufs {
  uint64_t *key[kMaxModes];
  uint32_t *idx[kMaxModes];
};

__global__ void k_cand_append(OtherModes om, double tau, CandBufs cb, StepCtl *ctl) {
  CPARLS_GUARD(ctl);
  double al[kMaxModes];
  load_alphas(om, al);
  int64_t total = 0;
  for (int j = 0; j < om.d; ++j) total += om.n[j];
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    int j = 0;
    int64_t idx = g;
    while (idx >= om.n[j]) { idx -= om.n[j]; ++j; }
    const double p = om.pt[j][idx];
    if (prod_with(om, al, j, p) > tau) {
      const unsigned long long pos = atomicAdd(&ctl->cand_acc[j], 1ull);
      cb.key[j][pos] = ~(uint64_t)__double_as_longlong(p);
      cb.idx[j][pos] = (uint32_t)idx;
    }
  }
}

__global__ void __launch_bounds__(kSmallSortThreads) k_cand_sort(CandBufs cb, StepCtl *ctl, int64_t step) {
  CPARLS_GUARD(ctl);
  const int j = blockIdx.x;
  const int64_t n64 = (int64_t)*(volatile unsigned long long *)&ctl->cand_acc[j];
  __syncthreads();   // every thread has read the count
  if (threadIdx.x == 0) {
    ctl->cand_acc[j] = 0ull;   // ready for the next step (stream-ordered)
    ctl->ncand[j] = n64;
  }
  if (n64 > kSmallSortMax) {
    if (threadIdx.x == 0) step_abort(ctl, step);
    return;
  }
  const int n = (int)n64;
  if (n <= 1) return;
  __shared__ uint64_t sk[kSmallSortMax];
  __shared__ uint32_t sv[kSmallSortMax];
  uint64_t *keys = cb.key[j];
  uint32_t *vals = cb.idx[j];
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

// ---------------------------------------------------------------- DIDX control
// Level 0 holds the candidates of mode m_1: nlist = ncand[0]; the DIDX list
// capacity (lcap) and the didx_cap limit are checked here and at every level.
__global__ void k_didx_start(StepCtl *ctl, int64_t lcap, int64_t cap, int64_t step) {
  CPARLS_GUARD(ctl);
  const int64_t n0 = ctl->ncand[0];
  ctl->nlist = n0;
  if (n0 > lcap || n0 > cap) step_abort(ctl, step);
}

// After the scan of a level's counts: the new length (ctl->scan_total) must fit
// the list buffers and didx_cap; otherwise the host-driven path (which grows
// the buffers, or reports ESAMPLE) takes the step.
__global__ void k_didx_check(StepCtl *ctl, int64_t lcap, int64_t cap, int64_t step) {
  CPARLS_GUARD(ctl);
  const int64_t nn = ctl->scan_total;
  if (nn > lcap || nn > cap) step_abort(ctl, step);
}
__global__ void k_didx_advance(StepCtl *ctl) {
  CPARLS_GUARD(ctl);
  ctl->nlist = ctl->scan_total;
}

// End of DIDX: s_det = list length.  The AMB-6 truncation (s_det > s) and the
// tau < 2^-63 drawable test run on the host path.
__global__ void k_didx_finish(StepCtl *ctl, int64_t s, int tiny_tau, int64_t step) {
  CPARLS_GUARD(ctl);
  const int64_t sdet = ctl->nlist;
  ctl->sdet = sdet;
  if (sdet > s || (tiny_tau && sdet > 0)) step_abort(ctl, step);
}

// ---------------------------------------------------------------- SIDX
constexpr int kSidxItems = 4;
constexpr int kSidxTile = kSidxThreads * kSidxItems;   // attempts per tile

// SIDX setup (Alg. 2 line 1; AMB-7): s_rnd = s - s_det; the random phase is
// skipped when 1 - p_det <= 1e-12 or every drawable row (q > 0 in every other
// mode) is deterministic (tau >= 2^-63: every DetSet row is drawable).
__global__ void k_sidx_prep(StepCtl *ctl, OtherModes om, int64_t s) {
  CPARLS_GUARD(ctl);
  const int64_t sdet = ctl->sdet;
  const int64_t s_rnd = s - sdet;
  double drawable_all = 1.0;
  for (int j = 0; j < om.d; ++j) drawable_all *= (double)om.md[j]->drawable;
  const int skip = s_rnd > 0 && (1.0 - ctl->pdet <= 1e-12 || drawable_all <= (double)sdet);
  ctl->s_rnd = s_rnd;
  ctl->skip = skip;
  ctl->have = skip ? 0 : s_rnd;
  ctl->attempts = 0;
  ctl->sidx_next_tile = 0;
  ctl->sidx_done = (s_rnd <= 0 || skip) ? 1 : 0;
  unsigned e = ctl->sidx_epoch + 1;
  if (e >= (1u << 30)) e = 1;   // epoch 0 = never published
  ctl->sidx_epoch = e;
}

// Tile state word: epoch (30 bits) | flag (2 bits: 1 aggregate, 2 inclusive
// prefix) | value (32 bits: accepted attempts).  Stale words of other epochs
// read as "not yet published", so the array is never cleared.
__device__ __forceinline__ unsigned long long tile_word(unsigned epoch, unsigned flag, unsigned value) {
  return ((unsigned long long)epoch << 34) | ((unsigned long long)flag << 32) | value;
}

// SIDX (Alg. 2) until s_rnd acceptances.  CTAs take tiles of
// kSidxTile consecutive attempts from a counter; thread i of a tile draws
// attempts a0 + 8i .. a0 + 8i + 7 (Philox4x32-10, key = seed, counter =
// (attempt, step, lane), AMB-10), accepts p <= tau; the tile's
// accepted count is published and its exclusive prefix found by looking back
// over the predecessor tiles (CUB-style decoupled look-back; predecessors are
// always held by running CTAs), so the accepted attempts land at their
// attempt-order positions (AMB-8) and the first s_rnd are kept.  The attempt
// cap (AMB-7) sends the step to the host path (which reports ESAMPLE).
__global__ void __launch_bounds__(kSidxThreads, 2) k_sidx_run(OtherModes om, double tau, uint32_t seed_lo,
                                                           uint32_t seed_hi, uint32_t step32, int64_t attempt_cap,
                                                           StepCtl *ctl, unsigned long long *tile_state,
                                                           int64_t tile_cap, uint64_t *__restrict__ rkey,
                                                           double *__restrict__ rp, int64_t step) {
  CPARLS_GUARD(ctl);
  if (ctl->sidx_done) return;   // s_rnd = 0 or AMB-7 skip
  const int64_t need = ctl->s_rnd;
  const int64_t cap_att = attempt_cap > 0 ? attempt_cap : 1024 * need + 65536;
  const unsigned epoch = ctl->sidx_epoch;
  __shared__ int64_t s_tile;
  __shared__ int64_t s_prefix;
  while (true) {
    if (threadIdx.x == 0) {
      const int done = *(volatile int *)&ctl->sidx_done;
      s_tile = done ? -1 : (int64_t)atomicAdd(&ctl->sidx_next_tile, 1ull);
    }
    __syncthreads();
    const int64_t t = s_tile;
    if (t < 0) break;
    const int64_t a0 = t * kSidxTile;
    if (a0 >= cap_att || t >= tile_cap) {   // attempt cap reached before s_rnd acceptances
      if (threadIdx.x == 0) {
        step_abort(ctl, step);
        *(volatile int *)&ctl->sidx_done = 1;
      }
      break;
    }
    // the thread's kSidxItems attempts advance together (one Philox call and
    // one binary-search level of every attempt per step: kSidxItems
    // independent L2 loads in flight per thread)
    uint64_t key[kSidxItems];
    double pv[kSidxItems];
    uint64_t a_[kSidxItems];
#pragma unroll
    for (int it = 0; it < kSidxItems; ++it) {
      a_[it] = (uint64_t)a0 + (uint64_t)threadIdx.x * kSidxItems + it;
      key[it] = 0;
      pv[it] = 1.0;
    }
    for (int lane = 0; lane < (om.d + 1) / 2; ++lane) {
      uint32_t wd[kSidxItems][4];
#pragma unroll
      for (int it = 0; it < kSidxItems; ++it) {
        const u32x4 x = philox4x32_10({(uint32_t)a_[it], (uint32_t)(a_[it] >> 32), step32, (uint32_t)lane}, seed_lo,
                                      seed_hi);
        wd[it][0] = x.x; wd[it][1] = x.y; wd[it][2] = x.z; wd[it][3] = x.w;
      }
      for (int jj = 0; jj < 2 && 2 * lane + jj < om.d; ++jj) {
        const int j = 2 * lane + jj;
        const uint64_t *C = om.C[j];
        const int64_t n = om.n[j];
        const uint64_t W = __ldg(C + n - 1);
        uint64_t t[kSidxItems];
        int64_t lo[kSidxItems];
#pragma unroll
        for (int it = 0; it < kSidxItems; ++it) {
          const uint64_t R = ((uint64_t)wd[it][2 * jj + 1] << 32) | wd[it][2 * jj];
          t[it] = __umul64hi(R, W);                                        // AMB-9
          lo[it] = 0;
        }
        // upper_bound (first C[i] > t) of all items in lockstep by
        // binary lifting: lo = #{i : C[i] <= t} (C is non-decreasing)
        int64_t step = 1;
        while (step * 2 <= n) step *= 2;
        for (; step > 0; step >>= 1) {
#pragma unroll
          for (int it = 0; it < kSidxItems; ++it)
            if (lo[it] + step <= n && __ldg(C + lo[it] + step - 1) <= t[it]) lo[it] += step;
        }
#pragma unroll
        for (int it = 0; it < kSidxItems; ++it) {
          const double v = __ldg(om.pt[j] + lo[it]);
          pv[it] = (j == 0) ? v : pv[it] * v;                              // AMB-5
          key[it] += (uint64_t)lo[it] * om.mult[j];
        }
      }
    }
    unsigned accm = 0;
    int cnt = 0;
#pragma unroll
    for (int it = 0; it < kSidxItems; ++it) {
      const bool acc = pv[it] <= tau && (int64_t)a_[it] < cap_att;
      accm |= (unsigned)acc << it;
      cnt += acc;
    }
    int64_t tot;
    const int64_t excl = block_excl_scan<int64_t>((int64_t)cnt, &tot);
    if (threadIdx.x < 32) {   // warp 0: publish, then look back 32 predecessors at a time
      const int lane = threadIdx.x;
      int64_t prefix = 0;
      if (t == 0) {
        if (lane == 0) atomicExch(tile_state + t, tile_word(epoch, 2u, (unsigned)tot));
      } else {
        if (lane == 0) atomicExch(tile_state + t, tile_word(epoch, 1u, (unsigned)tot));
        int64_t j = t - 1;   // window [j - 31, j], lane l reads tile j - l
        while (true) {
          const int64_t jt = j - lane;
          unsigned wf = 2u, wv = 0u;   // past tile 0: an empty inclusive prefix
          if (jt >= 0) {
            const unsigned long long w = *(volatile unsigned long long *)(tile_state + jt);
            wf = ((unsigned)(w >> 34) == epoch) ? ((unsigned)(w >> 32) & 3u) : 0u;
            wv = (unsigned)w;
          }
          const unsigned incl = __ballot_sync(0xffffffffu, wf == 2u);
          const int stop = incl ? __ffs(incl) - 1 : 31;          // nearest inclusive predecessor
          const unsigned unpub = __ballot_sync(0xffffffffu, wf == 0u) & (0xffffffffu >> (31 - stop));
          if (unpub) continue;                                   // some needed predecessor not published yet
          prefix += warp_sum<int64_t>(lane <= stop ? (int64_t)wv : 0);
          if (incl) break;
          j -= 32;
        }
        if (lane == 0) atomicExch(tile_state + t, tile_word(epoch, 2u, (unsigned)(prefix + tot)));
      }
      if (lane == 0) {
        s_prefix = prefix;
        if (prefix + tot >= need) *(volatile int *)&ctl->sidx_done = 1;
      }
    }
    __syncthreads();
    int64_t pos = s_prefix + excl;
#pragma unroll
    for (int it = 0; it < kSidxItems; ++it) {
      if ((accm >> it) & 1u) {
        if (pos < need) {
          rkey[pos] = key[it];
          rp[pos] = pv[it];
          if (pos == need - 1) ctl->attempts = (int64_t)a_[it] + 1;
        }
        ++pos;
      }
    }
    __syncthreads();
  }
}

// End of CIDX: s_bar = s_det + unique random rows; step statistics.
__global__ void k_sample_finish(StepCtl *ctl) {
  CPARLS_GUARD(ctl);
  const int64_t sbar = ctl->sdet + ctl->nuniq;
  ctl->sbar = sbar;
  ctl->st_sum_sbar += sbar;
  ctl->st_sum_attempts += ctl->attempts;
  ctl->st_sum_sdet += ctl->sdet;
  ctl->st_last_sbar = sbar;
  ctl->st_last_attempts = ctl->attempts;
}

// Leverage refresh setup (replaces unguarded memsets: an aborted step must not
// touch the mode's alpha / drawable count).
__global__ void k_lev_reset(ModeDev *md, const StepCtl *ctl) {
  CPARLS_GUARD(ctl);
  md->alpha = 0.0;
  md->drawable = 0;
}

// lambda of the model <- lambda of the solved mode (AMB-31)
__global__ void k_copy_lambda(double *dst, const double *src, int r, const StepCtl *ctl) {
  CPARLS_GUARD(ctl);
  for (int c = threadIdx.x; c < r; c += blockDim.x) dst[c] = src[c];
}

// per-step statistics of the solve (m_k, touched rows of mode k)
__global__ void k_solve_stats(StepCtl *ctl, int k, const int64_t *mk, const unsigned long long *touched) {
  CPARLS_GUARD(ctl);
  ctl->st_steps += 1;
  ctl->st_sum_mk += *mk;
  ctl->st_last_mk = *mk;
  ctl->st_touched[k] = (int64_t)*touched;
  ctl->st_sum_touched += (int64_t)*touched;
}

// fit = 1 - sqrt(max(0, ||X||^2 - 2<X,M> + ||M||^2)) / ||X|| after <X,M> was
// summed over the ranks (AMB-16)
__global__ void k_fit_combine(double *fit, double normX2, const StepCtl *ctl) {
  CPARLS_GUARD(ctl);
  double resid2 = normX2 - 2.0 * fit[1] + fit[2];
  if (resid2 < 0.0) resid2 = 0.0;
  fit[0] = 1.0 - sqrt(resid2) / sqrt(normX2);
}

// ---------------------------------------------------------------- sharded mode step
// The sampled rows of the other modes from their owners: rank p writes
// A_m(i_m,:) into zg[(j d + slot) ld ..] when it owns row i_m of mode m
// ([row_lo[m], row_hi[m])), zeros otherwise; an allreduce (one nonzero
// contribution per element: exact) gives every rank every sampled row.
__global__ void k_owned_rows(const uint64_t *__restrict__ skey, int64_t smax, const int64_t *sbar_dev,
                             OtherModes om, const int64_t *row_lo, const int64_t *row_hi, int ld,
                             double *__restrict__ zg, const StepCtl *ctl) {
  CPARLS_GUARD(ctl);
  const int64_t sbar = dcount(smax, sbar_dev);
  const int lane = threadIdx.x & 31;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < smax;
       j += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    uint64_t key = j < sbar ? skey[j] : 0ull;
    for (int m = 0; m < om.d; ++m) {
      uint64_t i;
      key = fastdivmod(key, om.div[m], i);
      const int mode = om.mode[m];
      const bool own = j < sbar && (int64_t)i >= row_lo[mode] && (int64_t)i < row_hi[mode];
      double *dst = zg + (j * (int64_t)om.d + m) * ld;
      for (int cc = lane; cc < ld; cc += 32) dst[cc] = own ? om.A[m][i * ld + cc] : 0.0;
    }
  }
}

// Heavy rows (cparls.cu plan_rows): every rank holds a partial RHS row for
// each.  Rank p copies its partials into block p of buf (P blocks of nh x ld);
// after an allgather every rank sums the P blocks in rank order -- int64 when
// the step's RHS is fixed point (exact), fp64 otherwise (fscale flag) -- the
// owner keeps the sum and the others zero their copies (M is zero outside the
// owned rows for the next RHS).
__global__ void k_heavy_gather(const double *__restrict__ M, const int64_t *__restrict__ rows, int64_t nh, int ld,
                               double *__restrict__ blk, const StepCtl *ctl) {
  CPARLS_GUARD(ctl);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nh * ld; t += (int64_t)gridDim.x * blockDim.x)
    blk[t] = M[rows[t / ld] * ld + t % ld];
}
__global__ void k_heavy_sum(double *__restrict__ M, const int64_t *__restrict__ rows,
                            const uint8_t *__restrict__ own, int64_t nh, int ld, const double *__restrict__ buf,
                            int P, const double *__restrict__ fscale, const StepCtl *ctl) {
  CPARLS_GUARD(ctl);
  const bool fixed = fscale && fscale[2 * kMaxRank] != 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nh * ld; t += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    if (fixed) {
      long long q = 0;
      for (int p = 0; p < P; ++p) q += __double_as_longlong(buf[(int64_t)p * nh * ld + t]);
      v = __longlong_as_double(q);
    } else {
      for (int p = 0; p < P; ++p) v += buf[(int64_t)p * nh * ld + t];
    }
    M[rows[t / ld] * ld + t % ld] = own[t / ld] ? v : 0.0;
  }
}

}  // namespace cparls
