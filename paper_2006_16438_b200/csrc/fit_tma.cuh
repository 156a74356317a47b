// fit_tma.cuh -- K10 exact fit (eq:fit P:867-875) with the factor-row gathers
// moved off the load/store pipe onto the bulk-copy (TMA) engine.
//
// k_fit_sub gathers one 224-byte A_{k*} row per nonzero (and the fiber's other
// rows per fiber) with 16-byte loads; ncu shows its L1 data pipe at ~73% of
// peak with the warps waiting on those loads (long_scoreboard), i.e. the
// gathers are issue/latency-bound in the LSU, not bound by DRAM (43%).  Here
// every lane issues `cp.async.bulk` copies of the rows its entry needs straight
// into a warp-private shared-memory stage, completing on an mbarrier; the warp
// computes on the previous stage while the next one is in flight, so two
// 32-entry batches of row copies per warp are outstanding and the LSU only
// sees the streamed key/out/value loads and 16-byte shared-memory reads.
//
// Measured on C4 (r = 25): 146 ms per fit against 69 ms for k_fit_sub -- the
// bulk-copy engine retires one 224-byte copy per ~18 SM cycles, so for
// row-sized gathers it is slower than the LSU path.  Kept opt-in
// (CPARLS_FIT_TMA=1) and parity-tested; k_fit_sub is the default.
//
// Same decomposition and arithmetic as k_fit_sub (fit.cuh): a warp takes a
// kFitChunk-entry chunk from the global counter; sub-warp s (8 lanes, 4
// columns per lane, ld <= 32) walks its own contiguous quarter; per fiber
// h = g * A_{m_1}(i_1,:) * ... with g = lambda * A_{slow}(i_slow,:) kept per
// sub-warp; acc_c += x_e * A_{k*}(out_e,c) * h_c; per chunk folded into a
// double-double.  The rare slow-mode row changes are loaded directly.
#pragma once
#include "common.cuh"
#include "fit.cuh"

namespace cparls {

constexpr int kFtSW = 8;                    // lanes per entry (4 columns each): ld <= 32
constexpr int kFtNS = 32 / kFtSW;           // sub-warps per warp
constexpr int kFtE = 32;                    // entries per warp batch (8 per sub-warp)
constexpr int kFtStages = 2;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16, both addresses 16-byte
// aligned), completing `bytes` of transaction count on bar
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Shared memory per warp: kFtStages x kFtE x DM rows of ld doubles (A_{k*}
// rows, then DM-1 fiber rows per entry).
template <int DM>
__host__ __device__ constexpr size_t fit_tma_warp_bytes(int ld) {
  return (size_t)kFtStages * kFtE * DM * ld * 8;
}

template <typename VT, int DM>
__global__ void __launch_bounds__(256, 1) k_fit_tma(const uint64_t *__restrict__ keys,
                                                   const int32_t *__restrict__ outidx,
                                                   const VT *__restrict__ vals, int64_t nnz, FitDecode fd,
                                                   const double *__restrict__ Ak, const double *__restrict__ lam,
                                                   int r, int ld, dd *__restrict__ part,
                                                   unsigned long long *__restrict__ work) {
  constexpr int SUB = kFitChunk / kFtNS;     // entries per sub-warp per chunk
  extern __shared__ __align__(128) unsigned char ft_smem[];
  __shared__ __align__(8) uint64_t bars[8][kFtStages];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int sl = lane & (kFtSW - 1), sbase = lane & ~(kFtSW - 1);
  const int c0 = 4 * sl;
  const bool colok = c0 < ld;
  const uint32_t RB = (uint32_t)ld * 8u;
  double *const stage0 = reinterpret_cast<double *>(ft_smem + fit_tma_warp_bytes<DM>(ld) * w);
  const size_t stage_d = (size_t)kFtE * DM * ld;   // doubles per stage
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kFtStages; ++s) mbar_init(&bars[w][s], 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t phase = 0;                        // bit s: parity of stage s's next completion
  double lam4[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) lam4[q] = (c0 + q < r) ? lam[c0 + q] : 0.0;
  const uint64_t pstream = l2_evict_first();
  const double *Aslow = fd.A[DM - 1];
  dd acc = {0.0, 0.0};
  while (true) {
    int64_t cb = 0;
    if (lane == 0) cb = (int64_t)atomicAdd(work, (unsigned long long)kFitChunk);
    cb = __shfl_sync(0xffffffffu, cb, 0);
    if (cb >= nnz) break;
    const int64_t s0 = cb + (int64_t)(lane / kFtSW) * SUB;
    const int64_t s1 = min(nnz, s0 + SUB);
    double h[4] = {0.0, 0.0, 0.0, 0.0};
    double g[4] = {0.0, 0.0, 0.0, 0.0};
    double cacc[4] = {0.0, 0.0, 0.0, 0.0};
    uint32_t cur_slow = 0xffffffffu;
    uint64_t ilast = ~0ull;                  // last key of the previously issued batch (this sub-warp)
    // stream data of the batch to issue next (loaded one batch ahead)
    uint64_t nkey = (s0 + sl < s1) ? ld_stream(keys + s0 + sl, pstream) : ~0ull;
    int32_t no = (s0 + sl < s1) ? ld_stream(outidx + s0 + sl, pstream) : 0;
    VT nx = (s0 + sl < s1) ? ld_stream(vals + s0 + sl, pstream) : VT(0);
    // the issued-but-not-computed batch: value, slow index, lead/valid masks
    double nxx = 0.0;
    uint32_t nslow = 0;
    unsigned nlm = 0, nvm = 0;
    constexpr int NB = SUB / kFtSW;          // batches per sub-warp per chunk
    for (int b = 0; b <= NB; ++b) {
      // batch b-1's data (issued last iteration) becomes the one to compute
      const double cx_ = nxx;
      const uint32_t cslow = nslow;
      const unsigned clm = nlm, cvm = nvm;
      // ---- issue batch b into stage b % kFtStages
      if (b < NB) {
        const int st = b % kFtStages;
        const int64_t e = s0 + (int64_t)b * kFtSW + sl;
        const bool valid = e < s1;
        const uint64_t key = nkey;
        const int32_t o = no;
        const double x = (double)nx;
        {
          const int64_t en = e + kFtSW;
          const bool vn = en < s1 && b + 1 < NB;
          nkey = vn ? ld_stream(keys + en, pstream) : ~0ull;
          no = vn ? ld_stream(outidx + en, pstream) : 0;
          nx = vn ? ld_stream(vals + en, pstream) : VT(0);
        }
        uint64_t prev = __shfl_up_sync(0xffffffffu, key, 1, kFtSW);
        if (sl == 0) prev = ilast;
        const bool lead = valid && key != prev;
        ilast = __shfl_sync(0xffffffffu, key, sbase + kFtSW - 1);
        uint32_t id[DM];
        {
          uint64_t t = key;
#pragma unroll
          for (int m = 0; m < DM; ++m) {
            uint64_t rem;
            t = divmod_fast(t, fd.n[m], fd.inv[m], rem, fd.fast);
            id[m] = (uint32_t)rem;
          }
        }
        nxx = x;
        nslow = id[DM - 1];
        nlm = __ballot_sync(0xffffffffu, lead);
        nvm = __ballot_sync(0xffffffffu, valid);
        // the stage's previous contents were read through the generic proxy
        fence_proxy_async_smem();
        double *rows = stage0 + (size_t)st * stage_d;
        const uint32_t bytes = valid ? RB * (lead ? (uint32_t)DM : 1u) : 0u;
        mbar_arrive_tx(&bars[w][st], bytes);
        if (valid) {
          bulk_g2s(rows + (size_t)lane * ld, Ak + (int64_t)o * ld, RB, &bars[w][st]);
          if (lead) {
#pragma unroll
            for (int m = 0; m + 1 < DM; ++m)
              bulk_g2s(rows + (size_t)(kFtE * (1 + m) + lane) * ld, fd.A[m] + (int64_t)id[m] * ld, RB,
                       &bars[w][st]);
          }
        }
      }
      // ---- compute batch b-1 from stage (b-1) % kFtStages
      if (b >= 1) {
        const int st = (b - 1) % kFtStages;
        mbar_wait(&bars[w][st], (phase >> st) & 1u);
        phase ^= 1u << st;
        const double *rows = stage0 + (size_t)st * stage_d;
        const unsigned lm = clm, vm = cvm;
#pragma unroll 2
        for (int u = 0; u < kFtSW; ++u) {
          const int src = sbase + u;
          const double xu = __shfl_sync(0xffffffffu, cx_, src);
          const uint32_t sid = __shfl_sync(0xffffffffu, cslow, src);
          if (!((vm >> src) & 1u)) continue;   // uniform within the sub-warp
          if ((lm >> src) & 1u) {
            if (sid != cur_slow) {             // rare: the slowest key mode moved
              cur_slow = sid;
              double2 q0 = make_double2(0.0, 0.0), q1 = make_double2(0.0, 0.0);
              if (colok) {
                const double2 *gr = reinterpret_cast<const double2 *>(Aslow + (int64_t)sid * ld + c0);
                q0 = __ldg(gr);
                q1 = __ldg(gr + 1);
              }
              g[0] = lam4[0] * q0.x; g[1] = lam4[1] * q0.y; g[2] = lam4[2] * q1.x; g[3] = lam4[3] * q1.y;
            }
            double hh[4] = {g[0], g[1], g[2], g[3]};
#pragma unroll
            for (int m = 0; m + 1 < DM; ++m) {
              if (colok) {
                const double *fr = rows + (size_t)(kFtE * (1 + m) + src) * ld + c0;
                const double2 f0 = *reinterpret_cast<const double2 *>(fr);
                const double2 f1 = *reinterpret_cast<const double2 *>(fr + 2);
                hh[0] *= f0.x; hh[1] *= f0.y; hh[2] *= f1.x; hh[3] *= f1.y;
              }
            }
            h[0] = hh[0]; h[1] = hh[1]; h[2] = hh[2]; h[3] = hh[3];
          }
          if (colok) {
            const double *ar = rows + (size_t)src * ld + c0;
            const double2 a0 = *reinterpret_cast<const double2 *>(ar);
            const double2 a1 = *reinterpret_cast<const double2 *>(ar + 2);
            cacc[0] = fma(xu * a0.x, h[0], cacc[0]);
            cacc[1] = fma(xu * a0.y, h[1], cacc[1]);
            cacc[2] = fma(xu * a1.x, h[2], cacc[2]);
            cacc[3] = fma(xu * a1.y, h[3], cacc[3]);
          }
        }
        __syncwarp();
      }
    }
    acc = dd_add_d(acc, (cacc[0] + cacc[1]) + (cacc[2] + cacc[3]));
  }
  acc = warp_sum_dd(acc);
  __shared__ dd ws[8];
  if (lane == 0) ws[w] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    dd tt = {0.0, 0.0};
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) tt = dd_add(tt, ws[i]);
    part[blockIdx.x] = tt;
  }
}

}  // namespace cparls
