// als.cuh -- N2: the exact CP-ALS baseline on the same sorted
// copies: M = X_(k) (A_{m_d} (.) ... (.) A_{m_1}) (full sparse
// MTTKRP), V = *_{m != k} A_m^T A_m, B = M V^+.
//
// Every copy's slowest key mode is a different mode (copy_order: copy c's
// slowest is mode (c+1) mod D), so the MTTKRP of mode k streams the copy c with
// slowest digit k: its nonzeros come grouped by the output row i_k, and a
// sub-warp accumulates the row in registers (4 columns per lane, as in
// k_fit_sub) -- per nonzero one A_c(out, :) row, per fiber the rows of the
// other key modes -- and writes it once.  Only the first and last row of each
// sub-warp's contiguous range can be shared with a neighbour; those two are
// added with fp64 atomics into the zeroed M, every other row is a plain store.
#pragma once
#include "common.cuh"
#include "fit.cuh"

namespace cparls {

template <typename VT, int SW, int DM, int U>
__global__ void __launch_bounds__(kFitThreads, 2) k_mttkrp(const uint64_t *__restrict__ keys,
                                                         const int32_t *__restrict__ outidx,
                                                         const VT *__restrict__ vals, int64_t nnz, FitDecode fd,
                                                         const double *__restrict__ Ac, int ld,
                                                         double *__restrict__ M, unsigned long long *__restrict__ work) {
  static_assert(SW >= 2 && SW <= 32 && (SW & (SW - 1)) == 0, "SW power of two");
  constexpr int NS = 32 / SW;
  constexpr int SUB = kFitChunk / NS;
  const int lane = threadIdx.x & 31;
  const int sl = lane & (SW - 1);
  const int sbase = lane & ~(SW - 1);
  const int c0 = 4 * sl;
  const bool colok = c0 < ld;
  const uint64_t pstream = l2_evict_first();
  while (true) {
    int64_t cb = 0;
    if (lane == 0) cb = (int64_t)atomicAdd(work, (unsigned long long)kFitChunk);
    cb = __shfl_sync(0xffffffffu, cb, 0);
    if (cb >= nnz) break;
    const int64_t s0 = cb + (int64_t)(lane / SW) * SUB;
    const int64_t s1 = min(nnz, s0 + SUB);
    double h[4] = {1.0, 1.0, 1.0, 1.0};
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    int64_t cur = -1;       // output row being accumulated
    int nflushed = 0;       // rows of this range already written
    uint64_t last_key = ~0ull;
    auto flush = [&](bool shared_row) {
      if (cur < 0 || !colok) return;
      double *dst = M + cur * ld + c0;
      if (shared_row) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (acc[q] != 0.0) atomicAdd(dst + q, acc[q]);
      } else {
        reinterpret_cast<double2 *>(dst)[0] = make_double2(acc[0], acc[1]);
        reinterpret_cast<double2 *>(dst)[1] = make_double2(acc[2], acc[3]);
      }
    };
    uint64_t nkey = (s0 + sl < s1) ? ld_stream(keys + s0 + sl, pstream) : ~0ull;
    int32_t no = (s0 + sl < s1) ? ld_stream(outidx + s0 + sl, pstream) : 0;
    VT nx = (s0 + sl < s1) ? ld_stream(vals + s0 + sl, pstream) : VT(0);
    for (int64_t b0 = 0; b0 < SUB; b0 += SW) {
      const int64_t e = s0 + b0 + sl;
      const bool valid = e < s1;
      const uint64_t key = nkey;
      const int32_t o = no;
      const double x = (double)nx;
      {
        const int64_t en = e + SW;
        const bool vn = en < s1 && b0 + SW < SUB;
        nkey = vn ? ld_stream(keys + en, pstream) : ~0ull;
        no = vn ? ld_stream(outidx + en, pstream) : 0;
        nx = vn ? ld_stream(vals + en, pstream) : VT(0);
      }
      uint64_t prev = __shfl_up_sync(0xffffffffu, key, 1, SW);
      if (sl == 0) prev = last_key;
      const bool lead = valid && key != prev;
      const unsigned lm = __ballot_sync(0xffffffffu, lead);
      const unsigned vm = __ballot_sync(0xffffffffu, valid);
      if (vm == 0u) break;
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
      last_key = __shfl_sync(0xffffffffu, key, sbase + SW - 1);
#pragma unroll
      for (int t0 = 0; t0 < SW; t0 += U) {
        double av[U][4];
        double hv[U][DM > 1 ? DM - 1 : 1][4];
        bool lead_[U], ok_[U];
        uint32_t tid[U];
        double xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int src = sbase + t0 + u;
          ok_[u] = (vm >> src) & 1u;
          lead_[u] = (lm >> src) & 1u;
          const int ou = __shfl_sync(0xffffffffu, o, src);
          xv[u] = __shfl_sync(0xffffffffu, x, src);
          const double2 *row = reinterpret_cast<const double2 *>(Ac + (int64_t)ou * ld + c0);
          double2 p0 = make_double2(0.0, 0.0), p1 = make_double2(0.0, 0.0);
          if (ok_[u] && colok) { p0 = __ldg(row); p1 = __ldg(row + 1); }
          av[u][0] = p0.x; av[u][1] = p0.y; av[u][2] = p1.x; av[u][3] = p1.y;
#pragma unroll
          for (int m = 0; m + 1 < DM; ++m) {
            const uint32_t im = __shfl_sync(0xffffffffu, id[m], src);
            const double2 *hr = reinterpret_cast<const double2 *>(fd.A[m] + (int64_t)im * ld + c0);
            double2 q0 = make_double2(0.0, 0.0), q1 = make_double2(0.0, 0.0);
            if (lead_[u] && colok) { q0 = __ldg(hr); q1 = __ldg(hr + 1); }
            hv[u][m][0] = q0.x; hv[u][m][1] = q0.y; hv[u][m][2] = q1.x; hv[u][m][3] = q1.y;
          }
          tid[u] = __shfl_sync(0xffffffffu, id[DM - 1], src);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (lead_[u]) {
            if ((int64_t)tid[u] != cur) {   // a new output row: write the finished one
              flush(nflushed == 0);
              nflushed += cur >= 0;
              cur = tid[u];
#pragma unroll
              for (int q = 0; q < 4; ++q) acc[q] = 0.0;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              double hh = 1.0;
#pragma unroll
              for (int m = 0; m + 1 < DM; ++m) hh *= hv[u][m][q];
              h[q] = hh;
            }
          }
          if (ok_[u]) {
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = fma(xv[u] * h[q], av[u][q], acc[q]);
          }
        }
      }
    }
    flush(true);   // the range's last row may continue in the next range
  }
}

// V = *_{m != k} G_m (Hadamard of the factor Grams)
struct GramList {
  int D, k;
  const double *GA[kMaxModes];
};
__global__ void k_hadamard_grams(int r, GramList gl, double *__restrict__ V) {
  for (int i = threadIdx.x; i < r * r; i += blockDim.x) {
    double v = 1.0;
    for (int m = 0; m < gl.D; ++m)
      if (m != gl.k) v *= gl.GA[m][i];
    V[i] = v;
  }
}

}  // namespace cparls
