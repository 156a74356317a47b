/*
 * cparls_oracle.h -- plain, slow, single-threaded fp64 CPU oracle of the
 * CP-ARLS-LEV hot path (arXiv 2006.16438).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2006_16438_b200/csrc, include/cparls.h).
 *
 * Citations: "P:L" = /root/reference/PAPER.md line L; "AMB-n" = the reading
 * listed in DESIGN.md "Readings of the paper".
 */
#ifndef CPARLS_ORACLE_H
#define CPARLS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- primitives (each pinned independently by tests/test_oracle_*.py) ---- */

/* Philox4x32-10 (AMB-10).  out[0..3] from counter c[0..3], key k[0..1]. */
void or_philox4x32_10(const uint32_t c[4], const uint32_t k[2], uint32_t out[4]);

/* eq:bijection (AMB-1) over the modes != k, ascending, 0-based:
 * key = sum_j idx[m_j] * prod_{l<j} dims[m_l].  idx has D entries; idx[k] ignored. */
uint64_t or_key(int D, const int64_t *dims, int k, const int64_t *idx);
void or_decode(int D, const int64_t *dims, int k, uint64_t key, int64_t *idx);

/* Jacobi eigendecomposition of a symmetric r x r matrix (row-major).
 * On return w[j] are eigenvalues, V(:,j) (column j of row-major V) vectors. */
void or_jacobi_eig(int r, const double *G, double *w, double *V);

/* Leverage scores (Def. leverages_scores) in the parity form
 * l_i = a_i G^+ a_i^T, G = A^T A, pseudo-inverse keeping eigenvalues
 * mu_j > r*eps*mu_max (AMB-11).  A is n x r row-major (ld = r).
 * Returns rank (number of kept eigenvalues). */
int or_leverage(int64_t n, int r, const double *A, double *ell);

/* Integer CDF (AMB-9): q_i = nearbyint(ldexp(pt_i, 62)), C = inclusive scan. */
void or_cdf(int64_t n, const double *pt, uint64_t *C);
/* Inverse-CDF draw (AMB-9): t = (R*W)>>64, first i with C[i] > t. */
int64_t or_draw(int64_t n, const uint64_t *C, uint64_t R);

/* ---- context: tensor + model + sampler state (mirrors include/cparls.h) ---- */
typedef struct or_ctx or_ctx;

typedef struct {
  int64_t s_det, s_rnd, s_bar, attempts;
  double p_det;
  int32_t skipped_random; /* AMB-7 flag */
} or_sample_info;

typedef struct {
  int64_t matched_nnz, touched_rows;
  int32_t rank_used, chol_fallback;
} or_solve_info;

/* coords: nnz x D row-major int64 (0-based); vals fp64.  Copies everything. */
or_ctx *or_create(int D, const int64_t *dims, int64_t nnz, const int64_t *coords,
                  const double *vals, int r);
void or_destroy(or_ctx *c);
/* Set factor k (n_k x r row-major); recomputes its leverage / p~ / CDF. */
int or_set_factor(or_ctx *c, int k, const double *A);
void or_get_factor(or_ctx *c, int k, double *A, double *lambda /* r or NULL */);
/* Lockstep hook: overwrite p~_k (and its CDF) with externally given bits. */
void or_set_ptilde(or_ctx *c, int k, const double *pt);
void or_get_ptilde(or_ctx *c, int k, double *pt);
/* Leverage of the current A_k into ell (n_k); returns rank; refreshes p~_k. */
int or_leverage_mode(or_ctx *c, int k, double *ell);

/* SkrpLev (Alg. 1) for mode k: DIDX -> SIDX -> CIDX.
 * tau < 0 means 1/s.  Returns 0 ok, 6 sampling failure (AMB-7 cap). */
int or_sample(or_ctx *c, int k, int64_t s, double tau, uint64_t seed, uint64_t step,
              or_sample_info *info);
/* Copy the current sample (det block key-asc, then random block key-asc). */
int64_t or_get_sample(or_ctx *c, int64_t cap, uint64_t *keys, int32_t *counts,
                      double *w2, double *p, uint8_t *is_det);
/* Sampled fibers of the current sample: per sample j the fiber length
 * len[j]; (out, value) of all matched nonzeros concatenated in sample order,
 * each fiber sorted by out.  Returns total matched (cap-limited copy). */
int64_t or_get_fibers(or_ctx *c, int64_t cap, int64_t *len, int64_t *out, double *val);

/* One sketched mode update: KrpSamp, TnsrSamp, solve, normalize,
 * leverage refresh.  Also stores G (r x r) and M (n_k x r) for inspection. */
int or_solve_mode(or_ctx *c, int k, or_solve_info *info);
void or_get_last_solve(or_ctx *c, double *G /* r*r or NULL */, double *M /* n_k*r or NULL */,
                       double *B /* n_k*r unnormalized or NULL */);

/* Exact fit (eq:fit) via the three-term identity (AMB-16). */
double or_fit(or_ctx *c);
/* Dense brute-force fit over all prod(n) cells (tiny tensors only). */
double or_fit_dense(or_ctx *c);

/* Exact CP-ALS update of mode k: B = MTTKRP * V^+, normalized. */
int or_als_update(or_ctx *c, int k);

/* Alg. 3 loop with step = t*D + k (AMB-10, AMB-17). */
int or_run(or_ctx *c, int iters, int64_t s, double tau, uint64_t seed, int fit_every,
           double *fit_trace);

/* Estimated fit (sec:estimating-fit; AMB-32): draw and freeze the
 * stratified sample (ceil(alpha s_fit) nonzeros with replacement in input COO
 * order, floor((1-alpha) s_fit) zero cells by rejection), Philox key = seed.
 * Returns 0, 1 (bad argument) or 6 (rejection attempt cap). */
int or_fit_sample(or_ctx *c, int64_t s_fit, double alpha, uint64_t seed, int64_t *n_nz, int64_t *n_z);
/* Copy the frozen sample (nonzero stratum first): coords (n x D), x, is_nz. */
int64_t or_get_fit_sample(or_ctx *c, int64_t cap, int64_t *coords, double *x, uint8_t *is_nz);
/* 1 - sqrt(F^)/||X||, F^ = sum_i phi_i (m_i - x_i)^2; *Fhat optional. */
double or_fit_estimate(or_ctx *c, double *Fhat);
/* Alg. 3 with its stopping rule (AMB-33): fit_kind 0 exact, 1 estimated;
 * trace per epoch; *epochs = epochs run. */
int or_run_until(or_ctx *c, int64_t s, double tau, uint64_t seed, int eta, int pi, double tol, int max_epochs,
                 int fit_kind, double *trace, int *epochs);

/* Randomized range finder initialization (sec:enron; AMB-34):
 * A_k = X_(k)(:, S) Omega for every mode, S = s_init fibers drawn uniformly
 * with replacement from the nonempty fibers (ascending canonical key),
 * Omega standard normal (Box-Muller on Philox).  lambda = 1. */
int or_init_rrf(or_ctx *c, int64_t s_init, uint64_t seed);
double or_rrf_omega(uint64_t seed, int k, uint64_t j, int c);
int64_t or_rrf_fiber(uint64_t seed, int k, uint64_t j, int64_t nfib);

/* Standalone DIDX on d given p~ vectors (for pins): writes up to cap keys
 * (ascending) and p; returns s_det (full count) or -1 on cap overflow. */
int64_t or_didx(int d, const int64_t *n, const double *const *pt, double tau, int64_t cap,
                uint64_t *keys, double *p, double *p_det);
int64_t or_didx_brute(int d, const int64_t *n, const double *const *pt, double tau, int64_t cap,
                      uint64_t *keys, double *p, double *p_det);

#ifdef __cplusplus
}
#endif
#endif
