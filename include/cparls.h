/*
 * cparls.h -- C ABI of the B200-native CP-ARLS-LEV hot path
 * (Larsen & Kolda, "Practical Leverage-Based Sampling for Low-Rank Tensor
 * Decomposition", arXiv 2006.16438).  "P:L" cites /root/reference/PAPER.md
 * line L; "AMB-n" cites the reading listed in DESIGN.md.
 *
 * Library: paper_2006_16438_b200/libcparls.so (sm_100a).  Plain C types only.
 *
 * Conventions (apply to every call):
 *  - Status: every call returns cparls_status; nothing aborts or throws across
 *    the ABI.  cparls_last_error(ctx) returns the message of the last failure.
 *    CPARLS_EINVAL / ERANGE / ESAMPLE / ENUMERIC / ESTATE leave the context
 *    usable; CPARLS_ECUDA / ENCCL poison it (only cparls_destroy is valid).
 *  - Ownership: the context owns ALL device memory it allocates (the per-mode
 *    sorted nonzero copies, factors, sampler state).  Input buffers of
 *    cparls_create / cparls_set_factor may be host or device pointers (detected
 *    with cudaPointerGetAttributes) and may be freed on return.  Output
 *    buffers are caller-owned HOST pointers unless stated otherwise.
 *  - Stream: all device work is ordered on opts.stream (a cudaStream_t, e.g.
 *    torch.cuda.current_stream().cuda_stream); NULL = legacy default stream.
 *    Within a call, small independent kernels may run on a context-owned side
 *    stream that forks from and joins back into opts.stream via events.
 *  - Determinism: with the default fixed-point RHS (rhs_path 0/1) repeated
 *    runs with the same inputs, seed and steps give bit-identical factors.
 *  - Modes are 0-based; "other modes" of mode k are m_1 < ... < m_d (d = D-1).
 *  - Row-major factors: A_k is n_k x r, element (i,c) at A[i*r + c].
 *  - Multi-GPU is SPMD (world_size > 1): every rank passes its own chunk of the
 *    COO and calls the same sequence with the same seed; samples are
 *    replicated, B rows are owned by the rank holding their nonzeros.
 */
#ifndef CPARLS_H
#define CPARLS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cparls_ctx cparls_ctx;   /* opaque */
typedef struct cparls_comm cparls_comm; /* opaque communicator (NCCL or in-process group) */

typedef enum {
  CPARLS_OK = 0,
  CPARLS_EINVAL = 1,   /* bad argument (mode out of range, r > 64, nnz < 0, ...)   */
  CPARLS_EOOM = 2,     /* device allocation failed                                  */
  CPARLS_ECUDA = 3,    /* CUDA runtime error (context poisoned)                     */
  CPARLS_ENCCL = 4,    /* NCCL error (context poisoned)                             */
  CPARLS_ENUMERIC = 5, /* non-finite factor / solve failure after fallback          */
  CPARLS_ESAMPLE = 6,  /* DIDX candidate cap or rejection-attempt cap exceeded      */
  CPARLS_ERANGE = 7,   /* key width: prod_{m!=k} n_m >= 2^63, or coord >= n_k       */
  CPARLS_ESTATE = 8    /* call order violated (e.g. solve_mode without sample)      */
} cparls_status;

/* Options of cparls_create.  ABI versioning: struct_size is the caller's
 * sizeof(cparls_opts); the library reads only the fields that fit in it and
 * takes the documented default (0 / NULL) for every later field, so fields
 * are only ever appended.  cparls_opts_init fills the defaults and
 * struct_size.  struct_size 0 or smaller than the first four fields: EINVAL. */
typedef struct {
  uint32_t struct_size;    /* sizeof(cparls_opts) as compiled by the caller              */
  int32_t rank;            /* r, 1 <= r <= 64                                         */
  double tau;              /* deterministic threshold tau: > 0 literal; 1 =
                              pure random; < 0 = 1/s at sample time  */
  int32_t value_dtype;     /* vals of cparls_create: 0 fp64, 1 fp32 (stored as given;
                              accumulation is always fp64)                           */
  int32_t index_dtype;     /* coords of cparls_create: 0 int32, 1 int64              */
  void *stream;            /* cudaStream_t                                            */
  int32_t world_size;      /* 1 = single GPU; > 1 = row-sharded SPMD     */
  int32_t world_rank;      /* this shard, 0 <= world_rank < world_size                */
  cparls_comm *comm;       /* required when world_size > 1 (cparls_comm_create_*)      */
  int64_t didx_cap;        /* max DIDX list length per level (0 -> default 1<<22)     */
  int64_t attempt_cap;     /* max SIDX attempts (0 -> 1024*s_rnd + 65536, AMB-7)      */
  int32_t rhs_path;        /* sampled RHS kernels: 0 auto (= 1), 1 fixed-point int64
                              reductions into M (rhs.cuh, AMB-35: deterministic,
                              per-column scale 2^e_c from a bound on |M|), 3 fp64
                              reductions into M (order of the additions not fixed).
                              Same math; B = M G^+ follows.  2 (round 1's bucketed
                              transposition, measured slower) and other values:
                              EINVAL.                                               */
  int64_t fit_samples;     /* s_fit > 0: draw the stratified fit sample at create
                              (sec:estimating-fit, AMB-32); 0 = none.
                              Single GPU only (EINVAL with world_size > 1).          */
  double fit_alpha;        /* nonzero fraction alpha of the sample (<= 0 -> 0.5)     */
  uint64_t fit_seed;       /* Philox key of the fit sample                           */
  int64_t sidx_window;     /* > 0: at most this many SIDX attempts are drawn per
                              window (AMB-8: the result does not depend on it; small
                              values exercise the multi-window continuation);
                              0 = sized from the expected attempt count             */
  int32_t sample_sort;     /* 1: order the combined sample by key before the solve
                              (the fibers are then walked in key order; same
                              sample set and weights); 0 = deterministic device
                              order (DIDX list, then random rows by first draw)     */
  int32_t fit_mode;        /* mode whose sorted copy the exact fit streams: -1 or any
                              value outside [0, D) = automatic (fewest gathers); the
                              fit does not depend on it beyond rounding            */
  int32_t rhs_hot_rows;    /* fixed-point RHS: rows of a mode whose entries are summed
                              per CTA in shared memory before reaching M (the rows of
                              largest degree; rhs.cuh).  -1 = automatic (as many as
                              fit in shared memory, used for a mode when they hold
                              at least 70% of its nonzeros); 0 = none; > 0 = at most
                              this many, always used.  M is bit-identical either way
                              (int64 sums).  Ignored for r > 32 and rhs_path 3.     */
} cparls_opts;

/* Fill *opts with the defaults (tau = -1, rank = 1, world_size = 1, fit_mode = -1,
 * rhs_hot_rows = -1, everything else 0/NULL) and struct_size = sizeof(cparls_opts). */
void cparls_opts_init(cparls_opts *opts);

typedef struct {
  int64_t s_det;     /* |DetSet|                                          */
  int64_t s_rnd;     /* s - s_det                                             */
  int64_t s_bar;     /* rows after combining                                  */
  int64_t attempts;  /* SIDX attempts consumed (index of last accepted + 1)           */
  double p_det;      /* sum_{i in DetSet} p_i                                 */
  int32_t skipped_random; /* AMB-7: random phase skipped (every drawable row is det) */
} cparls_sample_info;

typedef struct {
  int64_t matched_nnz;  /* nonzeros in the sampled fibers (m_k)                      */
  int64_t touched_rows; /* output rows receiving at least one matched nonzero         */
  int32_t rank_used;    /* rank of the sampled Gram kept by the solve                 */
  int32_t chol_fallback;/* 1 if Cholesky failed and the eigen pseudo-inverse was used */
} cparls_solve_info;

/* Per-phase device times (ms, accumulated since create or the last reset) and
 * counters of the algorithmic bytes each phase touched (DESIGN.md byte model).
 * ABI versioning: cparls_get_stats copies min(bytes, sizeof(cparls_stats)) and
 * sets struct_size to the library's sizeof(cparls_stats); fields are only
 * ever appended. */
typedef struct {
  uint32_t struct_size;      /* the library's sizeof(cparls_stats)                 */
  uint32_t reserved0;
  double ms_leverage, ms_sample, ms_gram, ms_lookup, ms_rhs, ms_solve, ms_fit;
  double bytes_leverage, bytes_sample, bytes_gram, bytes_lookup, bytes_rhs, bytes_solve, bytes_fit;
  int64_t mode_steps, fits, kernel_launches;
  int64_t last_matched_nnz, last_s_bar, last_attempts;
  int64_t touched_rows[8];   /* rows of A_k nonzero after its last solve, per mode */
  /* Device time (ms) and launch count of the hot kernels alone, from CUDA
   * events recorded around every launch on the context's stream (always on,
   * no host synchronisation; resolved when the stats are read or at the
   * context's next synchronisation).
   * Index: 0 = sampled RHS (k_rhs / k_rhs_agg), 1 = exact fit (k_fit_sub /
   * k_fit_thread), 2 = solve rows (k_solve_dmma / k_solve_rows_t),
   * 3 = leverage rows (k_lev_rows_w). */
  double kernel_ms[4];
  int64_t kernel_launches_by_id[4];
  int64_t sum_matched_nnz;   /* sum of m_k over the solves since the last reset   */
  int64_t host_syncs;        /* cudaStreamSynchronize calls made by the library   */
  double bytes_comm;         /* bytes this rank contributed to collectives (world_size > 1) */
  double create_ms[4];       /* cparls_create wall time: [0] setup + input copy to the
                                device, [1] per-mode sorted copies, [2] duplicates,
                                fiber counts, fit sample, [3] factors + leverage       */
  int32_t rhs_hot_rows[8];   /* per mode: rows summed in shared memory by the RHS
                                (cparls_opts.rhs_hot_rows; 0 = none)                */
  double rhs_hot_share[8];   /* per mode: fraction of this rank's nonzeros in them  */
  double build_ms[4];        /* create_ms[1] split: [0] cudaMalloc/cudaFree, [1] radix
                                sorts, [2] key/payload kernels + directory, [3] hot rows */
} cparls_stats;

/* Build the context: validates sizes (ERANGE if some prod_{m!=k} n_m >= 2^63 or
 * a coordinate is out of range), copies the COO to the device, builds for every
 * mode k the sorted-key copy of the nonzeros (per-mode linearized
 * "other-mode" indices; key = eq:bijection P:220-222, AMB-1), ||X||^2, and
 * initial factors U[0,1) from init_seed (AMB-21) with their leverage scores.
 * coords: nnz_local x nmodes row-major, 0-based; vals: nnz_local values. */
cparls_status cparls_create(cparls_ctx **out, int32_t nmodes, const int64_t *dims,
                            int64_t nnz_local, const void *coords, const void *vals,
                            const cparls_opts *opts, uint64_t init_seed);
cparls_status cparls_destroy(cparls_ctx *ctx);

/* Replace factor k (n_k x r row-major fp64, host or device) and recompute its
 * leverage scores / CDF.  lambda is reset to ones. */
cparls_status cparls_set_factor(cparls_ctx *ctx, int32_t mode, const double *A);
/* Copy factor k (n_k x r row-major fp64) and the model weights lambda (r, may
 * be NULL) into caller memory: device, pinned host (rows packed on the device,
 * then contiguous DMA into A) or pageable host (through a pinned double buffer
 * the context owns).  Synchronous. */
cparls_status cparls_get_factor(cparls_ctx *ctx, int32_t mode, double *A, double *lambda);

/* Leverage scores of A_k (Def. leverages_scores P:319-331 as l_i =
 * a_i (A^T A)^+ a_i^T), refreshing p~_k = l/rank (AMB-11) and the integer CDF
 * (AMB-9).  scores: n_k host doubles or NULL.  rank_out may be NULL. */
cparls_status cparls_leverage(cparls_ctx *ctx, int32_t mode, double *scores, int32_t *rank_out);
/* Copy p~_k (n_k host doubles); set p~_k from given bits (lockstep parity). */
cparls_status cparls_get_ptilde(cparls_ctx *ctx, int32_t mode, double *pt);
cparls_status cparls_set_ptilde(cparls_ctx *ctx, int32_t mode, const double *pt);

/* SkrpLev (Alg. 1) for solving mode k: DIDX (exact {p_i > tau},
 * P:688-735) -> SIDX (Alg. 2, Philox4x32-10 key=seed, counter=(attempt, step,
 * lane), AMB-8/10) -> CIDX (combine repeats, w^2 = c(1-p_det)/(s_rnd p),
 * P:526-542, AMB-3).  tau is opts.tau unless cparls_set_tau was called. */
cparls_status cparls_sample(cparls_ctx *ctx, int32_t mode, int64_t s, uint64_t seed,
                            uint64_t step, cparls_sample_info *info);
cparls_status cparls_set_tau(cparls_ctx *ctx, double tau);
/* Copy the current sample in canonical order: deterministic block (key asc)
 * then random block (key asc).  Returns s_bar in *n_out; copies min(cap,s_bar). */
cparls_status cparls_get_sample(cparls_ctx *ctx, int64_t cap, uint64_t *keys, int32_t *counts,
                                double *w2, double *p, uint8_t *is_det, int64_t *n_out);
/* Sampled fibers of the current sample (TnsrSamp) in canonical
 * sample order: len[j] per sample, then the matched (out, value) pairs, each
 * fiber sorted by out.  Copies min(cap, m_k) pairs; *m_out = m_k. */
cparls_status cparls_get_fibers(cparls_ctx *ctx, int64_t cap, int64_t *len, int64_t *out,
                                double *val, int64_t *m_out);

/* One sketched mode update (Alg. 3): KrpSamp + sampled Gram,
 * TnsrSamp lookup, RHS M = Xs^T diag(w^2) Z_S (AMB-14), r x r Cholesky solve
 * with eigen pseudo-inverse fallback (AMB-12), column normalization (lambda,
 * AMB-13), leverage refresh.  Requires a current sample of this mode (ESTATE). */
cparls_status cparls_solve_mode(cparls_ctx *ctx, int32_t mode, cparls_solve_info *info);
/* Debug/parity: sampled Gram G (r*r) and unnormalized solution B (n_k*r) of the
 * last solve (either may be NULL). */
cparls_status cparls_get_last_solve(cparls_ctx *ctx, double *G, double *B);

/* Exact fit 1 - ||X - M||/||X|| (eq:fit P:871-875) via ||X||^2 - 2<X,M> +
 * ||M||^2 (AMB-16) with the model [[lambda; A_1..A_D]] (AMB-31). */
cparls_status cparls_fit(cparls_ctx *ctx, double *fit);

/* Alg. 3: iters outer iterations, each cycling all modes with
 * step = (iter0 + t)*D + k; fit after every fit_every-th iteration (0 = never).
 * fit_trace: iters host doubles (NaN where no fit) or NULL.  iter0 lets a run
 * be resumed exactly (counter-based RNG). */
cparls_status cparls_run(cparls_ctx *ctx, int32_t iters, int64_t s, uint64_t seed, int32_t iter0,
                         int32_t fit_every, double *fit_trace);

/* Estimated fit: 1 - sqrt(F^)/||X|| over the frozen sample drawn
 * at create (opts.fit_samples > 0, else ESTATE).  Fhat may be NULL. */
cparls_status cparls_fit_estimate(cparls_ctx *ctx, double *fit, double *Fhat);
/* The frozen fit sample, nonzero stratum first: coords (cap x D, int64),
 * x (cap), is_nz (cap); *n = total size.  NULL arrays / cap 0 query n. */
cparls_status cparls_get_fit_sample(cparls_ctx *ctx, int64_t cap, int64_t *coords, double *x, uint8_t *is_nz,
                                    int64_t *n);
/* The model's value m_i at every fit-sample position (n = sample size host
 * doubles), the same arithmetic as the estimate (diagnostics). */
cparls_status cparls_fit_sample_model(cparls_ctx *ctx, double *m);
/* Alg. 3 with its stopping rule (AMB-33): epochs of eta outer
 * iterations (steps (e*eta + t)*D + k), a fit after each epoch (fit_kind 0
 * exact, 1 estimated), stop after pi consecutive epochs without
 * fit > best + tol, or after max_epochs.  trace: max_epochs host doubles (fit
 * per epoch); *epochs = epochs run. */
cparls_status cparls_run_until(cparls_ctx *ctx, int64_t s, uint64_t seed, int32_t eta, int32_t pi, double tol,
                               int32_t max_epochs, int32_t fit_kind, double *trace, int32_t *epochs);

/* Randomized range finder initialization (SURVEY 8(f) N4, sec:enron
 * P:1668-1701, AMB-34): every factor A_k = X_(k)(:, S) Omega, S = s_init
 * nonempty fibers drawn uniformly with replacement (ranked by canonical key),
 * Omega standard normal (Box-Muller on Philox, key = seed); lambda = 1, p~
 * refreshed.  Single GPU. */
cparls_status cparls_init_rrf(cparls_ctx *ctx, int64_t s_init, uint64_t seed);

/* Exact CP-ALS baseline on the same sorted copies:
 * one mode update = full sparse MTTKRP, V = *_{m != k} A_m^T A_m, B = M V^+
 * (AMB-12 pseudo-inverse), normalize (lambda), leverage refresh.  Single GPU,
 * D <= 4.  cparls_run_als: iters outer iterations over all modes, exact fit
 * every fit_every (trace as cparls_run). */
cparls_status cparls_als_update(cparls_ctx *ctx, int32_t mode);
cparls_status cparls_run_als(cparls_ctx *ctx, int32_t iters, int32_t fit_every, double *fit_trace);

/* ---- multi-GPU (SURVEY 8(e), P:1797-1801 sketches the distributed variant) ----
 * Row sharding: for every mode k the rows of B (and the nonzeros whose mode-k
 * index is one of them) are split into world_size contiguous blocks balanced
 * by nonzero count (cparls_plan_rows).  Sampling is replicated (same p~ bits,
 * seed, step on every rank: no communication); per mode step the ranks
 * allreduce the r x r Gram of their B rows and allgather the B rows; the fit
 * allreduces one scalar.  cparls_create routes each rank's COO chunk to the
 * row owners with one all-to-all per mode. */
/* NCCL: rank 0 creates the id, the caller broadcasts the 128 bytes (e.g. with
 * torch.distributed), every rank then creates its communicator. */
cparls_status cparls_comm_nccl_unique_id(uint8_t id[128]);
cparls_status cparls_comm_create_nccl(int32_t world_size, int32_t rank, const uint8_t id[128], cparls_comm **out);
/* In-process group of world_size shards on the current GPU, driven by
 * world_size host threads (one cparls_ctx each, opts.world_rank = its shard):
 * the shard simulator for single-GPU testing of the sharded path.  One object
 * is shared by all shards. */
cparls_status cparls_comm_create_local(int32_t world_size, cparls_comm **out);
cparls_status cparls_comm_destroy(cparls_comm *comm);
/* Host-only: row blocks of a mode from its global per-row nonzero counts deg[n]
 * (bound[p]..bound[p+1]-1 owned by rank p; bound has world_size+1 entries).
 * A heavy row (deg > total/world_size: a Zipf head row) has its nonzeros
 * spread over all ranks (by a hash of the other coordinates) and weighs
 * ceil(deg/world_size); its partial RHS rows are summed over the ranks every
 * mode step and the rank whose block contains it solves it.  heavy (n bytes,
 * may be NULL) receives 1 for the heavy rows. */
cparls_status cparls_plan_rows(int64_t n, const uint64_t *deg, int32_t world_size, int64_t *bound,
                               uint8_t *heavy);
/* Host-only: the rank cparls_create routes each nonzero to in the sharded
 * build of mode `mode` (coords: nnz x nmodes int64; bound/heavy from
 * cparls_plan_rows, heavy may be NULL): the owner of its row, or for a heavy
 * row a hash of its other coordinates.  rank_out: nnz int32. */
cparls_status cparls_route_nonzeros(int32_t nmodes, int32_t mode, int64_t nnz, const int64_t *coords,
                                    int32_t world_size, const int64_t *bound, const uint8_t *heavy, int32_t *rank_out);
/* Rows of mode `mode` owned by this rank. */
cparls_status cparls_owned_rows(const cparls_ctx *ctx, int32_t mode, int64_t *lo, int64_t *hi);

/* Copy the statistics into stats (min(bytes, sizeof(cparls_stats)) bytes, see
 * cparls_stats).  bytes < 8: EINVAL. */
cparls_status cparls_get_stats(cparls_ctx *ctx, void *stats, int64_t bytes);
cparls_status cparls_reset_stats(cparls_ctx *ctx);
/* Record per-phase CUDA events (adds small overhead). 0 off, 1 on. */
cparls_status cparls_set_profiling(cparls_ctx *ctx, int32_t on);
const char *cparls_last_error(const cparls_ctx *ctx);
/* Library/device description string (static). */
const char *cparls_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CPARLS_H */
