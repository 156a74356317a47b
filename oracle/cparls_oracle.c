/*
 * cparls_oracle.c -- plain CPU oracle of the CP-ARLS-LEV hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see cparls_oracle.h).  Single-threaded, fp64,
 * built with -O2 -ffp-contract=off.  Every reduction longer than r uses a
 * Neumaier-compensated sum.  No blocking, fusion or reordering beyond what
 * the paper's definitions / algorithms state; each function cites the
 * passage it follows ("P:L" = PAPER.md line L).  Shares no code with the
 * CUDA path.
 */
#include "cparls_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define OR_MAXD 8
#define OR_MAXR 64

/* ------------------------------------------------------------------ */
/* Neumaier compensated summation                                      */
/* ------------------------------------------------------------------ */
typedef struct { double s, c; } ksum;
static void kadd(ksum *a, double x) {
  double t = a->s + x;
  if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
  else a->c += (x - t) + a->s;
  a->s = t;
}
static double kval(const ksum *a) { return a->s + a->c; }

/* ------------------------------------------------------------------ */
/* O5: Philox4x32-10 (Salmon et al.; AMB-10)                           */
/* ------------------------------------------------------------------ */
void or_philox4x32_10(const uint32_t c[4], const uint32_t k[2], uint32_t out[4]) {
  uint32_t x0 = c[0], x1 = c[1], x2 = c[2], x3 = c[3];
  uint32_t k0 = k[0], k1 = k[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * x0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * x2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t y0 = hi1 ^ x1 ^ k0, y1 = lo1, y2 = hi0 ^ x3 ^ k1, y3 = lo0;
    x0 = y0; x1 = y1; x2 = y2; x3 = y3;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

/* ------------------------------------------------------------------ */
/* O1: eq:bijection, AMB-1: 0-based, ascending other modes,  */
/* first other mode fastest.                                            */
/* ------------------------------------------------------------------ */
uint64_t or_key(int D, const int64_t *dims, int k, const int64_t *idx) {
  uint64_t key = 0, mult = 1;
  for (int m = 0; m < D; ++m) {
    if (m == k) continue;
    key += (uint64_t)idx[m] * mult;
    mult *= (uint64_t)dims[m];
  }
  return key;
}

void or_decode(int D, const int64_t *dims, int k, uint64_t key, int64_t *idx) {
  for (int m = 0; m < D; ++m) {
    if (m == k) continue;
    idx[m] = (int64_t)(key % (uint64_t)dims[m]);
    key /= (uint64_t)dims[m];
  }
}

/* ------------------------------------------------------------------ */
/* Cyclic Jacobi eigendecomposition (textbook), used by O3 and O14.     */
/* ------------------------------------------------------------------ */
void or_jacobi_eig(int r, const double *G, double *w, double *V) {
  double *a = (double *)malloc(sizeof(double) * r * r);
  memcpy(a, G, sizeof(double) * r * r);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < r; ++j) V[i * r + j] = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < r; ++i) {
      diag += a[i * r + i] * a[i * r + i];
      for (int j = i + 1; j < r; ++j) off += a[i * r + j] * a[i * r + j];
    }
    if (off <= 1e-34 * diag || off == 0.0) break;
    for (int p = 0; p < r; ++p) {
      for (int q = p + 1; q < r; ++q) {
        double apq = a[p * r + q];
        if (apq == 0.0) continue;
        double app = a[p * r + p], aqq = a[q * r + q];
        double theta = (aqq - app) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < r; ++k) {          /* columns p,q */
          double akp = a[k * r + p], akq = a[k * r + q];
          a[k * r + p] = c * akp - s * akq;
          a[k * r + q] = s * akp + c * akq;
        }
        for (int k = 0; k < r; ++k) {          /* rows p,q */
          double apk = a[p * r + k], aqk = a[q * r + k];
          a[p * r + k] = c * apk - s * aqk;
          a[q * r + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < r; ++k) {
          double vkp = V[k * r + p], vkq = V[k * r + q];
          V[k * r + p] = c * vkp - s * vkq;
          V[k * r + q] = s * vkp + c * vkq;
        }
      }
    }
  }
  for (int i = 0; i < r; ++i) w[i] = a[i * r + i];
  free(a);
}

/* G = A^T A with compensated sums over rows (P:148 form). */
static void gram(int64_t n, int r, const double *A, double *G) {
  ksum *acc = (ksum *)calloc((size_t)r * r, sizeof(ksum));
  for (int64_t i = 0; i < n; ++i) {
    const double *a = A + i * r;
    for (int p = 0; p < r; ++p) {
      if (a[p] == 0.0) continue;
      for (int q = p; q < r; ++q) kadd(&acc[p * r + q], a[p] * a[q]);
    }
  }
  for (int p = 0; p < r; ++p)
    for (int q = p; q < r; ++q) G[p * r + q] = G[q * r + p] = kval(&acc[p * r + q]);
  free(acc);
}

/* Pseudo-inverse factors of symmetric PSD G: kept eigenpairs with
 * mu_j > r*eps*mu_max (AMB-11/12).  Returns the number kept. */
static int pinv_eig(int r, const double *G, double *w, double *V, int *keep) {
  or_jacobi_eig(r, G, w, V);
  double mumax = 0.0;
  for (int j = 0; j < r; ++j) if (w[j] > mumax) mumax = w[j];
  int rank = 0;
  for (int j = 0; j < r; ++j) {
    keep[j] = (mumax > 0.0 && w[j] > (double)r * DBL_EPSILON * mumax);
    rank += keep[j];
  }
  return rank;
}

/* ------------------------------------------------------------------ */
/* O3: leverage scores, Def. leverages_scores in the form   */
/* l_i = a_i G^+ a_i^T (BASELINE north_star), G = A^T A.                */
/* ------------------------------------------------------------------ */
int or_leverage(int64_t n, int r, const double *A, double *ell) {
  double G[OR_MAXR * OR_MAXR], w[OR_MAXR], V[OR_MAXR * OR_MAXR];
  int keep[OR_MAXR];
  gram(n, r, A, G);
  int rank = pinv_eig(r, G, w, V, keep);
  for (int64_t i = 0; i < n; ++i) {
    const double *a = A + i * r;
    double l = 0.0;
    for (int j = 0; j < r; ++j) {
      if (!keep[j]) continue;
      double t = 0.0;
      for (int p = 0; p < r; ++p) t += a[p] * V[p * r + j];
      l += t * t / w[j];
    }
    ell[i] = l;
  }
  return rank;
}

/* ------------------------------------------------------------------ */
/* O4 / O6: integer CDF and inverse-CDF draw (AMB-9)            */
/* ------------------------------------------------------------------ */
void or_cdf(int64_t n, const double *pt, uint64_t *C) {
  uint64_t run = 0;
  for (int64_t i = 0; i < n; ++i) {
    run += (uint64_t)nearbyint(ldexp(pt[i], 62));
    C[i] = run;
  }
}

int64_t or_draw(int64_t n, const uint64_t *C, uint64_t R) {
  uint64_t W = C[n - 1];
  uint64_t t = (uint64_t)(((unsigned __int128)R * W) >> 64);
  int64_t lo = 0, hi = n; /* first i with C[i] > t */
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (C[mid] > t) hi = mid; else lo = mid + 1;
  }
  return lo;
}

/* ------------------------------------------------------------------ */
/* Context                                                              */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t nb;      /* buckets (power of two) */
  int shift;
  int64_t *head;
  int64_t *next;
  uint64_t *key;
} or_index;

struct or_ctx {
  int D, r;
  int64_t dims[OR_MAXD];
  int64_t nnz;
  int64_t *coords;
  double *vals;
  or_index idx[OR_MAXD];
  double *A[OR_MAXD];
  double *pt[OR_MAXD];
  uint64_t *C[OR_MAXD];
  double alpha[OR_MAXD];
  int rank[OR_MAXD];
  double lambda[OR_MAXR];
  double normX2;
  /* current sample */
  int smode;
  int64_t sbar, sdet, scap;
  uint64_t *skeys;
  int32_t *scnt;
  double *sw2, *sp;
  uint8_t *sisdet;
  /* last solve */
  int lmode;
  double G[OR_MAXR * OR_MAXR];
  double *M, *B;
  /* frozen stratified fit sample */
  int64_t fs_nnz, fs_zero;   /* stratum sizes */
  int64_t *fs_coords;        /* (fs_nnz + fs_zero) x D */
  double *fs_x;
  double fs_phi_nz, fs_phi_z;
};

static uint64_t hash64(uint64_t k) { return k * 0x9E3779B97F4A7C15ull; }

/* O2: per-mode lookup structure ("precompute and store the
 * linearized indices ... for every mode"), here a chained hash table. */
static void build_index(or_ctx *c, int k) {
  or_index *ix = &c->idx[k];
  int64_t nb = 1; int lg = 0;
  while (nb < 2 * c->nnz + 2) { nb <<= 1; ++lg; }
  ix->nb = nb;
  ix->shift = 64 - lg;
  ix->head = (int64_t *)malloc(sizeof(int64_t) * nb);
  ix->next = (int64_t *)malloc(sizeof(int64_t) * (c->nnz + 1));
  ix->key = (uint64_t *)malloc(sizeof(uint64_t) * (c->nnz + 1));
  for (int64_t b = 0; b < nb; ++b) ix->head[b] = -1;
  for (int64_t e = 0; e < c->nnz; ++e) {
    uint64_t key = or_key(c->D, c->dims, k, c->coords + e * c->D);
    uint64_t b = ix->shift >= 64 ? 0 : hash64(key) >> ix->shift;
    ix->key[e] = key;
    ix->next[e] = ix->head[b];
    ix->head[b] = e;
  }
}

static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) - (x < y);
}

/* Fiber of `key` in mode k (TnsrSamp): nonzero ids sorted by
 * their mode-k coordinate.  Returns count; *ids malloc'd. */
static int64_t fiber(or_ctx *c, int k, uint64_t key, int64_t **ids) {
  or_index *ix = &c->idx[k];
  uint64_t b = ix->shift >= 64 ? 0 : hash64(key) >> ix->shift;
  int64_t cnt = 0, cap = 16;
  int64_t *v = (int64_t *)malloc(sizeof(int64_t) * 2 * cap);
  for (int64_t e = ix->head[b]; e >= 0; e = ix->next[e]) {
    if (ix->key[e] != key) continue;
    if (cnt == cap) { cap *= 2; v = (int64_t *)realloc(v, sizeof(int64_t) * 2 * cap); }
    v[2 * cnt] = c->coords[e * c->D + k];
    v[2 * cnt + 1] = e;
    ++cnt;
  }
  qsort(v, (size_t)cnt, 2 * sizeof(int64_t), cmp_i64); /* by out (unique in a fiber) */
  int64_t *out = (int64_t *)malloc(sizeof(int64_t) * (cnt + 1));
  for (int64_t i = 0; i < cnt; ++i) out[i] = v[2 * i + 1];
  free(v);
  *ids = out;
  return cnt;
}

/* O16: refresh p~_k = l(A_k)/rank, CDF and alpha (AMB-11). */
static int refresh_mode(or_ctx *c, int k, double *ell_out) {
  int64_t n = c->dims[k];
  double *ell = ell_out ? ell_out : (double *)malloc(sizeof(double) * n);
  int rank = or_leverage(n, c->r, c->A[k], ell);
  c->rank[k] = rank;
  double a = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    c->pt[k][i] = rank > 0 ? ell[i] / (double)rank : 0.0;
    if (c->pt[k][i] > a) a = c->pt[k][i];
  }
  c->alpha[k] = a;
  or_cdf(n, c->pt[k], c->C[k]);
  if (!ell_out) free(ell);
  return rank;
}

or_ctx *or_create(int D, const int64_t *dims, int64_t nnz, const int64_t *coords,
                  const double *vals, int r) {
  if (D < 2 || D > OR_MAXD || r < 1 || r > OR_MAXR) return NULL;
  or_ctx *c = (or_ctx *)calloc(1, sizeof(or_ctx));
  c->D = D; c->r = r; c->nnz = nnz;
  memcpy(c->dims, dims, sizeof(int64_t) * D);
  c->coords = (int64_t *)malloc(sizeof(int64_t) * (nnz * D + 1));
  c->vals = (double *)malloc(sizeof(double) * (nnz + 1));
  memcpy(c->coords, coords, sizeof(int64_t) * nnz * D);
  memcpy(c->vals, vals, sizeof(double) * nnz);
  ksum nx = {0, 0};
  for (int64_t e = 0; e < nnz; ++e) kadd(&nx, vals[e] * vals[e]);
  c->normX2 = kval(&nx);
  for (int k = 0; k < D; ++k) {
    build_index(c, k);
    c->A[k] = (double *)calloc((size_t)dims[k] * r, sizeof(double));
    c->pt[k] = (double *)calloc((size_t)dims[k], sizeof(double));
    c->C[k] = (uint64_t *)calloc((size_t)dims[k], sizeof(uint64_t));
  }
  for (int j = 0; j < r; ++j) c->lambda[j] = 1.0;
  c->smode = -1;
  c->lmode = -1;
  return c;
}

void or_destroy(or_ctx *c) {
  if (!c) return;
  for (int k = 0; k < c->D; ++k) {
    free(c->idx[k].head); free(c->idx[k].next); free(c->idx[k].key);
    free(c->A[k]); free(c->pt[k]); free(c->C[k]);
  }
  free(c->coords); free(c->vals);
  free(c->skeys); free(c->scnt); free(c->sw2); free(c->sp); free(c->sisdet);
  free(c->M); free(c->B);
  free(c->fs_coords); free(c->fs_x);
  free(c);
}

int or_set_factor(or_ctx *c, int k, const double *A) {
  memcpy(c->A[k], A, sizeof(double) * c->dims[k] * c->r);
  return refresh_mode(c, k, NULL);
}

void or_get_factor(or_ctx *c, int k, double *A, double *lambda) {
  memcpy(A, c->A[k], sizeof(double) * c->dims[k] * c->r);
  if (lambda) memcpy(lambda, c->lambda, sizeof(double) * c->r);
}

void or_set_ptilde(or_ctx *c, int k, const double *pt) {
  double a = 0.0;
  for (int64_t i = 0; i < c->dims[k]; ++i) {
    c->pt[k][i] = pt[i];
    if (pt[i] > a) a = pt[i];
  }
  c->alpha[k] = a;
  or_cdf(c->dims[k], c->pt[k], c->C[k]);
}

void or_get_ptilde(or_ctx *c, int k, double *pt) {
  memcpy(pt, c->pt[k], sizeof(double) * c->dims[k]);
}

int or_leverage_mode(or_ctx *c, int k, double *ell) { return refresh_mode(c, k, ell); }

/* ------------------------------------------------------------------ */
/* O7: p_i = prod_k p~_k(i_k) (eq:pi P:651-654), canonical order  */
/* left to right over ascending modes, no FMA (AMB-5).                  */
/* ------------------------------------------------------------------ */
static double canon_prob(int d, const double *const *pt, const int64_t *ii) {
  double p = pt[0][ii[0]];
  for (int j = 1; j < d; ++j) p = p * pt[j][ii[j]];
  return p;
}

/* ------------------------------------------------------------------ */
/* O8: DIDX: the exact set {i : p_i > tau}.      */
/* ------------------------------------------------------------------ */
typedef struct { uint64_t key; double p; } kp;
static int cmp_kp_key(const void *a, const void *b) {
  uint64_t x = ((const kp *)a)->key, y = ((const kp *)b)->key;
  return (x > y) - (x < y);
}
static int cmp_kp_pdesc(const void *a, const void *b) { /* AMB-6 */
  const kp *x = (const kp *)a, *y = (const kp *)b;
  if (x->p > y->p) return -1;
  if (x->p < y->p) return 1;
  return (x->key > y->key) - (x->key < y->key);
}

typedef struct { double v; int64_t i; } vi;
static int cmp_vi_desc(const void *a, const void *b) {
  const vi *x = (const vi *)a, *y = (const vi *)b;
  if (x->v > y->v) return -1;
  if (x->v < y->v) return 1;
  return (x->i > y->i) - (x->i < y->i);
}

static uint64_t key_of(int d, const int64_t *n, const int64_t *ii) {
  uint64_t key = 0, mult = 1;
  for (int j = 0; j < d; ++j) { key += (uint64_t)ii[j] * mult; mult *= (uint64_t)n[j]; }
  return key;
}

typedef struct {
  int d;
  const int64_t *n;
  const double *const *pt;
  double tau;
  double alpha[OR_MAXD];
  vi *cand[OR_MAXD];
  int64_t ncand[OR_MAXD];
  int64_t ii[OR_MAXD];
  kp *out;
  int64_t cnt, cap;
} didx_st;

/* Canonical product with position j taken as x and every other position
 * at its maximum alpha: the largest p_i any index with i_j fixed can have
 * (each fp multiply is monotone).  Exact pruning test of P:714-716. */
static double prod_with(const didx_st *st, int j, double x) {
  double p = (j == 0) ? x : st->alpha[0];
  for (int l = 1; l < st->d; ++l) p = p * ((l == j) ? x : st->alpha[l]);
  return p;
}

static void didx_rec(didx_st *st, int lvl, double pp) {
  for (int64_t t = 0; t < st->ncand[lvl]; ++t) {
    double x = st->cand[lvl][t].v;
    double q = (lvl == 0) ? x : pp * x;
    double bound = q;
    for (int l = lvl + 1; l < st->d; ++l) bound = bound * st->alpha[l];
    if (!(bound > st->tau)) break; /* candidates sorted descending: monotone */
    st->ii[lvl] = st->cand[lvl][t].i;
    if (lvl + 1 < st->d) {
      didx_rec(st, lvl + 1, q);
    } else {
      if (st->cnt < st->cap) {
        st->out[st->cnt].key = key_of(st->d, st->n, st->ii);
        st->out[st->cnt].p = q;
      }
      st->cnt++;
    }
  }
}

static int64_t didx_collect(int d, const int64_t *n, const double *const *pt, double tau,
                            int64_t cap, kp **res) {
  didx_st st;
  memset(&st, 0, sizeof(st));
  st.d = d; st.n = n; st.pt = pt; st.tau = tau;
  for (int j = 0; j < d; ++j) {
    double a = 0.0;
    for (int64_t i = 0; i < n[j]; ++i) if (pt[j][i] > a) a = pt[j][i];
    st.alpha[j] = a;
  }
  for (int j = 0; j < d; ++j) {
    st.cand[j] = (vi *)malloc(sizeof(vi) * (n[j] + 1));
    int64_t m = 0;
    for (int64_t i = 0; i < n[j]; ++i)
      if (prod_with(&st, j, pt[j][i]) > tau) { st.cand[j][m].v = pt[j][i]; st.cand[j][m].i = i; ++m; }
    qsort(st.cand[j], (size_t)m, sizeof(vi), cmp_vi_desc);
    st.ncand[j] = m;
  }
  st.cap = cap;
  st.out = (kp *)malloc(sizeof(kp) * (cap + 1));
  didx_rec(&st, 0, 1.0);
  for (int j = 0; j < d; ++j) free(st.cand[j]);
  int64_t got = st.cnt < cap ? st.cnt : cap;
  qsort(st.out, (size_t)got, sizeof(kp), cmp_kp_key);
  *res = st.out;
  return st.cnt;
}

static int64_t didx_brute_collect(int d, const int64_t *n, const double *const *pt, double tau,
                                  int64_t cap, kp **res) {
  uint64_t N = 1;
  for (int j = 0; j < d; ++j) N *= (uint64_t)n[j];
  kp *out = (kp *)malloc(sizeof(kp) * (cap + 1));
  int64_t cnt = 0;
  int64_t ii[OR_MAXD];
  for (uint64_t key = 0; key < N; ++key) {
    uint64_t t = key;
    for (int j = 0; j < d; ++j) { ii[j] = (int64_t)(t % (uint64_t)n[j]); t /= (uint64_t)n[j]; }
    double p = canon_prob(d, pt, ii);
    if (p > tau) {
      if (cnt < cap) { out[cnt].key = key; out[cnt].p = p; }
      ++cnt;
    }
  }
  *res = out;
  return cnt;
}

static int64_t didx_export(int64_t cnt, int64_t cap, kp *v, uint64_t *keys, double *p,
                           double *p_det) {
  if (cnt > cap) { free(v); return -1; }
  ksum s = {0, 0};
  for (int64_t i = 0; i < cnt; ++i) {
    if (keys) keys[i] = v[i].key;
    if (p) p[i] = v[i].p;
    kadd(&s, v[i].p);
  }
  if (p_det) *p_det = kval(&s);
  free(v);
  return cnt;
}

int64_t or_didx(int d, const int64_t *n, const double *const *pt, double tau, int64_t cap,
                uint64_t *keys, double *p, double *p_det) {
  kp *v;
  int64_t cnt = didx_collect(d, n, pt, tau, cap, &v);
  return didx_export(cnt, cap, v, keys, p, p_det);
}

int64_t or_didx_brute(int d, const int64_t *n, const double *const *pt, double tau, int64_t cap,
                      uint64_t *keys, double *p, double *p_det) {
  kp *v;
  int64_t cnt = didx_brute_collect(d, n, pt, tau, cap, &v);
  return didx_export(cnt, cap, v, keys, p, p_det);
}

/* ------------------------------------------------------------------ */
/* SkrpLev (Alg. 1) = DIDX -> SIDX (Alg. 2) -> CIDX          */
/* ------------------------------------------------------------------ */
static int cmp_u64(const void *a, const void *b) {
  uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return (x > y) - (x < y);
}

#define OR_DIDX_CAP 100000000LL

int or_sample(or_ctx *c, int k, int64_t s, double tau, uint64_t seed, uint64_t step,
              or_sample_info *info) {
  const int D = c->D, d = D - 1;
  if (tau < 0) tau = 1.0 / (double)s;                  /* tau = 1/s */
  int modes[OR_MAXD];
  int64_t n[OR_MAXD];
  const double *pts[OR_MAXD];
  uint64_t N = 1;
  for (int m = 0, j = 0; m < D; ++m) {
    if (m == k) continue;
    modes[j] = m; n[j] = c->dims[m]; pts[j] = c->pt[m]; N *= (uint64_t)n[j]; ++j;
  }
  memset(info, 0, sizeof(*info));

  /* DIDX: brute force over [N] when small, pruned otherwise. */
  kp *det = NULL;
  int64_t sdet = (N <= 10000000ull) ? didx_brute_collect(d, n, pts, tau, OR_DIDX_CAP, &det)
                                    : didx_collect(d, n, pts, tau, OR_DIDX_CAP, &det);
  if (sdet > OR_DIDX_CAP) { free(det); return 6; }
  if (sdet > s) {                                     /* P:812, AMB-6 */
    qsort(det, (size_t)sdet, sizeof(kp), cmp_kp_pdesc);
    sdet = s;
    qsort(det, (size_t)sdet, sizeof(kp), cmp_kp_key);
  }
  ksum pd = {0, 0};
  for (int64_t i = 0; i < sdet; ++i) kadd(&pd, det[i].p);
  double p_det = kval(&pd);

  /* SIDX (Alg. 2): rejection sampling in attempt order (AMB-8). */
  int64_t s_rnd = s - sdet;
  uint64_t *rk = (uint64_t *)malloc(sizeof(uint64_t) * (s_rnd > 0 ? s_rnd : 1));
  int64_t acc = 0, att = 0;
  int skipped = 0;
  if (s_rnd > 0) {
    /* AMB-7: skip when every drawable index is deterministic or 1-p_det tiny */
    double drawable = 1.0;
    for (int j = 0; j < d; ++j) {
      int64_t cnt = 0;
      for (int64_t i = 0; i < n[j]; ++i) cnt += (i == 0 ? c->C[modes[j]][0] : c->C[modes[j]][i] - c->C[modes[j]][i - 1]) > 0;
      drawable *= (double)cnt;
    }
    int64_t det_drawable = 0;
    for (int64_t i = 0; i < sdet; ++i) {
      int64_t ii[OR_MAXD];
      uint64_t t = det[i].key;
      int ok = 1;
      for (int j = 0; j < d; ++j) {
        ii[j] = (int64_t)(t % (uint64_t)n[j]); t /= (uint64_t)n[j];
        const uint64_t *C = c->C[modes[j]];
        uint64_t q = ii[j] == 0 ? C[0] : C[ii[j]] - C[ii[j] - 1];
        ok &= (q > 0);
      }
      det_drawable += ok;
    }
    if (1.0 - p_det <= 1e-12 || drawable <= (double)det_drawable) {
      skipped = 1;
    } else {
      int64_t cap_att = 1024 * s_rnd + 65536;
      uint32_t key2[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
      while (acc < s_rnd) {
        if (att >= cap_att) { free(det); free(rk); return 6; }
        uint64_t a = (uint64_t)att;
        uint32_t words[2 * OR_MAXD];
        for (int lane = 0; lane < (d + 1) / 2; ++lane) {
          uint32_t ctr[4] = {(uint32_t)a, (uint32_t)(a >> 32), (uint32_t)step, (uint32_t)lane};
          or_philox4x32_10(ctr, key2, words + 4 * lane);
        }
        int64_t ii[OR_MAXD];
        for (int j = 0; j < d; ++j) {
          uint32_t lo = words[4 * (j / 2) + 2 * (j % 2)];
          uint32_t hi = words[4 * (j / 2) + 2 * (j % 2) + 1];
          uint64_t R = ((uint64_t)hi << 32) | lo;
          ii[j] = or_draw(n[j], c->C[modes[j]], R);   /* i_k ~ Multi(p~_k) */
        }
        double p = canon_prob(d, pts, ii);
        if (p <= tau) rk[acc++] = key_of(d, n, ii);
        ++att;
      }
    }
  }

  /* CIDX: combine repeats, w^2 = c(1-p_det)/(s_rnd p) */
  qsort(rk, (size_t)acc, sizeof(uint64_t), cmp_u64);
  int64_t nuniq = 0;
  for (int64_t i = 0; i < acc; ++i) if (i == 0 || rk[i] != rk[i - 1]) ++nuniq;
  int64_t sbar = sdet + nuniq;
  free(c->skeys); free(c->scnt); free(c->sw2); free(c->sp); free(c->sisdet);
  c->skeys = (uint64_t *)malloc(sizeof(uint64_t) * (sbar + 1));
  c->scnt = (int32_t *)malloc(sizeof(int32_t) * (sbar + 1));
  c->sw2 = (double *)malloc(sizeof(double) * (sbar + 1));
  c->sp = (double *)malloc(sizeof(double) * (sbar + 1));
  c->sisdet = (uint8_t *)malloc(sbar + 1);
  for (int64_t i = 0; i < sdet; ++i) {
    c->skeys[i] = det[i].key; c->scnt[i] = 1; c->sw2[i] = 1.0; c->sp[i] = det[i].p; c->sisdet[i] = 1;
  }
  int64_t o = sdet;
  for (int64_t i = 0; i < acc;) {
    int64_t j = i;
    while (j < acc && rk[j] == rk[i]) ++j;
    int64_t ii[OR_MAXD];
    uint64_t t = rk[i];
    for (int l = 0; l < d; ++l) { ii[l] = (int64_t)(t % (uint64_t)n[l]); t /= (uint64_t)n[l]; }
    double p = canon_prob(d, pts, ii);
    double cnt = (double)(j - i);
    c->skeys[o] = rk[i];
    c->scnt[o] = (int32_t)(j - i);
    c->sw2[o] = (cnt * (1.0 - p_det)) / ((double)s_rnd * p);
    c->sp[o] = p;
    c->sisdet[o] = 0;
    ++o;
    i = j;
  }
  c->smode = k;
  c->sbar = sbar;
  c->sdet = sdet;
  info->s_det = sdet;
  info->s_rnd = s_rnd;
  info->s_bar = sbar;
  info->attempts = att;
  info->p_det = p_det;
  info->skipped_random = skipped;
  free(det);
  free(rk);
  return 0;
}

int64_t or_get_sample(or_ctx *c, int64_t cap, uint64_t *keys, int32_t *counts, double *w2,
                      double *p, uint8_t *is_det) {
  int64_t m = c->sbar < cap ? c->sbar : cap;
  for (int64_t i = 0; i < m; ++i) {
    if (keys) keys[i] = c->skeys[i];
    if (counts) counts[i] = c->scnt[i];
    if (w2) w2[i] = c->sw2[i];
    if (p) p[i] = c->sp[i];
    if (is_det) is_det[i] = c->sisdet[i];
  }
  return c->sbar;
}

int64_t or_get_fibers(or_ctx *c, int64_t cap, int64_t *len, int64_t *out, double *val) {
  int k = c->smode;
  int64_t tot = 0;
  for (int64_t j = 0; j < c->sbar; ++j) {
    int64_t *ids;
    int64_t cnt = fiber(c, k, c->skeys[j], &ids);
    if (len) len[j] = cnt;
    for (int64_t t = 0; t < cnt; ++t, ++tot) {
      if (tot < cap) {
        if (out) out[tot] = c->coords[ids[t] * c->D + k];
        if (val) val[tot] = c->vals[ids[t]];
      }
    }
    free(ids);
  }
  return tot;
}

/* ------------------------------------------------------------------ */
/* O14: B = M G^+ for all rows: the minimum-norm least-squares   */
/* solution, G^+ from the eigendecomposition with the cutoff            */
/* mu_j > r*eps*mu_max (AMB-11/12).  The plain definition: no Cholesky   */
/* shortcut (a pivot test is not rank revealing).  *fallback = rank < r. */
/* ------------------------------------------------------------------ */
static int solve_rows(int r, const double *G, int64_t n, const double *M, double *B,
                      int *fallback) {
  double w[OR_MAXR], V[OR_MAXR * OR_MAXR];
  int keep[OR_MAXR];
  int rank = pinv_eig(r, G, w, V, keep);
  *fallback = rank < r;
  for (int64_t i = 0; i < n; ++i) {
    const double *m = M + i * r;
    double *b = B + i * r;
    double t[OR_MAXR];
    for (int j = 0; j < r; ++j) {
      t[j] = 0.0;
      if (!keep[j]) continue;
      double v = 0.0;
      for (int p = 0; p < r; ++p) v += m[p] * V[p * r + j];
      t[j] = v / w[j];
    }
    for (int p = 0; p < r; ++p) {
      double v = 0.0;
      for (int j = 0; j < r; ++j) if (keep[j]) v += V[p * r + j] * t[j];
      b[p] = v;
    }
  }
  return rank;
}

/* O15: lambda = column norms of B, A_k = B / lambda (AMB-13). */
static void normalize_into(or_ctx *c, int k, const double *B) {
  int r = c->r;
  int64_t n = c->dims[k];
  ksum acc[OR_MAXR];
  memset(acc, 0, sizeof(acc));
  for (int64_t i = 0; i < n; ++i)
    for (int j = 0; j < r; ++j) kadd(&acc[j], B[i * r + j] * B[i * r + j]);
  for (int j = 0; j < r; ++j) c->lambda[j] = sqrt(kval(&acc[j]));
  for (int64_t i = 0; i < n; ++i)
    for (int j = 0; j < r; ++j)
      c->A[k][i * r + j] = c->lambda[j] > 0.0 ? B[i * r + j] / c->lambda[j] : 0.0;
}

/* One sketched mode update, Alg. 3 lines P:918-927. */
int or_solve_mode(or_ctx *c, int k, or_solve_info *info) {
  if (c->smode != k) return 8;
  const int D = c->D, r = c->r;
  int64_t nk = c->dims[k];
  memset(info, 0, sizeof(*info));
  /* KrpSamp and sampled Gram G = sum_j w_j^2 z_j z_j^T */
  double *Z = (double *)malloc(sizeof(double) * (c->sbar * r + 1));
  ksum Gs[OR_MAXR * OR_MAXR];
  memset(Gs, 0, sizeof(Gs));
  for (int64_t j = 0; j < c->sbar; ++j) {
    int64_t idx[OR_MAXD];
    or_decode(D, c->dims, k, c->skeys[j], idx);
    double *z = Z + j * r;
    int first = 1;
    for (int m = 0; m < D; ++m) {               /* eq:Zrow, left to right */
      if (m == k) continue;
      const double *a = c->A[m] + idx[m] * r;
      for (int q = 0; q < r; ++q) z[q] = first ? a[q] : z[q] * a[q];
      first = 0;
    }
    double w2 = c->sw2[j];
    for (int p = 0; p < r; ++p)
      for (int q = p; q < r; ++q) kadd(&Gs[p * r + q], (w2 * z[p]) * z[q]);
  }
  for (int p = 0; p < r; ++p)
    for (int q = p; q < r; ++q) c->G[p * r + q] = c->G[q * r + p] = kval(&Gs[p * r + q]);
  /* TnsrSamp + RHS M = Xs^T diag(w^2) Z_S (AMB-14) */
  free(c->M); free(c->B);
  c->M = (double *)calloc((size_t)nk * r + 1, sizeof(double));
  c->B = (double *)calloc((size_t)nk * r + 1, sizeof(double));
  ksum *Ms = (ksum *)calloc((size_t)nk * r + 1, sizeof(ksum));
  uint8_t *touched = (uint8_t *)calloc((size_t)nk + 1, 1);
  int64_t matched = 0;
  for (int64_t j = 0; j < c->sbar; ++j) {
    int64_t *ids;
    int64_t cnt = fiber(c, k, c->skeys[j], &ids);
    const double *z = Z + j * r;
    for (int64_t t = 0; t < cnt; ++t) {
      int64_t e = ids[t];
      int64_t out = c->coords[e * D + k];
      double coef = c->sw2[j] * c->vals[e];
      for (int q = 0; q < r; ++q) kadd(&Ms[out * r + q], coef * z[q]);
      touched[out] = 1;
    }
    matched += cnt;
    free(ids);
  }
  int64_t ntouched = 0;
  for (int64_t i = 0; i < nk; ++i) {
    ntouched += touched[i];
    for (int q = 0; q < r; ++q) c->M[i * r + q] = kval(&Ms[i * r + q]);
  }
  free(Ms); free(touched); free(Z);
  /* Solve */
  int fb = 0;
  info->rank_used = solve_rows(r, c->G, nk, c->M, c->B, &fb);
  info->chol_fallback = fb;
  info->matched_nnz = matched;
  info->touched_rows = ntouched;
  /* Normalize and refresh leverage */
  normalize_into(c, k, c->B);
  refresh_mode(c, k, NULL);
  c->lmode = k;
  return 0;
}

void or_get_last_solve(or_ctx *c, double *G, double *M, double *B) {
  int r = c->r;
  if (G) memcpy(G, c->G, sizeof(double) * r * r);
  if (c->lmode < 0) return;
  int64_t nk = c->dims[c->lmode];
  if (M) memcpy(M, c->M, sizeof(double) * nk * r);
  if (B) memcpy(B, c->B, sizeof(double) * nk * r);
}

/* ------------------------------------------------------------------ */
/* O17: exact fit (eq:fit P:871-875) by ||X||^2 - 2<X,M> + ||M||^2       */
/* (AMB-16); <X,M> over nonzeros, ||M||^2 = lambda^T (*_m A_m^T A_m) lambda */
/* ------------------------------------------------------------------ */
double or_fit(or_ctx *c) {
  const int D = c->D, r = c->r;
  ksum inner = {0, 0};
  for (int64_t e = 0; e < c->nnz; ++e) {
    const int64_t *ix = c->coords + e * D;
    double m = 0.0;
    for (int q = 0; q < r; ++q) {
      double t = c->lambda[q];
      for (int k = 0; k < D; ++k) t *= c->A[k][ix[k] * r + q];
      m += t;
    }
    kadd(&inner, c->vals[e] * m);
  }
  double H[OR_MAXR * OR_MAXR], Gk[OR_MAXR * OR_MAXR];
  for (int i = 0; i < r * r; ++i) H[i] = 1.0;
  for (int k = 0; k < D; ++k) {
    gram(c->dims[k], r, c->A[k], Gk);
    for (int i = 0; i < r * r; ++i) H[i] *= Gk[i];
  }
  ksum nm = {0, 0};
  for (int p = 0; p < r; ++p)
    for (int q = 0; q < r; ++q) kadd(&nm, c->lambda[p] * c->lambda[q] * H[p * r + q]);
  double resid2 = c->normX2 - 2.0 * kval(&inner) + kval(&nm);
  if (resid2 < 0.0) resid2 = 0.0;
  return 1.0 - sqrt(resid2) / sqrt(c->normX2);
}

double or_fit_dense(or_ctx *c) {
  const int D = c->D, r = c->r;
  int64_t N = 1;
  for (int k = 0; k < D; ++k) N *= c->dims[k];
  double *X = (double *)calloc((size_t)N, sizeof(double));
  for (int64_t e = 0; e < c->nnz; ++e) {
    int64_t lin = 0, mult = 1;
    for (int k = 0; k < D; ++k) { lin += c->coords[e * D + k] * mult; mult *= c->dims[k]; }
    X[lin] = c->vals[e];
  }
  ksum err = {0, 0};
  int64_t ix[OR_MAXD];
  for (int64_t lin = 0; lin < N; ++lin) {
    int64_t t = lin;
    for (int k = 0; k < D; ++k) { ix[k] = t % c->dims[k]; t /= c->dims[k]; }
    double m = 0.0;
    for (int q = 0; q < r; ++q) {
      double v = c->lambda[q];
      for (int k = 0; k < D; ++k) v *= c->A[k][ix[k] * r + q];
      m += v;
    }
    double dlt = X[lin] - m;
    kadd(&err, dlt * dlt);
  }
  free(X);
  return 1.0 - sqrt(kval(&err)) / sqrt(c->normX2);
}

/* ------------------------------------------------------------------ */
/* O18: exact CP-ALS update: B = MTTKRP V^+, V = *_{m!=k} G_m */
/* ------------------------------------------------------------------ */
int or_als_update(or_ctx *c, int k) {
  const int D = c->D, r = c->r;
  int64_t nk = c->dims[k];
  double V[OR_MAXR * OR_MAXR], Gm[OR_MAXR * OR_MAXR];
  for (int i = 0; i < r * r; ++i) V[i] = 1.0;
  for (int m = 0; m < D; ++m) {
    if (m == k) continue;
    gram(c->dims[m], r, c->A[m], Gm);
    for (int i = 0; i < r * r; ++i) V[i] *= Gm[i];
  }
  ksum *Ms = (ksum *)calloc((size_t)nk * r + 1, sizeof(ksum));
  for (int64_t e = 0; e < c->nnz; ++e) {
    const int64_t *ix = c->coords + e * D;
    double z[OR_MAXR];
    int first = 1;
    for (int m = 0; m < D; ++m) {
      if (m == k) continue;
      const double *a = c->A[m] + ix[m] * r;
      for (int q = 0; q < r; ++q) z[q] = first ? a[q] : z[q] * a[q];
      first = 0;
    }
    for (int q = 0; q < r; ++q) kadd(&Ms[ix[k] * r + q], c->vals[e] * z[q]);
  }
  free(c->M); free(c->B);
  c->M = (double *)calloc((size_t)nk * r + 1, sizeof(double));
  c->B = (double *)calloc((size_t)nk * r + 1, sizeof(double));
  for (int64_t i = 0; i < nk * r; ++i) c->M[i] = kval(&Ms[i]);
  free(Ms);
  memcpy(c->G, V, sizeof(double) * r * r);
  int fb;
  solve_rows(r, V, nk, c->M, c->B, &fb);
  normalize_into(c, k, c->B);
  refresh_mode(c, k, NULL);
  c->lmode = k;
  return 0;
}

/* ------------------------------------------------------------------ */
/* O19: Alg. 3 outer loop; step = t*D + k (AMB-10).        */
/* ------------------------------------------------------------------ */
int or_run(or_ctx *c, int iters, int64_t s, double tau, uint64_t seed, int fit_every,
           double *fit_trace) {
  for (int t = 0; t < iters; ++t) {
    for (int k = 0; k < c->D; ++k) {
      or_sample_info si;
      or_solve_info so;
      int st = or_sample(c, k, s, tau, seed, (uint64_t)t * c->D + k, &si);
      if (st) return st;
      st = or_solve_mode(c, k, &so);
      if (st) return st;
    }
    if (fit_trace) {
      if (fit_every > 0 && (t + 1) % fit_every == 0) fit_trace[t] = or_fit(c);
      else fit_trace[t] = NAN;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------ */
/* O20: estimated fit by stratified sampling (sec:estimating-fit,       */
/* P:964-989), AMB-32: ceil(alpha s_fit) nonzeros drawn uniformly WITH   */
/* replacement from the input COO order, floor((1-alpha) s_fit) zeros by */
/* rejection of uniform cells that are nonzeros (attempt order); draws   */
/* from Philox4x32-10 with key = seed, counter = (draw lo, draw hi,      */
/* 0x46495400, lane): nonzero draw i lane 0 words (0,1) -> e =            */
/* mulhi(R, nnz); zero attempt a, mode m: lane 1 + m/2, words            */
/* (2(m%2), 2(m%2)+1) -> i_m = mulhi(R, n_m).                            */
/* ------------------------------------------------------------------ */
static uint64_t mulhi64(uint64_t a, uint64_t b) { return (uint64_t)(((unsigned __int128)a * b) >> 64); }

static uint64_t fs_word(uint64_t seed, uint64_t ctr, uint32_t lane, int half) {
  uint32_t cc[4] = {(uint32_t)ctr, (uint32_t)(ctr >> 32), 0x46495400u, lane};
  uint32_t kk[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t o[4];
  or_philox4x32_10(cc, kk, o);
  return (uint64_t)o[2 * half] | ((uint64_t)o[2 * half + 1] << 32);
}

/* is (ii[0..D)) a nonzero of X?  (mode-0 fiber of its key, scanned) */
static int is_nonzero(or_ctx *c, const int64_t *ii) {
  int64_t *ids = NULL;
  int64_t n = fiber(c, 0, or_key(c->D, c->dims, 0, ii), &ids);
  int hit = 0;
  for (int64_t t = 0; t < n; ++t)
    if (c->coords[ids[t] * c->D] == ii[0]) { hit = 1; break; }
  free(ids);
  return hit;
}

int or_fit_sample(or_ctx *c, int64_t s_fit, double alpha, uint64_t seed, int64_t *n_nz, int64_t *n_z) {
  const int D = c->D;
  if (s_fit < 1 || !(alpha >= 0.0 && alpha <= 1.0)) return 1;
  int64_t nn = (int64_t)ceil(alpha * (double)s_fit);
  int64_t nz = (int64_t)floor((1.0 - alpha) * (double)s_fit);
  if (c->nnz == 0) nn = 0;
  double Nd = 1.0;
  for (int k = 0; k < D; ++k) Nd *= (double)c->dims[k];
  const double Nz = Nd - (double)c->nnz;
  if (!(Nz > 0.0)) nz = 0;   /* fully dense: no zero stratum */
  free(c->fs_coords); free(c->fs_x);
  c->fs_coords = (int64_t *)malloc(sizeof(int64_t) * ((nn + nz) * D + 1));
  c->fs_x = (double *)malloc(sizeof(double) * (nn + nz + 1));
  for (int64_t i = 0; i < nn; ++i) {
    int64_t e = (int64_t)mulhi64(fs_word(seed, (uint64_t)i, 0u, 0), (uint64_t)c->nnz);
    memcpy(c->fs_coords + i * D, c->coords + e * D, sizeof(int64_t) * D);
    c->fs_x[i] = c->vals[e];
  }
  const int64_t cap = 64 * nz + 65536;
  int64_t got = 0;
  for (uint64_t a = 0; got < nz; ++a) {
    if ((int64_t)a >= cap) return 6;
    int64_t ii[OR_MAXD];
    for (int m = 0; m < D; ++m) ii[m] = (int64_t)mulhi64(fs_word(seed, a, 1u + (uint32_t)(m / 2), m % 2),
                                                         (uint64_t)c->dims[m]);
    if (is_nonzero(c, ii)) continue;
    memcpy(c->fs_coords + (nn + got) * D, ii, sizeof(int64_t) * D);
    c->fs_x[nn + got] = 0.0;
    ++got;
  }
  c->fs_nnz = nn;
  c->fs_zero = nz;
  c->fs_phi_nz = nn > 0 ? (double)c->nnz / (double)nn : 0.0;
  c->fs_phi_z = nz > 0 ? Nz / (double)nz : 0.0;
  if (n_nz) *n_nz = nn;
  if (n_z) *n_z = nz;
  return 0;
}

int64_t or_get_fit_sample(or_ctx *c, int64_t cap, int64_t *coords, double *x, uint8_t *is_nz) {
  const int64_t n = c->fs_nnz + c->fs_zero;
  for (int64_t i = 0; i < n && i < cap; ++i) {
    if (coords) memcpy(coords + i * c->D, c->fs_coords + i * c->D, sizeof(int64_t) * c->D);
    if (x) x[i] = c->fs_x[i];
    if (is_nz) is_nz[i] = i < c->fs_nnz;
  }
  return n;
}

/* F^ = sum_i phi_i (m_i - x_i)^2; returns 1 - sqrt(F^)/||X||. */
double or_fit_estimate(or_ctx *c, double *Fhat) {
  const int D = c->D, r = c->r;
  ksum F = {0, 0};
  const int64_t n = c->fs_nnz + c->fs_zero;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t *ix = c->fs_coords + i * D;
    double m = 0.0;
    for (int q = 0; q < r; ++q) {
      double t = c->lambda[q];
      for (int k = 0; k < D; ++k) t *= c->A[k][ix[k] * r + q];
      m += t;
    }
    const double dlt = m - c->fs_x[i];
    const double phi = i < c->fs_nnz ? c->fs_phi_nz : c->fs_phi_z;
    kadd(&F, phi * (dlt * dlt));
  }
  double f = kval(&F);
  if (Fhat) *Fhat = f;
  if (f < 0.0) f = 0.0;
  return 1.0 - sqrt(f) / sqrt(c->normX2);
}

/* Alg. 3 with its stopping rule, AMB-33: epochs of
 * eta outer iterations; after each epoch the fit (0 exact, 1 estimated); an
 * epoch improves if fit > best + tol (best = best fit so far, initially
 * -inf), else a failure; stop after pi consecutive failures or max_epochs.
 * trace[e] = fit after epoch e; returns 0 and *epochs, or a status. */
int or_run_until(or_ctx *c, int64_t s, double tau, uint64_t seed, int eta, int pi, double tol, int max_epochs,
                 int fit_kind, double *trace, int *epochs) {
  double best = -INFINITY;
  int fails = 0, e = 0;
  for (e = 0; e < max_epochs; ++e) {
    for (int t = 0; t < eta; ++t) {
      const int64_t it = (int64_t)e * eta + t;
      for (int k = 0; k < c->D; ++k) {
        or_sample_info si;
        or_solve_info so;
        int st = or_sample(c, k, s, tau, seed, (uint64_t)it * c->D + k, &si);
        if (st) return st;
        st = or_solve_mode(c, k, &so);
        if (st) return st;
      }
    }
    const double f = fit_kind == 1 ? or_fit_estimate(c, NULL) : or_fit(c);
    if (trace) trace[e] = f;
    if (f > best + tol) { best = f; fails = 0; }
    else if (++fails >= pi) { ++e; break; }
  }
  if (epochs) *epochs = e;
  return 0;
}

/* ------------------------------------------------------------------ */
/* O21: randomized range finder initialization (sec:enron), */
/* AMB-34: for every mode k, A_k = X_(k)(:, S) Omega with S = s_init     */
/* fibers drawn uniformly WITH replacement from the nonempty mode-k      */
/* fibers ordered by canonical key (AMB-1), Omega(j, c) standard normal. */
/* Draw j of mode k: Philox key = seed, counter = (j lo, j hi,           */
/* 0x52524600 + k, lane); fiber u = mulhi(R, nfib) from lane 0xFFFF      */
/* words (0,1); Omega(j, c) from lane c/2: u1 = (w0|w1<<32 >> 11 + 1)    */
/* 2^-53, u2 = (w2|w3<<32 >> 11) 2^-53, rho = sqrt(-2 ln u1), c even ->   */
/* rho cos(2 pi u2), odd -> rho sin(2 pi u2) (Box-Muller).  lambda = 1.  */
/* ------------------------------------------------------------------ */
static void rrf_words(uint64_t seed, uint64_t j, int k, uint32_t lane, uint32_t o[4]) {
  uint32_t cc[4] = {(uint32_t)j, (uint32_t)(j >> 32), 0x52524600u + (uint32_t)k, lane};
  uint32_t kk[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  or_philox4x32_10(cc, kk, o);
}

double or_rrf_omega(uint64_t seed, int k, uint64_t j, int c) {
  uint32_t o[4];
  rrf_words(seed, j, k, (uint32_t)(c / 2), o);
  const uint64_t a = (uint64_t)o[0] | ((uint64_t)o[1] << 32), b = (uint64_t)o[2] | ((uint64_t)o[3] << 32);
  const double u1 = (double)((a >> 11) + 1) * 0x1p-53, u2 = (double)(b >> 11) * 0x1p-53;
  const double rho = sqrt(-2.0 * log(u1));
  const double th = 2.0 * 3.14159265358979323846 * u2;
  return (c % 2 == 0) ? rho * cos(th) : rho * sin(th);
}

int64_t or_rrf_fiber(uint64_t seed, int k, uint64_t j, int64_t nfib) {
  uint32_t o[4];
  rrf_words(seed, j, k, 0xFFFFu, o);
  return (int64_t)mulhi64((uint64_t)o[0] | ((uint64_t)o[1] << 32), (uint64_t)nfib);
}

static int cmp_u64_rrf(const void *a, const void *b) {
  uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return (x > y) - (x < y);
}

int or_init_rrf(or_ctx *c, int64_t s_init, uint64_t seed) {
  const int D = c->D, r = c->r;
  if (s_init < 1) return 1;
  for (int k = 0; k < D; ++k) {
    /* nonempty fibers of X_(k): distinct canonical keys, ascending */
    uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (c->nnz + 1));
    for (int64_t e = 0; e < c->nnz; ++e) keys[e] = c->idx[k].key[e];
    qsort(keys, (size_t)c->nnz, sizeof(uint64_t), cmp_u64_rrf);
    int64_t nf = 0;
    for (int64_t e = 0; e < c->nnz; ++e)
      if (e == 0 || keys[e] != keys[e - 1]) keys[nf++] = keys[e];
    const int64_t n = c->dims[k];
    ksum *acc = (ksum *)calloc((size_t)n * r + 1, sizeof(ksum));
    for (int64_t j = 0; j < s_init && nf > 0; ++j) {
      const uint64_t key = keys[or_rrf_fiber(seed, k, (uint64_t)j, nf)];
      int64_t *ids = NULL;
      const int64_t len = fiber(c, k, key, &ids);
      double om[OR_MAXR];
      for (int q = 0; q < r; ++q) om[q] = or_rrf_omega(seed, k, (uint64_t)j, q);
      for (int64_t t = 0; t < len; ++t) {
        const int64_t e = ids[t], i = c->coords[e * D + k];
        for (int q = 0; q < r; ++q) kadd(&acc[i * r + q], c->vals[e] * om[q]);
      }
      free(ids);
    }
    for (int64_t i = 0; i < n * r; ++i) c->A[k][i] = kval(&acc[i]);
    free(acc);
    free(keys);
    refresh_mode(c, k, NULL);
  }
  for (int q = 0; q < r; ++q) c->lambda[q] = 1.0;
  return 0;
}
