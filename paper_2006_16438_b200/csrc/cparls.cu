// cparls.cu -- host orchestrator and C ABI (include/cparls.h) of the B200-native
// CP-ARLS-LEV hot path.  All arithmetic of the method runs in the kernels of
// kernels.cuh; this file only sequences them, owns device memory and moves
// results across the ABI.  "P:L" cites /root/reference/PAPER.md line L.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <cub/device/device_radix_sort.cuh>
#include <thrust/execution_policy.h>
#include <thrust/merge.h>
#include <new>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/cparls.h"
#include "comm.cuh"
#include "kernels.cuh"
#include "sampler.cuh"

using namespace cparls;

namespace {

struct ModeIndex {
  uint64_t *key = nullptr;   // sorted eq:bijection keys over the other modes
  int32_t *out = nullptr;    // mode-k coordinate (row of B it updates)
  void *val = nullptr;       // value (fp32 or fp64)
  int64_t *dir = nullptr;    // dir[b] = first position with key >> shift >= b
  int shift = 0;
  int64_t nbkt = 0;
  int64_t nnz = 0;           // nonzeros of this rank's slice of mode k
  // order of the other modes in this copy's keys, fastest first (copy_order):
  // the slowest is mode (k+1) mod D, the rest by ascending n_m.  Sample keys
  // stay canonical (AMB-1) and are re-encoded by the lookup.
  int order[kMaxModes] = {};
  // hot rows of the fixed-point RHS (rhs.cuh k_rhs_hot): hot_n > 0 enables;
  // hot_slot (n_k entries, -1 = cold) and hot_rows (hot_n) are null when every
  // row is hot (slot = row)
  int32_t *hot_slot = nullptr;
  int32_t *hot_rows = nullptr;
  int hot_n = 0;
  double hot_share = 0.0;    // fraction of this copy's nonzeros in the hot rows
};

// other modes of k, ascending n_m (ties: lower mode first)
void copy_order(const cparls_ctx *c, int k, int *order);

struct DevScalars {
  double pdet;
  int64_t total;
  unsigned long long last_attempt;
  unsigned long long counter;
  unsigned long long bad;
  int64_t mk;
  unsigned long long touched;
  unsigned long long det_drawable;
  double fit[3];
  double normX2;
  double maxabs;                    // max |x| over the nonzeros (fixed-point RHS bound)
  unsigned long long dupmax;        // longest run of duplicate coordinates in a copy
  unsigned int done_count;          // k_gram_scales: blocks finished (the last resets it)
};

}  // namespace

// Named slots of the context's pinned scratch hscr (async device->host scalar
// copies read after a later synchronisation); every use has its own range.
constexpr int kHscrDrawable = 0;                     // [0, kMaxModes): drawable rows per other mode
constexpr int kHscrSidx = kHscrDrawable + kMaxModes; // 2: SIDX accepted total, last accepted attempt
constexpr int kHscrCand = kHscrSidx + 2;             // [.., +kMaxModes): DIDX candidate counts
constexpr int kHscrSlots = 64;
static_assert(kHscrCand + kMaxModes <= kHscrSlots, "pinned scratch layout");

struct cparls_ctx {
  int D = 0, r = 0, ld = 0;
  int64_t dims[kMaxModes] = {0};
  int64_t nnz = 0;
  int vf32 = 0;
  cudaStream_t st = nullptr;
  cparls_opts opts{};
  double tau = -1.0;
  bool poisoned = false;
  std::string err;
  double normX2 = 0.0;
  int64_t nmax = 0;
  ModeIndex idx[kMaxModes];
  double *A[kMaxModes] = {nullptr};
  double *pt[kMaxModes] = {nullptr};
  uint64_t *C[kMaxModes] = {nullptr};
  ModeDev *md[kMaxModes] = {nullptr};
  SolveDev *sd = nullptr;
  double *lam_model = nullptr;   // lambda of the model (AMB-31)
  DevScalars *dv = nullptr;
  StepCtl *ctl = nullptr;        // asynchronous mode step control (common.cuh)
  void *hctl = nullptr;          // pinned host copy of *ctl
  StepCtl ctl_seen{};            // device statistics already folded into stats
  int64_t s_cur = 0;             // s of the current sample (upper bound of s_bar)
  bool sample_pulled = false;    // host sbar/sdet/... hold the current sample's values
  unsigned long long *tile_state = nullptr;   // SIDX look-back tiles (sampler.cuh)
  double *fitbuf = nullptr;      // per-iteration fit values of an asynchronous run
  int64_t fitbuf_cap = 0;
  int64_t tile_cap = 0;
  // scratch
  double *M = nullptr;
  uint8_t *touched = nullptr;
  double *gpart = nullptr;
  int64_t gpart_blocks = 0;
  int nsm = 148;                 // SMs of the device (k_rhs_hot: one CTA each)
  double *Gtmp = nullptr;
  uint64_t *tile_u64 = nullptr;
  int64_t *i64part = nullptr;    // scan partials
  int64_t i64part_cap = 0;
  dd *ddpart = nullptr;
  // sample state
  int64_t scap = 0;
  int smode = -1;
  bool have_sample = false;
  int64_t sbar = 0, sdet = 0, s_rnd = 0, attempts = 0;
  double p_det = 0.0;
  int skipped = 0;
  uint64_t *skey = nullptr;
  double *sw2 = nullptr, *sp = nullptr;
  int32_t *scnt = nullptr;
  uint8_t *sisdet = nullptr;
  // canonical-order sort of the combined sample (second copies, swapped in)
  uint64_t *skey2 = nullptr;
  double *sw2_2 = nullptr, *sp2 = nullptr;
  int32_t *scnt2 = nullptr;
  uint8_t *sisdet2 = nullptr;
  uint32_t *sperm = nullptr, *sperm2 = nullptr, *shist = nullptr;
  double *Z = nullptr;
  int64_t *lo = nullptr, *len = nullptr, *off = nullptr;
  int64_t mk = 0;
  bool have_lookup = false;
  // DIDX
  int64_t ccap = 0;
  uint64_t *ckey[kMaxModes] = {nullptr};
  uint32_t *cidx[kMaxModes] = {nullptr};
  uint64_t *ckey_tmp = nullptr;
  uint32_t *cidx_tmp = nullptr;
  uint32_t *rhist = nullptr;
  int64_t lcap = 0;
  uint64_t *lkey[2] = {nullptr, nullptr};
  double *lpp[2] = {nullptr, nullptr};
  int64_t *lcnt = nullptr, *loff = nullptr;
  // SIDX / CIDX
  int64_t acap = 0;
  uint64_t *akey = nullptr;
  double *ap = nullptr;
  uint64_t *rkey = nullptr;
  double *rp = nullptr;
  unsigned long long *hkey = nullptr;
  uint32_t *hcnt = nullptr;
  double *hp = nullptr;
  uint32_t *hfirst = nullptr;   // first draw index per hash slot (deterministic combine)
  uint32_t *rslot = nullptr;    // per random draw: its slot
  int64_t *rflag = nullptr, *rpos = nullptr;
  bool sample_sort = false;      // opts.sample_sort
  uint64_t hsize = 0;
  // bookkeeping
  std::vector<void *> allocs;
  cparls_stats stats{};
  bool profiling = false;
  std::vector<cudaEvent_t> ev_pool;                             // free events
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_pending;
  int fit_mode = 0;
  int smode_last_solved = -1;
  // row sharding: this rank owns rows [row_lo, row_hi) of mode k
  Comm *comm = nullptr;
  int world = 1, wrank = 0;
  int64_t row_lo[kMaxModes] = {0}, row_hi[kMaxModes] = {0};
  std::vector<int64_t> bounds[kMaxModes];   // row blocks of every rank per mode
  std::vector<int64_t> heavy[kMaxModes];    // heavy rows (nonzeros spread over the ranks), ascending
  int64_t *heavy_dev[kMaxModes] = {nullptr};
  uint8_t *heavy_own[kMaxModes] = {nullptr};   // this rank owns heavy row h
  int64_t heavy_buf_n = 0;
  double *heavy_buf = nullptr;              // |heavy| x ld exchange buffer
  bool fac_dirty[kMaxModes] = {false};      // only the owned rows of A_k are current (world > 1)
  double *Zg = nullptr;                     // sampled other-mode rows from their owners (s x d x ld)
  int64_t *drow_lo = nullptr, *drow_hi = nullptr;   // owned row ranges of every mode (device)
  int64_t zg_cap = 0;
  // RHS output-row windows (see rhs.cuh)
  int64_t segcap = 0;
  int64_t *seg_lo = nullptr, *seg_len = nullptr, *seg_off = nullptr, *i64part_seg = nullptr;
  double *fx_scale = nullptr;   // fixed-point RHS scales 2^e_c, 2^-e_c (kernels.cuh)
  double dupmax = 1.0;
  bool rhs_fixed = true;        // int64 fixed-point RHS (rhs_path 0/1/2); false: fp64 reductions (rhs_path 3)
  bool fx_on = false;           // this solve's RHS is fixed point (M holds int64)
  // pinned double buffer for copies into pageable host memory (rows_to_host)
  void *stage[2] = {nullptr, nullptr};
  double *stage_dev[2] = {nullptr, nullptr};   // packed (ld -> r) rows on the device
  long long *hscr = nullptr;    // small pinned scratch: async scalar reads folded into later syncs
  double *cpart = nullptr;       // K6 block partials of sum_j w_j^2 |z_j| per column (fixed-point scales)
  ScanState scan;                // single-pass scans of the asynchronous step (prims.cuh)
  // auxiliary stream: G^+ (k_solve_prep) runs concurrently with the lookup and
  // the RHS of the same step (it needs only the sampled Gram)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  // frozen stratified fit sample (fitest.cuh, AMB-32)
  bool have_fs = false;
  int64_t fs_nnz = 0, fs_zero = 0;
  double fs_phi_nz = 0.0, fs_phi_z = 0.0;
  int32_t *fs_idx[kMaxModes] = {nullptr};
  double *fs_x = nullptr;
  int32_t *seg_j = nullptr;
  int64_t nfib[kMaxModes] = {0};
  uint32_t *deg[kMaxModes] = {nullptr};   // row degrees of each copy (single-sort build; else null)
};

struct cparls_comm {
  int kind = 0;   // 0 NCCL, 1 local group
  int world = 1, rank = 0;
  ncclComm_t nccl = nullptr;
  cparls::LocalGroup *group = nullptr;
};

namespace {

int64_t row_start(const cparls_ctx *c, int k, int q) { return c->bounds[k][q]; }

Comm *make_comm(cparls_comm *cc, int rank) {
  if (cc->kind == 0) {
    auto *n = new NcclComm();
    n->c = cc->nccl;
    n->owns = false;
    n->world = cc->world;
    n->rank = cc->rank;
    if (n->rank != rank) {
      delete n;
      throw ApiError(CPARLS_EINVAL, "NCCL communicator rank != opts.world_rank");
    }
    return n;
  }
  auto *l = new LocalComm();
  l->g = cc->group;
  l->world = cc->world;
  l->rank = rank;
  return l;
}

// host wall time of a scope added to *acc (ms)
struct WallAcc {
  double *acc;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit WallAcc(double *a) : acc(a) {}
  ~WallAcc() { *acc += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); }
};

void *dalloc(cparls_ctx *c, size_t bytes) {
  void *p = nullptr;
  if (bytes == 0) bytes = 16;
  WallAcc wa(&c->stats.build_ms[0]);
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw ApiError(CPARLS_EOOM, "cudaMalloc(" + std::to_string(bytes) + ") failed: " + cudaGetErrorString(e));
  }
  c->allocs.push_back(p);
  return p;
}
void dfree(cparls_ctx *c, void *p) {
  if (!p) return;
  auto it = std::find(c->allocs.begin(), c->allocs.end(), p);
  if (it != c->allocs.end()) c->allocs.erase(it);
  WallAcc wa(&c->stats.build_ms[0]);
  cudaFree(p);
}

template <typename T>
T *dalloc_t(cparls_ctx *c, int64_t n) {
  return static_cast<T *>(dalloc(c, sizeof(T) * (size_t)std::max<int64_t>(n, 1)));
}

bool is_device_ptr(const void *p) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Fold the step statistics the asynchronous kernels accumulated in the step
// control (StepCtl::st_*) into cparls_stats: the deltas since the last fold
// (SURVEY 8(d) byte model; ctl_seen holds the values already folded).
void fold_ctl_stats(cparls_ctx *c) {
  const StepCtl &h = *reinterpret_cast<const StepCtl *>(c->hctl);
  StepCtl &o = c->ctl_seen;
  const double v = c->vf32 ? 4.0 : 8.0;
  const int d = c->D - 1;
  const double dmk = (double)(h.st_sum_mk - o.st_sum_mk), dsb = (double)(h.st_sum_sbar - o.st_sum_sbar);
  const double datt = (double)(h.st_sum_attempts - o.st_sum_attempts);
  const double dtouch = (double)(h.st_sum_touched - o.st_sum_touched);
  c->stats.bytes_rhs += dmk * (4.0 + v) + dtouch * c->r * 8.0 * 2;
  c->stats.bytes_gram += dsb * (d * c->r * 8.0 + 16.0);
  c->stats.bytes_lookup += dsb * 16.0;
  c->stats.bytes_sample += datt * d * 8.0;
  c->stats.sum_matched_nnz += (int64_t)dmk;
  if (h.st_steps != o.st_steps) {
    c->stats.last_matched_nnz = h.st_last_mk;
    c->mk = h.st_last_mk;
    for (int k = 0; k < c->D; ++k) c->stats.touched_rows[k] = h.st_touched[k];
  }
  if (h.st_sum_sbar != o.st_sum_sbar || h.st_sum_attempts != o.st_sum_attempts) {
    c->stats.last_s_bar = h.st_last_sbar;
    c->stats.last_attempts = h.st_last_attempts;
  }
  o = h;
}

void ktimers_resolve(cparls_ctx *c);

// Stream synchronisation of the context: reads the step control back (the
// statistics of the asynchronous steps are folded) and resolves the per-kernel
// event timers (all recorded before this point on the stream, so complete).
// count = false for the synchronisations of the stats calls themselves.
void sync(cparls_ctx *c, bool count = true) {
  if (c->ctl) CK(cudaMemcpyAsync(c->hctl, c->ctl, sizeof(StepCtl), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  if (count) c->stats.host_syncs++;
  if (c->ctl) fold_ctl_stats(c);
  ktimers_resolve(c);
}

bool is_pinned_host(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// rows x r doubles of an ld-strided device matrix -> dst (r-strided), any
// memory kind.  Pageable destinations go through a pinned double buffer
// (DMA of chunk i+1 overlaps the host memcpy of chunk i); a pitched copy
// straight into pageable memory runs at ~1 GB/s.
void rows_to_host(cparls_ctx *c, double *dst, const double *src, int64_t rows, int r, int ld) {
  if (rows <= 0) return;
  const size_t pitch_d = sizeof(double) * ld, pitch_h = sizeof(double) * r;
  if (is_device_ptr(dst) || ld == r) {
    CK(cudaMemcpy2DAsync(dst, pitch_h, src, pitch_d, pitch_h, rows, cudaMemcpyDefault, c->st));
    sync(c);
    return;
  }
  constexpr size_t kStageBytes = size_t(32) << 20;
  const bool pinned = is_pinned_host(dst);
  if (pinned && !c->stage_dev[0]) {
    for (int b = 0; b < 2; ++b) c->stage_dev[b] = static_cast<double *>(dalloc(c, kStageBytes));
  }
  if (pinned) {   // rows packed on the device, then contiguous D2H copies straight into dst
    const int64_t per = std::max<int64_t>(1, (int64_t)(kStageBytes / pitch_h));
    for (int64_t r0 = 0, i = 0; r0 < rows; r0 += per, ++i) {
      const int b = (int)(i & 1);
      const int64_t nr = std::min(per, rows - r0);
      k_pack_rows<<<(unsigned)std::min<int64_t>(1184, ceil_div(nr * r, 256)), 256, 0, c->st>>>(
          src + r0 * ld, ld, r, nr, c->stage_dev[b]);
      CK_LAUNCH();
      CK(cudaMemcpyAsync(dst + r0 * r, c->stage_dev[b], (size_t)nr * pitch_h, cudaMemcpyDeviceToHost, c->st));
    }
    sync(c);
    return;
  }
  if (!c->stage[0]) {
    for (int b = 0; b < 2; ++b) {
      CK(cudaHostAlloc(&c->stage[b], kStageBytes, cudaHostAllocDefault));
      CK(cudaEventCreateWithFlags(&c->stage_ev[b], cudaEventDisableTiming));
      if (!c->stage_dev[b]) c->stage_dev[b] = static_cast<double *>(dalloc(c, kStageBytes));
    }
  }
  const int64_t per = std::max<int64_t>(1, (int64_t)(kStageBytes / pitch_h));
  const int64_t nch = (rows + per - 1) / per;
  auto drain = [&](int64_t i) {
    const int b = (int)(i & 1);
    CK(cudaEventSynchronize(c->stage_ev[b]));
    const int64_t r0 = i * per, nr = std::min(per, rows - r0);
    // host copy out of the pinned buffer on a few threads (first-touch page
    // faults of the destination dominate a single-threaded memcpy)
    char *d = reinterpret_cast<char *>(dst + r0 * r);
    const char *src_h = static_cast<const char *>(c->stage[b]);
    const size_t bytes = (size_t)nr * pitch_h;
    constexpr int kThreads = 8;
    const size_t part = (bytes + kThreads - 1) / kThreads;
    std::thread th[kThreads];
    for (int t = 0; t < kThreads; ++t) {
      const size_t o = std::min(bytes, (size_t)t * part), len = std::min(bytes, o + part) - o;
      th[t] = std::thread([=] { if (len) std::memcpy(d + o, src_h + o, len); });
    }
    for (auto &x : th) x.join();
  };
  for (int64_t i = 0; i < nch; ++i) {
    const int b = (int)(i & 1);
    if (i >= 2) drain(i - 2);
    const int64_t r0 = i * per, nr = std::min(per, rows - r0);
    // rows packed on the device first: one contiguous copy instead of a
    // 2D copy of nr r-wide rows (the copy engine moves those row by row)
    k_pack_rows<<<(unsigned)std::min<int64_t>(1184, ceil_div(nr * r, 256)), 256, 0, c->st>>>(src + r0 * ld, ld, r, nr,
                                                                                            c->stage_dev[b]);
    CK_LAUNCH();
    CK(cudaMemcpyAsync(c->stage[b], c->stage_dev[b], (size_t)nr * pitch_h, cudaMemcpyDeviceToHost, c->st));
    CK(cudaEventRecord(c->stage_ev[b], c->st));
  }
  for (int64_t i = std::max<int64_t>(0, nch - 2); i < nch; ++i) drain(i);
}

template <typename T>
T read_dev(cparls_ctx *c, const T *p) {
  T v;
  CK(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, c->st));
  sync(c);
  return v;
}

struct Phase {
  cparls_ctx *c;
  double *acc;
  cudaEvent_t a = nullptr, b = nullptr;
  Phase(cparls_ctx *c_, double *acc_) : c(c_), acc(acc_) {
    if (c->profiling) {
      CK(cudaEventCreate(&a));
      CK(cudaEventCreate(&b));
      CK(cudaEventRecord(a, c->st));
    }
  }
  void end() {
    if (c->profiling && a) {
      CK(cudaEventRecord(b, c->st));
      CK(cudaEventSynchronize(b));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, a, b));
      *acc += ms;
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      a = b = nullptr;
    }
  }
  ~Phase() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
};

// Always-on per-kernel device timers: an event pair around every launch of a
// hot kernel, resolved (synchronised and summed) only when stats are read.
enum { KT_RHS = 0, KT_FIT = 1, KT_SOLVE = 2, KT_LEV = 3, KT_N = 4 };
struct KTimer {
  cparls_ctx *c;
  int id;
  cudaStream_t st;
  cudaEvent_t a = nullptr, b = nullptr;
  KTimer(cparls_ctx *c_, int id_, cudaStream_t st_ = nullptr);
  void stop();
  ~KTimer();   // a timer never stopped (an exception in between) returns its events
};

cudaEvent_t ev_get(cparls_ctx *c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  return e;
}
KTimer::KTimer(cparls_ctx *c_, int id_, cudaStream_t st_) : c(c_), id(id_), st(st_ ? st_ : c_->st) {
  a = ev_get(c);
  b = ev_get(c);
  CK(cudaEventRecord(a, st));
}
void KTimer::stop() {
  CK(cudaEventRecord(b, st));
  c->ev_pending.push_back({id, {a, b}});
  c->stats.kernel_launches_by_id[id]++;
  a = b = nullptr;
  // bounded: a long run without synchronisation folds the finished pairs here
  if (c->ev_pending.size() >= 4096) {
    size_t keep = 0;
    for (auto &p : c->ev_pending) {
      if (cudaEventQuery(p.second.second) == cudaSuccess) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, p.second.first, p.second.second));
        c->stats.kernel_ms[p.first] += ms;
        c->ev_pool.push_back(p.second.first);
        c->ev_pool.push_back(p.second.second);
      } else {
        c->ev_pending[keep++] = p;
      }
    }
    cudaGetLastError();   // cudaErrorNotReady of the unfinished ones
    c->ev_pending.resize(keep);
  }
}
KTimer::~KTimer() {
  if (a) c->ev_pool.push_back(a);
  if (b) c->ev_pool.push_back(b);
}
// sum the elapsed times of all recorded launches into the stats
void ktimers_resolve(cparls_ctx *c) {
  for (auto &p : c->ev_pending) {
    CK(cudaEventSynchronize(p.second.second));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, p.second.first, p.second.second));
    c->stats.kernel_ms[p.first] += ms;
    c->ev_pool.push_back(p.second.first);
    c->ev_pool.push_back(p.second.second);
  }
  c->ev_pending.clear();
}

#define LAUNCHED(c, n) ((c)->stats.kernel_launches += (n))

inline int rmax_bucket(int r) { return r <= 4 ? 4 : r <= 8 ? 8 : r <= 16 ? 16 : r <= 28 ? 28 : r <= 32 ? 32 : 64; }

#define RSWITCH(r, ...)                                      \
  do {                                                       \
    switch (rmax_bucket(r)) {                                \
      case 4: { constexpr int RM = 4; __VA_ARGS__; } break;   \
      case 8: { constexpr int RM = 8; __VA_ARGS__; } break;   \
      case 16: { constexpr int RM = 16; __VA_ARGS__; } break; \
      case 28: { constexpr int RM = 28; __VA_ARGS__; } break; \
      case 32: { constexpr int RM = 32; __VA_ARGS__; } break; \
      default: { constexpr int RM = 64; __VA_ARGS__; } break; \
    }                                                        \
  } while (0)

// dynamic shared memory (doubles) of the row kernels; +RMAX slack covers the
// unconditional register loads of padded columns
size_t tile_d(int ld) { return (size_t)kRowThreads * (ld + 1); }
size_t gram_smem(int r, int ld) { return sizeof(double) * (tile_d(ld) + 64); }
size_t solve_smem(int r, int ld) { return sizeof(double) * ((size_t)r * ld + (size_t)kRowThreads * (ld + 2) + 64); }
// B = M G^+ and B^T B block partials: FP64 tensor-core kernel for r in 5..32
// (ld = 8..32), CUDA-core k_solve_rows_t otherwise or with CPARLS_SOLVE_DMMA=0
// returns the grid it launched (the number of BtB block partials in gpart)
int64_t launch_solve_rows(cparls_ctx *c, double *M, int64_t n, double *B, int64_t grid, int zero_m,
                          const double *fscale) {
  const int r = c->r, ld = c->ld;
  const bool dmma = r > 4 && ld <= 32 && ld % 8 == 0;
  if (dmma) {
    const bool pipe = CPARLS_SOLVE_PIPE != 0;
    const size_t sm = sizeof(double) * solve_dmma_smem_d(ld, pipe);
    if (pipe) grid = std::min<int64_t>(grid, c->nsm);   // one CTA per SM
#define SOLVE_DMMA(NTV)                                                                                          \
  do {                                                                                                           \
    if (pipe)                                                                                                    \
      k_solve_dmma<NTV, true><<<(unsigned)grid, kRowThreads, sm, c->st>>>(M, n, r, ld, c->sd, B, c->gpart,       \
                                                                         &c->dv->touched, zero_m, fscale,       \
                                                                         c->ctl);                               \
    else                                                                                                         \
      k_solve_dmma<NTV, false><<<(unsigned)grid, kRowThreads, sm, c->st>>>(M, n, r, ld, c->sd, B, c->gpart,      \
                                                                          &c->dv->touched, zero_m, fscale,      \
                                                                          c->ctl);                              \
  } while (0)
    switch (ld / 8) {
      case 1: SOLVE_DMMA(1); break;
      case 2: SOLVE_DMMA(2); break;
      case 3: SOLVE_DMMA(3); break;
      default: SOLVE_DMMA(4); break;
    }
#undef SOLVE_DMMA
  } else {
    RSWITCH(r, k_solve_rows_t<RM><<<(unsigned)grid, kRowThreads, solve_smem(r, ld), c->st>>>(
                   M, n, r, ld, c->sd, B, c->gpart, &c->dv->touched, zero_m, fscale, c->ctl));
  }
  return grid;
}
size_t krp_smem(int r, int ld) { return sizeof(double) * (tile_d(ld) + kRowThreads + 64); }
size_t prep_smem(int r) { return sizeof(double) * 4 * (size_t)r * r; }
size_t warp_tiles_d(int ld) { return (size_t)(kRowThreads / 32) * kWarpRows * warp_tile_stride(ld); }
// + 64 doubles of slack: the register loads of padded columns (c < RMAX) may
// run past the last row of the last tile
size_t lev_w_smem(int r, int ld) {
  const size_t rm = rmax_bucket(r);
  return sizeof(double) * (rm * rm + kMaxRank + warp_tiles_d(ld) + 64);
}

// allow the largest dynamic shared memory the kernel can take (opt-in limit
// minus its static shared memory)
template <typename F>
void max_dyn_smem(F func) {
  static int optin = -1;
  if (optin < 0) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  }
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, func));
  CK(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes));
}

template <int RM>
void set_attrs_rm() {
  max_dyn_smem(k_gram_rows_t<RM>);
  max_dyn_smem(k_solve_rows_t<RM>);
  max_dyn_smem(k_lev_rows_w<RM>);
  max_dyn_smem(k_fit_thread<float, RM>);
  max_dyn_smem(k_fit_thread<double, RM>);
}

void set_kernel_attrs(int r, int ld) {
  max_dyn_smem(k_solve_dmma<1>); max_dyn_smem(k_solve_dmma<2>); max_dyn_smem(k_solve_dmma<3>);
  max_dyn_smem(k_solve_dmma<4>);
  max_dyn_smem(k_solve_dmma<1, true>); max_dyn_smem(k_solve_dmma<2, true>); max_dyn_smem(k_solve_dmma<3, true>);
  max_dyn_smem(k_solve_dmma<4, true>);
  max_dyn_smem(k_rhs_hot<float>); max_dyn_smem(k_rhs_hot<double>);
  set_attrs_rm<4>(); set_attrs_rm<8>(); set_attrs_rm<16>(); set_attrs_rm<28>(); set_attrs_rm<32>();
  set_attrs_rm<64>();
  int prep = (int)prep_smem(r);
  CK(cudaFuncSetAttribute(k_lev_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, prep));
  CK(cudaFuncSetAttribute(k_norm_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, prep));
  CK(cudaFuncSetAttribute(k_solve_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, prep));
}

int64_t row_grid(cparls_ctx *c, int64_t ntiles) { return std::max<int64_t>(1, std::min<int64_t>(ntiles, c->gpart_blocks)); }

// ---------------------------------------------------------------- leverage
// rows -> p~, integer CDF (AMB-9/11).  lam != null also
// normalizes A_k in place by lam.
// Guarded by the context's step control (an aborted asynchronous step leaves
// the mode's factor, p~, CDF, alpha and drawable count untouched).
void lev_rows_and_cdf(cparls_ctx *c, int k, const double *lam) {
  const int64_t n = c->dims[k];
  const int64_t nt = ceil_div(n, kLevThreads);
  k_lev_reset<<<1, 1, 0, c->st>>>(c->md[k], c->ctl);
  CK_LAUNCH();
  {
    const unsigned g = (unsigned)row_grid(c, ceil_div(n, kWarpRows * (kRowThreads / 32)));
    CK(cudaMemsetAsync(c->tile_u64, 0, sizeof(uint64_t) * nt, c->st));
    KTimer kt(c, KT_LEV);
    RSWITCH(c->r, k_lev_rows_w<RM><<<g, kRowThreads, lev_w_smem(c->r, c->ld), c->st>>>(
                      c->A[k], n, c->r, c->ld, lam, c->md[k], c->pt[k], c->C[k],
                      reinterpret_cast<unsigned long long *>(c->tile_u64), &c->md[k]->alpha,
                      reinterpret_cast<unsigned long long *>(&c->md[k]->drawable), c->ctl));
    kt.stop();
  }
  CK_LAUNCH();
  k_scan_u64_single<<<1, kScanThreads, 0, c->st>>>(c->tile_u64, nt, c->ctl);
  CK_LAUNCH();
  k_cdf_final<<<(unsigned)nt, kLevThreads, 0, c->st>>>(c->C[k], n, c->tile_u64, c->ctl);
  CK_LAUNCH();
  LAUNCHED(c, 4);
  c->stats.bytes_leverage += (double)n * (c->r * 8.0 * (lam ? 2 : 1) + 16.0);
}

// Sharded leverage refresh: normalize and score the owned rows
// of A_k only, allgather p~_k (8 bytes per row instead of the factor rows),
// then every rank forms q and the integer CDF of all rows from the identical
// p~ bits (the same kernels as the set_ptilde path).
void lev_rows_sharded(cparls_ctx *c, int k, const double *lam) {
  const int64_t n = c->dims[k];
  const int64_t r0 = c->row_lo[k], nown = c->row_hi[k] - c->row_lo[k];
  const int64_t nt = ceil_div(n, kLevThreads);
  if (nown > 0) {
    const unsigned g = (unsigned)row_grid(c, ceil_div(nown, kWarpRows * (kRowThreads / 32)));
    KTimer kt(c, KT_LEV);
    RSWITCH(c->r, k_lev_rows_w<RM><<<g, kRowThreads, lev_w_smem(c->r, c->ld), c->st>>>(
                      c->A[k] + r0 * c->ld, nown, c->r, c->ld, lam, c->md[k], c->pt[k] + r0, c->C[k] + r0,
                      reinterpret_cast<unsigned long long *>(c->tile_u64), &c->md[k]->alpha,
                      reinterpret_cast<unsigned long long *>(&c->md[k]->drawable), c->ctl));
    kt.stop();
    CK_LAUNCH();
  }
  std::vector<int64_t> off(c->world + 1);
  for (int q = 0; q <= c->world; ++q) off[q] = q < c->world ? row_start(c, k, q) : n;
  c->comm->allgatherv_f64(c->pt[k], off, c->st);
  c->stats.bytes_comm += 8.0 * n;
  k_lev_reset<<<1, 1, 0, c->st>>>(c->md[k], c->ctl);
  k_q_from_pt<<<(unsigned)nt, kLevThreads, 0, c->st>>>(c->pt[k], n, c->C[k], c->tile_u64, &c->md[k]->alpha,
                                                       reinterpret_cast<unsigned long long *>(&c->md[k]->drawable),
                                                       c->ctl);
  CK_LAUNCH();
  k_scan_u64_single<<<1, kScanThreads, 0, c->st>>>(c->tile_u64, nt, c->ctl);
  CK_LAUNCH();
  k_cdf_final<<<(unsigned)nt, kLevThreads, 0, c->st>>>(c->C[k], n, c->tile_u64, c->ctl);
  CK_LAUNCH();
  LAUNCHED(c, 5);
  c->stats.bytes_leverage += (double)nown * (c->r * 8.0 * 2 + 16.0) + (double)n * 16.0;
  c->fac_dirty[k] = true;   // only the owned rows of A_k are current here
}

// Every rank gets every row of A_m (collective, SPMD): the per-epoch dense
// allgather for the exact fit, and the factor getters of a sharded run.
void gather_factor(cparls_ctx *c, int m) {
  if (c->world <= 1 || !c->fac_dirty[m]) return;
  std::vector<int64_t> off(c->world + 1);
  for (int q = 0; q <= c->world; ++q) off[q] = (q < c->world ? row_start(c, m, q) : c->dims[m]) * c->ld;
  c->comm->allgatherv_f64(c->A[m], off, c->st);
  c->stats.bytes_comm += 8.0 * c->dims[m] * c->ld;
  c->fac_dirty[m] = false;
}

void gram_of_rows(cparls_ctx *c, const double *A, int64_t n, double *G_out) {
  const int64_t grid = row_grid(c, ceil_div(n, kRowThreads));
  RSWITCH(c->r, k_gram_rows_t<RM><<<(unsigned)grid, kRowThreads, gram_smem(c->r, c->ld), c->st>>>(A, n, c->r, c->ld,
                                                                                                  c->gpart));
  CK_LAUNCH();
  k_pairs_reduce<<<pairs_reduce_grid(c->r), 256, 0, c->st>>>(c->gpart, grid, c->r, G_out);
  CK_LAUNCH();
  LAUNCHED(c, 2);
}

void leverage_full(cparls_ctx *c, int k) {
  gather_factor(c, k);
  Phase ph(c, &c->stats.ms_leverage);
  gram_of_rows(c, c->A[k], c->dims[k], c->Gtmp);
  k_lev_prep<<<1, kPrepThreads, prep_smem(c->r), c->st>>>(c->r, c->Gtmp, c->md[k], c->A[k], c->dims[k], c->ld);
  CK_LAUNCH();
  LAUNCHED(c, 1);
  c->stats.bytes_leverage += (double)c->dims[k] * c->r * 8.0;
  lev_rows_and_cdf(c, k, nullptr);
  ph.end();
}

void reset_lambda(cparls_ctx *c) {
  std::vector<double> ones(c->r, 1.0);
  CK(cudaMemcpyAsync(c->lam_model, ones.data(), sizeof(double) * c->r, cudaMemcpyHostToDevice, c->st));
  sync(c);
}

// The other modes of k (ascending, AMB-1); alpha / drawable counts are read by
// the kernels from the modes' ModeDev (no host copy).
OtherModes other_modes(cparls_ctx *c, int k) {
  OtherModes om{};
  om.d = c->D - 1;
  uint64_t mult = 1;
  for (int m = 0, j = 0; m < c->D; ++m) {
    if (m == k) continue;
    om.mode[j] = m;
    om.n[j] = c->dims[m];
    om.div[j] = make_fastdiv((uint64_t)c->dims[m]);
    om.pt[j] = c->pt[m];
    om.C[j] = c->C[m];
    om.A[j] = c->A[m];
    om.md[j] = c->md[m];
    om.mult[j] = mult;
    mult *= (uint64_t)c->dims[m];
    ++j;
  }
  return om;
}

void copy_order(const cparls_ctx *c, int k, int *order) {
  // slowest: mode (k+1) mod D, so every mode is the slowest key mode of exactly
  // one copy (the exact CP-ALS MTTKRP streams that copy, als.cuh); the others
  // by ascending n_m, fastest first
  const int slow = (k + 1) % c->D;
  int d = 0;
  for (int m = 0; m < c->D; ++m)
    if (m != k && m != slow) order[d++] = m;
  std::stable_sort(order, order + d, [&](int a, int b) { return c->dims[a] < c->dims[b]; });
  order[d] = slow;
}

KeyRemap key_remap(const cparls_ctx *c, int k) {
  KeyRemap rm{};
  rm.d = c->D - 1;
  rm.identity = 1;
  const int *order = c->idx[k].order;
  for (int j = 0, m = 0; m < c->D; ++m) {
    if (m == k) continue;
    rm.n[j] = c->dims[m];
    rm.div[j] = make_fastdiv((uint64_t)c->dims[m]);
    uint64_t mult = 1;
    for (int q = 0; q < rm.d && order[q] != m; ++q) mult *= (uint64_t)c->dims[order[q]];
    rm.cmult[j] = mult;
    rm.identity &= (order[j] == m);
    ++j;
  }
  return rm;
}

// ---------------------------------------------------------------- index build (K0)
// Hot rows of mode k for the fixed-point RHS (rhs.cuh k_rhs_hot): the rows of
// largest degree in this rank's copy (ties: lower row), as many as the
// shared-memory accumulators hold.
constexpr size_t kHotSmemBytes = 200 * 1024;

int hot_capacity(int r) { return r > 32 ? 0 : (int)(kHotSmemBytes / (8 * (size_t)r)); }

// The H (< n_k) rows of mode k of largest degree in this rank's copy (ties:
// lower row first) into rows_dst (device, H entries); returns the fraction of
// the copy's nonzeros they hold.
double top_rows_by_degree(cparls_ctx *c, int k, int64_t H, int32_t *rows_dst) {
  ModeIndex &ix = c->idx[k];
  const int64_t nk = c->dims[k];
  uint32_t *deg = dalloc_t<uint32_t>(c, nk);
  if (c->deg[k]) {   // from the run boundaries of the neighbouring copy
    CK(cudaMemcpyAsync(deg, c->deg[k], sizeof(uint32_t) * nk, cudaMemcpyDeviceToDevice, c->st));
  } else {
    CK(cudaMemsetAsync(deg, 0, sizeof(uint32_t) * nk, c->st));
    k_row_degree<<<(unsigned)std::min<int64_t>(4096, ceil_div(ix.nnz, 256)), 256, 0, c->st>>>(ix.out, ix.nnz, deg);
    CK_LAUNCH();
  }
  uint32_t *deg1 = dalloc_t<uint32_t>(c, nk);
  int32_t *rows0 = dalloc_t<int32_t>(c, nk), *rows1 = dalloc_t<int32_t>(c, nk);
  k_iota_u32<<<(unsigned)ceil_div(nk, 256), 256, 0, c->st>>>(reinterpret_cast<uint32_t *>(rows0), nk);
  CK_LAUNCH();
  cub::DoubleBuffer<uint32_t> kb(deg, deg1);
  cub::DoubleBuffer<int32_t> vb(rows0, rows1);
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, kb, vb, nk, 0, 32, c->st));
  void *tmp = dalloc(c, tb);
  CK(cub::DeviceRadixSort::SortPairsDescending(tmp, tb, kb, vb, nk, 0, 32, c->st));
  std::vector<uint32_t> top(H);
  CK(cudaMemcpyAsync(top.data(), kb.Current(), sizeof(uint32_t) * H, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(rows_dst, vb.Current(), sizeof(int32_t) * H, cudaMemcpyDeviceToDevice, c->st));
  sync(c);
  double hot = 0.0;
  for (uint32_t d : top) hot += d;
  dfree(c, tmp);
  dfree(c, deg);
  dfree(c, deg1);
  dfree(c, rows0);
  dfree(c, rows1);
  return ix.nnz > 0 ? hot / (double)ix.nnz : 0.0;
}

void build_hot_rows(cparls_ctx *c, int k) {
  ModeIndex &ix = c->idx[k];
  const int64_t nk = c->dims[k];
  const int req = c->opts.rhs_hot_rows;
  int64_t H = std::min<int64_t>(hot_capacity(c->r), nk);
  if (req > 0) H = std::min<int64_t>(H, req);
  if (req == 0 || H <= 0 || ix.nnz == 0 || c->opts.rhs_path == 3) return;
  if (H == nk) {   // every row hot: slot = row
    ix.hot_n = (int)H;
    ix.hot_share = 1.0;
    return;
  }
  int32_t *rows = dalloc_t<int32_t>(c, H);
  ix.hot_share = top_rows_by_degree(c, k, H, rows);
  if (req > 0 || ix.hot_share >= 0.7) {
    ix.hot_n = (int)H;
    ix.hot_rows = rows;
    ix.hot_slot = dalloc_t<int32_t>(c, nk);
    CK(cudaMemsetAsync(ix.hot_slot, 0xff, sizeof(int32_t) * nk, c->st));
    k_hot_slots<<<(unsigned)ceil_div(H, 256), 256, 0, c->st>>>(ix.hot_rows, (int)H, ix.hot_slot);
    CK_LAUNCH();
    sync(c);
  } else {
    dfree(c, rows);
  }
}

template <typename IT, typename VT>
void build_index_mode(cparls_ctx *c, int k, const IT *coords, const VT *vals, int64_t nnz) {
  ModeIndex &ix = c->idx[k];
  ix.nnz = nnz;
  sync(c);
  const double b0 = c->stats.build_ms[0] + c->stats.build_ms[1] + c->stats.build_ms[3];
  const auto tw0 = std::chrono::steady_clock::now();
  const unsigned g = (unsigned)std::max<int64_t>(1, ceil_div(nnz, 256));
  // pass 1: stable sort of nonzero ids by mode-k coordinate
  uint32_t *ok0 = dalloc_t<uint32_t>(c, nnz), *ok1 = dalloc_t<uint32_t>(c, nnz);
  uint32_t *id0 = dalloc_t<uint32_t>(c, nnz), *id1 = dalloc_t<uint32_t>(c, nnz);
  if (nnz > 0) {
    k_make_outkey<IT><<<g, 256, 0, c->st>>>(coords, nnz, c->D, k, ok0, id0);
    CK_LAUNCH();
  }
  int obits = 1;
  while ((int64_t(1) << obits) < c->dims[k]) ++obits;
  cub::DoubleBuffer<uint32_t> kb(ok0, ok1);
  cub::DoubleBuffer<uint32_t> vb(id0, id1);
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, nnz, 0, obits, c->st));
  void *tmp = dalloc(c, tb);
  {
    sync(c);
    WallAcc ws(&c->stats.build_ms[1]);
    CK(cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb, nnz, 0, obits, c->st));
    sync(c);
  }
  dfree(c, tmp);
  uint32_t *ids = vb.Current();
  dfree(c, kb.Current());
  dfree(c, kb.Alternate());
  // pass 2: stable sort by key
  KeySpec ks{};
  ks.D = c->D;
  ks.k = k;
  for (int m = 0; m < c->D; ++m) ks.dims[m] = c->dims[m];
  copy_order(c, k, ix.order);
  for (int j = 0; j < c->D - 1; ++j) ks.order[j] = ix.order[j];
  uint64_t *key0 = dalloc_t<uint64_t>(c, nnz), *key1 = dalloc_t<uint64_t>(c, nnz);
  if (nnz > 0) {
    k_make_keys<IT><<<g, 256, 0, c->st>>>(coords, nnz, ks, ids, key0);
    CK_LAUNCH();
  }
  long double Nk = 1;
  for (int m = 0; m < c->D; ++m)
    if (m != k) Nk *= (long double)c->dims[m];
  int kbits = 1;
  while ((long double)((unsigned long long)1 << kbits) < Nk && kbits < 63) ++kbits;
  cub::DoubleBuffer<uint64_t> kb2(key0, key1);
  cub::DoubleBuffer<uint32_t> vb2(ids, ids == id0 ? id1 : id0);
  tb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb2, vb2, nnz, 0, kbits, c->st));
  tmp = dalloc(c, tb);
  {
    sync(c);
    WallAcc ws(&c->stats.build_ms[1]);
    CK(cub::DeviceRadixSort::SortPairs(tmp, tb, kb2, vb2, nnz, 0, kbits, c->st));
    sync(c);
  }
  dfree(c, tmp);
  ix.key = kb2.Current();
  dfree(c, kb2.Alternate());
  uint32_t *fids = vb2.Current();
  dfree(c, vb2.Alternate());
  ix.out = dalloc_t<int32_t>(c, nnz);
  ix.val = dalloc(c, sizeof(VT) * (size_t)std::max<int64_t>(nnz, 1));
  if (nnz > 0) {
    k_gather_nz<IT, VT><<<g, 256, 0, c->st>>>(coords, vals, nnz, c->D, k, fids, ix.out, (VT *)ix.val);
    CK_LAUNCH();
  }
  sync(c);
  dfree(c, fids);
  // top-level directory on the high key bits
  int dbits = 1;
  while (dbits < 26 && (int64_t(1) << (dbits + 1)) <= std::max<int64_t>(nnz / 8, 2)) ++dbits;
  ix.shift = std::max(0, kbits - dbits);
  unsigned long long Nk1 = (unsigned long long)(Nk - 1);
  ix.nbkt = (int64_t)(Nk1 >> ix.shift) + 1;
  ix.dir = dalloc_t<int64_t>(c, ix.nbkt + 1);
  if (nnz > 0) {
    k_dir_fill<<<g, 256, 0, c->st>>>(ix.key, nnz, ix.shift, ix.dir, ix.nbkt);
    CK_LAUNCH();
  } else {
    CK(cudaMemsetAsync(ix.dir, 0, sizeof(int64_t) * (ix.nbkt + 1), c->st));
  }
  sync(c);
  {
    WallAcc wh(&c->stats.build_ms[3]);
    build_hot_rows(c, k);
  }
  const double tot = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tw0).count();
  c->stats.build_ms[2] += tot - (c->stats.build_ms[0] + c->stats.build_ms[1] + c->stats.build_ms[3] - b0);
}

// Row partition of mode k into world contiguous blocks balanced by nonzeros
// (SURVEY 8(e)).  A heavy row -- more nonzeros than a rank's share total/world
// (a Zipf head row) -- has its nonzeros spread over all ranks (heavy_rank) and
// weighs ceil(deg/world) in the plan; it is owned (solved) by the rank whose
// block contains it, after its partial RHS rows are summed over the ranks.
// bound[p] = first row whose exclusive prefix of the weights reaches
// p*W/world.  heavy (n flags, may be null) receives the heavy rows.
void plan_rows(int64_t n, const unsigned long long *deg, int world, int64_t *bound, uint8_t *heavy) {
  unsigned long long total = 0;
  for (int64_t i = 0; i < n; ++i) total += deg[i];
  const unsigned long long share = total / (unsigned long long)world;
  auto is_heavy = [&](int64_t i) { return world > 1 && deg[i] > share; };
  auto weight = [&](int64_t i) {
    return is_heavy(i) ? (deg[i] + (unsigned long long)world - 1) / (unsigned long long)world : deg[i];
  };
  unsigned long long W = 0;
  for (int64_t i = 0; i < n; ++i) {
    W += weight(i);
    if (heavy) heavy[i] = is_heavy(i) ? 1 : 0;
  }
  bound[0] = 0;
  unsigned long long run = 0;
  int64_t i = 0;
  for (int p = 1; p < world; ++p) {
    const unsigned long long t = (unsigned long long)(((unsigned __int128)W * p) / world);
    while (i < n && run < t) run += weight(i++);
    bound[p] = i;
  }
  bound[world] = n;
}

// Sharded build of mode k: global row degrees (allreduce), row blocks
// (plan_rows), all-to-all of the local COO chunk to the owners of the mode-k
// rows, then the usual sorted copy of the received slice.
template <typename IT, typename VT>
void route_and_build(cparls_ctx *c, int k, const IT *coords, const VT *vals) {
  const int P = c->world, D = c->D;
  const int64_t n = c->dims[k], nnz = c->nnz;
  unsigned long long *deg = dalloc_t<unsigned long long>(c, n);
  CK(cudaMemsetAsync(deg, 0, sizeof(unsigned long long) * n, c->st));
  if (nnz > 0) {
    k_coord_degree<IT><<<1184, 256, 0, c->st>>>(coords, nnz, D, k, deg);
    CK_LAUNCH();
  }
  c->comm->allreduce_u64(deg, n, c->st);
  std::vector<unsigned long long> hdeg(n);
  CK(cudaMemcpyAsync(hdeg.data(), deg, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost, c->st));
  sync(c);
  dfree(c, deg);
  std::vector<int64_t> bound(P + 1);
  std::vector<uint8_t> hv(n);
  plan_rows(n, hdeg.data(), P, bound.data(), hv.data());
  c->row_lo[k] = bound[c->wrank];
  c->row_hi[k] = bound[c->wrank + 1];
  c->bounds[k] = bound;
  // heavy rows of mode k: nonzeros spread over the ranks; partial RHS rows summed
  c->heavy[k].clear();
  for (int64_t i = 0; i < n; ++i)
    if (hv[i]) c->heavy[k].push_back(i);
  uint8_t *dheavy = dalloc_t<uint8_t>(c, n);
  CK(cudaMemcpyAsync(dheavy, hv.data(), n, cudaMemcpyHostToDevice, c->st));
  if (!c->heavy[k].empty()) {
    const int64_t nh = (int64_t)c->heavy[k].size();
    c->heavy_dev[k] = dalloc_t<int64_t>(c, nh);
    CK(cudaMemcpyAsync(c->heavy_dev[k], c->heavy[k].data(), sizeof(int64_t) * nh, cudaMemcpyHostToDevice, c->st));
    std::vector<uint8_t> own(nh);
    for (int64_t h = 0; h < nh; ++h) own[h] = c->heavy[k][h] >= c->row_lo[k] && c->heavy[k][h] < c->row_hi[k];
    c->heavy_own[k] = dalloc_t<uint8_t>(c, nh);
    CK(cudaMemcpyAsync(c->heavy_own[k], own.data(), nh, cudaMemcpyHostToDevice, c->st));
    c->heavy_buf_n = std::max(c->heavy_buf_n, nh);
  }
  // destination rank per local nonzero, stable order by destination
  int64_t *dbound = dalloc_t<int64_t>(c, P + 1);
  CK(cudaMemcpyAsync(dbound, bound.data(), sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice, c->st));
  uint32_t *dk0 = dalloc_t<uint32_t>(c, nnz), *dk1 = dalloc_t<uint32_t>(c, nnz);
  uint32_t *ix0 = dalloc_t<uint32_t>(c, nnz), *ix1 = dalloc_t<uint32_t>(c, nnz);
  unsigned long long *dcnt = dalloc_t<unsigned long long>(c, P);
  CK(cudaMemsetAsync(dcnt, 0, sizeof(unsigned long long) * P, c->st));
  if (nnz > 0) {
    k_dest_rank<IT><<<(unsigned)ceil_div(nnz, 256), 256, 0, c->st>>>(coords, nnz, D, k, dbound, P, dk0, ix0, dcnt,
                                                                     dheavy);
    CK_LAUNCH();
  }
  std::vector<unsigned long long> hcnt(P);
  CK(cudaMemcpyAsync(hcnt.data(), dcnt, sizeof(unsigned long long) * P, cudaMemcpyDeviceToHost, c->st));
  cub::DoubleBuffer<uint32_t> kb(dk0, dk1), vb(ix0, ix1);
  int dbits = 1;
  while ((1 << dbits) < P) ++dbits;
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, nnz, 0, dbits, c->st));
  void *tmp = dalloc(c, tb);
  CK(cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb, nnz, 0, dbits, c->st));
  // pack coords (D x IT) and vals in destination order
  IT *scoord = dalloc_t<IT>(c, nnz * D);
  VT *sval = dalloc_t<VT>(c, nnz);
  if (nnz > 0) {
    k_pack_nz<IT, VT><<<(unsigned)ceil_div(nnz, 256), 256, 0, c->st>>>(coords, vals, nnz, D, vb.Current(), scoord,
                                                                       sval);
    CK_LAUNCH();
  }
  sync(c);
  dfree(c, tmp); dfree(c, dk0); dfree(c, dk1); dfree(c, ix0); dfree(c, ix1); dfree(c, dcnt); dfree(c, dbound);
  dfree(c, dheavy);
  // exchange counts, then coordinates and values
  std::vector<int64_t> mine(P);
  for (int q = 0; q < P; ++q) mine[q] = (int64_t)hcnt[q];
  std::vector<int64_t> all = c->comm->allgather_host(mine, c->st);   // all[p*P + q] = count p -> q
  std::vector<int64_t> soff_c(P + 1, 0), roff_c(P + 1, 0), soff_v(P + 1, 0), roff_v(P + 1, 0);
  for (int q = 0; q < P; ++q) {
    soff_c[q + 1] = soff_c[q] + mine[q] * D * (int64_t)sizeof(IT);
    soff_v[q + 1] = soff_v[q] + mine[q] * (int64_t)sizeof(VT);
    const int64_t rc = all[(int64_t)q * P + c->wrank];
    roff_c[q + 1] = roff_c[q] + rc * D * (int64_t)sizeof(IT);
    roff_v[q + 1] = roff_v[q] + rc * (int64_t)sizeof(VT);
  }
  const int64_t nrecv = roff_v[P] / (int64_t)sizeof(VT);
  if (nrecv >= (int64_t(1) << 32)) throw ApiError(CPARLS_ERANGE, "a rank's slice of a mode exceeds 2^32 nonzeros");
  IT *rcoord = dalloc_t<IT>(c, nrecv * D);
  VT *rval = dalloc_t<VT>(c, nrecv);
  c->comm->alltoallv((const char *)scoord, soff_c, (char *)rcoord, roff_c, c->st);
  c->comm->alltoallv((const char *)sval, soff_v, (char *)rval, roff_v, c->st);
  sync(c);
  dfree(c, scoord);
  dfree(c, sval);
  build_index_mode<IT, VT>(c, k, rcoord, rval, nrecv);
  sync(c);
  dfree(c, rcoord);
  dfree(c, rval);
}

// Single-sort build of the per-mode copies (world_size 1, prod_m n_m < 2^64):
// scratch allocated once for all modes (cudaMalloc of tens of GB is slow, and
// slower still right after large frees), one stable radix sort per mode of
// the composite key with the value as payload (kernels.cuh k_make_comp), the
// sorted composite split in place into (key, out).  The sorted key and value
// buffers become the copy's; fresh scratch replaces them for the next mode.
struct BuildArena {
  uint64_t *comp[2] = {nullptr, nullptr};
  void *val[2] = {nullptr, nullptr};
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  int cbits = 64;
};

int key_bits(long double N) {   // bits of the largest value N - 1
  int b = 1;
  while (b < 64 && (long double)((unsigned long long)1 << b) < N) ++b;
  return b;
}

template <typename VT>
void arena_alloc(cparls_ctx *c, BuildArena &ar, int64_t nnz) {
  for (int i = 0; i < 2; ++i) {
    ar.comp[i] = dalloc_t<uint64_t>(c, nnz);
    ar.val[i] = dalloc(c, sizeof(VT) * (size_t)std::max<int64_t>(nnz, 1));
  }
  cub::DoubleBuffer<uint64_t> kb(ar.comp[0], ar.comp[1]);
  cub::DoubleBuffer<VT> vb((VT *)ar.val[0], (VT *)ar.val[1]);
  CK(cub::DeviceRadixSort::SortPairs(nullptr, ar.tmp_bytes, kb, vb, nnz, 0, ar.cbits, c->st));
  ar.tmp = dalloc(c, ar.tmp_bytes);
}

void build_directory(cparls_ctx *c, int k) {
  ModeIndex &ix = c->idx[k];
  const int64_t nnz = ix.nnz;
  long double Nk = 1;
  for (int m = 0; m < c->D; ++m)
    if (m != k) Nk *= (long double)c->dims[m];
  const int kbits = key_bits(Nk);
  int dbits = 1;
  while (dbits < 26 && (int64_t(1) << (dbits + 1)) <= std::max<int64_t>(nnz / 8, 2)) ++dbits;
  ix.shift = std::max(0, kbits - dbits);
  unsigned long long Nk1 = (unsigned long long)(Nk - 1);
  ix.nbkt = (int64_t)(Nk1 >> ix.shift) + 1;
  ix.dir = dalloc_t<int64_t>(c, ix.nbkt + 1);
  if (nnz > 0) {
    k_dir_fill<<<(unsigned)std::max<int64_t>(1, ceil_div(nnz, 256)), 256, 0, c->st>>>(ix.key, nnz, ix.shift, ix.dir,
                                                                                     ix.nbkt);
    CK_LAUNCH();
  } else {
    CK(cudaMemsetAsync(ix.dir, 0, sizeof(int64_t) * (ix.nbkt + 1), c->st));
  }
}

template <typename IT, typename VT>
void build_index_mode_comp(cparls_ctx *c, int k, const IT *coords, const VT *vals, int64_t nnz, BuildArena &ar,
                           bool last, bool comp_made = false) {
  ModeIndex &ix = c->idx[k];
  ix.nnz = nnz;
  sync(c);
  const double b0 = c->stats.build_ms[0] + c->stats.build_ms[1] + c->stats.build_ms[3];
  const auto tw0 = std::chrono::steady_clock::now();
  KeySpec ks{};
  ks.D = c->D;
  ks.k = k;
  for (int m = 0; m < c->D; ++m) ks.dims[m] = c->dims[m];
  copy_order(c, k, ix.order);
  for (int j = 0; j < c->D - 1; ++j) ks.order[j] = ix.order[j];
  const unsigned g = (unsigned)std::min<int64_t>(148 * 16, std::max<int64_t>(1, ceil_div(nnz, 256)));
  if (nnz > 0 && !comp_made) {
    k_make_comp<IT, VT><<<g, 256, 0, c->st>>>(coords, vals, nnz, ks, ar.comp[0], (VT *)ar.val[0]);
    CK_LAUNCH();
  }
  cub::DoubleBuffer<uint64_t> kb(ar.comp[0], ar.comp[1]);
  cub::DoubleBuffer<VT> vb((VT *)ar.val[0], (VT *)ar.val[1]);
  {
    sync(c);
    WallAcc ws(&c->stats.build_ms[1]);
    CK(cub::DeviceRadixSort::SortPairs(ar.tmp, ar.tmp_bytes, kb, vb, nnz, 0, ar.cbits, c->st));
    sync(c);
  }
  ix.out = dalloc_t<int32_t>(c, nnz);
  if (nnz > 0) {
    k_split_comp<<<g, 256, 0, c->st>>>(kb.Current(), nnz, make_fastdiv((uint64_t)c->dims[k]), ix.out);
    CK_LAUNCH();
  }
  ix.key = kb.Current();
  ix.val = vb.Current();
  const int ci = kb.Current() == ar.comp[0] ? 0 : 1;
  const int vi = (void *)vb.Current() == ar.val[0] ? 0 : 1;
  ar.comp[ci] = last ? nullptr : dalloc_t<uint64_t>(c, nnz);
  ar.val[vi] = last ? nullptr : dalloc(c, sizeof(VT) * (size_t)std::max<int64_t>(nnz, 1));
  build_directory(c, k);
  sync(c);
  const double tot = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tw0).count();
  c->stats.build_ms[2] += tot - (c->stats.build_ms[0] + c->stats.build_ms[1] + c->stats.build_ms[3] - b0);
}

// Row degrees of every mode from the copy whose slowest key mode it is
// (copy_order: mode (k+1) mod D in copy k), then the RHS hot rows.
void degrees_and_hot_rows(cparls_ctx *c) {
  const int D = c->D;
  for (int m = 0; m < D; ++m) {
    const int k = (m - 1 + D) % D;
    const ModeIndex &ix = c->idx[k];
    const int64_t n = c->dims[m];
    uint64_t stride = 1;
    for (int j = 0; j + 1 < D - 1; ++j) stride *= (uint64_t)c->dims[ix.order[j]];
    int64_t *beg = dalloc_t<int64_t>(c, n), *end = dalloc_t<int64_t>(c, n);
    CK(cudaMemsetAsync(beg, 0, sizeof(int64_t) * n, c->st));
    CK(cudaMemsetAsync(end, 0, sizeof(int64_t) * n, c->st));
    if (ix.nnz > 0) {
      k_slow_bounds<<<(unsigned)std::min<int64_t>(148 * 16, ceil_div(ix.nnz, 256)), 256, 0, c->st>>>(
          ix.key, ix.nnz, make_fastdiv(stride), beg, end);
      CK_LAUNCH();
    }
    c->deg[m] = dalloc_t<uint32_t>(c, n);
    k_bounds_deg<<<(unsigned)std::min<int64_t>(148 * 16, ceil_div(n, 256)), 256, 0, c->st>>>(beg, end, n, c->deg[m]);
    CK_LAUNCH();
    sync(c);
    dfree(c, beg);
    dfree(c, end);
  }
  WallAcc wh(&c->stats.build_ms[3]);
  for (int k = 0; k < D; ++k) build_hot_rows(c, k);
}

// Merge the sorted runs [rb[j], rb[j+1]) of (k, v) pairwise until one run is
// left (stable: on equal keys the earlier run first, i.e. input order).  The
// result ends in (k, v); (sk, sv) is scratch of the same size and the pointers
// are swapped so the caller's (k, v) hold the result.
template <typename VT>
void merge_runs(cparls_ctx *c, const std::vector<int64_t> &rb0, uint64_t *&k, VT *&v, uint64_t *&sk, VT *&sv) {
  std::vector<int64_t> rb = rb0;
  auto pol = thrust::cuda::par_nosync.on(c->st);
  while (rb.size() > 2) {
    std::vector<int64_t> nb{0};
    for (size_t j = 0; j + 1 < rb.size(); j += 2) {
      if (j + 2 < rb.size()) {
        thrust::merge_by_key(pol, k + rb[j], k + rb[j + 1], k + rb[j + 1], k + rb[j + 2], v + rb[j], v + rb[j + 1],
                             sk + rb[j], sv + rb[j]);
        nb.push_back(rb[j + 2]);
      } else {
        const int64_t n = rb[j + 1] - rb[j];
        CK(cudaMemcpyAsync(sk + rb[j], k + rb[j], sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, c->st));
        CK(cudaMemcpyAsync(sv + rb[j], v + rb[j], sizeof(VT) * n, cudaMemcpyDeviceToDevice, c->st));
        nb.push_back(rb[j + 1]);
      }
    }
    CK(cudaGetLastError());
    std::swap(k, sk);
    std::swap(v, sv);
    rb.swap(nb);
  }
}

// Copy k from composite keys already sorted (merge_runs): split, directory.
void finish_mode_presorted(cparls_ctx *c, int k, int64_t nnz, uint64_t *comp, void *val) {
  ModeIndex &ix = c->idx[k];
  ix.nnz = nnz;
  copy_order(c, k, ix.order);
  const unsigned g = (unsigned)std::min<int64_t>(148 * 16, std::max<int64_t>(1, ceil_div(nnz, 256)));
  ix.out = dalloc_t<int32_t>(c, nnz);
  if (nnz > 0) {
    k_split_comp<<<g, 256, 0, c->st>>>(comp, nnz, make_fastdiv((uint64_t)c->dims[k]), ix.out);
    CK_LAUNCH();
  }
  ix.key = comp;
  ix.val = val;
  build_directory(c, k);
  sync(c);
}

// Chunked host->device copy of the COO in flight on its own stream (cparls_create):
// chunk i covers nonzeros [end[i-1], end[i]) and is resident once ev[i] fires.
struct H2DChunks {
  static constexpr int64_t kMinSplit = int64_t(1) << 27;
  // chunk ends: 4 chunks of 40/30/20/10% above kMinSplit nonzeros (each chunk's
  // sorts take about as long as the next chunk's transfer, the last chunk is
  // small -- little left to sort after the transfer -- and 4 runs merge in 2
  // rounds); one chunk below
  static std::vector<int64_t> plan(int64_t nnz) {
    if (nnz < kMinSplit) return {nnz};
    const int64_t a = nnz / 10 * 4, b = a + nnz / 10 * 3, c = b + nnz / 10 * 2;
    return {a, b, c, nnz};
  }
  cudaStream_t cs = nullptr;
  cudaEvent_t ev0 = nullptr;
  std::vector<int64_t> end;
  std::vector<cudaEvent_t> ev;
  H2DChunks() { CK(cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming)); }
  ~H2DChunks() {   // every user of the chunks is ordered after them on c->st by then
    if (cs) cudaStreamSynchronize(cs);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    if (ev0) cudaEventDestroy(ev0);
    if (cs) cudaStreamDestroy(cs);
  }
  H2DChunks(const H2DChunks &) = delete;
  H2DChunks &operator=(const H2DChunks &) = delete;
  void wait_all(cudaStream_t st) const {
    if (!ev.empty()) CK(cudaStreamWaitEvent(st, ev.back(), 0));
  }
};

template <typename IT, typename VT>
void build_all(cparls_ctx *c, const IT *coords, const VT *vals, const H2DChunks *hc) {
  KeySpec ks{};
  ks.D = c->D;
  for (int m = 0; m < c->D; ++m) ks.dims[m] = c->dims[m];
  long double Nall = 1;
  for (int m = 0; m < c->D; ++m) Nall *= (long double)c->dims[m];
  const bool single_sort = c->world == 1 && Nall <= 18446744073709551615.0L && c->D >= 2;
  BuildArena ar;
  bool comp0_made = false;
  // create from host: every mode's composite keys of chunk i are made and
  // sorted while chunks > i are still crossing PCIe (sorted runs, one per
  // chunk and mode); the runs are merged once the input is complete
  // (merge_runs).  Stable throughout, so the copies equal those of the
  // single full sort bit for bit.
  std::vector<uint64_t *> rk;
  std::vector<VT *> rv;
  std::vector<int64_t> rb;
  if (single_sort && hc && c->nnz > 0 && hc->ev.size() > 1) {
    const int D = c->D;
    const int64_t nnz = c->nnz;
    const size_t pair = sizeof(uint64_t) + sizeof(VT);
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    const int64_t cmax = hc->end[0];
    const size_t need = pair * (size_t)nnz * (D + 1) + sizeof(int32_t) * (size_t)nnz * D + pair * (size_t)cmax * 2 +
                        (size_t(6) << 30);
    if (need < fr) {
      ar.cbits = key_bits(Nall);
      rk.resize(D);
      rv.resize(D);
      for (int k = 0; k < D; ++k) {
        rk[k] = dalloc_t<uint64_t>(c, nnz);
        rv[k] = (VT *)dalloc(c, sizeof(VT) * (size_t)nnz);
      }
      uint64_t *ck = dalloc_t<uint64_t>(c, cmax);
      VT *cv = (VT *)dalloc(c, sizeof(VT) * (size_t)cmax);
      size_t tb = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, ck, rk[0], cv, rv[0], cmax, 0, ar.cbits, c->st));
      void *tmp = dalloc(c, tb);
      KeySpec km[kMaxModes];
      for (int k = 0; k < D; ++k) {
        km[k] = KeySpec{};
        km[k].D = D;
        km[k].k = k;
        for (int m = 0; m < D; ++m) km[k].dims[m] = c->dims[m];
        int ord[kMaxModes];
        copy_order(c, k, ord);
        for (int j = 0; j < D - 1; ++j) km[k].order[j] = ord[j];
      }
      rb.push_back(0);
      int64_t e0 = 0;
      for (size_t i = 0; i < hc->ev.size(); ++i) {
        const int64_t n = hc->end[i] - e0;
        CK(cudaStreamWaitEvent(c->st, hc->ev[i], 0));
        const unsigned g = (unsigned)std::min<int64_t>(148 * 16, std::max<int64_t>(1, ceil_div(n, 256)));
        for (int k = 0; k < D; ++k) {
          k_make_comp<IT, VT><<<g, 256, 0, c->st>>>(coords + e0 * D, vals + e0, n, km[k], ck, cv);
          CK_LAUNCH();
          CK(cub::DeviceRadixSort::SortPairs(tmp, tb, ck, rk[k] + e0, cv, rv[k] + e0, n, 0, ar.cbits, c->st));
        }
        e0 = hc->end[i];
        rb.push_back(e0);
      }
      sync(c);
      dfree(c, tmp);
      dfree(c, ck);
      dfree(c, cv);
    }
  }
  if (hc) hc->wait_all(c->st);
  CK(cudaMemsetAsync(&c->dv->bad, 0, sizeof(unsigned long long), c->st));
  if (c->nnz > 0) {
    k_check_coords<IT><<<(unsigned)ceil_div(c->nnz, 256), 256, 0, c->st>>>(coords, c->nnz, ks, &c->dv->bad);
    CK_LAUNCH();
  }
  if (read_dev(c, &c->dv->bad) != 0) throw ApiError(CPARLS_ERANGE, "coordinate out of range [0, n_k)");
  // ||X||^2 (compensated; summed over ranks)
  const int nb = 296;
  k_sumsq<VT><<<nb, 256, 0, c->st>>>(vals, c->nnz, c->ddpart, &c->dv->maxabs);
  CK_LAUNCH();
  k_sum_dd_final<<<1, 32, 0, c->st>>>(c->ddpart, nb, &c->dv->normX2);
  CK_LAUNCH();
  if (c->world > 1) {
    c->comm->allreduce_f64(&c->dv->normX2, 1, c->st);
    c->comm->allreduce_f64(&c->dv->maxabs, 1, c->st);   // sum of the ranks' maxima: a common upper bound
  }
  c->normX2 = read_dev(c, &c->dv->normX2);
  if (single_sort && !rk.empty()) {
    // merge each mode's runs (the spare pair of buffers passes from mode to mode)
    uint64_t *sk = dalloc_t<uint64_t>(c, c->nnz);
    VT *sv = (VT *)dalloc(c, sizeof(VT) * (size_t)c->nnz);
    for (int k = 0; k < c->D; ++k) {
      c->row_lo[k] = 0;
      c->row_hi[k] = c->dims[k];
      {
        WallAcc ws(&c->stats.build_ms[1]);
        merge_runs<VT>(c, rb, rk[k], rv[k], sk, sv);
        sync(c);
      }
      finish_mode_presorted(c, k, c->nnz, rk[k], rv[k]);
    }
    sync(c);
    dfree(c, sk);
    dfree(c, sv);
    degrees_and_hot_rows(c);
    return;
  }
  if (single_sort) {
    if (!comp0_made) {
      ar.cbits = key_bits(Nall);
      arena_alloc<VT>(c, ar, c->nnz);
    }
    for (int k = 0; k < c->D; ++k) {
      c->row_lo[k] = 0;
      c->row_hi[k] = c->dims[k];
      build_index_mode_comp<IT, VT>(c, k, coords, vals, c->nnz, ar, k == c->D - 1, k == 0 && comp0_made);
    }
    sync(c);
    for (int i = 0; i < 2; ++i) {
      dfree(c, ar.comp[i]);
      dfree(c, ar.val[i]);
    }
    dfree(c, ar.tmp);
    degrees_and_hot_rows(c);
    return;
  }
  for (int k = 0; k < c->D; ++k) {
    if (c->world == 1) {
      c->row_lo[k] = 0;
      c->row_hi[k] = c->dims[k];
      build_index_mode<IT, VT>(c, k, coords, vals, c->nnz);
    } else {
      route_and_build<IT, VT>(c, k, coords, vals);
    }
  }
}

// the single-pass scan's tile states for n items (new memory is zeroed: epoch 0
// never matches a call's epoch >= 1)
void ensure_scan(cparls_ctx *c, int64_t n) {
  const int64_t need = ceil_div(std::max<int64_t>(n, 1), kScanTile) + 1;
  if (!c->scan.ticket) {
    c->scan.ticket = dalloc_t<unsigned long long>(c, 1);
    CK(cudaMemsetAsync(c->scan.ticket, 0, sizeof(unsigned long long), c->st));
  }
  if (need <= c->scan.cap) return;
  dfree(c, c->scan.flag);   // cudaFree waits for the kernels still using them
  dfree(c, c->scan.agg);
  dfree(c, c->scan.inc);
  c->scan.cap = std::max(need, 2 * c->scan.cap);
  c->scan.flag = dalloc_t<unsigned long long>(c, c->scan.cap);
  c->scan.agg = dalloc_t<int64_t>(c, c->scan.cap);
  c->scan.inc = dalloc_t<int64_t>(c, c->scan.cap);
  CK(cudaMemsetAsync(c->scan.flag, 0, sizeof(unsigned long long) * c->scan.cap, c->st));
}

// exclusive_scan_i64 over n items needs ceil(n / kScanTile) partials
void ensure_i64part(cparls_ctx *c, int64_t n) {
  const int64_t need = ceil_div(std::max<int64_t>(n, 1), kScanTile) + 64;
  if (need <= c->i64part_cap) return;
  dfree(c, c->i64part);   // cudaFree waits for the kernels still reading it
  c->i64part_cap = std::max(need, 2 * c->i64part_cap);
  c->i64part = dalloc_t<int64_t>(c, c->i64part_cap);
}

void alloc_sample_buffers(cparls_ctx *c, int64_t s) {
  if (s <= c->scap) return;
  int64_t cap = std::max<int64_t>(s, 1024);
  for (void *p : {(void *)c->skey, (void *)c->sw2, (void *)c->sp, (void *)c->scnt, (void *)c->sisdet, (void *)c->Z,
                  (void *)c->lo, (void *)c->len, (void *)c->off, (void *)c->rkey, (void *)c->rp, (void *)c->hkey,
                  (void *)c->hcnt, (void *)c->hp, (void *)c->skey2, (void *)c->sw2_2, (void *)c->sp2,
                  (void *)c->scnt2, (void *)c->sisdet2, (void *)c->sperm, (void *)c->sperm2, (void *)c->shist,
                  (void *)c->hfirst, (void *)c->rslot, (void *)c->rflag, (void *)c->rpos})
    dfree(c, p);
  c->skey = dalloc_t<uint64_t>(c, cap);
  c->sw2 = dalloc_t<double>(c, cap);
  c->sp = dalloc_t<double>(c, cap);
  c->scnt = dalloc_t<int32_t>(c, cap);
  c->sisdet = dalloc_t<uint8_t>(c, cap);
  c->Z = dalloc_t<double>(c, cap * c->ld);
  c->lo = dalloc_t<int64_t>(c, cap);
  c->len = dalloc_t<int64_t>(c, cap);
  c->off = dalloc_t<int64_t>(c, cap);
  c->rkey = dalloc_t<uint64_t>(c, cap);
  c->rp = dalloc_t<double>(c, cap);
  c->skey2 = dalloc_t<uint64_t>(c, cap);
  c->sw2_2 = dalloc_t<double>(c, cap);
  c->sp2 = dalloc_t<double>(c, cap);
  c->scnt2 = dalloc_t<int32_t>(c, cap);
  c->sisdet2 = dalloc_t<uint8_t>(c, cap);
  c->sperm = dalloc_t<uint32_t>(c, cap);
  c->sperm2 = dalloc_t<uint32_t>(c, cap);
  c->shist = dalloc_t<uint32_t>(c, 256 * (ceil_div(cap, kScanTile) + 1));
  uint64_t hs = 1;
  while (hs < (uint64_t)(2 * cap)) hs <<= 1;
  c->hsize = hs;
  c->hkey = dalloc_t<unsigned long long>(c, (int64_t)hs);
  c->hcnt = dalloc_t<uint32_t>(c, (int64_t)hs);
  c->hp = dalloc_t<double>(c, (int64_t)hs);
  c->hfirst = dalloc_t<uint32_t>(c, (int64_t)hs);
  CK(cudaMemsetAsync(c->hfirst, 0xFF, sizeof(uint32_t) * hs, c->st));
  c->rslot = dalloc_t<uint32_t>(c, cap);
  c->rflag = dalloc_t<int64_t>(c, cap);
  c->rpos = dalloc_t<int64_t>(c, cap);
  CK(cudaMemsetAsync(c->hkey, 0xFF, sizeof(unsigned long long) * hs, c->st));
  CK(cudaMemsetAsync(c->hcnt, 0, sizeof(uint32_t) * hs, c->st));
  ensure_i64part(c, cap);   // scans over the accepted draws and the sample (<= s)
  // SIDX look-back tiles of the asynchronous sampler: attempts <= the cap (AMB-7)
  const int64_t cap_att = c->opts.attempt_cap > 0 ? c->opts.attempt_cap : 1024 * cap + 65536;
  const int64_t tiles = ceil_div(cap_att, kSidxTile) + 2;
  if (tiles > c->tile_cap) {
    dfree(c, c->tile_state);
    c->tile_state = dalloc_t<unsigned long long>(c, tiles);
    CK(cudaMemsetAsync(c->tile_state, 0, sizeof(unsigned long long) * tiles, c->st));   // epoch 0: unpublished
    c->tile_cap = tiles;
  }
  c->scap = cap;
}

void ensure_list_cap(cparls_ctx *c, int64_t need) {
  if (need <= c->lcap) return;
  int64_t cap = std::max<int64_t>(need, c->lcap * 2);
  for (int i = 0; i < 2; ++i) {
    dfree(c, c->lkey[i]);
    dfree(c, c->lpp[i]);
  }
  dfree(c, c->lcnt);
  dfree(c, c->loff);
  for (int i = 0; i < 2; ++i) {
    c->lkey[i] = dalloc_t<uint64_t>(c, cap);
    c->lpp[i] = dalloc_t<double>(c, cap);
  }
  c->lcnt = dalloc_t<int64_t>(c, cap);
  c->loff = dalloc_t<int64_t>(c, cap);
  c->lcap = cap;
}

// ---------------------------------------------------------------- sampling
// DIDX: returns s_det; list in lkey[res]/lpp[res] (res returned via *which)
int64_t run_didx(cparls_ctx *c, const OtherModes &om, double tau, int *which) {
  const int d = om.d;
  int64_t ncand[kMaxModes] = {0};
  // candidates per mode (ordered compaction), then stable sort by p~ descending
  // every mode's candidates first (independent), then one read of all counts
  // (a sync per mode before)
  for (int j = 0; j < d; ++j) {
    const int64_t n = om.n[j];
    const int64_t nb = ceil_div(n, kScanTile);
    k_cand_count<<<(unsigned)nb, kScanThreads, 0, c->st>>>(om, j, tau, c->i64part);
    CK_LAUNCH();
    k_scan_part<<<1, kScanThreads, 0, c->st>>>(c->i64part, nb, &c->dv->total);
    CK_LAUNCH();
    k_cand_scatter<<<(unsigned)nb, kScanThreads, 0, c->st>>>(om, j, tau, c->i64part, c->ckey[j], c->cidx[j]);
    CK_LAUNCH();
    LAUNCHED(c, 3);
    CK(cudaMemcpyAsync(c->hscr + kHscrCand + j, &c->dv->total, sizeof(long long), cudaMemcpyDeviceToHost, c->st));
  }
  sync(c);
  for (int j = 0; j < d; ++j) {
    const int64_t n = om.n[j];
    const int64_t nc = c->hscr[kHscrCand + j];
    if (nc > 1) {
      int res = radix_sort_pairs(c->ckey[j], c->cidx[j], c->ckey_tmp, c->cidx_tmp, nc, 64, c->rhist, c->st,
                                 &c->stats.kernel_launches);
      if (res == 1) {
        CK(cudaMemcpyAsync(c->ckey[j], c->ckey_tmp, sizeof(uint64_t) * nc, cudaMemcpyDeviceToDevice, c->st));
        CK(cudaMemcpyAsync(c->cidx[j], c->cidx_tmp, sizeof(uint32_t) * nc, cudaMemcpyDeviceToDevice, c->st));
      }
    }
    c->stats.bytes_sample += (double)n * 8.0;
    ncand[j] = nc;
  }
  // level expansion (DetSet is a subset of the product of the
  // candidate sets); the exact canonical predicate decides membership.
  const int64_t n0 = ncand[0];
  ensure_list_cap(c, std::max<int64_t>(n0, 1));
  int cur = 0;
  if (n0 > 0) {
    k_didx_level0<<<(unsigned)ceil_div(n0, 256), 256, 0, c->st>>>(c->ckey[0], c->cidx[0], n0, c->lkey[0], c->lpp[0]);
    CK_LAUNCH();
    LAUNCHED(c, 1);
  }
  int64_t nlist = n0;
  const int64_t cap = c->opts.didx_cap > 0 ? c->opts.didx_cap : (int64_t(1) << 22);
  if (nlist > cap) throw ApiError(CPARLS_ESAMPLE, "DIDX list exceeds didx_cap");
  for (int l = 1; l < d && nlist > 0; ++l) {
    const int64_t ncl = ncand[l];
    if (ncl == 0) {
      nlist = 0;
      break;
    }
    ensure_i64part(c, nlist);
    k_didx_count<<<(unsigned)ceil_div(nlist, 256), 256, 0, c->st>>>(c->lpp[cur], nlist, c->ckey[l], ncl, om, l, tau,
                                                                    c->lcnt);
    CK_LAUNCH();
    exclusive_scan_i64(c->lcnt, c->loff, nlist, c->i64part, &c->dv->total, c->st);
    LAUNCHED(c, 4);
    const int64_t nn = read_dev(c, &c->dv->total);
    if (nn > cap) throw ApiError(CPARLS_ESAMPLE, "DIDX list exceeds didx_cap (" + std::to_string(nn) + ")");
    if (nn > c->lcap) {
      // grow, keeping the current level
      uint64_t *k0 = dalloc_t<uint64_t>(c, nlist);
      double *p0 = dalloc_t<double>(c, nlist);
      int64_t *cnt0 = dalloc_t<int64_t>(c, nlist), *off0 = dalloc_t<int64_t>(c, nlist);
      CK(cudaMemcpyAsync(k0, c->lkey[cur], 8 * nlist, cudaMemcpyDeviceToDevice, c->st));
      CK(cudaMemcpyAsync(p0, c->lpp[cur], 8 * nlist, cudaMemcpyDeviceToDevice, c->st));
      CK(cudaMemcpyAsync(cnt0, c->lcnt, 8 * nlist, cudaMemcpyDeviceToDevice, c->st));
      CK(cudaMemcpyAsync(off0, c->loff, 8 * nlist, cudaMemcpyDeviceToDevice, c->st));
      sync(c);
      ensure_list_cap(c, nn);
      CK(cudaMemcpyAsync(c->lkey[cur], k0, 8 * nlist, cudaMemcpyDeviceToDevice, c->st));
      CK(cudaMemcpyAsync(c->lpp[cur], p0, 8 * nlist, cudaMemcpyDeviceToDevice, c->st));
      CK(cudaMemcpyAsync(c->lcnt, cnt0, 8 * nlist, cudaMemcpyDeviceToDevice, c->st));
      CK(cudaMemcpyAsync(c->loff, off0, 8 * nlist, cudaMemcpyDeviceToDevice, c->st));
      sync(c);
      dfree(c, k0);
      dfree(c, p0);
      dfree(c, cnt0);
      dfree(c, off0);
    }
    if (nn > 0) {
      k_didx_emit<<<(unsigned)ceil_div(nlist * 32, 256), 256, 0, c->st>>>(c->lkey[cur], c->lpp[cur], nlist, c->lcnt,
                                                                          c->loff, c->ckey[l], c->cidx[l], om.mult[l],
                                                                          c->lkey[cur ^ 1], c->lpp[cur ^ 1]);
      CK_LAUNCH();
      LAUNCHED(c, 1);
    }
    cur ^= 1;
    nlist = nn;
  }
  *which = cur;
  return nlist;
}

void sample_host(cparls_ctx *c, int k, int64_t s, uint64_t seed, uint64_t step) {
  Phase ph(c, &c->stats.ms_sample);
  c->have_sample = false;
  c->have_lookup = false;
  if (s < 1) throw ApiError(CPARLS_EINVAL, "s must be >= 1");
  alloc_sample_buffers(c, s);
  double tau = c->tau;
  if (tau < 0) tau = 1.0 / (double)s;   // tau = 1/s
  OtherModes om = other_modes(c, k);
  const int d = om.d;
  // drawable counts (rows with q > 0): copied into pinned scratch now, read
  // after the p_det sync below (stream order), no sync of their own
  long long *drawable = c->hscr + kHscrDrawable;
  for (int j = 0; j < d; ++j)
    CK(cudaMemcpyAsync(&drawable[j], &c->md[om.mode[j]]->drawable, sizeof(long long), cudaMemcpyDeviceToHost,
                       c->st));
  // ---- DIDX
  int which = 0;
  int64_t sdet = run_didx(c, om, tau, &which);
  uint64_t *dkey = c->lkey[which];
  double *dp = c->lpp[which];
  if (sdet > s) {
    // keep the s largest p (ties: smaller key first), AMB-6
    ensure_list_cap(c, sdet);
    dkey = c->lkey[which];
    dp = c->lpp[which];
    uint64_t *k1 = dalloc_t<uint64_t>(c, sdet), *k2 = dalloc_t<uint64_t>(c, sdet);
    uint32_t *v1 = dalloc_t<uint32_t>(c, sdet), *v2 = dalloc_t<uint32_t>(c, sdet);
    uint32_t *h = dalloc_t<uint32_t>(c, 256 * (ceil_div(sdet, kScanTile) + 1));
    unsigned g = (unsigned)ceil_div(sdet, 256);
    CK(cudaMemcpyAsync(k1, dkey, 8 * sdet, cudaMemcpyDeviceToDevice, c->st));
    k_iota_u32<<<g, 256, 0, c->st>>>(v1, sdet);
    int res = radix_sort_pairs(k1, v1, k2, v2, sdet, 64, h, c->st, &c->stats.kernel_launches);
    uint32_t *perm = res ? v2 : v1;
    uint64_t *pk = res ? k1 : k2;   // free key buffer
    k_gather_kp<<<g, 256, 0, c->st>>>(dkey, dp, perm, sdet, c->lkey[which ^ 1], c->lpp[which ^ 1]);
    k_pbits_desc<<<g, 256, 0, c->st>>>(c->lpp[which ^ 1], sdet, pk);
    uint32_t *vv = res ? v1 : v2;
    k_iota_u32<<<g, 256, 0, c->st>>>(vv, sdet);
    uint64_t *ko = (pk == k1) ? k2 : k1;
    uint32_t *vo = (vv == v1) ? v2 : v1;
    int res2 = radix_sort_pairs(pk, vv, ko, vo, sdet, 64, h, c->st, &c->stats.kernel_launches);
    uint32_t *perm2 = res2 ? vo : vv;
    k_gather_kp<<<g, 256, 0, c->st>>>(c->lkey[which ^ 1], c->lpp[which ^ 1], perm2, sdet, dkey, dp);
    CK_LAUNCH();
    sync(c);
    dfree(c, k1); dfree(c, k2); dfree(c, v1); dfree(c, v2); dfree(c, h);
    sdet = s;
  }
  // p_det = sum_{DetSet} p_i (compensated)
  const int nbs = 64;
  k_sum_dd<<<nbs, 256, 0, c->st>>>(dp, sdet, c->ddpart);
  k_sum_dd_final<<<1, 32, 0, c->st>>>(c->ddpart, nbs, &c->dv->pdet);
  CK_LAUNCH();
  LAUNCHED(c, 2);
  double p_det = read_dev(c, &c->dv->pdet);
  if (sdet > 0) {
    k_det_emit<<<(unsigned)ceil_div(sdet, 256), 256, 0, c->st>>>(dkey, dp, sdet, c->skey, c->sw2, c->sp, c->scnt,
                                                                 c->sisdet);
    CK_LAUNCH();
    LAUNCHED(c, 1);
  }
  // ---- SIDX (Alg. 2)
  int64_t s_rnd = s - sdet;
  int64_t det_drawable = sdet;   // tau >= 2^-63 => every det index has q > 0
  if (tau < 1.0842021724855044e-19 && sdet > 0) {
    std::vector<uint64_t> hk(sdet);
    CK(cudaMemcpyAsync(hk.data(), dkey, 8 * sdet, cudaMemcpyDeviceToHost, c->st));
    std::vector<std::vector<double>> hp(d);
    for (int j = 0; j < d; ++j) {
      hp[j].resize(om.n[j]);
      CK(cudaMemcpyAsync(hp[j].data(), om.pt[j], 8 * om.n[j], cudaMemcpyDeviceToHost, c->st));
    }
    sync(c);
    det_drawable = 0;
    for (int64_t i = 0; i < sdet; ++i) {
      uint64_t t = hk[i];
      bool ok = true;
      for (int j = 0; j < d; ++j) {
        uint64_t ii = t % (uint64_t)om.n[j];
        t /= (uint64_t)om.n[j];
        ok &= hp[j][ii] > 1.0842021724855044e-19;
      }
      det_drawable += ok;
    }
  }
  double drawable_all = 1.0;
  for (int j = 0; j < d; ++j) drawable_all *= (double)drawable[j];
  int skipped = 0;
  int64_t attempts = 0;
  int64_t have = 0;
  if (s_rnd > 0) {
    if (1.0 - p_det <= 1e-12 || drawable_all <= (double)det_drawable) {
      skipped = 1;   // AMB-7
    } else {
      const int64_t cap_att = c->opts.attempt_cap > 0 ? c->opts.attempt_cap : 1024 * s_rnd + 65536;
      uint64_t a0 = 0;
      const uint32_t slo = (uint32_t)seed, shi = (uint32_t)(seed >> 32);
      while (have < s_rnd) {
        if ((int64_t)a0 >= cap_att) throw ApiError(CPARLS_ESAMPLE, "SIDX attempt cap reached");
        double accp = std::max(1.0 - p_det, 1e-3);
        int64_t want = (int64_t)std::ceil((double)(s_rnd - have) / accp * 1.08) + 4096;
        int64_t win = std::min<int64_t>(std::max<int64_t>(want, 4096), c->acap);
        win = std::min<int64_t>(win, cap_att - (int64_t)a0);
        if (c->opts.sidx_window > 0) win = std::min<int64_t>(win, c->opts.sidx_window);   // AMB-8: result-neutral
        int64_t nb = ceil_div(win, kSidxThreads);
        k_sidx_gen<<<(unsigned)nb, kSidxThreads, 0, c->st>>>(om, a0, win, tau, slo, shi, (uint32_t)step, c->akey,
                                                             c->ap, c->i64part);
        CK_LAUNCH();
        k_scan_part<<<1, kScanThreads, 0, c->st>>>(c->i64part, nb, &c->dv->total);
        CK_LAUNCH();
        k_sidx_scatter<<<(unsigned)nb, kSidxThreads, 0, c->st>>>(c->akey, c->ap, win, c->i64part, have, s_rnd, a0,
                                                                 c->rkey, c->rp, &c->dv->last_attempt);
        CK_LAUNCH();
        LAUNCHED(c, 3);
        // total and last_attempt (adjacent) in one read
        static_assert(offsetof(DevScalars, last_attempt) == offsetof(DevScalars, total) + 8, "layout");
        CK(cudaMemcpyAsync(c->hscr + kHscrSidx, &c->dv->total, 16, cudaMemcpyDeviceToHost, c->st));
        sync(c);
        const int64_t got = c->hscr[kHscrSidx];
        have += std::min<int64_t>(got, s_rnd - have);
        a0 += (uint64_t)win;
        c->stats.bytes_sample += (double)win * d * 8.0;
        if (have >= s_rnd) attempts = (int64_t)(unsigned long long)c->hscr[kHscrSidx + 1] + 1;
      }
    }
  }
  // ---- CIDX (combine repeats)
  int64_t nuniq = 0;
  if (have > 0) {
    // deterministic combine: unique rows in first-draw order (AMB-35)
    const unsigned gb = (unsigned)ceil_div(have, 256);
    k_cidx_insert_first<<<gb, 256, 0, c->st>>>(c->rkey, c->rp, have, c->hkey, c->hcnt, c->hp, c->hfirst,
                                               c->hsize - 1);
    CK_LAUNCH();
    k_cidx_first_flags<<<gb, 256, 0, c->st>>>(c->rkey, have, c->hkey, c->hfirst, c->hsize - 1, c->rflag, c->rslot);
    CK_LAUNCH();
    exclusive_scan_i64(c->rflag, c->rpos, have, c->i64part, &c->dv->total, c->st);
    k_cidx_emit_first<<<gb, 256, 0, c->st>>>(c->rflag, c->rpos, c->rslot, have, c->hkey, c->hcnt, c->hp,
                                             c->hfirst, &c->dv->pdet, s_rnd, sdet, c->skey, c->sw2, c->sp,
                                             c->scnt, c->sisdet);
    CK_LAUNCH();
    LAUNCHED(c, 6);
    nuniq = (int64_t)read_dev(c, &c->dv->total);
  }
  // The device order is already deterministic (DIDX list order, then the
  // random rows in first-draw order), so Z, the sampled Gram and the solve are
  // bit-reproducible (AMB-35).  CPARLS_SAMPLE_SORT=1 additionally sorts the
  // sample by key (walks factor rows and the fiber directory in key order).
  if (c->sample_sort && sdet + nuniq > 1) {
    const int64_t n = sdet + nuniq;
    int end_bit = 0;
    {
      unsigned __int128 prod = 1;
      for (int j = 0; j < d; ++j) prod *= (unsigned __int128)om.n[j];
      while (end_bit < 64 && (((unsigned __int128)1) << end_bit) < prod) ++end_bit;
    }
    const unsigned g = (unsigned)ceil_div(n, 256);
    k_iota_u32<<<g, 256, 0, c->st>>>(c->sperm, n);
    CK_LAUNCH();
    int res = radix_sort_pairs(c->skey, c->sperm, c->skey2, c->sperm2, n, end_bit, c->shist, c->st,
                               &c->stats.kernel_launches);
    if (res) std::swap(c->skey, c->skey2);   // sorted keys
    const uint32_t *perm = res ? c->sperm2 : c->sperm;
    k_sample_permute<<<g, 256, 0, c->st>>>(perm, n, c->sw2, c->sp, c->scnt, c->sisdet, c->sw2_2, c->sp2, c->scnt2,
                                           c->sisdet2);
    CK_LAUNCH();
    std::swap(c->sw2, c->sw2_2);
    std::swap(c->sp, c->sp2);
    std::swap(c->scnt, c->scnt2);
    std::swap(c->sisdet, c->sisdet2);
    LAUNCHED(c, 2);
  }
  c->smode = k;
  c->sdet = sdet;
  c->s_rnd = s_rnd;
  c->sbar = sdet + nuniq;
  c->p_det = p_det;
  c->attempts = attempts;
  c->skipped = skipped;
  c->have_sample = true;
  c->s_cur = s;
  ph.end();
}

// ---------------------------------------------------------------- asynchronous sampling
// SkrpLev (Alg. 1) for mode k with every size on the device
// (StepCtl, sampler.cuh): no host synchronisation.  The rare branches (more
// than kSmallSortMax candidates of a mode, a DIDX level beyond the list
// buffers or didx_cap, the AMB-6 truncation, tau < 2^-63, the SIDX attempt
// cap) raise ctl->abort; the host then redoes the step with sample_host.
void sample_async(cparls_ctx *c, int k, int64_t s, uint64_t seed, uint64_t step) {
  if (s < 1) throw ApiError(CPARLS_EINVAL, "s must be >= 1");
  alloc_sample_buffers(c, s);
  double tau = c->tau;
  if (tau < 0) tau = 1.0 / (double)s;   // tau = 1/s
  OtherModes om = other_modes(c, k);
  const int d = om.d;
  StepCtl *ctl = c->ctl;
  const int64_t st64 = (int64_t)step;
  Phase ph(c, &c->stats.ms_sample);
  // ---- DIDX candidates of every other mode, sorted by p~ descending
  {
    CandBufs cb{};
    int64_t total = 0;
    for (int j = 0; j < d; ++j) {
      cb.key[j] = c->ckey[j];
      cb.idx[j] = c->cidx[j];
      total += om.n[j];
      c->stats.bytes_sample += (double)om.n[j] * 8.0;
    }
    k_cand_append<<<(unsigned)std::min<int64_t>(148 * 8, ceil_div(total, 256)), 256, 0, c->st>>>(om, tau, cb, ctl);
    CK_LAUNCH();
    k_cand_sort<<<(unsigned)d, kSmallSortThreads, 0, c->st>>>(cb, ctl, st64);
    CK_LAUNCH();
    LAUNCHED(c, 2);
  }
  // ---- DIDX levels: the exact canonical predicate decides membership
  const int64_t cap = c->opts.didx_cap > 0 ? c->opts.didx_cap : (int64_t(1) << 22);
  const int64_t lcap = c->lcap;
  ensure_i64part(c, lcap);
  const unsigned gl = (unsigned)ceil_div(kSmallSortMax, 256);
  const unsigned gs = 148 * 4;
  k_didx_level0<<<gl, 256, 0, c->st>>>(c->ckey[0], c->cidx[0], 0, c->lkey[0], c->lpp[0], &ctl->ncand[0], ctl);
  CK_LAUNCH();
  k_didx_start<<<1, 1, 0, c->st>>>(ctl, lcap, cap, st64);
  CK_LAUNCH();
  LAUNCHED(c, 2);
  int cur = 0;
  for (int l = 1; l < d; ++l) {
    k_didx_count<<<gs, 256, 0, c->st>>>(c->lpp[cur], lcap, c->ckey[l], 0, om, l, tau, c->lcnt, &ctl->nlist,
                                        &ctl->ncand[l], ctl);
    CK_LAUNCH();
    ensure_scan(c, lcap);
    exclusive_scan_i64_1p(c->lcnt, c->loff, lcap, &ctl->nlist, &ctl->scan_total, c->scan, c->st, ctl);
    k_didx_check<<<1, 1, 0, c->st>>>(ctl, lcap, cap, st64);
    CK_LAUNCH();
    k_didx_emit<<<gs, 256, 0, c->st>>>(c->lkey[cur], c->lpp[cur], lcap, c->lcnt, c->loff, c->ckey[l], c->cidx[l],
                                       om.mult[l], c->lkey[cur ^ 1], c->lpp[cur ^ 1], &ctl->nlist, ctl);
    CK_LAUNCH();
    k_didx_advance<<<1, 1, 0, c->st>>>(ctl);
    CK_LAUNCH();
    LAUNCHED(c, 5);
    cur ^= 1;
  }
  k_didx_finish<<<1, 1, 0, c->st>>>(ctl, s, tau < 1.0842021724855044e-19 ? 1 : 0, st64);
  CK_LAUNCH();
  // p_det = sum_{DetSet} p_i (compensated, the host path's reduction order)
  const int nbs = 64;
  k_sum_dd<<<nbs, 256, 0, c->st>>>(c->lpp[cur], 0, c->ddpart, &ctl->sdet, ctl);
  CK_LAUNCH();
  k_sum_dd_final<<<1, 32, 0, c->st>>>(c->ddpart, nbs, &ctl->pdet, ctl);
  CK_LAUNCH();
  const unsigned gsamp = (unsigned)ceil_div(s, 256);
  k_det_emit<<<gsamp, 256, 0, c->st>>>(c->lkey[cur], c->lpp[cur], 0, c->skey, c->sw2, c->sp, c->scnt, c->sisdet,
                                       &ctl->sdet, ctl);
  CK_LAUNCH();
  LAUNCHED(c, 4);
  // ---- SIDX (Alg. 2): one persistent kernel until s_rnd acceptances
  k_sidx_prep<<<1, 1, 0, c->st>>>(ctl, om, s);
  CK_LAUNCH();
  {
    const unsigned gsidx = (unsigned)std::min<int64_t>(148 * 4, ceil_div(s, kSidxTile) + 8);
    k_sidx_run<<<gsidx, kSidxThreads, 0, c->st>>>(om, tau, (uint32_t)seed, (uint32_t)(seed >> 32), (uint32_t)step,
                                                  c->opts.attempt_cap, ctl, c->tile_state, c->tile_cap, c->rkey,
                                                  c->rp, st64);
    CK_LAUNCH();
  }
  // ---- CIDX: unique rows in first-draw order (AMB-35)
  k_cidx_insert_first<<<gsamp, 256, 0, c->st>>>(c->rkey, c->rp, 0, c->hkey, c->hcnt, c->hp, c->hfirst, c->hsize - 1,
                                                 &ctl->have, ctl);
  CK_LAUNCH();
  k_cidx_first_flags<<<gsamp, 256, 0, c->st>>>(c->rkey, 0, c->hkey, c->hfirst, c->hsize - 1, c->rflag, c->rslot,
                                               &ctl->have, ctl);
  CK_LAUNCH();
  ensure_scan(c, s);
  exclusive_scan_i64_1p(c->rflag, c->rpos, s, &ctl->have, &ctl->nuniq, c->scan, c->st, ctl);
  k_cidx_emit_first<<<gsamp, 256, 0, c->st>>>(c->rflag, c->rpos, c->rslot, 0, c->hkey, c->hcnt, c->hp, c->hfirst,
                                              &ctl->pdet, 0, 0, c->skey, c->sw2, c->sp, c->scnt, c->sisdet, ctl);
  CK_LAUNCH();
  k_sample_finish<<<1, 1, 0, c->st>>>(ctl);
  CK_LAUNCH();
  LAUNCHED(c, 8);
  c->smode = k;
  c->s_cur = s;
  c->have_sample = true;
  c->have_lookup = false;
  c->sample_pulled = false;
  ph.end();
}

// The sample scalars of the host path into the step control (the solve reads
// them there).  The stream is idle after sync(), so the control block can be
// rewritten whole.
void push_sample_state(cparls_ctx *c) {
  sync(c);
  StepCtl h = *reinterpret_cast<const StepCtl *>(c->hctl);
  h.sdet = c->sdet;
  h.s_rnd = c->s_rnd;
  h.skip = c->skipped;
  h.have = c->skipped ? 0 : c->s_rnd;
  h.nuniq = c->sbar - c->sdet;
  h.sbar = c->sbar;
  h.attempts = c->attempts;
  h.pdet = c->p_det;
  h.st_sum_sbar += c->sbar;       // (the host path counted its own sampling bytes)
  h.st_sum_sdet += c->sdet;
  h.st_last_sbar = c->sbar;
  h.st_last_attempts = c->attempts;
  c->ctl_seen.st_sum_attempts = h.st_sum_attempts;
  CK(cudaMemcpyAsync(c->ctl, &h, sizeof(StepCtl), cudaMemcpyHostToDevice, c->st));
  sync(c);
}

// Sample scalars of the current sample from the device (after an
// asynchronous sample) into the host fields the getters use.
void pull_sample_state(cparls_ctx *c) {
  if (c->sample_pulled) return;
  sync(c);
  const StepCtl &h = *reinterpret_cast<const StepCtl *>(c->hctl);
  if (h.abort) throw ApiError(CPARLS_ESTATE, "the asynchronous step was aborted");
  c->sdet = h.sdet;
  c->s_rnd = h.s_rnd;
  c->sbar = h.sbar;
  c->p_det = h.pdet;
  c->attempts = h.attempts;
  c->skipped = h.skip;
  c->sample_pulled = true;
}

// Clears an abort raised by an asynchronous step; returns that step, or -1.
int64_t clear_abort(cparls_ctx *c) {
  sync(c);
  const StepCtl &h = *reinterpret_cast<const StepCtl *>(c->hctl);
  if (!h.abort) return -1;
  const int64_t step = h.abort_step;
  CK(cudaMemsetAsync(&c->ctl->abort, 0, sizeof(int), c->st));
  sync(c);
  return step;
}

// cparls_sample: the asynchronous sampler, then (after one synchronisation)
// the host-driven one if it aborted.
void sample_impl(cparls_ctx *c, int k, int64_t s, uint64_t seed, uint64_t step, cparls_sample_info *info) {
  c->have_sample = false;
  if (s < 1) throw ApiError(CPARLS_EINVAL, "s must be >= 1");
  const bool async_ok = !c->sample_sort;
  if (async_ok) {
    sample_async(c, k, s, seed, step);
    if (clear_abort(c) >= 0) {
      sample_host(c, k, s, seed, step);
      push_sample_state(c);
    }
  } else {
    sample_host(c, k, s, seed, step);
    push_sample_state(c);
  }
  c->sample_pulled = false;
  pull_sample_state(c);
  c->stats.last_s_bar = c->sbar;
  c->stats.last_attempts = c->attempts;
  if (info) {
    info->s_det = c->sdet;
    info->s_rnd = c->s_rnd;
    info->s_bar = c->sbar;
    info->attempts = c->attempts;
    info->p_det = c->p_det;
    info->skipped_random = c->skipped;
  }
}

// ---------------------------------------------------------------- solve
// TnsrSamp lookup of the current sample's fibers; s_bar on the
// device (at most s_cur).
void lookup_impl(cparls_ctx *c, int k) {
  ModeIndex &ix = c->idx[k];
  const int64_t smax = std::max<int64_t>(c->s_cur, 1);
  k_lookup<<<(unsigned)ceil_div(smax, 256), 256, 0, c->st>>>(c->skey, smax, ix.key, ix.dir, ix.shift, ix.nbkt,
                                                             key_remap(c, k), c->lo, c->len, &c->ctl->sbar, c->ctl);
  CK_LAUNCH();
  ensure_scan(c, smax);
  exclusive_scan_i64_1p(c->len, c->off, smax, &c->ctl->sbar, &c->dv->mk, c->scan, c->st, c->ctl);
  LAUNCHED(c, 2);
  c->have_lookup = true;
}

// per-column fixed-point scales 2^e_c of the sampled RHS (kernels.cuh, AMB-35)
// One sketched mode update (Alg. 3) from the current sample, every
// size on the device: KrpSamp + sampled Gram, lookup, RHS, B = M G^+,
// normalize, leverage refresh.  No host synchronisation.
void solve_impl(cparls_ctx *c, int k, cparls_solve_info *info) {
  if (!c->have_sample || c->smode != k) throw ApiError(CPARLS_ESTATE, "solve_mode without a current sample of this mode");
  const int r = c->r, ld = c->ld;
  const int64_t nk = c->dims[k];
  const int64_t smax = std::max<int64_t>(c->s_cur, 1);   // s_bar <= s
  StepCtl *ctl = c->ctl;
  OtherModes om = other_modes(c, k);
  // sharded run: the sampled rows of the other modes from their
  // owners (only the owned rows of a factor are current on a rank)
  // per step the cheaper of: the sampled rows (s x d rows from their owners) or
  // the other modes' dense factors (only those not yet gathered)
  const double *zg = nullptr;
  int64_t dense_rows = 0;
  for (int j = 0; j < om.d; ++j)
    if (c->fac_dirty[om.mode[j]]) dense_rows += om.n[j];
  if (c->world > 1 && dense_rows <= smax * (int64_t)om.d) {
    for (int j = 0; j < om.d; ++j) gather_factor(c, om.mode[j]);
  } else if (c->world > 1) {
    const int64_t need = smax * (int64_t)om.d * ld;
    if (need > c->zg_cap) {
      dfree(c, c->Zg);
      c->zg_cap = need;
      c->Zg = dalloc_t<double>(c, need);
    }
    k_owned_rows<<<(unsigned)std::min<int64_t>(ceil_div(smax * 32, 256), 148 * 16), 256, 0, c->st>>>(
        c->skey, smax, &ctl->sbar, om, c->drow_lo, c->drow_hi, ld, c->Zg, ctl);
    CK_LAUNCH();
    c->comm->allreduce_f64(c->Zg, (size_t)need, c->st);
    c->stats.bytes_comm += 8.0 * need;
    zg = c->Zg;
  }
  // K6: KrpSamp + sampled Gram (every block writes its partial; s_bar = 0 gives G = 0)
  {
    Phase ph(c, &c->stats.ms_gram);
    // Z rows (+ column-sum partials of the fixed-point scales), then the Gram pass over Z
    const int64_t kgrid = std::min<int64_t>(kKrpBlocks, std::max<int64_t>(1, ceil_div(smax, 4 * (kKrpThreads / 32))));
    double *cp = c->rhs_fixed ? c->cpart : nullptr;
#define KRP(DM, QR, HI)                                                                                            \
  k_krp_rows<DM, QR, HI><<<(unsigned)kgrid, kKrpThreads, 0, c->st>>>(c->skey, c->sw2, smax, om, r, ld, c->Z, cp,    \
                                                                      &ctl->sbar, ctl, zg)
    if (r > 32) KRP(kMaxModes - 1, 1, true);
    else if (om.d <= 2) KRP(2, 4, false);
    else if (om.d == 3) KRP(3, 4, false);
    else KRP(kMaxModes - 1, 1, false);
#undef KRP
    CK_LAUNCH();
    const int64_t grid = row_grid(c, ceil_div(smax, kRowThreads));
    RSWITCH(r, k_gram_rows_t<RM><<<(unsigned)grid, kRowThreads, krp_smem(r, ld), c->st>>>(
                   c->Z, smax, r, ld, c->gpart, c->sw2, &ctl->sbar, ctl));
    CK_LAUNCH();
    if (c->rhs_fixed)   // the Gram and the fixed-point scales of the atomic RHS
      k_gram_scales<<<gram_scales_grid(r), 256, 0, c->st>>>(c->gpart, c->cpart, grid, kgrid, r, c->sd->G,
                                                             c->cpart + (int64_t)kKrpBlocks * r,
                                                             &c->dv->maxabs, c->dupmax, c->fx_scale,
                                                             &c->dv->done_count, ctl);
    else
      k_pairs_reduce<<<pairs_reduce_grid(r), 256, 0, c->st>>>(c->gpart, grid, r, c->sd->G, ctl);
    CK_LAUNCH();
    LAUNCHED(c, 3);
    ph.end();
  }
  // G^+ of the sampled Gram (K9's r x r part) on the auxiliary stream,
  // overlapping the lookup and the RHS; joined before B = M G^+
  CK(cudaEventRecord(c->ev_fork, c->st));
  CK(cudaStreamWaitEvent(c->aux, c->ev_fork, 0));
  k_solve_prep<<<1, kPrepThreads, prep_smem(r), c->aux>>>(r, c->sd, ctl);
  CK_LAUNCH();
  LAUNCHED(c, 1);
  CK(cudaEventRecord(c->ev_join, c->aux));
  // K7: lookup of the sampled fibers
  {
    Phase ph(c, &c->stats.ms_lookup);
    lookup_impl(c, k);
    ph.end();
  }
  // this rank's rows of B (all rows on one GPU); M is zero elsewhere
  const int64_t r0 = c->row_lo[k], nown = c->row_hi[k] - c->row_lo[k];
  const int path = c->opts.rhs_path;
  c->fx_on = c->rhs_fixed && path != 3;
  {
    // K8: sampled RHS (int64 fixed-point / fp64 red per entry in L2-sized
    // output-row windows, rhs.cuh)
    Phase ph(c, &c->stats.ms_rhs);
#ifndef CPARLS_RHS_WIN_MB
#define CPARLS_RHS_WIN_MB 96
#endif
    constexpr int win_mb = CPARLS_RHS_WIN_MB;   // output-row window of M kept in L2 (rhs.cuh)
    constexpr int grid_mult = 8;   // CTAs per SM
    const int64_t RW = std::max<int64_t>(1, (int64_t(win_mb) << 20) / ((int64_t)ld * 8));
    const int nwin = (int)ceil_div(nk, RW);
    const int64_t nseg_max = (int64_t)nwin * smax;
    const int64_t *soff = c->off, *slo = c->lo;
    const int32_t *sj = nullptr;
    const int64_t *nseg_dev = &ctl->sbar;
    if (nwin > 1) {
      if (nseg_max > c->segcap) {
        dfree(c, c->seg_lo); dfree(c, c->seg_len); dfree(c, c->seg_off); dfree(c, c->seg_j);
        dfree(c, c->i64part_seg);
        c->segcap = nseg_max;
        c->seg_lo = dalloc_t<int64_t>(c, nseg_max);
        c->seg_len = dalloc_t<int64_t>(c, nseg_max);
        c->seg_off = dalloc_t<int64_t>(c, nseg_max);
        c->seg_j = dalloc_t<int32_t>(c, nseg_max);
        c->i64part_seg = dalloc_t<int64_t>(c, ceil_div(nseg_max, kScanTile) + 16);
      }
      k_win_bounds<<<(unsigned)ceil_div(nseg_max, 256), 256, 0, c->st>>>(c->lo, c->len, smax, c->idx[k].out, nwin, RW,
                                                                         c->seg_lo, c->seg_len, c->seg_j,
                                                                         &ctl->sbar, &ctl->nseg, ctl);
      CK_LAUNCH();
      ensure_scan(c, nseg_max);
      exclusive_scan_i64_1p(c->seg_len, c->seg_off, nseg_max, &ctl->nseg, nullptr, c->scan, c->st, ctl);
      LAUNCHED(c, 2);
      soff = c->seg_off;
      slo = c->seg_lo;
      sj = c->seg_j;
      nseg_dev = &ctl->nseg;
    }
    CK(cudaMemsetAsync(&c->dv->counter, 0, sizeof(unsigned long long), c->st));
    const int grid = 148 * grid_mult;
    const int64_t per_warp = 512;
#define RHS(VT, HI)                                                                                               \
  if (c->fx_on) RHS2(VT, HI, true); else RHS2(VT, HI, false)
#define RHS2(VT, HI, FX)                                                                                           \
  k_rhs<VT, HI, FX><<<grid, kRhsThreads, 0, c->st>>>(soff, slo, sj, nseg_max, &c->dv->mk, &c->dv->counter,          \
                                                     c->idx[k].out, (const VT *)c->idx[k].val, c->sw2, c->Z, r, ld,  \
                                                     c->M, per_warp, c->fx_scale, nseg_dev, ctl)
    KTimer kt(c, KT_RHS);
    const ModeIndex &ix = c->idx[k];
    if (c->fx_on && ix.hot_n > 0 && r <= 32) {   // hot rows summed per CTA in shared memory
      const size_t hsm = 8 * (size_t)ix.hot_n * r;
#define RHS_HOT(VT)                                                                                               \
  k_rhs_hot<VT><<<c->nsm, kRhsHotThreads, hsm, c->st>>>(soff, slo, sj, nseg_max, &c->dv->mk, &c->dv->counter,      \
                                                     ix.out, (const VT *)ix.val, c->sw2, c->Z, r, ld, c->M,       \
                                                     per_warp, c->fx_scale, ix.hot_slot, ix.hot_rows, ix.hot_n,  \
                                                     nseg_dev, ctl)
      if (c->vf32) RHS_HOT(float); else RHS_HOT(double);
#undef RHS_HOT
    } else if (c->vf32) { if (r > 32) RHS(float, true); else RHS(float, false); }
    else { if (r > 32) RHS(double, true); else RHS(double, false); }
    kt.stop();
#undef RHS2
#undef RHS
    CK_LAUNCH();
    LAUNCHED(c, 1);
    ph.end();
  }
  // K9: solve + normalize + leverage refresh
  // sharded: the heavy rows' partial RHS rows summed over the ranks (plan_rows)
  if (c->world > 1 && !c->heavy[k].empty()) {
    const int64_t nh = (int64_t)c->heavy[k].size(), blk = nh * ld;
    if (!c->heavy_buf) c->heavy_buf = dalloc_t<double>(c, c->heavy_buf_n * ld * c->world);
    k_heavy_gather<<<(unsigned)ceil_div(blk, 256), 256, 0, c->st>>>(c->M, c->heavy_dev[k], nh, ld,
                                                                    c->heavy_buf + blk * c->wrank, ctl);
    CK_LAUNCH();
    std::vector<int64_t> off(c->world + 1);
    for (int q = 0; q <= c->world; ++q) off[q] = blk * q;
    c->comm->allgatherv_f64(c->heavy_buf, off, c->st);
    k_heavy_sum<<<(unsigned)ceil_div(blk, 256), 256, 0, c->st>>>(c->M, c->heavy_dev[k], c->heavy_own[k], nh, ld,
                                                                 c->heavy_buf, c->world,
                                                                 c->fx_on ? c->fx_scale : nullptr, ctl);
    CK_LAUNCH();
    c->stats.bytes_comm += 8.0 * blk * c->world;
  }
  {
    Phase ph(c, &c->stats.ms_solve);
    {
      CK(cudaStreamWaitEvent(c->st, c->ev_join, 0));   // G^+ from the auxiliary stream
      const int64_t grid = row_grid(c, ceil_div(std::max<int64_t>(nown, 1), kRowThreads));
      CK(cudaMemsetAsync(&c->dv->touched, 0, sizeof(unsigned long long), c->st));
      KTimer kts(c, KT_SOLVE);
      const int64_t sgrid =
          launch_solve_rows(c, c->M + r0 * ld, nown, c->A[k] + r0 * ld, grid, 1, c->fx_on ? c->fx_scale : nullptr);
      kts.stop();
      CK_LAUNCH();
      k_pairs_reduce<<<pairs_reduce_grid(r), 256, 0, c->st>>>(c->gpart, sgrid, r, c->sd->BtB, ctl);
      CK_LAUNCH();
    }
    if (c->world > 1) {
      // Gram of B over all ranks' owned rows (r x r): lambda and the leverage W
      c->comm->allreduce_f64(c->sd->BtB, (size_t)r * r, c->st);
      c->comm->allreduce_u64(&c->dv->touched, 1, c->st);
    }
    // (single GPU: the short-mode test reads every row of B)
    k_norm_prep<<<1, kPrepThreads, prep_smem(r), c->st>>>(r, c->sd, c->md[k], ctl, c->A[k],
                                                          c->world == 1 ? c->dims[k] : 0, ld);
    CK_LAUNCH();
    LAUNCHED(c, 3);
    if (c->world > 1) lev_rows_sharded(c, k, c->sd->lambda);
    else lev_rows_and_cdf(c, k, c->sd->lambda);
    k_copy_lambda<<<1, 64, 0, c->st>>>(c->lam_model, c->sd->lambda, r, ctl);
    CK_LAUNCH();
    c->stats.bytes_solve += (double)nk * r * 8.0 * 3;
    ph.end();
  }
  if (c->world > 1) c->comm->allreduce_u64(reinterpret_cast<unsigned long long *>(&c->dv->mk), 1, c->st);
  k_solve_stats<<<1, 1, 0, c->st>>>(ctl, k, &c->dv->mk, &c->dv->touched);
  CK_LAUNCH();
  LAUNCHED(c, 2);
  c->stats.mode_steps++;
  if (info) {
    int ru = 0, fb = 0;
    CK(cudaMemcpyAsync(&ru, &c->sd->rank_used, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(&fb, &c->sd->chol_fallback, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    sync(c);   // folds the step counters
    info->matched_nnz = c->stats.last_matched_nnz;
    info->touched_rows = c->stats.touched_rows[k];
    info->rank_used = ru;
    info->chol_fallback = fb;
  }
  c->have_sample = false;   // a sample is consumed by its solve (factors changed)
  c->smode_last_solved = k;
}

// ---------------------------------------------------------------- exact CP-ALS (N2)
// One exact ALS mode update: full MTTKRP from the copy whose slowest
// key mode is k (als.cuh), V = *_{m != k} G_m, B = M V^+ (the same solve and
// AMB-12 pseudo-inverse as the sketched path), normalize, leverage refresh.
void als_update_impl(cparls_ctx *c, int k) {
  if (c->world > 1) throw ApiError(CPARLS_EINVAL, "exact CP-ALS update: single GPU only");
  const int r = c->r, ld = c->ld;
  const int64_t nk = c->dims[k];
  int cm = -1;
  for (int m = 0; m < c->D; ++m)
    if (m != k && c->idx[m].order[c->D - 2] == k) cm = m;
  if (cm < 0) throw ApiError(CPARLS_ESTATE, "no copy with slowest key mode k");
  Phase ph(c, &c->stats.ms_rhs);
  FitDecode fd{};
  fd.d = c->D - 1;
  long double N = 1;
  for (int j = 0; j < fd.d; ++j) {
    const int m = c->idx[cm].order[j];
    fd.n[j] = c->dims[m];
    fd.inv[j] = 1.0 / (double)c->dims[m];
    fd.A[j] = c->A[m];
    N *= (long double)c->dims[m];
  }
  fd.fast = N < 9007199254740992.0L;
  const ModeIndex &ix = c->idx[cm];
  if (ix.nnz > 0) {
    CK(cudaMemsetAsync(&c->dv->counter, 0, sizeof(unsigned long long), c->st));
    const int nb = 148 * 2;
    KTimer kt(c, KT_RHS);
#define MTT(VT, SW, DM)                                                                                        \
  k_mttkrp<VT, SW, DM, (SW >= CPARLS_FIT_U ? CPARLS_FIT_U : SW)><<<nb, kFitThreads, 0, c->st>>>(                \
      ix.key, ix.out, (const VT *)ix.val, ix.nnz, fd, c->A[cm], ld, c->M, &c->dv->counter)
#define MTTD(VT, SW)                        \
  do {                                      \
    if (fd.d == 1) MTT(VT, SW, 1);          \
    else if (fd.d == 2) MTT(VT, SW, 2);     \
    else if (fd.d == 3) MTT(VT, SW, 3);     \
    else throw ApiError(CPARLS_EINVAL, "exact CP-ALS update: D <= 4"); \
  } while (0)
#define MTTV(VT)                            \
  do {                                      \
    if (ld <= 8) MTTD(VT, 2);               \
    else if (ld <= 32) MTTD(VT, 8);         \
    else MTTD(VT, 16);                      \
  } while (0)
    if (c->vf32) MTTV(float); else MTTV(double);
#undef MTTV
#undef MTTD
#undef MTT
    kt.stop();
    CK_LAUNCH();
  }
  GramList gl{};
  gl.D = c->D;
  gl.k = k;
  for (int m = 0; m < c->D; ++m) gl.GA[m] = c->md[m]->GA;
  k_hadamard_grams<<<1, 256, 0, c->st>>>(r, gl, c->sd->G);
  CK_LAUNCH();
  ph.end();
  Phase ph2(c, &c->stats.ms_solve);
  k_solve_prep<<<1, kPrepThreads, prep_smem(r), c->st>>>(r, c->sd);
  CK_LAUNCH();
  const int64_t grid = row_grid(c, ceil_div(std::max<int64_t>(nk, 1), kRowThreads));
  CK(cudaMemsetAsync(&c->dv->touched, 0, sizeof(unsigned long long), c->st));
  KTimer kts(c, KT_SOLVE);
  const int64_t sgrid = launch_solve_rows(c, c->M, nk, c->A[k], grid, 1, nullptr);
  kts.stop();
  CK_LAUNCH();
  k_pairs_reduce<<<pairs_reduce_grid(r), 256, 0, c->st>>>(c->gpart, sgrid, r, c->sd->BtB);
  CK_LAUNCH();
  k_norm_prep<<<1, kPrepThreads, prep_smem(r), c->st>>>(r, c->sd, c->md[k], nullptr, c->A[k], nk, ld);
  CK_LAUNCH();
  LAUNCHED(c, 8);
  lev_rows_and_cdf(c, k, c->sd->lambda);
  CK(cudaMemcpyAsync(c->lam_model, c->sd->lambda, sizeof(double) * r, cudaMemcpyDeviceToDevice, c->st));
  sync(c);
  c->have_sample = false;
  c->smode_last_solved = k;
  c->stats.mode_steps++;
  ph2.end();
}

// ---------------------------------------------------------------- RRF initialization (N4)
void init_rrf_impl(cparls_ctx *c, int64_t s_init, uint64_t seed) {
  if (c->world > 1) throw ApiError(CPARLS_EINVAL, "RRF initialization: single GPU only");
  if (s_init < 1) throw ApiError(CPARLS_EINVAL, "s_init >= 1");
  const int r = c->r, ld = c->ld;
  for (int k = 0; k < c->D; ++k) {
    const ModeIndex &ix = c->idx[k];
    const int64_t nnz = ix.nnz, nk = c->dims[k];
    CK(cudaMemsetAsync(c->M, 0, sizeof(double) * nk * ld, c->st));
    if (nnz > 0) {
      int64_t *flag = dalloc_t<int64_t>(c, nnz), *pos = dalloc_t<int64_t>(c, nnz);
      int64_t *part = dalloc_t<int64_t>(c, ceil_div(nnz, kScanTile) + 16);
      k_fiber_flags<<<1184, 256, 0, c->st>>>(ix.key, nnz, flag);
      CK_LAUNCH();
      exclusive_scan_i64(flag, pos, nnz, part, &c->dv->total, c->st);
      const int64_t nfib = read_dev(c, &c->dv->total);
      dfree(c, part);
      int64_t *fstart = dalloc_t<int64_t>(c, nfib);
      uint64_t *fkey = dalloc_t<uint64_t>(c, nfib);
      KeyToCanon kc{};
      kc.d = c->D - 1;
      bool identity = true;
      for (int j = 0; j < kc.d; ++j) {
        const int m = ix.order[j];
        kc.n[j] = c->dims[m];
        uint64_t mult = 1;   // canonical: other modes ascending, first fastest
        for (int q = 0; q < m; ++q)
          if (q != k) mult *= (uint64_t)c->dims[q];
        kc.cmult[j] = mult;
      }
      {
        int jj = 0;
        for (int m = 0; m < c->D; ++m)
          if (m != k) identity &= (ix.order[jj++] == m);
      }
      k_fiber_list<<<1184, 256, 0, c->st>>>(ix.key, nnz, flag, pos, kc, fstart, fkey);
      CK_LAUNCH();
      dfree(c, flag);
      dfree(c, pos);
      uint32_t *perm = nullptr;
      if (!identity && nfib > 1) {   // rank the fibers by canonical key
        uint64_t *k2 = dalloc_t<uint64_t>(c, nfib);
        uint32_t *v1 = dalloc_t<uint32_t>(c, nfib), *v2 = dalloc_t<uint32_t>(c, nfib);
        k_iota_u32<<<(unsigned)ceil_div(nfib, 256), 256, 0, c->st>>>(v1, nfib);
        CK_LAUNCH();
        cub::DoubleBuffer<uint64_t> kb(fkey, k2);
        cub::DoubleBuffer<uint32_t> vb(v1, v2);
        size_t tb = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, nfib, 0, 64, c->st));
        void *tmp = dalloc(c, tb);
        CK(cub::DeviceRadixSort::SortPairs(tmp, tb, kb, vb, nfib, 0, 64, c->st));
        sync(c);
        dfree(c, tmp);
        perm = vb.Current();
        dfree(c, vb.Alternate());
        dfree(c, k2);
      }
      k_rrf_scatter<<<(unsigned)std::min<int64_t>(ceil_div(s_init * 32, 256), 148 * 64), 256, 0, c->st>>>(
          s_init, seed, k, nfib, perm, fstart, nnz, ix.out, ix.val, c->vf32 ? 1 : 0, r, ld, c->M);
      CK_LAUNCH();
      sync(c);
      dfree(c, fstart);
      dfree(c, fkey);
      if (perm) dfree(c, perm);
    }
    CK(cudaMemcpyAsync(c->A[k], c->M, sizeof(double) * nk * ld, cudaMemcpyDeviceToDevice, c->st));
    CK(cudaMemsetAsync(c->M, 0, sizeof(double) * nk * ld, c->st));
  }
  c->have_sample = false;
  reset_lambda(c);
  for (int k = 0; k < c->D; ++k) leverage_full(c, k);
  sync(c);
}

// ---------------------------------------------------------------- estimated fit (N1)
FitSampleDev fs_dev(cparls_ctx *c) {
  FitSampleDev fs{};
  fs.D = c->D;
  for (int m = 0; m < c->D; ++m) { fs.dims[m] = c->dims[m]; fs.idx[m] = c->fs_idx[m]; }
  fs.x = c->fs_x;
  return fs;
}

// Draw and freeze the stratified sample (AMB-32) from the COO
// input (device pointers) and the mode-0 sorted copy (membership of zeros).
template <typename IT, typename VT>
void draw_fit_sample(cparls_ctx *c, const IT *coords, const VT *vals, int64_t s_fit, double alpha, uint64_t seed) {
  if (!(alpha > 0.0)) alpha = 0.5;
  if (alpha > 1.0) throw ApiError(CPARLS_EINVAL, "fit_alpha must be in (0, 1]");
  int64_t nn = (int64_t)std::ceil(alpha * (double)s_fit);
  int64_t nz = (int64_t)std::floor((1.0 - alpha) * (double)s_fit);
  if (c->nnz == 0) nn = 0;
  double Nd = 1.0;
  for (int m = 0; m < c->D; ++m) Nd *= (double)c->dims[m];
  const double Nz = Nd - (double)c->nnz;
  if (!(Nz > 0.0)) nz = 0;
  const int64_t tot = nn + nz;
  for (int m = 0; m < c->D; ++m) c->fs_idx[m] = dalloc_t<int32_t>(c, tot);
  c->fs_x = dalloc_t<double>(c, tot);
  FitSampleDev fs = fs_dev(c);
  if (nn > 0) {
    k_fs_nz<IT, VT><<<(unsigned)ceil_div(nn, 256), 256, 0, c->st>>>(coords, vals, c->nnz, nn, seed, fs);
    CK_LAUNCH();
  }
  if (nz > 0) {
    MemberIndex mi{};
    const ModeIndex &ix = c->idx[0];
    mi.key = ix.key; mi.out = ix.out; mi.dir = ix.dir; mi.shift = ix.shift; mi.nbkt = ix.nbkt;
    mi.d = c->D - 1;
    uint64_t mult = 1;
    for (int j = 0; j < mi.d; ++j) { mi.order[j] = ix.order[j]; mi.mult[j] = mult; mult *= (uint64_t)c->dims[ix.order[j]]; }
    const int64_t cap = 64 * nz + 65536;
    const int64_t wmax = std::min<int64_t>(nz + nz / 16 + 4096, int64_t(1) << 26);
    int64_t *flag = dalloc_t<int64_t>(c, wmax), *pos = dalloc_t<int64_t>(c, wmax);
    int32_t *cell = dalloc_t<int32_t>(c, wmax * c->D);
    int64_t *part = dalloc_t<int64_t>(c, ceil_div(wmax, kScanTile) + 16);
    int64_t have = 0;
    uint64_t a0 = 0;
    while (have < nz) {
      if ((int64_t)a0 >= cap) throw ApiError(CPARLS_ESAMPLE, "fit sample: zero-rejection attempt cap reached");
      const int64_t win = std::min<int64_t>(wmax, std::min<int64_t>(cap - (int64_t)a0, (nz - have) + (nz - have) / 16 + 4096));
      const unsigned g = (unsigned)ceil_div(win, 256);
      k_fs_zero_gen<<<g, 256, 0, c->st>>>(mi, c->D, fs, seed, a0, win, flag, cell);
      CK_LAUNCH();
      exclusive_scan_i64(flag, pos, win, part, &c->dv->total, c->st);
      k_fs_zero_scatter<<<g, 256, 0, c->st>>>(flag, pos, win, cell, c->D, nn + have, nz - have, fs,
                                               &c->dv->last_attempt, a0);
      CK_LAUNCH();
      have += std::min<int64_t>(read_dev(c, &c->dv->total), nz - have);
      a0 += (uint64_t)win;
    }
    sync(c);
    dfree(c, flag); dfree(c, pos); dfree(c, cell); dfree(c, part);
  }
  c->fs_nnz = nn;
  c->fs_zero = nz;
  c->fs_phi_nz = nn > 0 ? (double)c->nnz / (double)nn : 0.0;
  c->fs_phi_z = nz > 0 ? Nz / (double)nz : 0.0;
  c->have_fs = true;
}

double fit_estimate_impl(cparls_ctx *c, double *Fhat) {
  if (!c->have_fs) throw ApiError(CPARLS_ESTATE, "no fit sample (cparls_opts.fit_samples = 0)");
  Phase ph(c, &c->stats.ms_fit);
  FitDecode fa{};
  fa.d = c->D;
  for (int m = 0; m < c->D; ++m) fa.A[m] = c->A[m];
  const int64_t tot = c->fs_nnz + c->fs_zero;
  const int nb = 148 * 8;
  KTimer kt(c, KT_FIT);
  if (c->ld <= 8) k_fit_est<2><<<nb, 256, 0, c->st>>>(fs_dev(c), c->fs_nnz, tot, c->fs_phi_nz, c->fs_phi_z, fa,
                                                      c->lam_model, c->r, c->ld, c->ddpart);
  else if (c->ld <= 32) k_fit_est<8><<<nb, 256, 0, c->st>>>(fs_dev(c), c->fs_nnz, tot, c->fs_phi_nz, c->fs_phi_z,
                                                            fa, c->lam_model, c->r, c->ld, c->ddpart);
  else k_fit_est<16><<<nb, 256, 0, c->st>>>(fs_dev(c), c->fs_nnz, tot, c->fs_phi_nz, c->fs_phi_z, fa,
                                            c->lam_model, c->r, c->ld, c->ddpart);
  kt.stop();
  CK_LAUNCH();
  k_fit_est_final<<<1, 256, 0, c->st>>>(c->ddpart, nb, c->normX2, c->dv->fit);
  CK_LAUNCH();
  LAUNCHED(c, 2);
  double hv[2];
  CK(cudaMemcpyAsync(hv, c->dv->fit, sizeof(hv), cudaMemcpyDeviceToHost, c->st));
  sync(c);
  if (Fhat) *Fhat = hv[1];
  c->stats.fits++;
  ph.end();
  return hv[0];
}

// Launch the exact fit (eq:fit) on stream st from the factors
// A[0..D) and the model's lambda: <X,M> partials into part (dd[nb]), then
// k_fit_final -> out[0] = fit (single GPU), out[1] = <X,M>, out[2] = ||M||^2.
// blocks_per_sm: CTAs of the persistent fit kernel per SM (2 = all warp slots).
// Key decoding of copy k (its order, fastest digit first) with the factors A.
FitDecode fit_decode(const cparls_ctx *c, int k, double *const *A) {
  FitDecode fd{};
  fd.d = c->D - 1;
  long double N = 1;
  for (int j = 0; j < fd.d; ++j) {   // the copy's key order (fastest first)
    const int m = c->idx[k].order[j];
    fd.n[j] = c->dims[m];
    fd.inv[j] = 1.0 / (double)c->dims[m];
    fd.A[j] = A ? A[m] : nullptr;
    N *= (long double)c->dims[m];
  }
  fd.fast = N < 9007199254740992.0L;   // keys < 2^53
  return fd;
}

void fit_launch(cparls_ctx *c, cudaStream_t st, double *const *A, const double *lam, const FitModes &fm,
                dd *part, unsigned long long *counter, double *out, int blocks_per_sm) {
  const int k = c->fit_mode;
  const FitDecode fd = fit_decode(c, k, A);
  int nb = 148 * 4;
  KTimer kt(c, KT_FIT, st);
  if (fd.d <= 3) {
    // sub-warp per entry, 4 columns per lane (k_fit_sub)
    nb = 148 * std::max(1, std::min(CPARLS_FIT_MINB, blocks_per_sm));
    CK(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st));
#define FITS(VT, SW, DM)                                                                                         \
  k_fit_sub<VT, SW, DM, (SW >= CPARLS_FIT_U ? CPARLS_FIT_U : SW)><<<nb, kFitThreads, 0, st>>>(c->idx[k].key, c->idx[k].out, (const VT *)c->idx[k].val, \
                                                          c->idx[k].nnz, fd, A[k], lam, c->r, c->ld, part, counter, c->ctl)
#define FITSD(VT, SW)                          \
  do {                                         \
    if (fd.d == 1) FITS(VT, SW, 1);            \
    else if (fd.d == 2) FITS(VT, SW, 2);       \
    else FITS(VT, SW, 3);                      \
  } while (0)
#define FITSV(VT)                                        \
  do {                                                   \
    if (c->ld <= 8) FITSD(VT, 2);                        \
    else if (c->ld <= 32) FITSD(VT, 8);                  \
    else FITSD(VT, 16);                                  \
  } while (0)
    if (c->vf32) FITSV(float); else FITSV(double);
#undef FITSV
#undef FITSD
#undef FITS
  } else {
    const size_t smem = sizeof(double) * kFitThreads * (size_t)(c->r | 1);
    if (c->vf32)
      RSWITCH(c->r, k_fit_thread<float, RM><<<nb, kFitThreads, smem, st>>>(
                        c->idx[k].key, c->idx[k].out, (const float *)c->idx[k].val, c->idx[k].nnz, fd, A[k],
                        lam, c->r, c->ld, part, c->ctl));
    else
      RSWITCH(c->r, k_fit_thread<double, RM><<<nb, kFitThreads, smem, st>>>(
                        c->idx[k].key, c->idx[k].out, (const double *)c->idx[k].val, c->idx[k].nnz, fd, A[k],
                        lam, c->r, c->ld, part, c->ctl));
  }
  kt.stop();
  CK_LAUNCH();
  k_fit_final<<<1, 256, 0, st>>>(part, nb, fm, lam, c->r, c->normX2, out, c->ctl);
  CK_LAUNCH();
  LAUNCHED(c, 2);
  c->stats.fits++;
  c->stats.bytes_fit += (double)c->idx[k].nnz * (8.0 + 4.0 + (c->vf32 ? 4.0 : 8.0));
}

FitModes fit_modes(cparls_ctx *c, double *const *GA) {
  FitModes fm{};
  fm.D = c->D;
  for (int m = 0; m < c->D; ++m) fm.GA[m] = GA ? GA[m] : c->md[m]->GA;
  return fm;
}

// The exact fit enqueued on the context's stream: fit value at dv->fit[0]
// (over all ranks); guarded like the mode steps.
void fit_enqueue(cparls_ctx *c) {
  Phase ph(c, &c->stats.ms_fit);
  for (int m = 0; m < c->D; ++m) gather_factor(c, m);   // dense factors once per fit (per epoch)
  fit_launch(c, c->st, c->A, c->lam_model, fit_modes(c, nullptr), c->ddpart, &c->dv->counter, c->dv->fit, 8);
  if (c->world > 1) {
    // <X,M> is a sum over the ranks' slices of the fit mode
    c->comm->allreduce_f64(&c->dv->fit[1], 1, c->st);
    k_fit_combine<<<1, 1, 0, c->st>>>(c->dv->fit, c->normX2, c->ctl);
    CK_LAUNCH();
  }
  ph.end();
}

double fit_impl(cparls_ctx *c) {
  fit_enqueue(c);
  return read_dev(c, &c->dv->fit[0]);
}

// Alg. 3 iterations iter0 .. iter0+iters-1 (steps (iter0 + t) D + k, AMB-10)
// enqueued without host synchronisation: every mode step samples and solves
// on the device (sample_async, solve_impl) and every fit_every-th iteration's
// exact fit is copied to fitbuf[t] on the device.  One synchronisation at the
// end; a step that aborted (a rare branch, sampler.cuh) is redone with the
// host-driven sampler and the rest is enqueued again from the next step.
void run_async(cparls_ctx *c, int32_t iters, int64_t s, uint64_t seed, int32_t iter0, int32_t fit_every,
               double *trace) {
  if (iters < 0) throw ApiError(CPARLS_EINVAL, "iters < 0");
  if (s < 1) throw ApiError(CPARLS_EINVAL, "s must be >= 1");
  if (fit_every > 0 && iters >= fit_every && c->normX2 <= 0.0)
    throw ApiError(CPARLS_ENUMERIC, "||X|| = 0: fit undefined");
  const int D = c->D;
  if (iters > c->fitbuf_cap) {
    dfree(c, c->fitbuf);
    c->fitbuf_cap = std::max<int64_t>(iters, 64);
    c->fitbuf = dalloc_t<double>(c, c->fitbuf_cap);
  }
  if (iters > 0) CK(cudaMemsetAsync(c->fitbuf, 0xFF, sizeof(double) * iters, c->st));   // NaN: no fit
  const bool async_ok = !c->sample_sort;
  auto one_step = [&](int64_t g, bool host_sampler) {
    const int t = (int)(g / D), k = (int)(g % D);
    const uint64_t step = (uint64_t)(iter0 + t) * D + k;   // AMB-10
    if (host_sampler) {
      c->have_sample = false;
      sample_host(c, k, s, seed, step);
      push_sample_state(c);
    } else {
      sample_async(c, k, s, seed, step);
    }
    solve_impl(c, k, nullptr);
    if (k == D - 1 && fit_every > 0 && (t + 1) % fit_every == 0) {
      fit_enqueue(c);
      CK(cudaMemcpyAsync(c->fitbuf + t, &c->dv->fit[0], sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    }
  };
  const int64_t G = (int64_t)iters * D;
  int64_t g0 = 0;
  while (true) {
    for (int64_t g = g0; g < G; ++g) one_step(g, !async_ok);
    if (trace && iters > 0)
      CK(cudaMemcpyAsync(trace, c->fitbuf, sizeof(double) * iters, cudaMemcpyDeviceToHost, c->st));
    const int64_t ab = clear_abort(c);   // the run's one synchronisation (unless a step aborted)
    if (ab < 0) break;
    const int64_t ga = ab - (int64_t)iter0 * D;
    if (ga < 0 || ga >= G) throw ApiError(CPARLS_ECUDA, "asynchronous step abort outside the run");
    one_step(ga, true);
    g0 = ga + 1;
  }
  c->have_sample = false;
}

cparls_status fail(cparls_ctx *c, int st, const std::string &msg) {
  if (c) {
    c->err = msg;
    if (st == CPARLS_ECUDA || st == CPARLS_ENCCL) c->poisoned = true;
  }
  return (cparls_status)st;
}

template <typename F>
cparls_status guarded(cparls_ctx *c, F &&f) {
  if (c && c->poisoned) return fail(c, CPARLS_ECUDA, "context poisoned by an earlier CUDA error: " + c->err);
  try {
    f();
    return CPARLS_OK;
  } catch (const ApiError &e) {
    return fail(c, e.status, e.what());
  } catch (const CudaError &e) {
    if (e.code == cudaErrorMemoryAllocation) return fail(c, CPARLS_EOOM, e.what());
    return fail(c, CPARLS_ECUDA, e.what());
  } catch (const std::bad_alloc &) {
    return fail(c, CPARLS_EOOM, "host allocation failed");
  } catch (const std::exception &e) {
    return fail(c, CPARLS_ECUDA, e.what());
  }
}

void check_mode(cparls_ctx *c, int32_t mode) {
  if (mode < 0 || mode >= c->D) throw ApiError(CPARLS_EINVAL, "mode out of range");
}

}  // namespace

// =====================================================================
// C ABI
// =====================================================================
extern "C" {

static thread_local std::string g_create_err;

void cparls_opts_init(cparls_opts *o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->struct_size = (uint32_t)sizeof(cparls_opts);
  o->rank = 1;
  o->tau = -1.0;
  o->world_size = 1;
  o->fit_mode = -1;
  o->rhs_hot_rows = -1;
}

cparls_status cparls_create(cparls_ctx **out, int32_t nmodes, const int64_t *dims, int64_t nnz_local,
                            const void *coords, const void *vals, const cparls_opts *opts_in, uint64_t init_seed) {
  if (!out || !dims || !opts_in) return CPARLS_EINVAL;
  *out = nullptr;
  // versioned options: the caller's struct_size bytes over the defaults
  if (opts_in->struct_size < offsetof(cparls_opts, value_dtype)) return CPARLS_EINVAL;
  cparls_opts ob;
  cparls_opts_init(&ob);
  std::memcpy(&ob, opts_in, std::min<size_t>(opts_in->struct_size, sizeof(cparls_opts)));
  ob.struct_size = (uint32_t)sizeof(cparls_opts);
  const cparls_opts *opts = &ob;
  const auto t0 = std::chrono::steady_clock::now();
  auto since = [&t0] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); };
  double t_h2d = 0, t_build = 0, t_aux = 0;
  cparls_ctx *c = new (std::nothrow) cparls_ctx();
  if (!c) return CPARLS_EOOM;
  cparls_status st = guarded(c, [&] {
    if (nmodes < 2 || nmodes > kMaxModes) throw ApiError(CPARLS_EINVAL, "nmodes must be in [2, 8]");
    if (opts->rank < 1 || opts->rank > kMaxRank) throw ApiError(CPARLS_EINVAL, "rank must be in [1, 64]");
    if (opts->rhs_path < 0 || opts->rhs_path > 3 || opts->rhs_path == 2)
      throw ApiError(CPARLS_EINVAL, "rhs_path must be 0, 1 or 3");
    if (nnz_local < 0) throw ApiError(CPARLS_EINVAL, "nnz < 0");
    if (nnz_local >= (int64_t(1) << 32)) throw ApiError(CPARLS_ERANGE, "nnz_local must be < 2^32 per GPU");
    if (nnz_local > 0 && (!coords || !vals)) throw ApiError(CPARLS_EINVAL, "null coords/vals");
    if (opts->world_size < 1 || opts->world_rank < 0 || opts->world_rank >= opts->world_size)
      throw ApiError(CPARLS_EINVAL, "bad world_size / world_rank");
    if (opts->world_size > 1) {
      if (!opts->comm) throw ApiError(CPARLS_EINVAL, "world_size > 1 needs opts.comm");
      if (opts->comm->world != opts->world_size) throw ApiError(CPARLS_EINVAL, "comm size != world_size");
      c->comm = make_comm(opts->comm, opts->world_rank);
    }
    c->world = opts->world_size;
    c->wrank = opts->world_rank;
    c->D = nmodes;
    c->r = opts->rank;
    // row stride of the factor-shaped matrices (A_k, M, Z): r rounded up to 8
    // doubles (64-byte rows; r <= 4: 4).  On C4 (r = 25) 32 against 28 measured
    // k_rhs 5.38 -> 5.13 ms and the fit 69.2 -> 65.7 ms: a 256-byte row covers
    // exactly two 128-byte lines.
    c->ld = c->r <= 4 ? 4 : (c->r + 7) & ~7;
    c->nnz = nnz_local;
    c->vf32 = opts->value_dtype == 1;
    c->opts = *opts;
    c->tau = opts->tau;
    c->sample_sort = opts->sample_sort == 1;
    c->rhs_fixed = opts->rhs_path != 3;
    c->st = static_cast<cudaStream_t>(opts->stream);
    for (int m = 0; m < nmodes; ++m) {
      if (dims[m] < 1) throw ApiError(CPARLS_EINVAL, "dims must be >= 1");
      if (dims[m] >= (int64_t(1) << 31)) throw ApiError(CPARLS_ERANGE, "n_k must be < 2^31");
      c->dims[m] = dims[m];
      c->nmax = std::max(c->nmax, dims[m]);
    }
    for (int k = 0; k < nmodes; ++k) {
      long double Nk = 1;
      for (int m = 0; m < nmodes; ++m)
        if (m != k) Nk *= (long double)dims[m];
      if (Nk >= 9223372036854775808.0L) throw ApiError(CPARLS_ERANGE, "prod_{m!=k} n_m >= 2^63");
    }
    set_kernel_attrs(c->r, c->ld);
    CK(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    CK(cudaHostAlloc(reinterpret_cast<void **>(&c->hscr), kHscrSlots * sizeof(long long), cudaHostAllocDefault));
    c->dv = dalloc_t<DevScalars>(c, 1);
    c->ctl = dalloc_t<StepCtl>(c, 1);
    CK(cudaMemsetAsync(c->ctl, 0, sizeof(StepCtl), c->st));
    CK(cudaHostAlloc(&c->hctl, sizeof(StepCtl), cudaHostAllocDefault));
    std::memset(c->hctl, 0, sizeof(StepCtl));
    CK(cudaMemsetAsync(c->dv, 0, sizeof(DevScalars), c->st));
    c->sd = dalloc_t<SolveDev>(c, 1);
    CK(cudaMemsetAsync(c->sd, 0, sizeof(SolveDev), c->st));
    c->lam_model = dalloc_t<double>(c, kMaxRank);
    c->ddpart = dalloc_t<dd>(c, 4096);
    c->gpart_blocks = 148 * 2;
    {
      int dev = 0;
      CK(cudaGetDevice(&dev));
      CK(cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, dev));
    }
    c->gpart = dalloc_t<double>(c, c->gpart_blocks * (int64_t)c->r * c->r);
    c->cpart = dalloc_t<double>(c, (kKrpBlocks + 1) * (int64_t)c->r);   // + the column sums
    c->Gtmp = dalloc_t<double>(c, kMaxRank * kMaxRank);
    c->tile_u64 = dalloc_t<uint64_t>(c, ceil_div(c->nmax, kLevThreads) + 1);
    c->i64part_cap = ceil_div(c->nmax, kScanTile) + 65536 + 64;   // also the SIDX window partials (<= acap / kSidxThreads)
    c->i64part = dalloc_t<int64_t>(c, c->i64part_cap);
    // COO to device if needed
    const size_t isz = opts->index_dtype == 1 ? 8 : 4, vsz = c->vf32 ? 4 : 8;
    const void *dco = coords, *dva = vals;
    void *own_c = nullptr, *own_v = nullptr;
    // host COO: copied in chunks on a copy stream, each chunk's completion an
    // event the build waits on, so the build's allocations and its first key
    // pass run under the PCIe transfer (build_all)
    H2DChunks hc;
    const bool hc_c = nnz_local > 0 && !is_device_ptr(coords), hc_v = nnz_local > 0 && !is_device_ptr(vals);
    if (hc_c) own_c = dalloc(c, isz * nmodes * nnz_local);
    if (hc_v) own_v = dalloc(c, vsz * nnz_local);
    if (hc_c || hc_v) {
      CK(cudaStreamCreateWithFlags(&hc.cs, cudaStreamNonBlocking));
      CK(cudaEventRecord(hc.ev0, c->st));   // after the context's own memsets
      CK(cudaStreamWaitEvent(hc.cs, hc.ev0, 0));
      const std::vector<int64_t> ends = H2DChunks::plan(nnz_local);
      for (size_t i = 0, e0 = 0; i < ends.size(); e0 = ends[i++]) {
        const int64_t n = ends[i] - (int64_t)e0;
        if (hc_c)
          CK(cudaMemcpyAsync((char *)own_c + isz * nmodes * e0, (const char *)coords + isz * nmodes * e0,
                             isz * nmodes * n, cudaMemcpyHostToDevice, hc.cs));
        if (hc_v)
          CK(cudaMemcpyAsync((char *)own_v + vsz * e0, (const char *)vals + vsz * e0, vsz * n, cudaMemcpyHostToDevice,
                             hc.cs));
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CK(cudaEventRecord(ev, hc.cs));
        hc.end.push_back(e0 + n);
        hc.ev.push_back(ev);
      }
      if (hc_c) dco = own_c;
      if (hc_v) dva = own_v;
    }
    const H2DChunks *hcp = hc.ev.empty() ? nullptr : &hc;
    t_h2d = since();
    if (isz == 4 && vsz == 4) build_all<int32_t, float>(c, (const int32_t *)dco, (const float *)dva, hcp);
    else if (isz == 4) build_all<int32_t, double>(c, (const int32_t *)dco, (const double *)dva, hcp);
    else if (vsz == 4) build_all<int64_t, float>(c, (const int64_t *)dco, (const float *)dva, hcp);
    else build_all<int64_t, double>(c, (const int64_t *)dco, (const double *)dva, hcp);
    sync(c);
    t_build = since();
    c->drow_lo = dalloc_t<int64_t>(c, kMaxModes);
    c->drow_hi = dalloc_t<int64_t>(c, kMaxModes);
    CK(cudaMemcpyAsync(c->drow_lo, c->row_lo, sizeof(int64_t) * kMaxModes, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->drow_hi, c->row_hi, sizeof(int64_t) * kMaxModes, cudaMemcpyHostToDevice, c->st));
    sync(c);
    {   // duplicate coordinates bound the fixed-point RHS scale (kernels.cuh)
      CK(cudaMemsetAsync(&c->dv->dupmax, 0, sizeof(unsigned long long), c->st));
      for (int k = 0; k < nmodes; ++k)
        if (c->idx[k].nnz > 0) {
          k_dup_runs<<<1184, 256, 0, c->st>>>(c->idx[k].key, c->idx[k].out, c->idx[k].nnz, &c->dv->dupmax);
          CK_LAUNCH();
        }
      if (c->world > 1) c->comm->allreduce_u64(&c->dv->dupmax, 1, c->st);   // (sum: an upper bound)
      c->dupmax = std::max<double>(1.0, (double)read_dev(c, &c->dv->dupmax));
      c->fx_scale = dalloc_t<double>(c, 2 * kMaxRank + 1);
    }
    if (opts->fit_samples > 0) {
      if (c->world > 1) throw ApiError(CPARLS_EINVAL, "fit_samples needs world_size == 1");
      if (isz == 4 && vsz == 4)
        draw_fit_sample<int32_t, float>(c, (const int32_t *)dco, (const float *)dva, opts->fit_samples,
                                        opts->fit_alpha, opts->fit_seed);
      else if (isz == 4)
        draw_fit_sample<int32_t, double>(c, (const int32_t *)dco, (const double *)dva, opts->fit_samples,
                                         opts->fit_alpha, opts->fit_seed);
      else if (vsz == 4)
        draw_fit_sample<int64_t, float>(c, (const int64_t *)dco, (const float *)dva, opts->fit_samples,
                                        opts->fit_alpha, opts->fit_seed);
      else
        draw_fit_sample<int64_t, double>(c, (const int64_t *)dco, (const double *)dva, opts->fit_samples,
                                         opts->fit_alpha, opts->fit_seed);
    }
    dfree(c, own_c);
    dfree(c, own_v);
    // factors, p~, CDF
    for (int k = 0; k < nmodes; ++k) {
      c->A[k] = dalloc_t<double>(c, c->dims[k] * c->ld);
      c->pt[k] = dalloc_t<double>(c, c->dims[k]);
      c->C[k] = dalloc_t<uint64_t>(c, c->dims[k]);
      c->md[k] = dalloc_t<ModeDev>(c, 1);
      CK(cudaMemsetAsync(c->md[k], 0, sizeof(ModeDev), c->st));
      int64_t tot = c->dims[k] * c->ld;
      k_init_uniform<<<(unsigned)ceil_div(tot, 256), 256, 0, c->st>>>(c->A[k], c->dims[k], c->r, c->ld, k,
                                                                      (uint32_t)init_seed);
      CK_LAUNCH();
    }
    c->M = dalloc_t<double>(c, c->nmax * c->ld);
    CK(cudaMemsetAsync(c->M, 0, sizeof(double) * c->nmax * c->ld, c->st));
    // DIDX candidate buffers: slot j holds the candidates of the j-th OTHER
    // mode of whichever mode is being sampled, so every slot takes max n_m
    int64_t cc = c->nmax;
    for (int m = 0; m < nmodes; ++m) {
      c->ckey[m] = dalloc_t<uint64_t>(c, cc);
      c->cidx[m] = dalloc_t<uint32_t>(c, cc);
    }
    c->ckey_tmp = dalloc_t<uint64_t>(c, cc);
    c->cidx_tmp = dalloc_t<uint32_t>(c, cc);
    c->rhist = dalloc_t<uint32_t>(c, 256 * (ceil_div(cc, kScanTile) + 1));
    c->ccap = cc;
    ensure_list_cap(c, 1 << 16);
    c->acap = int64_t(1) << 22;
    c->akey = dalloc_t<uint64_t>(c, c->acap);
    c->ap = dalloc_t<double>(c, c->acap);
    alloc_sample_buffers(c, 1 << 17);
    // fit streams the mode copy with the fewest fibers (longest runs of equal
    // keys: most reuse of the fiber vector h), ties -> smaller n_k
    for (int m = 0; m < nmodes; ++m) {
      CK(cudaMemsetAsync(&c->dv->counter, 0, sizeof(unsigned long long), c->st));
      if (c->idx[m].nnz > 0) {
        k_count_fibers<<<592, 256, 0, c->st>>>(c->idx[m].key, c->idx[m].nnz, &c->dv->counter);
        CK_LAUNCH();
      }
      if (c->world > 1) c->comm->allreduce_u64(&c->dv->counter, 1, c->st);   // same fit mode on all ranks
      c->nfib[m] = (int64_t)read_dev(c, &c->dv->counter);
    }
    int64_t nnz_global = c->nnz;
    if (c->world > 1) {
      std::vector<int64_t> all = c->comm->allgather_host({c->nnz}, c->st);
      nnz_global = 0;
      for (int64_t v : all) nnz_global += v;
    }
    // per nonzero one A_{k*} row; per fiber one row of every other key mode but
    // the slowest (whose row is cached while the copy sweeps it); expected miss
    // traffic grows with the sizes of the randomly gathered factors
    {
      double best = 0;
      for (int m = 0; m < nmodes; ++m) {
        double fib = 0;
        for (int j = 0; j + 1 < nmodes - 1; ++j) fib += (double)c->dims[c->idx[m].order[j]];
        const double cost = (double)nnz_global * (double)c->dims[m] + (double)c->nfib[m] * fib;
        if (m == 0 || cost < best) { best = cost; c->fit_mode = m; }
      }
      if (opts->fit_mode >= 0 && opts->fit_mode < nmodes) c->fit_mode = opts->fit_mode;
    }
    sync(c);
    t_aux = since();
    reset_lambda(c);
    for (int k = 0; k < nmodes; ++k) leverage_full(c, k);
    sync(c);
    c->stats.create_ms[0] = t_h2d;
    c->stats.create_ms[1] = t_build - t_h2d;
    c->stats.create_ms[2] = t_aux - t_build;
    c->stats.create_ms[3] = since() - t_aux;
    for (int k = 0; k < c->D && k < 8; ++k) {
      c->stats.rhs_hot_rows[k] = c->idx[k].hot_n;
      c->stats.rhs_hot_share[k] = c->idx[k].hot_share;
    }
  });
  if (st != CPARLS_OK) {
    g_create_err = c->err;
    for (void *p : c->allocs) cudaFree(p);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->aux) cudaStreamDestroy(c->aux);
    if (c->hscr) cudaFreeHost(c->hscr);
    if (c->hctl) cudaFreeHost(c->hctl);
    delete c->comm;
    delete c;
    return st;
  }
  *out = c;
  return CPARLS_OK;
}

cparls_status cparls_destroy(cparls_ctx *c) {
  if (!c) return CPARLS_OK;
  if (!c->poisoned) cudaStreamSynchronize(c->st);
  for (auto &p : c->ev_pending) { cudaEventDestroy(p.second.first); cudaEventDestroy(p.second.second); }
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  for (void *p : c->allocs) cudaFree(p);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->aux) cudaStreamDestroy(c->aux);
  if (c->hscr) cudaFreeHost(c->hscr);
  if (c->hctl) cudaFreeHost(c->hctl);
  for (int b = 0; b < 2; ++b) {
    if (c->stage[b]) cudaFreeHost(c->stage[b]);
    if (c->stage_ev[b]) cudaEventDestroy(c->stage_ev[b]);
  }
  delete c->comm;
  delete c;
  return CPARLS_OK;
}

cparls_status cparls_set_factor(cparls_ctx *c, int32_t mode, const double *A) {
  if (!c || !A) return CPARLS_EINVAL;
  return guarded(c, [&] {
    check_mode(c, mode);
    const int64_t n = c->dims[mode];
    CK(cudaMemcpy2DAsync(c->A[mode], sizeof(double) * c->ld, A, sizeof(double) * c->r, sizeof(double) * c->r, n,
                         is_device_ptr(A) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->st));
    c->have_sample = false;
    c->fac_dirty[mode] = false;   // every row given
    reset_lambda(c);
    leverage_full(c, mode);
    sync(c);
  });
}

cparls_status cparls_get_factor(cparls_ctx *c, int32_t mode, double *A, double *lambda) {
  if (!c) return CPARLS_EINVAL;
  return guarded(c, [&] {
    check_mode(c, mode);
    gather_factor(c, mode);   // sharded: collective when only the owned rows are current
    if (A) rows_to_host(c, A, c->A[mode], c->dims[mode], c->r, c->ld);
    if (lambda) CK(cudaMemcpyAsync(lambda, c->lam_model, sizeof(double) * c->r, cudaMemcpyDefault, c->st));
    sync(c);
  });
}

cparls_status cparls_leverage(cparls_ctx *c, int32_t mode, double *scores, int32_t *rank_out) {
  if (!c) return CPARLS_EINVAL;
  return guarded(c, [&] {
    check_mode(c, mode);
    leverage_full(c, mode);
    int rank = 0;
    CK(cudaMemcpyAsync(&rank, &c->md[mode]->rank, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    if (scores)
      CK(cudaMemcpyAsync(scores, c->pt[mode], sizeof(double) * c->dims[mode], cudaMemcpyDeviceToHost, c->st));
    sync(c);
    if (scores)
      for (int64_t i = 0; i < c->dims[mode]; ++i) scores[i] *= (double)rank;   // l = p~ * rank
    if (rank_out) *rank_out = rank;
  });
}

cparls_status cparls_get_ptilde(cparls_ctx *c, int32_t mode, double *pt) {
  if (!c || !pt) return CPARLS_EINVAL;
  return guarded(c, [&] {
    check_mode(c, mode);
    CK(cudaMemcpyAsync(pt, c->pt[mode], sizeof(double) * c->dims[mode], cudaMemcpyDeviceToHost, c->st));
    sync(c);
  });
}

cparls_status cparls_set_ptilde(cparls_ctx *c, int32_t mode, const double *pt) {
  if (!c || !pt) return CPARLS_EINVAL;
  return guarded(c, [&] {
    check_mode(c, mode);
    const int64_t n = c->dims[mode];
    CK(cudaMemcpyAsync(c->pt[mode], pt, sizeof(double) * n,
                       is_device_ptr(pt) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->st));
    const int64_t nt = ceil_div(n, kLevThreads);
    CK(cudaMemsetAsync(&c->md[mode]->alpha, 0, sizeof(double), c->st));
    CK(cudaMemsetAsync(&c->md[mode]->drawable, 0, sizeof(long long), c->st));
    k_q_from_pt<<<(unsigned)nt, kLevThreads, 0, c->st>>>(c->pt[mode], n, c->C[mode], c->tile_u64,
                                                         &c->md[mode]->alpha,
                                                         reinterpret_cast<unsigned long long *>(&c->md[mode]->drawable));
    CK_LAUNCH();
    k_scan_u64_single<<<1, kScanThreads, 0, c->st>>>(c->tile_u64, nt);
    CK_LAUNCH();
    k_cdf_final<<<(unsigned)nt, kLevThreads, 0, c->st>>>(c->C[mode], n, c->tile_u64);
    CK_LAUNCH();
    c->have_sample = false;
    sync(c);
  });
}

cparls_status cparls_set_tau(cparls_ctx *c, double tau) {
  if (!c) return CPARLS_EINVAL;
  c->tau = tau;
  return CPARLS_OK;
}

cparls_status cparls_sample(cparls_ctx *c, int32_t mode, int64_t s, uint64_t seed, uint64_t step,
                            cparls_sample_info *info) {
  if (!c) return CPARLS_EINVAL;
  return guarded(c, [&] {
    check_mode(c, mode);
    sample_impl(c, mode, s, seed, step, info);
  });
}

namespace {
std::vector<int64_t> canonical_order(const std::vector<uint64_t> &k, const std::vector<uint8_t> &det) {
  std::vector<int64_t> o(k.size());
  std::iota(o.begin(), o.end(), 0);
  std::sort(o.begin(), o.end(), [&](int64_t a, int64_t b) {
    if (det[a] != det[b]) return det[a] > det[b];
    return k[a] < k[b];
  });
  return o;
}
}  // namespace

cparls_status cparls_get_sample(cparls_ctx *c, int64_t cap, uint64_t *keys, int32_t *counts, double *w2, double *p,
                                uint8_t *is_det, int64_t *n_out) {
  if (!c) return CPARLS_EINVAL;
  return guarded(c, [&] {
    pull_sample_state(c);
    const int64_t n = c->sbar;
    if (n_out) *n_out = n;
    std::vector<uint64_t> hk(n);
    std::vector<int32_t> hc(n);
    std::vector<double> hw(n), hp(n);
    std::vector<uint8_t> hd(n);
    if (n > 0) {
      CK(cudaMemcpyAsync(hk.data(), c->skey, 8 * n, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(hc.data(), c->scnt, 4 * n, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(hw.data(), c->sw2, 8 * n, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(hp.data(), c->sp, 8 * n, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(hd.data(), c->sisdet, n, cudaMemcpyDeviceToHost, c->st));
      sync(c);
    }
    auto o = canonical_order(hk, hd);
    int64_t m = std::min(cap, n);
    for (int64_t i = 0; i < m; ++i) {
      int64_t j = o[i];
      if (keys) keys[i] = hk[j];
      if (counts) counts[i] = hc[j];
      if (w2) w2[i] = hw[j];
      if (p) p[i] = hp[j];
      if (is_det) is_det[i] = hd[j];
    }
  });
}

cparls_status cparls_get_fibers(cparls_ctx *c, int64_t cap, int64_t *len, int64_t *out, double *val,
                                int64_t *m_out) {
  if (!c) return CPARLS_EINVAL;
  return guarded(c, [&] {
    if (c->smode < 0 || c->sbar < 0) throw ApiError(CPARLS_ESTATE, "no sample");
    pull_sample_state(c);
    const int k = c->smode;
    if (!c->have_lookup) lookup_impl(c, k);
    const int64_t n = c->sbar;
    int64_t mk = read_dev(c, &c->dv->mk);
    if (m_out) *m_out = mk;
    std::vector<uint64_t> hk(n);
    std::vector<uint8_t> hd(n);
    std::vector<int64_t> hl(n), ho(n);
    const bool entries = (out || val) && cap > 0;   // lengths only otherwise
    std::vector<int64_t> go(entries ? mk : 0);
    std::vector<double> gv(entries ? mk : 0);
    if (n > 0) {
      CK(cudaMemcpyAsync(hk.data(), c->skey, 8 * n, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(hd.data(), c->sisdet, n, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(hl.data(), c->len, 8 * n, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(ho.data(), c->off, 8 * n, cudaMemcpyDeviceToHost, c->st));
    }
    if (mk > 0 && entries) {
      int64_t *dO = dalloc_t<int64_t>(c, mk);
      double *dV = dalloc_t<double>(c, mk);
      if (c->vf32)
        k_gather_fibers<float><<<(unsigned)n, 128, 0, c->st>>>(c->off, c->lo, c->len, n, c->idx[k].out,
                                                                (const float *)c->idx[k].val, dO, dV);
      else
        k_gather_fibers<double><<<(unsigned)n, 128, 0, c->st>>>(c->off, c->lo, c->len, n, c->idx[k].out,
                                                                 (const double *)c->idx[k].val, dO, dV);
      CK_LAUNCH();
      CK(cudaMemcpyAsync(go.data(), dO, 8 * mk, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(gv.data(), dV, 8 * mk, cudaMemcpyDeviceToHost, c->st));
      sync(c);
      dfree(c, dO);
      dfree(c, dV);
    }
    sync(c);
    auto o = canonical_order(hk, hd);
    int64_t w = 0;
    for (int64_t i = 0; i < n; ++i) {
      int64_t j = o[i];
      if (len) len[i] = hl[j];
      if (!entries) continue;
      for (int64_t t = 0; t < hl[j]; ++t, ++w) {
        if (w < cap) {
          if (out) out[w] = go[ho[j] + t];
          if (val) val[w] = gv[ho[j] + t];
        }
      }
    }
  });
}

cparls_status cparls_solve_mode(cparls_ctx *c, int32_t mode, cparls_solve_info *info) {
  if (!c) return CPARLS_EINVAL;
  return guarded(c, [&] {
    check_mode(c, mode);
    solve_impl(c, mode, info);
  });
}

cparls_status cparls_get_last_solve(cparls_ctx *c, double *G, double *B) {
  if (!c) return CPARLS_EINVAL;
  return guarded(c, [&] {
    const int r = c->r;
    if (G) CK(cudaMemcpyAsync(G, c->sd->G, sizeof(double) * r * r, cudaMemcpyDeviceToHost, c->st));
    if (B) {
      int k = c->smode_last_solved;
      if (k < 0) throw ApiError(CPARLS_ESTATE, "no solve yet");
      gather_factor(c, k);
      std::vector<double> lam(r);
      CK(cudaMemcpy2DAsync(B, sizeof(double) * r, c->A[k], sizeof(double) * c->ld, sizeof(double) * r, c->dims[k],
                           cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(lam.data(), c->sd->lambda, sizeof(double) * r, cudaMemcpyDeviceToHost, c->st));
      sync(c);
      for (int64_t i = 0; i < c->dims[k]; ++i)
        for (int q = 0; q < r; ++q) B[i * r + q] *= lam[q];
    }
    sync(c);
  });
}

cparls_status cparls_fit(cparls_ctx *c, double *fit) {
  if (!c) return CPARLS_EINVAL;
  return guarded(c, [&] {
    if (c->normX2 <= 0.0) throw ApiError(CPARLS_ENUMERIC, "||X|| = 0: fit undefined");
    double f = fit_impl(c);
    if (fit) *fit = f;
  });
}

cparls_status cparls_run(cparls_ctx *c, int32_t iters, int64_t s, uint64_t seed, int32_t iter0, int32_t fit_every,
                         double *fit_trace) {
  if (!c) return CPARLS_EINVAL;
  return guarded(c, [&] { run_async(c, iters, s, seed, iter0, fit_every, fit_trace); });
}

cparls_status cparls_fit_estimate(cparls_ctx *c, double *fit, double *Fhat) {
  if (!c) return CPARLS_EINVAL;
  return guarded(c, [&] {
    if (c->normX2 <= 0.0) throw ApiError(CPARLS_ENUMERIC, "||X|| = 0: fit undefined");
    const double f = fit_estimate_impl(c, Fhat);
    if (fit) *fit = f;
  });
}

cparls_status cparls_fit_sample_model(cparls_ctx *c, double *m) {
  if (!c || !m) return CPARLS_EINVAL;
  return guarded(c, [&] {
    if (!c->have_fs) throw ApiError(CPARLS_ESTATE, "no fit sample (cparls_opts.fit_samples = 0)");
    FitDecode fa{};
    fa.d = c->D;
    for (int k = 0; k < c->D; ++k) fa.A[k] = c->A[k];
    const int64_t tot = c->fs_nnz + c->fs_zero;
    double *dm = dalloc_t<double>(c, tot);
    const int nb = 148 * 8;
    if (c->ld <= 8) k_fit_est_model<2><<<nb, 256, 0, c->st>>>(fs_dev(c), tot, fa, c->lam_model, c->r, c->ld, dm);
    else if (c->ld <= 32) k_fit_est_model<8><<<nb, 256, 0, c->st>>>(fs_dev(c), tot, fa, c->lam_model, c->r, c->ld, dm);
    else k_fit_est_model<16><<<nb, 256, 0, c->st>>>(fs_dev(c), tot, fa, c->lam_model, c->r, c->ld, dm);
    CK_LAUNCH();
    CK(cudaMemcpyAsync(m, dm, sizeof(double) * tot, cudaMemcpyDeviceToHost, c->st));
    sync(c);
    dfree(c, dm);
  });
}

cparls_status cparls_get_fit_sample(cparls_ctx *c, int64_t cap, int64_t *coords, double *x, uint8_t *is_nz,
                                    int64_t *n) {
  if (!c) return CPARLS_EINVAL;
  return guarded(c, [&] {
    if (!c->have_fs) throw ApiError(CPARLS_ESTATE, "no fit sample (cparls_opts.fit_samples = 0)");
    const int64_t tot = c->fs_nnz + c->fs_zero;
    if (n) *n = tot;
    const int64_t m = std::min(cap, tot);
    if (m <= 0) return;
    std::vector<int32_t> col(m);
    for (int d = 0; d < c->D; ++d) {
      CK(cudaMemcpyAsync(col.data(), c->fs_idx[d], sizeof(int32_t) * m, cudaMemcpyDeviceToHost, c->st));
      sync(c);
      if (coords)
        for (int64_t i = 0; i < m; ++i) coords[i * c->D + d] = col[i];
    }
    if (x) {
      CK(cudaMemcpyAsync(x, c->fs_x, sizeof(double) * m, cudaMemcpyDeviceToHost, c->st));
      sync(c);
    }
    if (is_nz)
      for (int64_t i = 0; i < m; ++i) is_nz[i] = i < c->fs_nnz;
  });
}

cparls_status cparls_run_until(cparls_ctx *c, int64_t s, uint64_t seed, int32_t eta, int32_t pi, double tol,
                               int32_t max_epochs, int32_t fit_kind, double *trace, int32_t *epochs) {
  if (!c) return CPARLS_EINVAL;
  return guarded(c, [&] {
    if (eta < 1 || pi < 1 || max_epochs < 0) throw ApiError(CPARLS_EINVAL, "eta, pi >= 1; max_epochs >= 0");
    if (c->normX2 <= 0.0) throw ApiError(CPARLS_ENUMERIC, "||X|| = 0: fit undefined");
    if (fit_kind == 1 && !c->have_fs) throw ApiError(CPARLS_ESTATE, "estimated fit needs opts.fit_samples > 0");
    double best = -INFINITY;
    int fails = 0, e = 0;
    for (e = 0; e < max_epochs; ++e) {
      // eta iterations (steps (e eta + t) D + k, AMB-10) without host synchronisation
      run_async(c, eta, s, seed, e * eta, 0, nullptr);
      const double f = fit_kind == 1 ? fit_estimate_impl(c, nullptr) : fit_impl(c);
      if (trace) trace[e] = f;
      if (f > best + tol) {   // AMB-33: improvement over the best fit so far
        best = f;
        fails = 0;
      } else if (++fails >= pi) {
        ++e;
        break;
      }
    }
    if (epochs) *epochs = e;
  });
}

cparls_status cparls_init_rrf(cparls_ctx *c, int64_t s_init, uint64_t seed) {
  if (!c) return CPARLS_EINVAL;
  return guarded(c, [&] { init_rrf_impl(c, s_init, seed); });
}

cparls_status cparls_als_update(cparls_ctx *c, int32_t mode) {
  if (!c) return CPARLS_EINVAL;
  return guarded(c, [&] {
    check_mode(c, mode);
    als_update_impl(c, mode);
  });
}

cparls_status cparls_run_als(cparls_ctx *c, int32_t iters, int32_t fit_every, double *fit_trace) {
  if (!c) return CPARLS_EINVAL;
  return guarded(c, [&] {
    if (iters < 0) throw ApiError(CPARLS_EINVAL, "iters < 0");
    for (int t = 0; t < iters; ++t) {
      for (int k = 0; k < c->D; ++k) als_update_impl(c, k);
      double f = NAN;
      if (fit_every > 0 && (t + 1) % fit_every == 0) {
        if (c->normX2 <= 0.0) throw ApiError(CPARLS_ENUMERIC, "||X|| = 0: fit undefined");
        f = fit_impl(c);
      }
      if (fit_trace) fit_trace[t] = f;
    }
  });
}

cparls_status cparls_comm_nccl_unique_id(uint8_t id[128]) {
  if (!id) return CPARLS_EINVAL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess) return CPARLS_ENCCL;
  std::memcpy(id, &u, 128);
  return CPARLS_OK;
}

cparls_status cparls_comm_create_nccl(int32_t world_size, int32_t rank, const uint8_t id[128], cparls_comm **out) {
  if (!out || !id || world_size < 1 || rank < 0 || rank >= world_size) return CPARLS_EINVAL;
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  auto *cc = new (std::nothrow) cparls_comm();
  if (!cc) return CPARLS_EOOM;
  cc->kind = 0;
  cc->world = world_size;
  cc->rank = rank;
  if (ncclCommInitRank(&cc->nccl, world_size, u, rank) != ncclSuccess) {
    delete cc;
    return CPARLS_ENCCL;
  }
  *out = cc;
  return CPARLS_OK;
}

cparls_status cparls_comm_create_local(int32_t world_size, cparls_comm **out) {
  if (!out || world_size < 1) return CPARLS_EINVAL;
  auto *cc = new (std::nothrow) cparls_comm();
  if (!cc) return CPARLS_EOOM;
  cc->kind = 1;
  cc->world = world_size;
  cc->group = new cparls::LocalGroup(world_size);
  *out = cc;
  return CPARLS_OK;
}

cparls_status cparls_comm_destroy(cparls_comm *cc) {
  if (!cc) return CPARLS_OK;
  if (cc->kind == 0 && cc->nccl) ncclCommDestroy(cc->nccl);
  delete cc->group;
  delete cc;
  return CPARLS_OK;
}

cparls_status cparls_plan_rows(int64_t n, const uint64_t *deg, int32_t world_size, int64_t *bound, uint8_t *heavy) {
  if (n < 0 || world_size < 1 || !bound || (n > 0 && !deg)) return CPARLS_EINVAL;
  plan_rows(n, reinterpret_cast<const unsigned long long *>(deg), world_size, bound, heavy);
  return CPARLS_OK;
}

cparls_status cparls_route_nonzeros(int32_t nmodes, int32_t mode, int64_t nnz, const int64_t *coords,
                                    int32_t world_size, const int64_t *bound, const uint8_t *heavy, int32_t *rank_out) {
  if (nmodes < 2 || nmodes > kMaxModes || mode < 0 || mode >= nmodes || nnz < 0 || world_size < 1 || !bound ||
      (nnz > 0 && (!coords || !rank_out)))
    return CPARLS_EINVAL;
  for (int64_t e = 0; e < nnz; ++e)
    rank_out[e] = route_rank<int64_t>(coords + e * nmodes, nmodes, mode, bound, world_size, heavy);
  return CPARLS_OK;
}

cparls_status cparls_owned_rows(const cparls_ctx *c, int32_t mode, int64_t *lo, int64_t *hi) {
  if (!c || mode < 0 || mode >= c->D) return CPARLS_EINVAL;
  if (lo) *lo = c->row_lo[mode];
  if (hi) *hi = c->row_hi[mode];
  return CPARLS_OK;
}

cparls_status cparls_get_stats(cparls_ctx *c, void *s, int64_t bytes) {
  if (!c || !s || bytes < 8) return CPARLS_EINVAL;
  return guarded(c, [&] {
    sync(c, false);   // folds a pending step's counters and the kernel timers
    c->stats.struct_size = (uint32_t)sizeof(cparls_stats);
    std::memcpy(s, &c->stats, (size_t)std::min<int64_t>(bytes, (int64_t)sizeof(cparls_stats)));
  });
}

cparls_status cparls_reset_stats(cparls_ctx *c) {
  if (!c) return CPARLS_EINVAL;
  return guarded(c, [&] {
    sync(c, false);   // a pending step's counters belong to the old stats
    const cparls_stats keep = c->stats;
    c->stats = cparls_stats{};
    // create-time facts survive a reset
    std::memcpy(c->stats.create_ms, keep.create_ms, sizeof(keep.create_ms));
    std::memcpy(c->stats.rhs_hot_rows, keep.rhs_hot_rows, sizeof(keep.rhs_hot_rows));
    std::memcpy(c->stats.rhs_hot_share, keep.rhs_hot_share, sizeof(keep.rhs_hot_share));
    std::memcpy(c->stats.build_ms, keep.build_ms, sizeof(keep.build_ms));
    c->ctl_seen = *reinterpret_cast<const StepCtl *>(c->hctl);
  });
}

cparls_status cparls_set_profiling(cparls_ctx *c, int32_t on) {
  if (!c) return CPARLS_EINVAL;
  c->profiling = on != 0;
  return CPARLS_OK;
}

const char *cparls_last_error(const cparls_ctx *c) {
  if (!c) return g_create_err.c_str();
  return c->err.c_str();
}

const char *cparls_version(void) { return "cparls 0.1 (sm_100a, CP-ARLS-LEV hot path)"; }

}  // extern "C"
