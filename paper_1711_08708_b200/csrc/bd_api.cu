// C-ABI implementation of the bidomain PCG hot path (see include/bidomain_b200.h).
//
// One private non-blocking stream per context; every public call orders
// itself after the caller's stream with an event and hands back with another,
// so callers see plain stream semantics while the PCG loop can be captured
// into a CUDA graph (conditional WHILE node) on the private stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <future>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include <unistd.h>

#include "../../include/bidomain_b200.h"
#include "bd_assembly.cuh"
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include "bd_device.cuh"
#include "bd_host.hpp"

using namespace bd;
using dev::Ctl;

#define BD_VERSION "bidomain_b200 0.1 sm_100a"

struct bd_ctx {
  int device = 0;
  cudaStream_t user = nullptr;    // caller's stream (may be the legacy default)
  cudaStream_t stream = nullptr;  // private stream all work runs on
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  std::string err;
  int64_t launches = 0;
  int nsm = 148;
  size_t l2_persist = 0;  // bytes of L2 set aside for persisting accesses (0: none)
  // profiling
  bool profile = false;
  std::vector<std::pair<cudaEvent_t, int>> marks;
  std::vector<cudaEvent_t> pool;
  double prof_ms[8] = {0};
  int64_t prof_launch[8] = {0};
  // utility control block (dot / mean readbacks)
  Ctl util{};
  double* h_pin = nullptr;  // pinned readback scratch (64 doubles)
};

struct bd_csr {
  bd_ctx* ctx;
  int64_t nrows, ncols, nnz;
  int* rowptr = nullptr;
  int* col = nullptr;
  double* val = nullptr;
  int G = 8;
  // entry-major ELL copy for bd_spmv when rows are short and near-uniform
  int ell_w = 0;
  int* ell_col = nullptr;
  double* ell_val = nullptr;
  dev::Csr dev() const { return dev::Csr{(int)nrows, rowptr, col, val}; }
};

struct DevTri {
  int n = 0;
  int* rowptr = nullptr;
  int* col = nullptr;
  double* val = nullptr;
  int* tasks = nullptr;
  int ntasks = 0;
  int nvb = 0;
  int64_t depth = 0;
  int64_t nnz = 0;
  dev::Tri dev() const { return dev::Tri{n, rowptr, col, val, tasks, ntasks}; }
};

struct DevTile {
  int* part_task_ptr = nullptr;
  int* part_step_ptr = nullptr;
  int* step_task_ptr = nullptr;
  int* task_row = nullptr;
  double* task_diag = nullptr;
  int* ell_col = nullptr;
  double* ell_val = nullptr;
  int max_part_rows = 0;
  int max_part_steps = 0;
  int nsteps = 0;
  dev::TileDev dev() const {
    return dev::TileDev{part_task_ptr, part_step_ptr, step_task_ptr, task_row, task_diag,
                        ell_col,       ell_val,       max_part_rows, max_part_steps};
  }
};

constexpr int kTileStages = 8;

struct DevEll {
  int* task_row = nullptr;
  double* task_diag = nullptr;
  int* ell_col = nullptr;
  double* ell_val = nullptr;
  int ntasks = 0;
  int nchunks = 0;
  int grid = 0;
  dev::EllTri dev() const { return dev::EllTri{task_row, task_diag, ell_col, ell_val, ntasks}; }
};

constexpr int kClusterParts = 16;
constexpr int kClusterStages = 3;
constexpr int kClusterStagesDeep = 10;

struct DevCluster {
  int* lvl_ptr = nullptr;
  int* task_row = nullptr;
  double* task_diag = nullptr;
  double* ell_val = nullptr;
  short* ell_code = nullptr;
  int* exp_ptr = nullptr;
  int* exp_src = nullptr;
  int* exp_dst = nullptr;
  int nlevels = 0, W = 4, wmax = 0, rmax = 0, emax = 0, E = 8;
  size_t smem = 0;
  bool deep = false;
  int64_t ntasks = 0;
  dev::ClusterDev dev() const {
    return dev::ClusterDev{lvl_ptr, task_row, task_diag, ell_val, ell_code, exp_ptr,
                           exp_src, exp_dst, nlevels, W, wmax, rmax, emax};
  }
};

struct DevDTile {
  int* tile_row_ptr = nullptr;
  int* tile_step_ptr = nullptr;
  int* step_row = nullptr;
  int* task_row = nullptr;
  double* task_diag = nullptr;
  int* ell_col = nullptr;
  double* ell_val = nullptr;
  int ntiles = 0, tmax = 0, grid = 0, threads = 64;
  dev::DTileDev dev() const {
    return dev::DTileDev{tile_row_ptr, tile_step_ptr, step_row, task_row, task_diag,
                         ell_col,      ell_val,       ntiles,   tmax};
  }
};

struct DevBTile {
  int* tile_nr = nullptr;
  int* task_row = nullptr;
  unsigned short* ent_rp = nullptr;
  unsigned short* ent_slot = nullptr;
  double* ent_val = nullptr;
  int* in_col = nullptr;
  double* inv = nullptr;
  int ntiles = 0, rs = 0, xs = 0, is = 0, es = 0, rps = 0, grid = 0, threads = 256, sleep_ns = 0,
      prefetch = 1, poll_depth = 3;
  double* inbox = nullptr;  // shared per inner (not owned here)
  int* dst = nullptr;
  int dmax = 0;
  int exw = 8;  // max external entries per row
  size_t smem = 0;
  bool pipe = false;      // k_trsv_ptile (pipelined; needs opos / tile-ordered rhs)
  int* opos = nullptr;    // forward schedule: slot of each row in the backward tile order
  bool reg = false;       // k_trsv_rtile instead of k_trsv_btile
  bool tile_rhs = false;  // k_trsv_rtile with the right-hand side pre-gathered in tile order
  bool reg_smem = false;  // k_trsv_rtile with the inverse staged in shared memory
  bool rpipe = false;     // k_trsv_rpipe: packed per-tile records through a TMA ring
  bool rpipe_wide = false;  // BD_RPIPE_WIDE=1: force the two-inputs-per-thread instantiation (tests)
  unsigned char* rec = nullptr;
  int recb = 0, depth = 2;
  dev::BTileDev dev() const {
    return dev::BTileDev{tile_nr, task_row, ent_rp,   ent_slot, ent_val, in_col, inv,
                         ntiles,  rs,       xs,       is,       es,      rps,    sleep_ns,
                         prefetch, poll_depth, inbox,    dst,      dmax,     exw,
                         rec,     recb,     depth,    INT32_MAX};
  }
};

struct DevSuper {
  int dchunk = 16;           // rows per dense-phase slice (BD_SUPER_DCHUNK)
  double* pinv = nullptr;    // panel inverses of the big supernodes' dense blocks
  int* sn_pan = nullptr;
  int* task_kind = nullptr;  // forward: split external phases (nullptr: none)
  int* task_arg = nullptr;
  int* sn_cnt = nullptr;
  int* sn_start = nullptr;
  int* sn_size = nullptr;
  int* task_sn = nullptr;
  int* task_w = nullptr;  // lanes per small supernode of each task (nullptr: 32)
  double* sinv = nullptr;      // whole-block inverses of the largest supernodes
  long long* sn_inv = nullptr;
  int ntasks = 0;
  int grid = 0;
};

struct bd_inner {
  bd_ctx* ctx;
  int kind;
  int64_t n;
  int G = 8;
  int prof_cls = 2;  // profile class of its triangular passes (2 bulk, 3 Schur)
  int fold_fill = 0; // BD_FOLD_FILL (see inner_solve_g)
  DevTri L, U;
  bool super = false;
  DevSuper SL, SU;
  bool cluster = false;
  DevCluster CL, CU;
  bool dtile = false;
  DevDTile DL, DU;
  bool btile = false;
  DevBTile BL, BU;
  double* rtmp = nullptr;
  bool prefilled = false;     // the caller's previous kernel reset y_int (consumed by the next solve)
  double* post_fill = nullptr;  // polled forward output of the NEXT inner solve, reset by this solve's
  int64_t post_fill_n = 0;      // backward pass (consumed by the next solve of this inner)
  bd_inner* post_fill_owner = nullptr;
  double* rhs_pre = nullptr;  // btile: pre-evaluated non-scalar right-hand side
  double* rext = nullptr;  // supernodal forward: precomputed external phases (n)
  double* dense = nullptr; // exact inner, small n: explicit inverse (P A P^T)^{-1}, row-major
  // tiled cooperative schedule (IC(0) factors with short rows)
  bool tiled = false;
  bool persist = false;
  DevEll EL, EU;
  int TG = 8, tparts = 0, tthreads = 0, tstages = 8, trows = 128;
  bool rows_mode = false;
  size_t tsmem = 0;
  DevTile TL, TU;
  int* perm = nullptr;        // exact: new -> old
  double* inv = nullptr;      // jacobi
  double* y_int = nullptr;    // forward output (sentinel between solves)
  double* bt_f = nullptr;     // k_trsv_ptile: forward right-hand side in tile order
  double* bt_b = nullptr;     // k_trsv_ptile: backward right-hand side in tile order
  double* inbox = nullptr;    // k_trsv_rtile inbox mode: per-tile input slots (sentinel between passes)
  int64_t inbox_len = 0;
  double* x_int = nullptr;    // internal backward output for standalone / exact
  HostCsr hlower;
  std::vector<int32_t> hperm;
  int restarts = 0;
  Ctl ctl{};                  // standalone control block
};

struct bd_system {
  bd_ctx* ctx;
  bd_csr* S1;
  bd_csr* Si;
  int64_t n, m;
  double* mass = nullptr;
  double* mh = nullptr;
  double gamma;
  Ctl ctl{};
  double* tmp = nullptr;  // n+m scratch
  // entry-major ELL copy of [S_1 | S_i] for Λ (W = 0: not built, CSR kernels)
  int ell_w = 0;
  int* ell_col = nullptr;
  double* ell_v1 = nullptr;
  double* ell_v2 = nullptr;
  unsigned long long* track = nullptr;  // bd_step_track flags (lazy)
};

struct bd_prec {
  bd_system* sys;
  bd_inner* bulk;
  bd_inner* schur;
  double beta;
  int64_t cnt[3] = {0, 0, 0};
  Ctl ctl{};       // PCG control block (flags on)
  Ctl ctl_nf{};    // same storage, flags off (standalone applies, final normalise)
  double *traw, *z2raw, *corr, *sbuf;  // P^{-1} scratch
  double* zsc = nullptr;               // zero scalar slots (PCG-internal RhsSchur)
  double *x, *r, *z, *d, *q;           // PCG vectors (n+m)
  int hist_cap = 0;
  // CUDA graph of one PCG iteration inside a WHILE node
  cudaGraphExec_t gexec = nullptr;
  cudaGraph_t graph = nullptr;
  bool use_graph = true;
};

// ---------------------------------------------------------------------------
namespace {

// The message of the last failing call, per calling thread: the bulk and
// Schur inners of one preconditioner are set up on two threads at once
// (precond.py), and each caller reads its own error right after its call.
thread_local std::string tl_err;

bd_status fail(bd_ctx* ctx, bd_status st, const std::string& msg) {
  (void)ctx;
  tl_err = msg;
  return st;
}

#define CK(ctx, expr)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail((ctx), BD_ECUDA, std::string(#expr ": ") + cudaGetErrorString(e_));  \
  } while (0)

#define LAUNCHED(ctx)                                                                   \
  do {                                                                                  \
    (ctx)->launches++;                                                                  \
    cudaError_t e_ = cudaGetLastError();                                                \
    if (e_ != cudaSuccess)                                                              \
      return fail((ctx), BD_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

#define TRY(expr)                 \
  do {                            \
    bd_status st_ = (expr);       \
    if (st_ != BD_OK) return st_; \
  } while (0)

// BD_POISON=1: every library allocation starts as all-ones bytes (a NaN
// pattern), so a kernel that reads device memory nothing wrote turns the
// results into NaN and the parity tests catch it (tests/test_gpu_poison.py;
// the pool's compute-sanitizer is closed).
static bool poison_allocs() {
  static const bool on = getenv("BD_POISON") && atoi(getenv("BD_POISON")) != 0;
  return on;
}

template <class T>
cudaError_t dalloc(T** p, int64_t count) {
  const size_t bytes = sizeof(T) * (size_t)std::max<int64_t>(count, 1);
  cudaError_t e = cudaMalloc((void**)p, bytes);
  if (e == cudaSuccess && poison_allocs()) e = cudaMemset(*p, 0xFF, bytes);
  return e;
}

static double wall_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static void setup_log(const char* what, double t0) {
  if (getenv("BD_DEBUG")) std::fprintf(stderr, "[bd] setup %s %.2f s\n", what, wall_s() - t0);
}

int grid_for(bd_ctx* ctx, int64_t items, int per_block) {
  const int64_t need = (items + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)ctx->nsm * 8));
}

int pick_g(double avg) {
  int g = 4;
  while (g < 32 && g < avg) g <<= 1;
  return g;
}

// Caller-stream handoff.
struct Scope {
  bd_ctx* c;
  explicit Scope(bd_ctx* ctx) : c(ctx) {
    cudaEventRecord(c->ev_in, c->user);
    cudaStreamWaitEvent(c->stream, c->ev_in, 0);
  }
  ~Scope() {
    cudaEventRecord(c->ev_out, c->stream);
    cudaStreamWaitEvent(c->user, c->ev_out, 0);
  }
};

void prof_mark(bd_ctx* ctx, int cls) {
  if (!ctx->profile) return;
  cudaEvent_t e;
  if (ctx->pool.empty()) {
    cudaEventCreate(&e);
  } else {
    e = ctx->pool.back();
    ctx->pool.pop_back();
  }
  cudaEventRecord(e, ctx->stream);
  ctx->marks.push_back({e, cls});
  ctx->prof_launch[cls]++;
}

void prof_collect(bd_ctx* ctx) {
  if (ctx->marks.size() < 2) {
    for (auto& m : ctx->marks) ctx->pool.push_back(m.first);
    ctx->marks.clear();
    return;
  }
  cudaEventSynchronize(ctx->marks.back().first);
  for (size_t i = 1; i < ctx->marks.size(); ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->marks[i - 1].first, ctx->marks[i].first);
    ctx->prof_ms[ctx->marks[i].second] += ms;
  }
  for (auto& m : ctx->marks) ctx->pool.push_back(m.first);
  ctx->marks.clear();
}

cudaError_t ctl_alloc(Ctl* c, int64_t partials, int hist_cap, int use_flags) {
  cudaError_t e;
  if ((e = dalloc(&c->sc, dev::NSLOTS))) return e;
  if ((e = dalloc(&c->fl, dev::NFLAGS))) return e;
  if ((e = dalloc(&c->partials, std::max<int64_t>(partials, 4096) * 2))) return e;
  if ((e = dalloc(&c->ctr, dev::NCTR))) return e;
  if ((e = cudaMemset(c->sc, 0, sizeof(double) * dev::NSLOTS))) return e;
  if ((e = cudaMemset(c->fl, 0, sizeof(int) * dev::NFLAGS))) return e;
  if ((e = cudaMemset(c->ctr, 0, sizeof(unsigned) * dev::NCTR))) return e;
  c->hist_cap = hist_cap;
  if (hist_cap > 0) {
    if ((e = dalloc(&c->res_hist, hist_cap))) return e;
    if ((e = dalloc(&c->prec_hist, hist_cap))) return e;
  } else {
    c->res_hist = c->prec_hist = nullptr;
  }
  c->use_flags = use_flags;
  return cudaSuccess;
}

void ctl_free(Ctl* c, bool own_hist = true) {
  cudaFree(c->sc);
  cudaFree(c->fl);
  cudaFree(c->partials);
  cudaFree(c->ctr);
  if (own_hist) {
    cudaFree(c->res_hist);
    cudaFree(c->prec_hist);
  }
}

// ---- device Tri upload ------------------------------------------------------
bd_status upload_tri(bd_ctx* ctx, const HostCsr& t, bool lower, int G, DevTri* out) {
  std::vector<int32_t> level;
  out->depth = row_levels(t, lower, &level);
  std::vector<int32_t> tasks;
  build_schedule(level, out->depth, 32 / G, &tasks);
  out->n = (int)t.n;
  out->nnz = t.nnz();
  out->ntasks = (int)tasks.size();
  out->nvb = (int)((tasks.size() + (dev::TPB / G) - 1) / (dev::TPB / G));
  std::vector<int> rp(t.n + 1);
  for (int64_t i = 0; i <= t.n; ++i) rp[i] = (int)t.indptr[i];
  CK(ctx, dalloc(&out->rowptr, t.n + 1));
  CK(ctx, dalloc(&out->col, t.nnz()));
  CK(ctx, dalloc(&out->val, t.nnz()));
  CK(ctx, dalloc(&out->tasks, (int64_t)tasks.size()));
  CK(ctx, cudaMemcpy(out->rowptr, rp.data(), sizeof(int) * rp.size(), cudaMemcpyHostToDevice));
  CK(ctx, cudaMemcpy(out->col, t.indices.data(), sizeof(int) * t.nnz(), cudaMemcpyHostToDevice));
  CK(ctx, cudaMemcpy(out->val, t.values.data(), sizeof(double) * t.nnz(), cudaMemcpyHostToDevice));
  CK(ctx, cudaMemcpy(out->tasks, tasks.data(), sizeof(int) * tasks.size(), cudaMemcpyHostToDevice));
  return BD_OK;
}

void free_tri(DevTri* t) {
  cudaFree(t->rowptr);
  cudaFree(t->col);
  cudaFree(t->val);
  cudaFree(t->tasks);
}

template <class T>
cudaError_t upload_vec(T** dst, const std::vector<T>& v) {
  cudaError_t e = dalloc(dst, (int64_t)v.size());
  if (e) return e;
  if (v.empty()) return cudaSuccess;
  return cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice);
}

bd_status upload_tile(bd_ctx* ctx, const TileSchedule& ts, DevTile* out) {
  CK(ctx, upload_vec(&out->part_task_ptr, ts.part_task_ptr));
  CK(ctx, upload_vec(&out->part_step_ptr, ts.part_step_ptr));
  CK(ctx, upload_vec(&out->step_task_ptr, ts.step_task_ptr));
  CK(ctx, upload_vec(&out->task_row, ts.task_row));
  CK(ctx, upload_vec(&out->task_diag, ts.task_diag));
  CK(ctx, upload_vec(&out->ell_col, ts.ell_col));
  CK(ctx, upload_vec(&out->ell_val, ts.ell_val));
  out->max_part_rows = ts.max_part_rows;
  out->max_part_steps = ts.max_part_steps;
  out->nsteps = (int)ts.step_task_ptr.size() - 1;
  return BD_OK;
}

void free_tile(DevTile* t) {
  cudaFree(t->part_task_ptr);
  cudaFree(t->part_step_ptr);
  cudaFree(t->step_task_ptr);
  cudaFree(t->task_row);
  cudaFree(t->task_diag);
  cudaFree(t->ell_col);
  cudaFree(t->ell_val);
}

// Build the tiled schedules of an IC(0)-like factor; leaves p->tiled false if
// a row is too long or the part does not fit in shared memory.
bd_status setup_tiles(bd_inner* p, const HostCsr& lower, const HostCsr& upper,
                      const double* coords, int dim) {
  bd_ctx* ctx = p->ctx;
  const char* env = getenv("BD_NO_TILE");
  if (env && env[0] == '1') return BD_OK;
  int64_t maxoff = 0;
  for (int64_t i = 0; i < lower.n; ++i)
    maxoff = std::max<int64_t>(maxoff, lower.indptr[i + 1] - lower.indptr[i] - 1);
  for (int64_t i = 0; i < upper.n; ++i)
    maxoff = std::max<int64_t>(maxoff, upper.indptr[i + 1] - upper.indptr[i] - 1);
  int G = 4;
  while (G < maxoff) G <<= 1;
  if (G > 16) return BD_OK;
  int threads = std::min(1024, 128 * G);
  if (const char* e = getenv("BD_TILE_THREADS")) threads = atoi(e);
  int R = threads / G;
  if (p->rows_mode) {
    R = getenv("BD_TILE_ROWS") ? atoi(getenv("BD_TILE_ROWS")) : 128;
    threads = 512;
  }
  int parts = (int)std::max<int64_t>(1, std::min<int64_t>(ctx->nsm, lower.n / 1024));
  if (const char* e = getenv("BD_TILE_PARTS")) parts = std::max(1, atoi(e));
  std::vector<int32_t> part;
  if (coords && dim > 0)
    partition_coords(lower.n, dim, coords, parts, &part);
  else
    partition_rows(lower, parts, &part);
  TileSchedule tl, tu;
  if (!build_tile_schedule(lower, true, part, parts, G, R, &tl, p->rows_mode)) return BD_OK;
  if (!build_tile_schedule(upper, false, part, parts, G, R, &tu, p->rows_mode)) return BD_OK;
  const int mrows = std::max(tl.max_part_rows, tu.max_part_rows);
  const int msteps = std::max(tl.max_part_steps, tu.max_part_steps);
  const int stages = getenv("BD_TILE_D") ? atoi(getenv("BD_TILE_D")) : kTileStages;
  const size_t smem = p->rows_mode ? dev::tile2_smem_bytes(mrows, msteps, R, G, stages)
                                   : dev::tile_smem_bytes(mrows, msteps, threads, G, stages);
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  if (smem + 1024 > (size_t)max_smem) return BD_OK;  // 1 KB headroom for static smem
  TRY(upload_tile(ctx, tl, &p->TL));
  TRY(upload_tile(ctx, tu, &p->TU));
  p->TL.max_part_rows = p->TU.max_part_rows = mrows;
  p->TL.max_part_steps = p->TU.max_part_steps = msteps;
  p->TG = G;
  p->tparts = parts;
  p->tthreads = threads;
  p->tsmem = smem;
  p->tstages = stages;
  p->trows = R;
  p->tiled = true;
  return BD_OK;
}

// ELL, level-ordered schedule for the persistent sync-free kernel.
bd_status build_ell(bd_ctx* ctx, const HostCsr& t, bool lower, int G, DevEll* out) {
  std::vector<int32_t> level, tasks;
  const int64_t depth = row_levels(t, lower, &level);
  build_schedule(level, depth, 32 / G, &tasks);
  const int64_t nt = (int64_t)tasks.size();
  std::vector<double> diag(nt, 1.0), val(nt * G, 0.0);
  std::vector<int32_t> col(nt * G, -1);
  for (int64_t k = 0; k < nt; ++k) {
    const int32_t row = tasks[k];
    if (row < 0) continue;
    int cnt = 0;
    for (int64_t q = t.indptr[row]; q < t.indptr[row + 1]; ++q) {
      const int32_t cidx = t.indices[q];
      if (cidx == row) {
        diag[k] = t.values[q];
        continue;
      }
      if (cnt == G) return BD_EINVAL;
      col[k * G + cnt] = cidx;
      val[k * G + cnt] = t.values[q];
      ++cnt;
    }
  }
  CK(ctx, upload_vec(&out->task_row, tasks));
  CK(ctx, upload_vec(&out->task_diag, diag));
  CK(ctx, upload_vec(&out->ell_col, col));
  CK(ctx, upload_vec(&out->ell_val, val));
  out->ntasks = (int)nt;
  const int rpc = dev::TPB / G;
  out->nchunks = (int)((nt + rpc - 1) / rpc);
  // ~3 levels of rows in flight
  const int64_t rows_flight = 3 * std::max<int64_t>(1, t.n / std::max<int64_t>(1, depth));
  const char* env = getenv("BD_PERSIST_LEVELS");
  const int64_t lv = env ? std::max(1, atoi(env)) : 3;
  const int64_t want = (lv * std::max<int64_t>(1, t.n / std::max<int64_t>(1, depth)) + rpc - 1) / rpc;
  (void)rows_flight;
  out->grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)ctx->nsm * 8));
  out->grid = std::min(out->grid, out->nchunks);
  return BD_OK;
}

void free_ell(DevEll* e) {
  cudaFree(e->task_row);
  cudaFree(e->task_diag);
  cudaFree(e->ell_col);
  cudaFree(e->ell_val);
}

// Supernodes of a lower CSR factor (diagonal last): maximal runs of rows whose
// mutual dependencies form a dense triangle; then level-ordered task lists
// for the forward (L) and backward (U = L^T) passes.
bd_status build_super(bd_ctx* ctx, const HostCsr& L, DevSuper* fw, DevSuper* bw) {
  const int64_t n = L.n;
  std::vector<int32_t> start, size, sn_of(n);
  int32_t c0 = 0;
  for (int64_t i = 0; i < n; ++i) {
    bool join = false;
    const int64_t k = i - c0;
    if (i > 0 && k < dev::SN_MAX) {
      const int64_t e = L.indptr[i + 1], off = e - 1 - L.indptr[i];
      if (off >= k && k > 0)
        join = L.indices[e - 1 - k] == c0 && L.indices[e - 2] == (int32_t)(i - 1);
    }
    if (!join) {
      if (i > 0) size.push_back((int32_t)(i - c0));
      c0 = (int32_t)i;
      start.push_back(c0);
    }
    sn_of[i] = (int32_t)start.size() - 1;
  }
  size.push_back((int32_t)(n - c0));
  const int64_t ns = (int64_t)start.size();
  // forward levels: external columns (< start) point to earlier supernodes
  std::vector<int32_t> lvf(ns, 0), lvb(ns, 0);
  for (int64_t s = 0; s < ns; ++s) {
    int32_t lv = 0;
    for (int64_t i = start[s]; i < start[s] + size[s]; ++i)
      for (int64_t q = L.indptr[i]; q < L.indptr[i + 1]; ++q) {
        const int32_t j = L.indices[q];
        if (j < start[s]) lv = std::max(lv, lvf[sn_of[j]] + 1);
      }
    lvf[s] = lv;
  }
  // backward levels: supernode s depends on the supernodes of rows j > end that
  // have s-rows in their pattern (U = L^T): propagate from L's rows
  {
    // dependency t -> s for every external entry (i in t, j in s, j < start[t])
    std::vector<std::vector<int32_t>> users(ns);
    for (int64_t t = 0; t < ns; ++t)
      for (int64_t i = start[t]; i < start[t] + size[t]; ++i)
        for (int64_t q = L.indptr[i]; q < L.indptr[i + 1]; ++q) {
          const int32_t j = L.indices[q];
          if (j < start[t]) {
            auto& u = users[sn_of[j]];
            if (u.empty() || u.back() != (int32_t)t) u.push_back((int32_t)t);
          }
        }
    for (int64_t s = ns - 1; s >= 0; --s) {
      int32_t lv = 0;
      for (int32_t t : users[s]) lv = std::max(lv, lvb[t] + 1);
      lvb[s] = lv;
    }
  }
  // external entries of each supernode's rows (forward: columns < start)
  std::vector<int64_t> ext(ns, 0);
  for (int64_t sn = 0; sn < ns; ++sn)
    for (int64_t i = start[sn]; i < start[sn] + size[sn]; ++i)
      ext[sn] += L.indptr[i + 1] - L.indptr[i] - 1 - (i - start[sn]);
  // backward (U = L^T): the external entries of row j are L's entries (i, j)
  // below j's supernode
  std::vector<int64_t> extb(ns, 0);
  for (int64_t sn = 0; sn < ns; ++sn)
    for (int64_t i = start[sn]; i < start[sn] + size[sn]; ++i)
      for (int64_t q = L.indptr[i]; q < L.indptr[i + 1]; ++q)
        if (L.indices[q] < start[sn]) ++extb[sn_of[L.indices[q]]];
  const int64_t split_min = getenv("BD_SUPER_SPLIT") ? atoll(getenv("BD_SUPER_SPLIT")) : 8192;
  // whole-block inverses from this many rows (used below and by the dense-phase split)
  const int64_t inv_min = getenv("BD_SUPER_INV_MIN") ? atoll(getenv("BD_SUPER_INV_MIN")) : 128;
  // split the dense GEMV of supernodes of at least this many rows (0: never)
  const int64_t dsplit_min_env = getenv("BD_SUPER_DSPLIT") ? atoll(getenv("BD_SUPER_DSPLIT")) : 128;
  const int64_t dsplit_min = dsplit_min_env > 0 ? dsplit_min_env : (int64_t)1 << 40;
  // (config 1, ms per step: 16 rows 8.72, 32 8.90, 64 9.16, 128 9.50; no
  // slicing 12.45: profiles/r02_cfg1_relax_sweep.txt)
  const int dch = std::max(16, std::min(256, getenv("BD_SUPER_DCHUNK") ? atoi(getenv("BD_SUPER_DCHUNK"))
                                                                       : 16));
  fw->dchunk = bw->dchunk = dch;
  // dense block of supernode sn: D[k][j] (j <= k) = L[start+k][start+j], the
  // last k+1 entries of the row (diagonal last)
  auto dense = [&](int64_t c0, int64_t k, int64_t j) -> long double {
    return L.values[L.indptr[c0 + k + 1] - 1 - k + j];
  };
  auto order = [&](const std::vector<int32_t>& lv, DevSuper* out, bool split,
                   const std::vector<int64_t>& ext) -> bd_status {
    std::vector<int32_t> idx(ns);
    std::iota(idx.begin(), idx.end(), 0);
    // lanes per small supernode: one warp each by default; BD_SUPER_PACK=1
    // packs 32/W of them per warp, W the next power of two >= the size (at
    // least 4) -- measured neutral-to-slower on cfg1 (18.3 vs 17.9 ms/step)
    const bool pack = getenv("BD_SUPER_PACK") && atoi(getenv("BD_SUPER_PACK")) != 0;
    auto lanes = [&](int32_t s) -> int {
      if (!pack || size[s] > 16) return 32;
      return size[s] > 8 ? 16 : size[s] > 4 ? 8 : 4;
    };
    // level order; within a level, small supernodes grouped by lane width
    std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) {
      return lv[a] != lv[b] ? lv[a] < lv[b] : lanes(a) < lanes(b);
    });
    std::vector<int32_t> st(ns), sz(ns), tasks;
    for (int64_t k = 0; k < ns; ++k) {
      st[k] = start[idx[k]];
      sz[k] = size[idx[k]];
    }
    // tasks: a big supernode alone, or up to 16 small ones of the same level.
    // Forward: a big supernode with a heavy external phase (the separators of
    // a nested-dissection factor, whose rows carry the fill of their whole
    // subtree) gets its external phase split into SN_CHUNK-row chunk tasks
    // placed right before it, so many CTAs stream it; the supernode's own task
    // then waits for its chunks and does the dense phase.
    std::vector<int32_t> kind, arg, tw;
    bool any_split = false, any_pack = false;
    for (int64_t k = 0; k < ns;) {
      if (sz[k] > 32) {
        if (split && ext[idx[k]] >= split_min) {
          const int nch = (sz[k] + dev::SN_CHUNK - 1) / dev::SN_CHUNK;
          for (int ch = 0; ch < nch; ++ch) {
            tasks.push_back((int32_t)k);
            kind.push_back(1);
            arg.push_back(ch * dev::SN_CHUNK);
          }
          // the dense phase: one task, or (big supernodes with a whole-block
          // inverse) DCH-row slices of its GEMV spread over several CTAs
          // (kind 3: arg = ext chunks | slice << 8 | slices << 16)
          const int nd = (inv_min > 0 && sz[k] >= inv_min && sz[k] >= dsplit_min)
                             ? (int)((sz[k] + dch - 1) / dch)
                             : 0;
          if (nd > 1) {
            for (int q = 0; q < nd; ++q) {
              tasks.push_back((int32_t)k);
              kind.push_back(3);
              arg.push_back(nch | (q << 8) | (nd << 16));
            }
          } else {
            tasks.push_back((int32_t)k);
            kind.push_back(2);
            arg.push_back(nch);
          }
          any_split = true;
        } else {
          tasks.push_back((int32_t)k);
          kind.push_back(0);
          arg.push_back(0);
        }
        tw.resize(tasks.size(), 32);
        ++k;
        continue;
      }
      // up to 16 warps x 32/W supernodes of one level and lane width W
      const int W = lanes(idx[k]);
      tasks.push_back((int32_t)k);
      kind.push_back(0);
      arg.push_back(0);
      tw.push_back(W);
      any_pack |= W < 32;
      int64_t e = k + 1;
      while (e < ns && e - k < 16 * (32 / W) && sz[e] <= 32 && lv[idx[e]] == lv[idx[k]] &&
             lanes(idx[e]) == W)
        ++e;
      k = e;
    }
    tasks.push_back((int32_t)ns);
    // inverses of the 32x32 diagonal blocks of every panel of the big
    // supernodes, in solve order (forward: rows ascending, B = D[P][P];
    // backward, U = L^T: rows descending, B[l][m] = D[q-m][q-l] with
    // q = ns-1-p0), each padded to 32x32, in long double
    if (!getenv("BD_SUPER_NOPINV")) {
      std::vector<int32_t> pan(ns, -1);
      std::vector<double> pinv;
      std::vector<long double> B(32 * 32), X(32 * 32);
      const bool fwd = out == fw;
      for (int64_t k = 0; k < ns; ++k) {
        if (sz[k] <= 32) continue;
        pan[k] = (int32_t)(pinv.size() / 1024);
        const int64_t c0 = st[k], nsz = sz[k];
        for (int64_t p0 = 0; p0 < nsz; p0 += 32) {
          const int pn = (int)std::min<int64_t>(32, nsz - p0);
          for (int l = 0; l < pn; ++l)
            for (int m = 0; m <= l; ++m)
              B[l * 32 + m] = fwd ? dense(c0, p0 + l, p0 + m)
                                  : dense(c0, nsz - 1 - p0 - m, nsz - 1 - p0 - l);
          std::fill(X.begin(), X.end(), 0.0L);
          for (int l = 0; l < pn; ++l) {  // X = B^{-1}, lower triangular
            for (int m = 0; m <= l; ++m) {
              long double acc = (l == m) ? 1.0L : 0.0L;
              for (int j = m; j < l; ++j) acc -= B[l * 32 + j] * X[j * 32 + m];
              X[l * 32 + m] = acc / B[l * 32 + l];
            }
          }
          for (int q = 0; q < 1024; ++q) pinv.push_back((double)X[q]);
        }
      }
      if (!pinv.empty()) {
        CK(ctx, upload_vec(&out->pinv, pinv));
        CK(ctx, upload_vec(&out->sn_pan, pan));
      }
    }
    // whole diagonal-block inverses (solve order, packed lower rows) for the
    // supernodes of at least BD_SUPER_INV_MIN rows: their dense phase becomes
    // one GEMV instead of ns/32 dependent panel steps
    {
      std::vector<long long> off(ns, -1);
      long long tot = 0;
      std::vector<int64_t> which;
      for (int64_t k = 0; k < ns; ++k)
        if (inv_min > 0 && sz[k] >= inv_min && sz[k] > 32) {
          off[k] = tot;
          tot += (long long)sz[k] * (sz[k] + 1) / 2;
          which.push_back(k);
        }
      if (tot > 0) {
        std::vector<double> sinv((size_t)tot);
        const bool fwd = out == fw;
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t w = 0; w < (int64_t)which.size(); ++w) {
          const int64_t k = which[w], c0 = st[k], m = sz[k];
          std::vector<long double> B((size_t)m * m), X((size_t)m * m, 0.0L);
          for (int64_t l = 0; l < m; ++l)
            for (int64_t q = 0; q <= l; ++q)
              B[l * m + q] = fwd ? dense(c0, l, q) : dense(c0, m - 1 - q, m - 1 - l);
          // X = B^{-1} column by column (forward substitution)
          for (int64_t q = 0; q < m; ++q)
            for (int64_t l = q; l < m; ++l) {
              long double acc = (l == q) ? 1.0L : 0.0L;
              for (int64_t j = q; j < l; ++j) acc -= B[l * m + j] * X[j * m + q];
              X[l * m + q] = acc / B[l * m + l];
            }
          double* dst = sinv.data() + off[k];
          for (int64_t l = 0; l < m; ++l)
            for (int64_t q = 0; q <= l; ++q) dst[l * (l + 1) / 2 + q] = (double)X[l * m + q];
        }
        CK(ctx, upload_vec(&out->sinv, sinv));
        CK(ctx, upload_vec(&out->sn_inv, off));
      }
    }
    CK(ctx, upload_vec(&out->sn_start, st));
    CK(ctx, upload_vec(&out->sn_size, sz));
    CK(ctx, upload_vec(&out->task_sn, tasks));
    if (any_pack) CK(ctx, upload_vec(&out->task_w, tw));
    if (any_split) {
      CK(ctx, upload_vec(&out->task_kind, kind));
      CK(ctx, upload_vec(&out->task_arg, arg));
      std::vector<int32_t> zeros(ns, 0);
      CK(ctx, upload_vec(&out->sn_cnt, zeros));
    }
    out->ntasks = (int)tasks.size() - 1;
    out->grid = (int)std::max<int64_t>(1, std::min<int64_t>(out->ntasks, (int64_t)ctx->nsm * 2));
    return BD_OK;
  };
  TRY(order(lvf, fw, !getenv("BD_SUPER_NOSPLIT"), ext));
  TRY(order(lvb, bw, !getenv("BD_SUPER_NOSPLIT") &&
                         !(getenv("BD_SUPER_SPLITB") && atoi(getenv("BD_SUPER_SPLITB")) == 0),
            extb));
  if (getenv("BD_DEBUG")) {
    int64_t big = 0, maxsz = 0, rows_big = 0;
    for (int64_t s = 0; s < ns; ++s) {
      maxsz = std::max<int64_t>(maxsz, size[s]);
      if (size[s] >= 32) {
        ++big;
        rows_big += size[s];
      }
    }
    const int32_t df = *std::max_element(lvf.begin(), lvf.end()) + 1;
    const int32_t db = *std::max_element(lvb.begin(), lvb.end()) + 1;
    std::fprintf(stderr,
                 "[bd] supernodes n=%lld count=%lld (>=32 rows: %lld covering %lld rows) max=%lld "
                 "levels fwd=%d bwd=%d\n",
                 (long long)n, (long long)ns, (long long)big, (long long)rows_big,
                 (long long)maxsz, df, db);
  }
  return BD_OK;
}

void free_super(DevSuper* s) {
  cudaFree(s->pinv);
  cudaFree(s->sn_pan);
  cudaFree(s->task_kind);
  cudaFree(s->task_arg);
  cudaFree(s->sn_cnt);
  cudaFree(s->sn_start);
  cudaFree(s->sn_size);
  cudaFree(s->task_sn);
  cudaFree(s->task_w);
  cudaFree(s->sinv);
  cudaFree(s->sn_inv);
}

bd_status upload_cluster(bd_ctx* ctx, const ClusterSchedule& cs, DevCluster* out) {
  CK(ctx, upload_vec(&out->lvl_ptr, cs.lvl_ptr));
  CK(ctx, upload_vec(&out->task_row, cs.task_row));
  CK(ctx, upload_vec(&out->task_diag, cs.task_diag));
  CK(ctx, upload_vec(&out->ell_val, cs.ell_val));
  std::vector<short> code(cs.ell_code.begin(), cs.ell_code.end());
  CK(ctx, upload_vec(&out->ell_code, code));
  CK(ctx, upload_vec(&out->exp_ptr, cs.exp_ptr));
  CK(ctx, upload_vec(&out->exp_src, cs.exp_src));
  CK(ctx, upload_vec(&out->exp_dst, cs.exp_dst));
  out->nlevels = cs.nlevels;
  out->W = cs.W;
  out->wmax = cs.wmax;
  out->rmax = cs.rmax;
  out->emax = std::max(cs.emax, 4);
  out->E = cs.E;
  out->ntasks = (int64_t)cs.task_row.size();
  out->smem = dev::cl_smem_bytes(out->rmax, out->emax, out->wmax, out->W, out->E,
                                 kClusterStagesDeep, out->nlevels);
  out->deep = true;
  if (out->smem + 1024 > 232448) {
    out->deep = false;
    out->smem = dev::cl_smem_bytes(out->rmax, out->emax, out->wmax, out->W, out->E, kClusterStages,
                                   out->nlevels);
  }
  return BD_OK;
}

void free_cluster(DevCluster* c) {
  cudaFree(c->lvl_ptr);
  cudaFree(c->task_row);
  cudaFree(c->task_diag);
  cudaFree(c->ell_val);
  cudaFree(c->ell_code);
  cudaFree(c->exp_ptr);
  cudaFree(c->exp_src);
  cudaFree(c->exp_dst);
}

// Cluster-wavefront schedules for an IC(0)-like factor; leaves p->cluster false
// (with the reason under BD_DEBUG) when the structure does not qualify.
bd_status setup_cluster(bd_inner* p, const HostCsr& lower, const HostCsr& upper,
                        const double* coords, int dim) {
  bd_ctx* ctx = p->ctx;
  const int P = kClusterParts;
  if (lower.n < 64 * P) return BD_OK;
  std::vector<int32_t> part;
  if (coords && dim > 0)
    partition_coords(lower.n, dim, coords, P, &part);
  else
    partition_rows(lower, P, &part);
  int E = 4;
  for (int64_t i = 0; i < lower.n; ++i)
    while (E < lower.indptr[i + 1] - lower.indptr[i] - 1) E <<= 1;
  for (int64_t i = 0; i < upper.n; ++i)
    while (E < upper.indptr[i + 1] - upper.indptr[i] - 1) E <<= 1;
  if (E > 8) return BD_OK;
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  ClusterSchedule cl, cu;
  std::string why;
  bool ok = build_cluster_schedule(lower, true, part, P, E, 4, 4096, 8192, &cl, &why) &&
            build_cluster_schedule(upper, false, part, P, E, 4, 4096, 8192, &cu, &why);
  if (ok) {
    TRY(upload_cluster(ctx, cl, &p->CL));
    TRY(upload_cluster(ctx, cu, &p->CU));
    if (std::max(p->CL.smem, p->CU.smem) + 1024 > (size_t)max_smem) {
      ok = false;
      why = "shared memory";
    }
  }
  if (getenv("BD_DEBUG"))
    std::fprintf(stderr, "[bd] cluster schedule n=%lld: %s (levels %d, rmax %d, wmax %d, smem %zu)\n",
                 (long long)lower.n, ok ? "ok" : why.c_str(), cl.nlevels, cl.rmax, cl.wmax,
                 std::max(p->CL.smem, p->CU.smem));
  if (!ok) return BD_OK;
  CK(ctx, dalloc(&p->rtmp, std::max(p->CL.ntasks, p->CU.ntasks)));
  p->cluster = true;
  p->G = E;
  return BD_OK;
}

template <int E, class Rhs>
bd_status launch_cluster(bd_inner* p, const DevCluster& cd, const Rhs& rhs, double* xg,
                         const Ctl& c) {
  bd_ctx* ctx = p->ctx;
  auto kern = cd.deep ? dev::k_trsv_cluster<E, kClusterStagesDeep, Rhs>
                     : dev::k_trsv_cluster<E, kClusterStages, Rhs>;
  CK(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cd.smem));
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kClusterParts;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kClusterParts);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = cd.smem;
  cfg.stream = ctx->stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(ctx, cudaLaunchKernelEx(&cfg, kern, cd.dev(), rhs, xg, p->rtmp, c));
  LAUNCHED(ctx);
  return BD_OK;
}

bd_status upload_dtile(bd_ctx* ctx, const DTileSchedule& ds, DevDTile* out) {
  CK(ctx, upload_vec(&out->tile_row_ptr, ds.tile_row_ptr));
  CK(ctx, upload_vec(&out->tile_step_ptr, ds.tile_step_ptr));
  CK(ctx, upload_vec(&out->step_row, ds.step_row));
  CK(ctx, upload_vec(&out->task_row, ds.task_row));
  CK(ctx, upload_vec(&out->task_diag, ds.task_diag));
  CK(ctx, upload_vec(&out->ell_col, ds.ell_col));
  CK(ctx, upload_vec(&out->ell_val, ds.ell_val));
  out->ntiles = (int)ds.tile_row_ptr.size() - 1;
  out->tmax = ds.tmax;
  out->threads = std::max(32, (ds.tmax + 31) / 32 * 32);  // one row per thread (<= 256)
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::k_trsv_dtile<8, dev::RhsGather>,
                                                out->threads, 0);
  out->grid = (int)std::min<int64_t>(out->ntiles, (int64_t)ctx->nsm * std::max(1, per_sm));
  return BD_OK;
}

void free_dtile(DevDTile* d) {
  cudaFree(d->tile_row_ptr);
  cudaFree(d->tile_step_ptr);
  cudaFree(d->step_row);
  cudaFree(d->task_row);
  cudaFree(d->task_diag);
  cudaFree(d->ell_col);
  cudaFree(d->ell_val);
}

bd_status setup_dtile(bd_inner* p, const HostCsr& lower, const HostCsr& upper,
                      const double* coords, int dim) {
  bd_ctx* ctx = p->ctx;
  const int target = getenv("BD_DTILE_ROWS") ? atoi(getenv("BD_DTILE_ROWS")) : 64;
  const char* part = getenv("BD_TILE_PART");
  const bool grid = !(part && std::string(part) == "rcb");
  int ntiles = (int)std::max<int64_t>(1, lower.n / target);
  std::vector<int32_t> tile;
  // Row orderings that concatenate coordinate-sorted blocks (the heart-first
  // numbering of bd/mesh.py:252-263: heart vertices, then torso vertices, each
  // in lattice order) make lattice tiles that mix the blocks cyclic.  Detect
  // the blocks as the descents of the lexicographic coordinate order and keep
  // them in separate tiles (partition_grid's class argument).
  std::vector<int32_t> cls;
  if (coords && dim > 0) {
    int nd = 0;
    cls.assign(lower.n, 0);
    for (int64_t i = 1; i < lower.n; ++i) {
      bool less = false;  // coords[i] < coords[i-1] lexicographically
      for (int a = 0; a < dim; ++a) {
        const double x = coords[i * dim + a], y = coords[(i - 1) * dim + a];
        if (x != y) {
          less = x < y;
          break;
        }
      }
      nd += less;
      cls[i] = nd;
    }
    if (nd == 0 || nd > 8) cls.clear();
  }
  if (coords && dim > 0 && grid)
    ntiles = partition_grid(lower.n, dim, coords, target, cls.empty() ? nullptr : &cls, &tile);
  else if (coords && dim > 0)
    partition_coords(lower.n, dim, coords, ntiles, &tile);
  else
    partition_rows(lower, ntiles, &tile);
  int E = 4;
  for (int64_t i = 0; i < lower.n; ++i)
    while (E < lower.indptr[i + 1] - lower.indptr[i] - 1) E <<= 1;
  for (int64_t i = 0; i < upper.n; ++i)
    while (E < upper.indptr[i + 1] - upper.indptr[i] - 1) E <<= 1;
  if (E > 8) return BD_OK;
  DTileSchedule dl, du;
  std::string why;
  bool ok = build_dtile_schedule(lower, true, tile, ntiles, E, &dl, &why) &&
            build_dtile_schedule(upper, false, tile, ntiles, E, &du, &why);
  if (!ok && coords && dim > 0 && grid) {
    ntiles = (int)std::max<int64_t>(1, lower.n / target);
    partition_coords(lower.n, dim, coords, ntiles, &tile);
    ok = build_dtile_schedule(lower, true, tile, ntiles, E, &dl, &why) &&
         build_dtile_schedule(upper, false, tile, ntiles, E, &du, &why);
  }
  if (ok && (std::max(dl.tmax, du.tmax) > dev::DT_MAX_ROWS ||
             std::max(dl.smax, du.smax) > dev::DT_MAX_STEPS)) {
    ok = false;
    why = "tile too large";
  }
  if (getenv("BD_DEBUG"))
    std::fprintf(stderr, "[bd] dtile n=%lld tiles=%d: %s (tmax %d, smax %d)\n", (long long)lower.n,
                 ntiles, ok ? "ok" : why.c_str(), dl.tmax, dl.smax);
  if (!ok) return BD_OK;
  TRY(upload_dtile(ctx, dl, &p->DL));
  TRY(upload_dtile(ctx, du, &p->DU));
  p->G = E;
  p->dtile = true;
  return BD_OK;
}

bd_status upload_btile(bd_ctx* ctx, const BTileSchedule& bs, DevBTile* out) {
  // re-lay the schedule out with fixed per-tile strides; external entries as
  // a compact per-tile list (row ranges, input slots, values)
  const int nt = (int)bs.tile_row_ptr.size() - 1;
  const int ex = bs.Ex, rs = (bs.tmax + 3) & ~3, xs = (bs.xmax + 3) & ~3;  // 16-byte int rows
  const int64_t is = dev::bt_even(rs * (rs + 1) / 2);
  const int rps = dev::bt_round8(rs + 1);
  int emax = 0;
#pragma omp parallel for reduction(max : emax) schedule(static)
  for (int t = 0; t < nt; ++t) {
    int cnt = 0;
    for (int64_t k = bs.tile_row_ptr[t]; k < bs.tile_row_ptr[t + 1]; ++k)
      for (int e = 0; e < ex; ++e) cnt += bs.ext_col[k * ex + e] >= 0;
    emax = std::max(emax, cnt);
  }
  const int es = dev::bt_round8(std::max(emax, 1));
  out->exw = ex;
  if (emax > 65535 || bs.xmax > 65535) return fail(ctx, BD_EINVAL, "btile: tile too large");
  std::vector<int32_t> nr(nt), row((size_t)nt * rs, -1), in((size_t)nt * xs, -1);
  std::vector<uint16_t> rp((size_t)nt * rps, 0), slot((size_t)nt * es, 0);
  std::vector<double> val((size_t)nt * es, 0.0), inv((size_t)nt * is, 0.0);
  // tiles fill disjoint ranges: host threads
#pragma omp parallel for schedule(dynamic, 64)
  for (int t = 0; t < nt; ++t) {
    const int r0 = bs.tile_row_ptr[t], n_ = bs.tile_row_ptr[t + 1] - r0;
    nr[t] = n_;
    int cnt = 0;
    for (int k = 0; k < rs + 1 && k < rps; ++k) {
      rp[(size_t)t * rps + k] = (uint16_t)cnt;
      if (k >= n_) continue;
      row[(size_t)t * rs + k] = bs.task_row[r0 + k];
      for (int e = 0; e < ex; ++e) {
        const int32_t sl = bs.ext_col[(size_t)(r0 + k) * ex + e];
        if (sl < 0) continue;
        slot[(size_t)t * es + cnt] = (uint16_t)sl;
        val[(size_t)t * es + cnt] = bs.ext_val[(size_t)(r0 + k) * ex + e];
        ++cnt;
      }
    }
    const int x0 = bs.tile_in_ptr[t], nx = bs.tile_in_ptr[t + 1] - x0;
    for (int j = 0; j < nx; ++j) in[(size_t)t * xs + j] = bs.in_col[x0 + j];
    // packed row-major (k(k+1)/2 + l) -> packed column-major (l*n - l(l-1)/2 + k - l)
    const int64_t i0 = bs.tile_inv_ptr[t];
    for (int k = 0; k < n_; ++k)
      for (int l = 0; l <= k; ++l)
        inv[(size_t)t * is + (size_t)l * n_ - (size_t)l * (l - 1) / 2 + (k - l)] =
            bs.inv[i0 + (int64_t)k * (k + 1) / 2 + l];
  }
  CK(ctx, upload_vec(&out->tile_nr, nr));
  CK(ctx, upload_vec(&out->task_row, row));
  CK(ctx, upload_vec(&out->ent_rp, rp));
  CK(ctx, upload_vec(&out->ent_slot, slot));
  CK(ctx, upload_vec(&out->ent_val, val));
  CK(ctx, upload_vec(&out->in_col, in));
  CK(ctx, upload_vec(&out->inv, inv));
  out->ntiles = nt;
  out->rs = rs;
  out->xs = xs;
  out->is = (int)is;
  out->es = es;
  out->rps = rps;
  out->threads = std::min(256, std::max(32, dev::BT_LANES * ((bs.tmax + 7) / 8 * 8)));
  out->threads = std::max(out->threads, std::min(256, (rs + 31) / 32 * 32));
  if (getenv("BD_BTILE_THREADS"))
    out->threads = std::max((rs + 31) / 32 * 32,
                            std::min(256, atoi(getenv("BD_BTILE_THREADS")) / 32 * 32));
  out->threads = std::max(out->threads, ((xs + 1) / 2 + 31) / 32 * 32);  // <= 2 inputs per thread
  out->sleep_ns = getenv("BD_BTILE_SLEEP") ? atoi(getenv("BD_BTILE_SLEEP")) : 0;
  out->prefetch = getenv("BD_BTILE_PREFETCH") ? atoi(getenv("BD_BTILE_PREFETCH")) : 1;
  out->poll_depth = getenv("BD_BTILE_POLL") ? atoi(getenv("BD_BTILE_POLL")) : 1;
  out->smem = dev::bt_smem(rs, xs, (int)is, es, rps);
  auto kg = dev::k_trsv_btile<dev::RhsGather>;
  auto kv = dev::k_trsv_btile<dev::RhsVec>;
  auto ks = dev::k_trsv_btile<dev::RhsSchur>;
  // the attribute is per kernel and device, shared by every schedule: only
  // ever raise it (check-and-set under a lock: two inners may be set up on
  // two threads at once)
  {
    static std::mutex mu;
    static size_t smem_attr[64] = {};
    int dev_id = 0;
    CK(ctx, cudaGetDevice(&dev_id));
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = smem_attr[dev_id & 63];
    if (out->smem > cur) {
      const int sm = (int)out->smem;
      CK(ctx, cudaFuncSetAttribute(kg, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      CK(ctx, cudaFuncSetAttribute(kv, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      CK(ctx, cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      cur = out->smem;
    }
  }
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ks, out->threads, out->smem);
  {
    // "auto" (default) | "reg" | "rsmem" | "regt" | "pipe" | "smem" (k_trsv_btile)
    const char* kern = getenv("BD_BTILE_KERNEL");
    std::string kn = kern ? kern : "auto";
    if (kn == "auto") {
      // Latency-bound passes (few tiles per level of the tile DAG) want the
      // register inverse (shortest on-path compute); throughput-bound ones
      // (wide levels, e.g. config 3) want more tiles in flight per SM, i.e.
      // the inverse staged in shared memory (6 CTAs/SM instead of 4).
      // Measured crossover: cfg2 ~230 tiles/level -> reg,
      // 192x192x96 ~470 and cfg3 ~900 -> rsmem.
      std::vector<int32_t> row_tile(bs.task_row.empty() ? 0 : 1 + *std::max_element(
                                                                    bs.task_row.begin(), bs.task_row.end()), -1);
      for (int t = 0; t < nt; ++t)
        for (int64_t q = bs.tile_row_ptr[t]; q < bs.tile_row_ptr[t + 1]; ++q) row_tile[bs.task_row[q]] = t;
      std::vector<int32_t> lev(nt, 0);
      int depth = 0;
      for (int t = 0; t < nt; ++t) {  // task order is topological
        int l = 0;
        for (int32_t j = bs.tile_in_ptr[t]; j < bs.tile_in_ptr[t + 1]; ++j)
          l = std::max(l, lev[row_tile[bs.in_col[j]]] + 1);
        lev[t] = l;
        depth = std::max(depth, l + 1);
      }
      const double width = (double)nt / std::max(1, depth);
      // k_trsv_rpipe (TMA ring) beats both in both regimes (cfg2 pair 379 -> 307 us,
      // cfg3 1534 -> 1330 us); the others remain selectable
      kn = (rs <= dev::RT_ROWS && xs <= 512 && ex <= 16) ? "rpipe" : (width > 350.0 ? "rsmem" : "reg");
      if (getenv("BD_DEBUG"))
        std::fprintf(stderr, "[bd] btile auto: %d tiles, tile-DAG depth %d, %.0f tiles/level -> %s\n", nt,
                     depth, width, kn.c_str());
    }
    if (ex > 8 && kn == "smem") kn = "reg";  // k_trsv_btile handles <= 8 external entries per row
    if (kn == "pipe" && rs <= dev::RT_ROWS && xs <= 512 && ex <= 8) {
      out->pipe = true;
      out->threads = 256;
      out->smem = dev::pt_smem(rs, xs, (int)is, es, rps);
      CK(ctx, cudaFuncSetAttribute(dev::k_trsv_ptile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)out->smem));
      CK(ctx, cudaFuncSetAttribute(dev::k_trsv_ptile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)out->smem));
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::k_trsv_ptile<true>, 256, out->smem);
    } else if (kn == "rpipe" && rs <= dev::RT_ROWS && xs <= 512 && ex <= 16) {
      // one packed record per tile (dev::rp_layout), fetched by one TMA bulk copy
      const dev::RpLayout lay = dev::rp_layout(rs, xs, dev::RP_INV, es, rps);
      std::vector<unsigned char> rec((size_t)nt * lay.bytes, 0);
#pragma omp parallel for schedule(static)
      for (int t = 0; t < nt; ++t) {
        unsigned char* r = rec.data() + (size_t)t * lay.bytes;
        std::memcpy(r, &nr[t], 4);
        std::memcpy(r + lay.o_row, &row[(size_t)t * rs], 4 * (size_t)rs);
        std::memcpy(r + lay.o_in, &in[(size_t)t * xs], 4 * (size_t)xs);
        std::memcpy(r + lay.o_rp, &rp[(size_t)t * rps], 2 * (size_t)rps);
        std::memcpy(r + lay.o_slot, &slot[(size_t)t * es], 2 * (size_t)es);
        std::memcpy(r + lay.o_val, &val[(size_t)t * es], 8 * (size_t)es);
        // the inverse in the threads' order (dev::rp_inv_base): thread 4k + g, block j
        // <- inv[k][g + 4j] of the packed column-major copy
        double* iv = reinterpret_cast<double*>(r + lay.o_inv);
        const int n_ = nr[t];
        for (int j = 0; j < 16; ++j)
          for (int th = 16 * j; th < 256; ++th) {
            const int k = th >> 2, l = (th & 3) + 4 * j;
            if (l <= k && k < n_)
              iv[dev::rp_inv_base(j) - 16 * j + th] =
                  inv[(size_t)t * is + (size_t)l * n_ - (size_t)l * (l - 1) / 2 + (k - l)];
          }
      }
      CK(ctx, upload_vec(&out->rec, rec));
      out->recb = lay.bytes;
      out->depth = 2;  // compile-time in the kernel (three slots measured no gain)
      out->reg = true;
      out->rpipe = true;
      out->rpipe_wide = getenv("BD_RPIPE_WIDE") && atoi(getenv("BD_RPIPE_WIDE")) != 0;
      out->threads = 256;
      out->smem = dev::rp_smem(out->recb, out->depth, xs);
      auto pg = dev::k_trsv_rpipe<false, false, dev::RhsGather>;
      auto pv = dev::k_trsv_rpipe<false, false, dev::RhsVec>;
      auto ps = dev::k_trsv_rpipe<false, false, dev::RhsSchur>;
      auto wg = dev::k_trsv_rpipe<true, false, dev::RhsGather>;
      auto wv = dev::k_trsv_rpipe<true, false, dev::RhsVec>;
      auto ws = dev::k_trsv_rpipe<true, false, dev::RhsSchur>;
      auto tg = dev::k_trsv_rpipe<false, true, dev::RhsGather>;
      auto tv = dev::k_trsv_rpipe<false, true, dev::RhsVec>;
      {
        static std::mutex mu2;
        static size_t attr2[64] = {};
        int dev_id = 0;
        CK(ctx, cudaGetDevice(&dev_id));
        std::lock_guard<std::mutex> lk(mu2);
        size_t& cur = attr2[dev_id & 63];
        if (out->smem > cur) {
          const int sm = (int)out->smem;
          CK(ctx, cudaFuncSetAttribute(pg, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
          CK(ctx, cudaFuncSetAttribute(pv, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
          CK(ctx, cudaFuncSetAttribute(ps, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
          CK(ctx, cudaFuncSetAttribute(wg, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
          CK(ctx, cudaFuncSetAttribute(wv, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
          CK(ctx, cudaFuncSetAttribute(ws, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
          CK(ctx, cudaFuncSetAttribute(tg, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
          CK(ctx, cudaFuncSetAttribute(tv, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
          cur = out->smem;
        }
      }
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ps, 256, out->smem);
      // the records hold everything the kernel reads: drop the separate arrays
      // (task_row / tile_nr stay for the debug helpers)
      cudaFree(out->inv), out->inv = nullptr;
      cudaFree(out->ent_val), out->ent_val = nullptr;
      cudaFree(out->ent_slot), out->ent_slot = nullptr;
      cudaFree(out->ent_rp), out->ent_rp = nullptr;
      cudaFree(out->in_col), out->in_col = nullptr;
    } else if (kn != "smem" && rs <= dev::RT_ROWS && xs <= 512 && ex <= 16) {
      out->reg = true;
      out->reg_smem = kn == "rsmem";
      out->tile_rhs = kn == "regt";
      out->threads = 256;
      out->smem = dev::rt_smem(xs, es, rps, out->reg_smem ? (int)is : 0);
      if (out->reg_smem)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, dev::k_trsv_rtile<true, false, dev::RhsSchur>, 256, out->smem);
      else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, dev::k_trsv_rtile<false, false, dev::RhsSchur>, 256, out->smem);
    }
  }
  if (getenv("BD_BTILE_PERSM")) per_sm = std::max(1, std::min(per_sm, atoi(getenv("BD_BTILE_PERSM"))));
  out->grid = (int)std::min<int64_t>(out->ntiles, (int64_t)ctx->nsm * std::max(1, per_sm));
  if (getenv("BD_DEBUG"))
    std::fprintf(stderr, "[bd] btile launch: %d threads, %zu B smem, %d CTAs/SM, grid %d, "
                 "entries/tile max %d\n", out->threads, out->smem, per_sm, out->grid, emax);
  return BD_OK;
}

void free_btile(DevBTile* d) {
  cudaFree(d->rec);
  cudaFree(d->dst);
  cudaFree(d->opos);
  cudaFree(d->tile_nr);
  cudaFree(d->task_row);
  cudaFree(d->ent_rp);
  cudaFree(d->ent_slot);
  cudaFree(d->ent_val);
  cudaFree(d->in_col);
  cudaFree(d->inv);
}

bd_status setup_btile(bd_inner* p, const HostCsr& lower, const HostCsr& upper,
                      const double* coords, int dim) {
  bd_ctx* ctx = p->ctx;
  const double t_s = wall_s();
  const int target = getenv("BD_BTILE_ROWS") ? atoi(getenv("BD_BTILE_ROWS")) : 64;
  const char* part = getenv("BD_TILE_PART");  // "grid" (default) | "rcb"
  const bool grid = !(part && std::string(part) == "rcb");
  int ntiles = (int)std::max<int64_t>(1, lower.n / target);
  std::vector<int32_t> tile;
  // Row orderings that concatenate coordinate-sorted blocks (the heart-first
  // numbering of bd/mesh.py:252-263: heart vertices, then torso vertices, each
  // in lattice order) make lattice tiles that mix the blocks cyclic.  Detect
  // the blocks as the descents of the lexicographic coordinate order and keep
  // them in separate tiles (partition_grid's class argument).
  std::vector<int32_t> cls;
  if (coords && dim > 0) {
    int nd = 0;
    cls.assign(lower.n, 0);
    for (int64_t i = 1; i < lower.n; ++i) {
      bool less = false;  // coords[i] < coords[i-1] lexicographically
      for (int a = 0; a < dim; ++a) {
        const double x = coords[i * dim + a], y = coords[(i - 1) * dim + a];
        if (x != y) {
          less = x < y;
          break;
        }
      }
      nd += less;
      cls[i] = nd;
    }
    if (nd == 0 || nd > 8) cls.clear();
  }
  if (coords && dim > 0 && grid)
    ntiles = partition_grid(lower.n, dim, coords, target, cls.empty() ? nullptr : &cls, &tile);
  else if (coords && dim > 0)
    partition_coords(lower.n, dim, coords, ntiles, &tile);
  else
    partition_rows(lower, ntiles, &tile);
  setup_log("tiles", t_s);
  int E = 4;
  for (int64_t i = 0; i < lower.n; ++i)
    while (E < lower.indptr[i + 1] - lower.indptr[i] - 1) E <<= 1;
  for (int64_t i = 0; i < upper.n; ++i)
    while (E < upper.indptr[i + 1] - upper.indptr[i] - 1) E <<= 1;
  DTileSchedule dl, du;
  BTileSchedule bl, bu;
  std::string why;
  // forward and backward schedules are independent: build them concurrently
  auto build_pair = [&](const std::vector<int32_t>& tl, int nt) {
    std::string why_u;
    auto fu = std::async(std::launch::async, [&] {
      return build_dtile_schedule(upper, false, tl, nt, E, &du, &why_u);
    });
    const bool okl = build_dtile_schedule(lower, true, tl, nt, E, &dl, &why);
    const bool oku = fu.get();
    if (okl && !oku) why = why_u;
    return okl && oku;
  };
  bool ok = build_pair(tile, ntiles);
  if (!ok && coords && dim > 0 && grid) {  // e.g. a cyclic tile graph: fall back to RCB tiles
    ntiles = (int)std::max<int64_t>(1, lower.n / target);
    partition_coords(lower.n, dim, coords, ntiles, &tile);
    ok = build_pair(tile, ntiles);
  }
  setup_log("dtile schedules", t_s);
  ok = ok && build_btile_schedule(dl, &bl, &why) && build_btile_schedule(du, &bu, &why);
  setup_log("btile schedules", t_s);
  if (ok && (std::max(bl.tmax, bu.tmax) > 256 || std::max(bl.Ex, bu.Ex) > 16 ||
             (std::max(bl.Ex, bu.Ex) > 8 && std::max(bl.tmax, bu.tmax) > dev::RT_ROWS) ||
             std::max(bl.xmax, bu.xmax) > 512 ||
             std::max(bl.tmax, bu.tmax) > (int)std::sqrt(2.0 * 24000))) {
    ok = false;
    why = "tile too large or too many external entries";
  }
  if (getenv("BD_DEBUG"))
    std::fprintf(stderr, "[bd] btile n=%lld tiles=%d: %s (tmax %d, Ex %d/%d, inv %.1f MB)\n",
                 (long long)lower.n, ntiles, ok ? "ok" : why.c_str(), bl.tmax, bl.Ex, bu.Ex,
                 8e-6 * (double)(bl.inv.size() + bu.inv.size()));
  if (!ok) return BD_OK;
  TRY(upload_btile(ctx, bl, &p->BL));
  TRY(upload_btile(ctx, bu, &p->BU));
  setup_log("btile upload", t_s);
  // inbox mode (BD_BTILE_INBOX=1; measured 1.5% slower than polling the output
  // vector): per pass, the inbox slots (consumer tile, input slot)
  // fed by each row
  const char* ib = getenv("BD_BTILE_INBOX");
  if (p->BL.reg && p->BU.reg && !p->BL.tile_rhs && !p->BL.reg_smem && ib && atoi(ib) == 1) {
    bool ok = true;
    for (int pass = 0; pass < 2 && ok; ++pass) {
      const BTileSchedule& bs = pass ? bu : bl;
      DevBTile& db = pass ? p->BU : p->BL;
      std::vector<std::vector<int32_t>> need(lower.n);
      const int nt = db.ntiles;
      for (int c = 0; c < nt; ++c)
        for (int32_t j = 0; j < bs.tile_in_ptr[c + 1] - bs.tile_in_ptr[c]; ++j)
          need[bs.in_col[bs.tile_in_ptr[c] + j]].push_back((int32_t)((int64_t)c * db.xs + j));
      int dmax = 1;
      for (const auto& v : need) dmax = std::max<int>(dmax, (int)v.size());
      if (dmax > 8 || (int64_t)nt * db.xs >= INT32_MAX) {
        ok = false;
        break;
      }
      std::vector<int32_t> dst((size_t)nt * db.rs * dmax, -1);
      for (int t = 0; t < nt; ++t)
        for (int64_t q = bs.tile_row_ptr[t]; q < bs.tile_row_ptr[t + 1]; ++q) {
          const auto& v = need[bs.task_row[q]];
          const size_t base = ((size_t)t * db.rs + (size_t)(q - bs.tile_row_ptr[t])) * dmax;
          for (size_t d = 0; d < v.size(); ++d) dst[base + d] = v[d];
        }
      CK(ctx, upload_vec(&db.dst, dst));
      db.dmax = dmax;
      p->inbox_len = std::max<int64_t>(p->inbox_len, (int64_t)nt * db.xs);
    }
    if (ok) {
      if (dalloc(&p->inbox, p->inbox_len)) return fail(ctx, BD_ECUDA, "btile: inbox allocation");
      p->BL.inbox = p->BU.inbox = p->inbox;
    } else {
      p->BL.dmax = p->BU.dmax = 0;
    }
  }
  if ((p->BL.pipe && p->BU.pipe) || (p->BL.tile_rhs && p->BU.tile_rhs)) {
    // forward rows -> their slot in the backward pass's tile order
    std::vector<int32_t> pos_u(lower.n, -1), opos((size_t)p->BL.ntiles * p->BL.rs, 0);
    for (int t = 0; t < p->BU.ntiles; ++t)
      for (int64_t q = bu.tile_row_ptr[t]; q < bu.tile_row_ptr[t + 1]; ++q)
        pos_u[bu.task_row[q]] = (int32_t)((int64_t)t * p->BU.rs + (q - bu.tile_row_ptr[t]));
    for (int t = 0; t < p->BL.ntiles; ++t)
      for (int64_t q = bl.tile_row_ptr[t]; q < bl.tile_row_ptr[t + 1]; ++q)
        opos[(size_t)t * p->BL.rs + (q - bl.tile_row_ptr[t])] = pos_u[bl.task_row[q]];
    CK(ctx, upload_vec(&p->BL.opos, opos));
    if (dalloc(&p->bt_f, (int64_t)p->BL.ntiles * p->BL.rs) ||
        dalloc(&p->bt_b, (int64_t)p->BU.ntiles * p->BU.rs))
      return fail(ctx, BD_ECUDA, "btile: out of device memory");
    CK(ctx, cudaMemset(p->bt_b, 0, sizeof(double) * (size_t)p->BU.ntiles * p->BU.rs));
  } else {
    p->BL.pipe = p->BU.pipe = false;
    p->BL.tile_rhs = p->BU.tile_rhs = false;
  }
  // BD_RHS_PRE=1: heavy right-hand sides (the Schur solve's r_v - S_i t)
  // evaluated by one streaming kernel before the forward pass instead of
  // inside its tiles; measured 0.5-1 % slower at cfg2, so off by default
  if (getenv("BD_RHS_PRE") && atoi(getenv("BD_RHS_PRE")) != 0)
    if (dalloc(&p->rhs_pre, lower.n)) return fail(ctx, BD_ECUDA, "btile: out of device memory");
  p->btile = true;
  return BD_OK;
}

static bool g_tile_trace_on = false;  // bd_debug_tile_trace set a buffer: launch the tracing instantiation

template <class Rhs>
bd_status launch_btile(bd_inner* p, const DevBTile& b, const Rhs& rhs, double* xg, const Ctl& c,
                       int ctr_task, int ctr_done, double* reset, double* r0 = nullptr,
                       double* r1 = nullptr, int64_t r1n = INT32_MAX) {
  bd_ctx* ctx = p->ctx;
  dev::BTileDev T = b.dev();
  T.reset1_n = (int)std::min<int64_t>(r1n, INT32_MAX);
  if (b.rpipe && !reset && (b.xs > 256 || b.rpipe_wide))
    dev::k_trsv_rpipe<true, false, Rhs><<<b.grid, b.threads, b.smem, ctx->stream>>>(
        T, rhs, xg, c, ctr_task, ctr_done, r0, r1);
  else if (b.rpipe && !reset && g_tile_trace_on && Rhs::kScalar) {
    // per-tile timestamps (tools/btile_trace.py): scalar right-hand sides only
    if constexpr (Rhs::kScalar)
      dev::k_trsv_rpipe<false, true, Rhs><<<b.grid, b.threads, b.smem, ctx->stream>>>(
          T, rhs, xg, c, ctr_task, ctr_done, r0, r1);
  } else if (b.rpipe && !reset) {
    // The polled output vector as a persisting L2 window (BD_L2_PERSIST=0: off), so the
    // record stream (400 MB per pass) does not evict the lines the tiles spin on
    static const int persist = getenv("BD_L2_PERSIST") ? atoi(getenv("BD_L2_PERSIST")) : 1;
    // about five polled vectors alternate over one PCG iteration (the forward / backward
    // outputs of the two inners): they share the set-aside; when they do not fit (config 3:
    // 68 MB each) a fractional window measured 2 % slower than none, so it is left out
    const double win = sizeof(double) * (double)p->n;
    const float hit = (float)std::min(1.0, (double)ctx->l2_persist / (5.0 * win) * 1.12);
    if (persist && ctx->l2_persist && hit >= 0.5f) {
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeAccessPolicyWindow;
      at[0].val.accessPolicyWindow.base_ptr = xg;
      at[0].val.accessPolicyWindow.num_bytes = sizeof(double) * (size_t)p->n;
      at[0].val.accessPolicyWindow.hitRatio = hit;
      at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      cudaLaunchConfig_t cf = {};
      cf.gridDim = dim3(b.grid);
      cf.blockDim = dim3(b.threads);
      cf.dynamicSmemBytes = b.smem;
      cf.stream = ctx->stream;
      cf.attrs = at;
      cf.numAttrs = 1;
      CK(ctx, cudaLaunchKernelEx(&cf, dev::k_trsv_rpipe<false, false, Rhs>, T, rhs, xg, c, ctr_task, ctr_done,
                                 r0, r1));
    } else {
      dev::k_trsv_rpipe<false, false, Rhs><<<b.grid, b.threads, b.smem, ctx->stream>>>(
          T, rhs, xg, c, ctr_task, ctr_done, r0, r1);
    }
  } else if (b.reg && b.reg_smem && !reset)
    dev::k_trsv_rtile<true, false, Rhs><<<b.grid, b.threads, b.smem, ctx->stream>>>(
        T, rhs, xg, c, ctr_task, ctr_done, nullptr, nullptr, nullptr, r0, r1);
  else if (b.reg && !reset)
    dev::k_trsv_rtile<false, false, Rhs><<<b.grid, b.threads, b.smem, ctx->stream>>>(
        T, rhs, xg, c, ctr_task, ctr_done, nullptr, nullptr, nullptr, r0, r1);
  else
    dev::k_trsv_btile<Rhs><<<b.grid, b.threads, b.smem, ctx->stream>>>(T, rhs, xg, c, ctr_task,
                                                                       ctr_done, reset);
  LAUNCHED(ctx);
  return BD_OK;
}

template <int G, class Rhs>
bd_status launch_tiled(bd_inner* p, const DevTile& t, const Rhs& rhs, double* xg, const Ctl& c,
                       int ctr, int fin, int slot, int slot2, int64_t nmean) {
  bd_ctx* ctx = p->ctx;
  if (p->rows_mode) {
    auto kr = dev::k_trsv_rows<G, kTileStages, Rhs>;
    CK(ctx, cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->tsmem));
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cudaLaunchConfig_t cf = {};
    cf.gridDim = dim3(p->tparts);
    cf.blockDim = dim3(p->tthreads);
    cf.dynamicSmemBytes = p->tsmem;
    cf.stream = ctx->stream;
    cf.attrs = at;
    cf.numAttrs = 1;
    CK(ctx, cudaLaunchKernelEx(&cf, kr, t.dev(), rhs, xg, c, ctr, fin, slot, slot2, nmean, p->trows));
    LAUNCHED(ctx);
    return BD_OK;
  }
  auto kern = p->tstages >= 16 ? dev::k_trsv_tiled<G, 16, Rhs> : dev::k_trsv_tiled<G, kTileStages, Rhs>;
  CK(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p->tsmem));
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p->tparts);
  cfg.blockDim = dim3(p->tthreads);
  cfg.dynamicSmemBytes = p->tsmem;
  cfg.stream = ctx->stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(ctx, cudaLaunchKernelEx(&cfg, kern, t.dev(), rhs, xg, c, ctr, fin, slot, slot2, nmean));
  LAUNCHED(ctx);
  return BD_OK;
}

bd_status launch_dot(bd_ctx* ctx, const double* x, const double* y, int64_t n, const Ctl& c,
                     int ctr, int fin, int slot, int slot2, int64_t nmean);

// ---- inner solve dispatch -----------------------------------------------------
// Solve P x = rhs for one inner preconditioner inside control block c.
// x_int: polled internal output (sentinel-filled here); out (nullable):
// scatter target in the original ordering; fin/slot/slot2: optional mean of
// the output.
template <int G, class Rhs>
bd_status inner_solve_g(bd_inner* p, const Rhs& rhs, double* x_int, double* out, const Ctl& c,
                        int ctr0, int fin, int slot, int slot2, int64_t nmean) {
  bd_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  if (p->kind == BD_INNER_JACOBI) {
    const int grid = grid_for(ctx, p->n, dev::TPB / G);
    dev::k_jacobi<G, Rhs><<<grid, dev::TPB, 0, st>>>((int)p->n, p->inv, rhs, out ? out : x_int, c,
                                                      ctr0, fin, slot, slot2, nmean);
    LAUNCHED(ctx);
    return BD_OK;
  }
  if (p->dense) {
    // small exact inner: y = rhs (permuted order), x = X y, out[perm] = x
    const int grid = grid_for(ctx, p->n, dev::TPB / G);
    dev::k_rhs_eval<G, Rhs><<<grid, dev::TPB, 0, st>>>((int)p->n, rhs, p->y_int, c);
    LAUNCHED(ctx);
    dev::k_dense_gemv<<<grid_for(ctx, p->n, 8), 256, 0, st>>>(p->n, p->dense, p->y_int, x_int, out,
                                                             p->perm, c);
    LAUNCHED(ctx);
    if (fin >= 0) TRY(launch_dot(ctx, x_int, nullptr, p->n, c, ctr0 + 1, fin, slot, slot2, nmean));
    return BD_OK;
  }
  if (p->btile && p->BL.tile_rhs) {
    double* xg = (out && !p->perm) ? out : x_int;
    const DevBTile& bl = p->BL;
    const DevBTile& bu = p->BU;
    dev::k_tile_rhs<Rhs><<<grid_for(ctx, (int64_t)bl.ntiles * bl.rs, dev::TPB), dev::TPB, 0, st>>>(
        bl.task_row, (int64_t)bl.ntiles * bl.rs, rhs, p->bt_f, p->y_int, p->n, c);
    LAUNCHED(ctx);
    dev::k_trsv_rtile<false, true, Rhs><<<bl.grid, 256, bl.smem, st>>>(
        bl.dev(), rhs, p->y_int, c, ctr0, ctr0 + 1, p->bt_f, bl.opos, p->bt_b);
    LAUNCHED(ctx);
    dev::k_fill<<<grid_for(ctx, p->n, dev::TPB), dev::TPB, 0, st>>>(xg, p->n, dev::SENTINEL, c);
    LAUNCHED(ctx);
    dev::k_trsv_rtile<false, true, dev::RhsGather><<<bu.grid, 256, bu.smem, st>>>(
        bu.dev(), dev::RhsGather{nullptr}, xg, c, ctr0 + 2, ctr0 + 3, p->bt_b, nullptr, nullptr);
    LAUNCHED(ctx);
    if (fin >= 0) TRY(launch_dot(ctx, xg, nullptr, p->n, c, ctr0 + 1, fin, slot, slot2, nmean));
    return BD_OK;
  }
  if (p->btile && p->BL.pipe) {
    double* xg = (out && !p->perm) ? out : x_int;
    const DevBTile& bl = p->BL;
    const DevBTile& bu = p->BU;
    dev::k_tile_rhs<Rhs><<<grid_for(ctx, (int64_t)bl.ntiles * bl.rs, dev::TPB), dev::TPB, 0, st>>>(
        bl.task_row, (int64_t)bl.ntiles * bl.rs, rhs, p->bt_f, p->y_int, p->n, c);
    LAUNCHED(ctx);
    dev::k_trsv_ptile<true><<<bl.grid, 256, bl.smem, st>>>(bl.dev(), bl.opos, p->bt_f, p->y_int,
                                                           p->bt_b, c, ctr0, ctr0 + 1);
    LAUNCHED(ctx);
    dev::k_fill<<<grid_for(ctx, p->n, dev::TPB), dev::TPB, 0, st>>>(xg, p->n, dev::SENTINEL, c);
    LAUNCHED(ctx);
    dev::k_trsv_ptile<false><<<bu.grid, 256, bu.smem, st>>>(bu.dev(), nullptr, p->bt_b, xg, nullptr, c,
                                                            ctr0 + 2, ctr0 + 3);
    LAUNCHED(ctx);
    if (fin >= 0) TRY(launch_dot(ctx, xg, nullptr, p->n, c, ctr0 + 1, fin, slot, slot2, nmean));
    return BD_OK;
  }
  if (p->btile) {
    double* xg = (out && !p->perm) ? out : x_int;
    // sentinel fills right before each pass: besides resetting the polled
    // buffers they leave them L2-resident, so polls and publishes hit L2
    // (folding the resets into the passes measured ~30% slower passes)
    // (inbox mode: only the inboxes are polled, so only they are reset)
    const bool ib = p->BL.inbox != nullptr;
    const int64_t nf1 = ib ? (int64_t)p->BL.ntiles * p->BL.xs : p->n;
    const int64_t nf2 = ib ? (int64_t)p->BU.ntiles * p->BU.xs : p->n;
    if constexpr (!Rhs::kScalar) {
      if (p->rhs_pre) {
        if (rhs.ell_w && !rhs.perm && rhs.si.nrows == p->n) {
          const int grid = grid_for(ctx, p->n, dev::TPB);
#define SCHUR_RHS_ELL(WW)                                                                          \
  case WW:                                                                                         \
    dev::k_schur_rhs_ell<WW><<<grid, dev::TPB, 0, st>>>(rhs.ell_col, rhs.ell_v2, rhs.ell_n,         \
                                                        (int)p->n, rhs.traw, rhs.sc, rhs.rv,        \
                                                        p->rhs_pre, c);                            \
    break;
          switch (rhs.ell_w) {
            SCHUR_RHS_ELL(8)
            SCHUR_RHS_ELL(16)
            SCHUR_RHS_ELL(24)
            default:
              dev::k_schur_rhs_ell<32><<<grid, dev::TPB, 0, st>>>(rhs.ell_col, rhs.ell_v2, rhs.ell_n,
                                                                  (int)p->n, rhs.traw, rhs.sc, rhs.rv,
                                                                  p->rhs_pre, c);
          }
#undef SCHUR_RHS_ELL
        } else {
          dev::k_rhs_eval<G, Rhs><<<grid_for(ctx, p->n, dev::TPB / G), dev::TPB, 0, st>>>(
              (int)p->n, rhs, p->rhs_pre, c);
        }
        LAUNCHED(ctx);
      }
    }
    // BD_FOLD_FILL: 1 = the forward pass resets the backward's output rows
    // (no fill before the backward); 2 = also the backward pass resets the
    // forward output it gathers (y_int stays sentinel between solves)
    const int fold = (ib || !p->BL.reg || !p->BU.reg) ? 0 : p->fold_fill;
    const bool prefilled = p->prefilled;  // y_int was reset by the kernel just before this solve
    p->prefilled = false;
    if (fold < 2 && !prefilled) {
      dev::k_fill<<<grid_for(ctx, nf1, dev::TPB), dev::TPB, 0, st>>>(ib ? p->inbox : p->y_int, nf1,
                                                                    dev::SENTINEL, c);
      LAUNCHED(ctx);
    }
    prof_mark(ctx, 5);  // (profile classes: fills and dots are vector work,
                        //  the two passes alone are the triangular-solve class)
    if (!Rhs::kScalar && p->rhs_pre)
      TRY(launch_btile(p, p->BL, dev::RhsVec{p->rhs_pre, (int)p->n, nullptr, nullptr}, p->y_int, c,
                       ctr0, ctr0 + 1, nullptr, fold ? xg : nullptr));
    else
      TRY(launch_btile(p, p->BL, rhs, p->y_int, c, ctr0, ctr0 + 1, nullptr, fold ? xg : nullptr));
    prof_mark(ctx, p->prof_cls);
    if (fold < 1) {
      dev::k_fill<<<grid_for(ctx, nf2, dev::TPB), dev::TPB, 0, st>>>(ib ? p->inbox : xg, nf2,
                                                                    dev::SENTINEL, c);
      LAUNCHED(ctx);
    }
    prof_mark(ctx, 5);
    {
      double* pf = (fold < 2 && p->BU.reg) ? p->post_fill : nullptr;
      const int64_t pfn = p->post_fill_n;
      p->post_fill = nullptr;
      TRY(launch_btile(p, p->BU, dev::RhsGather{p->y_int}, xg, c, ctr0 + 2, ctr0 + 3, nullptr, nullptr,
                       fold >= 2 ? p->y_int : pf, fold >= 2 ? (int64_t)INT32_MAX : pfn));
      if (pf && p->post_fill_owner) p->post_fill_owner->prefilled = true;
      p->post_fill_owner = nullptr;
    }
    prof_mark(ctx, p->prof_cls);
    if (fin >= 0) TRY(launch_dot(ctx, xg, nullptr, p->n, c, ctr0 + 1, fin, slot, slot2, nmean));
    prof_mark(ctx, 5);
    return BD_OK;
  }
  if (p->dtile) {
    double* xg = (out && !p->perm) ? out : x_int;
    dev::k_fill<<<grid_for(ctx, p->n, dev::TPB), dev::TPB, 0, st>>>(p->y_int, p->n, dev::SENTINEL, c);
    LAUNCHED(ctx);
    if (p->G == 4)
      dev::k_trsv_dtile<4, Rhs><<<p->DL.grid, p->DL.threads, 0, st>>>(p->DL.dev(), rhs, p->y_int, c,
                                                                       ctr0, ctr0 + 1);
    else
      dev::k_trsv_dtile<8, Rhs><<<p->DL.grid, p->DL.threads, 0, st>>>(p->DL.dev(), rhs, p->y_int, c,
                                                                       ctr0, ctr0 + 1);
    LAUNCHED(ctx);
    dev::k_fill<<<grid_for(ctx, p->n, dev::TPB), dev::TPB, 0, st>>>(xg, p->n, dev::SENTINEL, c);
    LAUNCHED(ctx);
    if (p->G == 4)
      dev::k_trsv_dtile<4, dev::RhsGather><<<p->DU.grid, p->DU.threads, 0, st>>>(
          p->DU.dev(), dev::RhsGather{p->y_int}, xg, c, ctr0 + 2, ctr0 + 3);
    else
      dev::k_trsv_dtile<8, dev::RhsGather><<<p->DU.grid, p->DU.threads, 0, st>>>(
          p->DU.dev(), dev::RhsGather{p->y_int}, xg, c, ctr0 + 2, ctr0 + 3);
    LAUNCHED(ctx);
    if (fin >= 0) TRY(launch_dot(ctx, xg, nullptr, p->n, c, ctr0 + 1, fin, slot, slot2, nmean));
    return BD_OK;
  }
  if (p->cluster) {
    double* xg = (out && !p->perm) ? out : x_int;
    if (p->G == 4) {
      TRY(launch_cluster<4>(p, p->CL, rhs, p->y_int, c));
      TRY(launch_cluster<4>(p, p->CU, dev::RhsGather{p->y_int}, xg, c));
    } else {
      TRY(launch_cluster<8>(p, p->CL, rhs, p->y_int, c));
      TRY(launch_cluster<8>(p, p->CU, dev::RhsGather{p->y_int}, xg, c));
    }
    if (fin >= 0) TRY(launch_dot(ctx, xg, nullptr, p->n, c, ctr0 + 1, fin, slot, slot2, nmean));
    return BD_OK;
  }
  if (p->super) {
    // exact factor: supernodal forward / backward passes
    dev::k_fill<<<grid_for(ctx, p->n, dev::TPB), dev::TPB, 0, st>>>(p->y_int, p->n, dev::SENTINEL, c);
    LAUNCHED(ctx);
    dev::SuperTri tl{(int)p->n,        p->L.rowptr,  p->L.col,    p->L.val, p->SL.sn_start,
                     p->SL.sn_size,     p->SL.task_sn, p->SL.ntasks, nullptr,
                     p->SL.task_kind,   p->SL.task_arg, p->SL.sn_cnt, p->rext,
                     p->SL.pinv,        p->SL.sn_pan,  p->SL.task_w, p->SL.sinv, p->SL.sn_inv,
                     p->SL.dchunk};
    dev::k_trsv_super<true, Rhs><<<p->SL.grid, 512, 0, st>>>(tl, rhs, p->y_int, nullptr, c, ctr0,
                                                              ctr0 + 1);
    LAUNCHED(ctx);
    dev::k_fill<<<grid_for(ctx, p->n, dev::TPB), dev::TPB, 0, st>>>(x_int, p->n, dev::SENTINEL, c);
    LAUNCHED(ctx);
    dev::SuperTri tu{(int)p->n,        p->U.rowptr,  p->U.col,    p->U.val, p->SU.sn_start,
                     p->SU.sn_size,     p->SU.task_sn, p->SU.ntasks, p->perm,
                     p->SU.task_kind,   p->SU.task_arg, p->SU.sn_cnt, p->rext,
                     p->SU.pinv,        p->SU.sn_pan,  p->SU.task_w, p->SU.sinv, p->SU.sn_inv,
                     p->SU.dchunk};
    dev::k_trsv_super<false, dev::RhsGather><<<p->SU.grid, 512, 0, st>>>(
        tu, dev::RhsGather{p->y_int}, x_int, out, c, ctr0 + 2, ctr0 + 3);
    LAUNCHED(ctx);
    if (fin >= 0) TRY(launch_dot(ctx, x_int, nullptr, p->n, c, ctr0 + 1, fin, slot, slot2, nmean));
    return BD_OK;
  }
  if (p->persist) {
    double* xg = (out && !p->perm) ? out : x_int;
    dev::k_fill<<<grid_for(ctx, p->n, dev::TPB), dev::TPB, 0, st>>>(p->y_int, p->n, dev::SENTINEL, c);
    LAUNCHED(ctx);
    dev::k_trsv_persist<G, Rhs><<<p->EL.grid, dev::TPB, 0, st>>>(
        p->EL.dev(), rhs, p->y_int, c, ctr0, ctr0 + 1, p->EL.nchunks, -1, 0, -1, 1);
    LAUNCHED(ctx);
    dev::k_fill<<<grid_for(ctx, p->n, dev::TPB), dev::TPB, 0, st>>>(xg, p->n, dev::SENTINEL, c);
    LAUNCHED(ctx);
    dev::k_trsv_persist<G, dev::RhsGather><<<p->EU.grid, dev::TPB, 0, st>>>(
        p->EU.dev(), dev::RhsGather{p->y_int}, xg, c, ctr0 + 2, ctr0 + 3, p->EU.nchunks, -1, slot,
        slot2, nmean);
    LAUNCHED(ctx);
    // the mean of the output as a separate fixed-order pass: a per-chunk block
    // reduction inside the solve would sit on its critical path
    if (fin >= 0) TRY(launch_dot(ctx, xg, nullptr, p->n, c, ctr0 + 1, fin, slot, slot2, nmean));
    return BD_OK;
  }
  if (p->tiled) {
    double* xg = (out && !p->perm) ? out : x_int;
    switch (p->TG) {
      case 4:
        TRY(launch_tiled<4>(p, p->TL, rhs, p->y_int, c, ctr0, -1, 0, -1, 1));
        TRY(launch_tiled<4>(p, p->TU, dev::RhsGather{p->y_int}, xg, c, ctr0 + 3, fin, slot, slot2,
                            nmean));
        break;
      case 8:
        TRY(launch_tiled<8>(p, p->TL, rhs, p->y_int, c, ctr0, -1, 0, -1, 1));
        TRY(launch_tiled<8>(p, p->TU, dev::RhsGather{p->y_int}, xg, c, ctr0 + 3, fin, slot, slot2,
                            nmean));
        break;
      default:
        TRY(launch_tiled<16>(p, p->TL, rhs, p->y_int, c, ctr0, -1, 0, -1, 1));
        TRY(launch_tiled<16>(p, p->TU, dev::RhsGather{p->y_int}, xg, c, ctr0 + 3, fin, slot,
                             slot2, nmean));
    }
    return BD_OK;
  }
  dev::k_fill<<<grid_for(ctx, p->n, dev::TPB), dev::TPB, 0, st>>>(x_int, p->n, dev::SENTINEL, c);
  LAUNCHED(ctx);
  dev::k_trsv_fwd<G, true, Rhs><<<p->L.nvb, dev::TPB, 0, st>>>(p->L.dev(), rhs, p->y_int, c, ctr0,
                                                               ctr0 + 1, p->L.nvb);
  LAUNCHED(ctx);
  dev::k_trsv_bwd<G, false><<<p->U.nvb, dev::TPB, 0, st>>>(p->U.dev(), p->y_int, x_int, out, p->perm,
                                                           c, ctr0 + 2, ctr0 + 3, p->U.nvb, fin,
                                                           slot, slot2, nmean);
  LAUNCHED(ctx);
  return BD_OK;
}

template <class Rhs>
bd_status inner_solve(bd_inner* p, const Rhs& rhs, double* x_int, double* out, const Ctl& c,
                      int ctr0, int fin = -1, int slot = 0, int slot2 = -1, int64_t nmean = 1) {
  switch (p->G) {
    case 4: return inner_solve_g<4>(p, rhs, x_int, out, c, ctr0, fin, slot, slot2, nmean);
    case 8: return inner_solve_g<8>(p, rhs, x_int, out, c, ctr0, fin, slot, slot2, nmean);
    case 16: return inner_solve_g<16>(p, rhs, x_int, out, c, ctr0, fin, slot, slot2, nmean);
    default: return inner_solve_g<32>(p, rhs, x_int, out, c, ctr0, fin, slot, slot2, nmean);
  }
}

// ---- operator -----------------------------------------------------------------
bd_status launch_lambda(bd_system* s, const double* x, double* q, const Ctl& c, int with_dot) {
  bd_ctx* ctx = s->ctx;
  const char* lv = getenv("BD_LAMBDA");
  if (s->ell_w && !(lv && lv[0] != 'e')) {
    const dev::LamEll L{s->ell_col, s->ell_v1, s->ell_v2};
    const int grid = grid_for(ctx, s->n, dev::TPB);
#define LAMBDA_ELL(WW)                                                                         \
  case WW:                                                                                     \
    dev::k_lambda_ell<WW><<<grid, dev::TPB, 0, ctx->stream>>>(L, x, q, s->mh, s->gamma,         \
                                                             (int)s->n, (int)s->m, c, with_dot); \
    break;
    switch (s->ell_w) {
      LAMBDA_ELL(8)
      LAMBDA_ELL(16)
      LAMBDA_ELL(24)
      LAMBDA_ELL(32)
    }
#undef LAMBDA_ELL
    LAUNCHED(ctx);
    return BD_OK;
  }
  if (!(lv && lv[0] == '1')) {
    // entries per row ~ nnz/n: 3D P1 ~15 -> 8 lanes x 2, 2D ~7 -> 4 lanes x 2
    const double avg = s->n ? (double)s->S1->nnz / s->n : 1.0;
    auto s1 = s->S1->dev();
    auto si = s->Si->dev();
    if (avg <= 8.0) {
      const int grid = grid_for(ctx, s->n, dev::TPB / 4);
      dev::k_lambda2<4, 2><<<grid, dev::TPB, 0, ctx->stream>>>(s1, si, x, q, s->mh, s->gamma,
                                                              (int)s->n, (int)s->m, c, with_dot);
    } else {
      const int grid = grid_for(ctx, s->n, dev::TPB / 8);
      dev::k_lambda2<8, 2><<<grid, dev::TPB, 0, ctx->stream>>>(s1, si, x, q, s->mh, s->gamma,
                                                              (int)s->n, (int)s->m, c, with_dot);
    }
    LAUNCHED(ctx);
    return BD_OK;
  }
  const int G = s->S1->G;
  const int grid = grid_for(ctx, s->n, dev::TPB / G);
  auto s1 = s->S1->dev();
  auto si = s->Si->dev();
#define LAMBDA_CASE(GG)                                                                       \
  case GG:                                                                                    \
    dev::k_lambda<GG><<<grid, dev::TPB, 0, ctx->stream>>>(s1, si, x, q, s->mh, s->gamma,      \
                                                          (int)s->n, (int)s->m, c, with_dot); \
    break;
  switch (G) {
    LAMBDA_CASE(4)
    LAMBDA_CASE(8)
    LAMBDA_CASE(16)
    default:
      dev::k_lambda<32><<<grid, dev::TPB, 0, ctx->stream>>>(s1, si, x, q, s->mh, s->gamma, (int)s->n,
                                                            (int)s->m, c, with_dot);
  }
#undef LAMBDA_CASE
  LAUNCHED(ctx);
  return BD_OK;
}

bd_status launch_dot(bd_ctx* ctx, const double* x, const double* y, int64_t n, const Ctl& c,
                     int ctr, int fin, int slot, int slot2, int64_t nmean) {
  dev::k_dot<<<grid_for(ctx, n, dev::TPB), dev::TPB, 0, ctx->stream>>>(x, y, n, c, ctr, fin, slot,
                                                                       slot2, nmean);
  LAUNCHED(ctx);
  return BD_OK;
}

// The polled forward output of an inner's blocked-tile solve, if the kernel
// right before that solve may reset it (BD_PREFILL=0 keeps the separate fill).
int prefill_level() {  // BD_PREFILL: 0 off, 1 bulk solves, 2 (default) + the Schur solve
  static const int lv = getenv("BD_PREFILL") ? atoi(getenv("BD_PREFILL")) : 2;
  return lv;
}
double* fill_target(bd_inner* p) {
  const bool on = prefill_level() >= 1;
  if (!on || !p->btile || p->BL.inbox || !p->BL.reg || !p->BU.reg || p->fold_fill >= 2) return nullptr;
  return p->y_int;
}

bd_status launch_corr(bd_prec* p, const double* s, const Ctl& c) {
  bd_ctx* ctx = p->sys->ctx;
  bd_system* sy = p->sys;
  if (sy->ell_w && !getenv("BD_NO_CORR_ELL")) {
    const dev::LamEll L{sy->ell_col, sy->ell_v1, sy->ell_v2};
    const int grid = grid_for(ctx, sy->m, dev::TPB);
    // the second bulk solve follows: its forward output is reset here
    double* ft = fill_target(p->bulk);
    const int64_t nf = ft ? p->bulk->n : 0;
    switch (sy->ell_w) {
      case 8: dev::k_corr_ell<8><<<grid, dev::TPB, 0, ctx->stream>>>(L, (int)sy->n, (int)sy->m, s, p->corr, c, sy->n, ft, nf); break;
      case 16: dev::k_corr_ell<16><<<grid, dev::TPB, 0, ctx->stream>>>(L, (int)sy->n, (int)sy->m, s, p->corr, c, sy->n, ft, nf); break;
      case 24: dev::k_corr_ell<24><<<grid, dev::TPB, 0, ctx->stream>>>(L, (int)sy->n, (int)sy->m, s, p->corr, c, sy->n, ft, nf); break;
      default: dev::k_corr_ell<32><<<grid, dev::TPB, 0, ctx->stream>>>(L, (int)sy->n, (int)sy->m, s, p->corr, c, sy->n, ft, nf); break;
    }
    LAUNCHED(ctx);
    if (ft) p->bulk->prefilled = true;
    return BD_OK;
  }
  {
    const double avg = p->sys->m ? (double)p->sys->Si->nnz / p->sys->m : 1.0;
    auto si2 = p->sys->Si->dev();
    if (avg <= 8.0) {
      dev::k_corr2<4, 2><<<grid_for(ctx, p->sys->m, dev::TPB / 4), dev::TPB, 0, ctx->stream>>>(
          si2, s, p->corr, c, p->sys->n);
    } else {
      dev::k_corr2<8, 2><<<grid_for(ctx, p->sys->m, dev::TPB / 8), dev::TPB, 0, ctx->stream>>>(
          si2, s, p->corr, c, p->sys->n);
    }
    LAUNCHED(ctx);
    return BD_OK;
  }
  const int G = p->sys->Si->G;
  const int grid = grid_for(ctx, p->sys->m, dev::TPB / G);
  auto si = p->sys->Si->dev();
  switch (G) {
    case 4: dev::k_corr<4><<<grid, dev::TPB, 0, ctx->stream>>>(si, s, p->corr, c, p->sys->n); break;
    case 8: dev::k_corr<8><<<grid, dev::TPB, 0, ctx->stream>>>(si, s, p->corr, c, p->sys->n); break;
    case 16: dev::k_corr<16><<<grid, dev::TPB, 0, ctx->stream>>>(si, s, p->corr, c, p->sys->n); break;
    default: dev::k_corr<32><<<grid, dev::TPB, 0, ctx->stream>>>(si, s, p->corr, c, p->sys->n);
  }
  LAUNCHED(ctx);
  return BD_OK;
}

// P_Λ^{-1} r (bd/precond.py:298-312) with sc[MU1], sc[C1] already holding
// mean(r_u) and mean(r_u)/beta.  zu: output u-block; zv_int: polled Schur
// output (sentinel-filled); zv_out: nullable scatter copy of it.
// in_pcg (the PCG loop, whose next step deflates z_u, bd/krylov.py:41-43):
// the two bulk solves skip their output means (constants on z_u that the
// deflation removes; S_i t = S_i t_raw because S_i 𝟙 = 0), and the tail
// forms z_u = t_raw − z2_raw together with the partials of rho (no k_rho).
// The standalone apply keeps the reference's recentring (bd_blocklu_apply).
bd_status enqueue_pinv(bd_prec* p, const double* r, double* zu, double* zv_int, double* zv_out,
                       const Ctl& c, bool in_pcg) {
  bd_system* s = p->sys;
  bd_ctx* ctx = s->ctx;
  const int64_t n = s->n, m = s->m;
  // t = bulk^{-1}(r_u - mu1), recentred lazily by its consumers
  prof_mark(ctx, 5);
  {
    dev::RhsVec rhs{r, (int)n, c.sc + dev::S_MU1, p->bulk->perm};
    double* xi = p->bulk->perm ? p->bulk->x_int : p->traw;
    double* out = p->bulk->perm ? p->traw : nullptr;
    if (p->bulk->kind == BD_INNER_JACOBI) {
      xi = p->traw;
      out = nullptr;
    }
    // the Schur solve follows directly (in the PCG no dot in between): the bulk solve's
    // backward pass resets the Schur solve's polled forward output on its way
    if (in_pcg && prefill_level() >= 2 && p->bulk != p->schur && p->bulk->btile && p->bulk->BU.rpipe) {
      if (double* ft = fill_target(p->schur)) {
        p->bulk->post_fill = ft;
        p->bulk->post_fill_n = m;
        p->bulk->post_fill_owner = p->schur;
      }
    }
    if (in_pcg)
      TRY(inner_solve(p->bulk, rhs, xi, out, c, dev::C_BULK1_S));
    else
      TRY(inner_solve(p->bulk, rhs, xi, out, c, dev::C_BULK1_S, dev::FIN_MEAN, dev::S_MT, -1, n));
    p->bulk->post_fill = nullptr;
    p->bulk->post_fill_owner = nullptr;
  }
  prof_mark(ctx, 2);
  // s = K^{-1}(r_v - S_i t[:m])
  {
    dev::RhsSchur rhs{s->Si->dev(), p->traw, in_pcg ? p->zsc : c.sc, r + n, p->schur->perm};
    if (s->ell_w && !getenv("BD_NO_CORR_ELL")) {  // the ELL copy for the streaming pre-evaluation
      rhs.ell_col = s->ell_col;
      rhs.ell_v2 = s->ell_v2;
      rhs.ell_w = s->ell_w;
      rhs.ell_n = (int)s->n;
    }
    double* xi = zv_int;
    double* out = zv_out;
    if (p->schur->perm) {
      xi = p->schur->x_int;
      out = zv_out ? zv_out : zv_int;
    }
    if (p->schur->kind == BD_INNER_JACOBI) {
      xi = zv_out ? zv_out : zv_int;
      out = nullptr;
    }
    TRY(inner_solve(p->schur, rhs, xi, out, c, dev::C_SCH_S));
  }
  prof_mark(ctx, 3);
  // correction = pad(S_i s); mu2 = mean(correction)
  const double* sv = zv_out ? zv_out : zv_int;
  TRY(launch_corr(p, sv, c));
  prof_mark(ctx, 4);
  {
    dev::RhsVec rhs{p->corr, (int)m, c.sc + dev::S_MU2, p->bulk->perm};
    double* xi = p->bulk->perm ? p->bulk->x_int : p->z2raw;
    double* out = p->bulk->perm ? p->z2raw : nullptr;
    if (p->bulk->kind == BD_INNER_JACOBI) {
      xi = p->z2raw;
      out = nullptr;
    }
    if (in_pcg)
      TRY(inner_solve(p->bulk, rhs, xi, out, c, dev::C_BULK2_S));
    else
      TRY(inner_solve(p->bulk, rhs, xi, out, c, dev::C_BULK2_S, dev::FIN_MEAN, dev::S_M2, -1, n));
  }
  prof_mark(ctx, 2);
  if (in_pcg) {
    dev::k_combine_rho<<<grid_for(ctx, n + m, dev::TPB), dev::TPB, 0, ctx->stream>>>(
        p->traw, p->z2raw, zu, zv_out ? zv_out : zv_int, r, n, n + m, c);
  } else {
    dev::k_combine<<<grid_for(ctx, n, dev::TPB), dev::TPB, 0, ctx->stream>>>(p->traw, p->z2raw, zu, n,
                                                                          c);
  }
  LAUNCHED(ctx);
  prof_mark(ctx, 5);
  return BD_OK;
}

// One PCG loop iteration (bd/krylov.py:100-131).
bd_status enqueue_iteration(bd_prec* p) {
  bd_system* s = p->sys;
  bd_ctx* ctx = s->ctx;
  const int64_t n = s->n, nm = s->n + s->m;
  const Ctl& c = p->ctl;
  TRY(launch_lambda(s, p->d, p->q, c, 1));
  prof_mark(ctx, 0);
  double* ft = fill_target(p->bulk);  // the first bulk solve follows: its forward output is reset here
  dev::k_update<<<grid_for(ctx, nm, dev::TPB), dev::TPB, 0, ctx->stream>>>(p->x, p->r, p->d, p->q, n,
                                                                           nm, c, ft, ft ? p->bulk->n : 0);
  LAUNCHED(ctx);
  if (ft) p->bulk->prefilled = true;
  prof_mark(ctx, 1);
  TRY(enqueue_pinv(p, p->r, p->z, p->z + n, nullptr, c, true));  // rho in its tail
  dev::k_dupdate<<<grid_for(ctx, nm, dev::TPB), dev::TPB, 0, ctx->stream>>>(p->z, p->d, n, nm, c);
  LAUNCHED(ctx);
  prof_mark(ctx, 5);
  return BD_OK;
}

__global__ void k_loop_cond(cudaGraphConditionalHandle h, const int* fl) {
  const volatile int* f = fl;
  cudaGraphSetConditional(h, (f[dev::F_DONE] || f[dev::F_STOP]) ? 0u : 1u);
}

bd_status build_graph(bd_prec* p) {
  bd_ctx* ctx = p->sys->ctx;
  if (p->gexec) {
    cudaGraphExecDestroy(p->gexec);
    cudaGraphDestroy(p->graph);
    p->gexec = nullptr;
    p->graph = nullptr;
  }
  cudaGraph_t g;
  CK(ctx, cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  CK(ctx, cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  CK(ctx, cudaGraphAddNode(&node, g, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  CK(ctx, cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0,
                                        cudaStreamCaptureModeThreadLocal));
  const int64_t saved = ctx->launches;
  bd_status st = enqueue_iteration(p);
  k_loop_cond<<<1, 1, 0, ctx->stream>>>(h, p->ctl.fl);
  cudaGraph_t captured = nullptr;
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &captured);
  ctx->launches = saved;
  if (st != BD_OK) return st;
  CK(ctx, e);
  CK(ctx, cudaGraphInstantiate(&p->gexec, g, nullptr, nullptr, 0));
  p->graph = g;
  return BD_OK;
}

int64_t iteration_launches(bd_prec* p) {
  // Λ, update, 2 bulk solves + schur solve (3 kernels each, 1 for jacobi),
  // corr, combine, rho, dupdate
  auto per = [](bd_inner* in) { return in->kind == BD_INNER_JACOBI ? 1 : 3; };
  return 2 + 2 * per(p->bulk) + per(p->schur) + 1 + 1 + 2;
}

}  // namespace

// ===========================================================================
extern "C" {

const char* bd_version(void) { return BD_VERSION; }

bd_status bd_ctx_create(int device, void* stream, bd_ctx** out) {
  if (!out) return BD_EINVAL;
  *out = nullptr;
  bd_ctx* c = new bd_ctx();
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete c;
    return BD_ECUDA;
  }
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, device);
  // L2 set-aside for the persisting window of the triangular passes' polled vectors
  // (launch_btile; the limit cannot be set during graph capture)
  if (!(getenv("BD_L2_PERSIST") && atoi(getenv("BD_L2_PERSIST")) == 0)) {
    int max_persist = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device);
    if (max_persist > 0)
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize,
                         std::min<size_t>((size_t)max_persist,
                                          (size_t)(getenv("BD_L2_PERSIST_MB") ? atoi(getenv("BD_L2_PERSIST_MB")) : 48)
                                              << 20));
    cudaDeviceGetLimit(&c->l2_persist, cudaLimitPersistingL2CacheSize);
    cudaGetLastError();
  }
  c->user = (cudaStream_t)stream;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming) != cudaSuccess ||
      cudaMallocHost((void**)&c->h_pin, 64 * sizeof(double)) != cudaSuccess ||
      ctl_alloc(&c->util, (int64_t)c->nsm * 8, 0, 0) != cudaSuccess) {
    delete c;
    return BD_ECUDA;
  }
  *out = c;
  return BD_OK;
}

bd_status bd_ctx_destroy(bd_ctx* c) {
  if (!c) return BD_OK;
  cudaStreamSynchronize(c->stream);
  ctl_free(&c->util);
  for (auto& m : c->marks) cudaEventDestroy(m.first);
  for (auto e : c->pool) cudaEventDestroy(e);
  cudaFreeHost(c->h_pin);
  cudaEventDestroy(c->ev_in);
  cudaEventDestroy(c->ev_out);
  cudaStreamDestroy(c->stream);
  delete c;
  return BD_OK;
}

bd_status bd_ctx_set_stream(bd_ctx* c, void* stream) {
  if (!c) return BD_EINVAL;
  c->user = (cudaStream_t)stream;
  return BD_OK;
}

bd_status bd_ctx_synchronize(bd_ctx* c) {
  if (!c) return BD_EINVAL;
  CK(c, cudaStreamSynchronize(c->stream));
  return BD_OK;
}

const char* bd_last_error(bd_ctx* c) { return c ? tl_err.c_str() : "null context"; }

int64_t bd_launch_count(bd_ctx* c) { return c ? c->launches : 0; }

bd_status bd_profile_enable(bd_ctx* c, int enable) {
  if (!c) return BD_EINVAL;
  c->profile = enable != 0;
  std::fill(c->prof_ms, c->prof_ms + 8, 0.0);
  std::fill(c->prof_launch, c->prof_launch + 8, 0);
  return BD_OK;
}

bd_status bd_profile_read(bd_ctx* c, double* times_ms, int64_t* launches, int cap) {
  if (!c) return BD_EINVAL;
  prof_collect(c);
  for (int i = 0; i < std::min(cap, 8); ++i) {
    if (times_ms) times_ms[i] = c->prof_ms[i];
    if (launches) launches[i] = c->prof_launch[i];
  }
  return BD_OK;
}

// ---- CSR ------------------------------------------------------------------
bd_status bd_csr_create(bd_ctx* ctx, int64_t nrows, int64_t ncols, int64_t nnz,
                        const int64_t* indptr, const int32_t* indices, const double* values,
                        bd_csr** out) {
  if (!ctx || !out || nrows < 0 || ncols < 0 || nnz < 0 || !indptr)
    return fail(ctx, BD_EINVAL, "bd_csr_create: bad arguments");
  if (nnz >= (int64_t)INT32_MAX || nrows >= (int64_t)INT32_MAX)
    return fail(ctx, BD_EINVAL, "bd_csr_create: matrix too large for int32 indexing");
  if (indptr[0] != 0 || indptr[nrows] != nnz)
    return fail(ctx, BD_EINVAL, "bd_csr_create: inconsistent indptr");
  bd_csr* a = new bd_csr();
  a->ctx = ctx;
  a->nrows = nrows;
  a->ncols = ncols;
  a->nnz = nnz;
  a->G = pick_g(nrows ? (double)nnz / nrows : 1.0);
  std::vector<int> rp(nrows + 1);
  for (int64_t i = 0; i <= nrows; ++i) rp[i] = (int)indptr[i];
  if (dalloc(&a->rowptr, nrows + 1) || dalloc(&a->col, nnz) || dalloc(&a->val, nnz) ||
      cudaMemcpy(a->rowptr, rp.data(), sizeof(int) * rp.size(), cudaMemcpyHostToDevice) ||
      (nnz && cudaMemcpy(a->col, indices, sizeof(int) * nnz, cudaMemcpyHostToDevice)) ||
      (nnz && cudaMemcpy(a->val, values, sizeof(double) * nnz, cudaMemcpyHostToDevice))) {
    bd_csr_destroy(a);
    return fail(ctx, BD_ECUDA, "bd_csr_create: device allocation/copy failed");
  }
  {  // ELL copy (P1 stencils: <= 32 entries per row, little padding)
    int64_t maxlen = 0;
    for (int64_t i = 0; i < nrows; ++i) maxlen = std::max<int64_t>(maxlen, indptr[i + 1] - indptr[i]);
    const int W = maxlen <= 8 ? 8 : maxlen <= 16 ? 16 : maxlen <= 24 ? 24 : maxlen <= 32 ? 32 : 0;
    if (W && nnz > 0 && (double)W * nrows <= 1.5 * (double)nnz && !getenv("BD_NO_SPMV_ELL")) {
      std::vector<int> ec((size_t)W * nrows, -1);
      std::vector<double> ev((size_t)W * nrows, 0.0);
      for (int64_t i = 0; i < nrows; ++i)
        for (int64_t q = indptr[i]; q < indptr[i + 1]; ++q) {
          ec[(size_t)(q - indptr[i]) * nrows + i] = indices[q];
          ev[(size_t)(q - indptr[i]) * nrows + i] = values[q];
        }
      if (dalloc(&a->ell_col, (int64_t)W * nrows) || dalloc(&a->ell_val, (int64_t)W * nrows) ||
          cudaMemcpy(a->ell_col, ec.data(), sizeof(int) * ec.size(), cudaMemcpyHostToDevice) ||
          cudaMemcpy(a->ell_val, ev.data(), sizeof(double) * ev.size(), cudaMemcpyHostToDevice)) {
        bd_csr_destroy(a);
        return fail(ctx, BD_ECUDA, "bd_csr_create: ELL allocation/copy failed");
      }
      a->ell_w = W;
    }
  }
  *out = a;
  return BD_OK;
}

bd_status bd_csr_destroy(bd_csr* a) {
  if (!a) return BD_OK;
  cudaFree(a->ell_col);
  cudaFree(a->ell_val);
  cudaFree(a->rowptr);
  cudaFree(a->col);
  cudaFree(a->val);
  delete a;
  return BD_OK;
}

bd_status bd_spmv(bd_csr* a, const double* x, double* y, double alpha, double beta) {
  if (!a) return BD_EINVAL;
  bd_ctx* ctx = a->ctx;
  Scope sc(ctx);
  if (a->ell_w) {
    const int grid = grid_for(ctx, a->nrows, dev::TPB);
    switch (a->ell_w) {
      case 8: dev::k_spmv_ell<8><<<grid, dev::TPB, 0, ctx->stream>>>(a->nrows, a->ell_col, a->ell_val, x, y, alpha, beta); break;
      case 16: dev::k_spmv_ell<16><<<grid, dev::TPB, 0, ctx->stream>>>(a->nrows, a->ell_col, a->ell_val, x, y, alpha, beta); break;
      case 24: dev::k_spmv_ell<24><<<grid, dev::TPB, 0, ctx->stream>>>(a->nrows, a->ell_col, a->ell_val, x, y, alpha, beta); break;
      default: dev::k_spmv_ell<32><<<grid, dev::TPB, 0, ctx->stream>>>(a->nrows, a->ell_col, a->ell_val, x, y, alpha, beta);
    }
    LAUNCHED(ctx);
    return BD_OK;
  }
  const int grid = grid_for(ctx, a->nrows, dev::TPB / a->G);
  switch (a->G) {
    case 4: dev::k_spmv<4><<<grid, dev::TPB, 0, ctx->stream>>>(a->dev(), x, y, alpha, beta); break;
    case 8: dev::k_spmv<8><<<grid, dev::TPB, 0, ctx->stream>>>(a->dev(), x, y, alpha, beta); break;
    case 16: dev::k_spmv<16><<<grid, dev::TPB, 0, ctx->stream>>>(a->dev(), x, y, alpha, beta); break;
    default: dev::k_spmv<32><<<grid, dev::TPB, 0, ctx->stream>>>(a->dev(), x, y, alpha, beta);
  }
  LAUNCHED(ctx);
  return BD_OK;
}

bd_status bd_spmv_split(bd_csr* a, const double* x, int64_t nsplit, const double* x_ghost,
                        double* y, double alpha, double beta) {
  if (!a || !x || !y || nsplit < 0 || (nsplit < a->ncols && !x_ghost)) return BD_EINVAL;
  bd_ctx* ctx = a->ctx;
  Scope sc(ctx);
  const int grid = grid_for(ctx, a->nrows, dev::TPB);
  const int ns = (int)std::min<int64_t>(nsplit, 0x7fffffff);
  if (!a->ell_w) {  // irregular / small blocks: CSR rows, one thread each
    if (a->nrows == 0) return BD_OK;
    dev::k_spmv_csr_split<<<grid, dev::TPB, 0, ctx->stream>>>(a->nrows, a->rowptr, a->col, a->val, x,
                                                              x_ghost, ns, y, alpha, beta);
    LAUNCHED(ctx);
    return BD_OK;
  }
  switch (a->ell_w) {
    case 8: dev::k_spmv_ell<8><<<grid, dev::TPB, 0, ctx->stream>>>(a->nrows, a->ell_col, a->ell_val, x, y, alpha, beta, x_ghost, ns); break;
    case 16: dev::k_spmv_ell<16><<<grid, dev::TPB, 0, ctx->stream>>>(a->nrows, a->ell_col, a->ell_val, x, y, alpha, beta, x_ghost, ns); break;
    case 24: dev::k_spmv_ell<24><<<grid, dev::TPB, 0, ctx->stream>>>(a->nrows, a->ell_col, a->ell_val, x, y, alpha, beta, x_ghost, ns); break;
    default: dev::k_spmv_ell<32><<<grid, dev::TPB, 0, ctx->stream>>>(a->nrows, a->ell_col, a->ell_val, x, y, alpha, beta, x_ghost, ns);
  }
  LAUNCHED(ctx);
  return BD_OK;
}

// ---- vector utilities -------------------------------------------------------
static bd_status util_reduce(bd_ctx* ctx, int64_t n, const double* x, const double* y, int fin,
                             int64_t nmean, double* out) {
  Scope sc(ctx);
  TRY(launch_dot(ctx, x, y, n, ctx->util, dev::C_DOT, fin, dev::S_TMP0, -1, nmean));
  CK(ctx, cudaMemcpyAsync(ctx->h_pin, ctx->util.sc + dev::S_TMP0, sizeof(double),
                          cudaMemcpyDeviceToHost, ctx->stream));
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  *out = ctx->h_pin[0];
  return BD_OK;
}

bd_status bd_dot(bd_ctx* ctx, int64_t n, const double* x, const double* y, double* out) {
  if (!ctx || !out || n < 0) return BD_EINVAL;
  if (n == 0) {
    *out = 0.0;
    return BD_OK;
  }
  return util_reduce(ctx, n, x, y, dev::FIN_STORE0, 1, out);
}

bd_status bd_mean(bd_ctx* ctx, int64_t n, const double* x, double* out) {
  if (!ctx || !out || n <= 0) return fail(ctx, BD_EINVAL, "bd_mean: empty vector");
  return util_reduce(ctx, n, x, nullptr, dev::FIN_MEAN, n, out);
}

// ---- system ---------------------------------------------------------------------
bd_status bd_system_create(bd_ctx* ctx, bd_csr* S1, bd_csr* Si, const double* mass,
                           const double* heart_mass, double gamma, bd_system** out) {
  if (!ctx || !S1 || !Si || !mass || !heart_mass || !out)
    return fail(ctx, BD_EINVAL, "bd_system_create: null argument");
  if (S1->nrows != S1->ncols || Si->nrows != Si->ncols || Si->nrows > S1->nrows)
    return fail(ctx, BD_EINVAL, "bd_system_create: block shapes do not match");
  bd_system* s = new bd_system();
  s->ctx = ctx;
  s->S1 = S1;
  s->Si = Si;
  s->n = S1->nrows;
  s->m = Si->nrows;
  s->gamma = gamma;
  if (dalloc(&s->mass, s->n) || dalloc(&s->mh, s->m) || dalloc(&s->tmp, s->n + s->m) ||
      cudaMemcpy(s->mass, mass, sizeof(double) * s->n, cudaMemcpyHostToDevice) ||
      cudaMemcpy(s->mh, heart_mass, sizeof(double) * s->m, cudaMemcpyHostToDevice) ||
      ctl_alloc(&s->ctl, (int64_t)ctx->nsm * 8, 0, 0)) {
    bd_system_destroy(s);
    return fail(ctx, BD_ECUDA, "bd_system_create: device allocation failed");
  }
  CK(ctx, cudaDeviceSynchronize());
  // entry-major ELL copy for Λ when rows are short and near-uniform
  {
    std::vector<int32_t> rp(s->n + 1);
    CK(ctx, cudaMemcpy(rp.data(), S1->dev().rowptr, sizeof(int32_t) * (s->n + 1),
                       cudaMemcpyDeviceToHost));
    int64_t maxlen = 0;
    for (int64_t i = 0; i < s->n; ++i) maxlen = std::max<int64_t>(maxlen, rp[i + 1] - rp[i]);
    const int W = maxlen <= 8 ? 8 : maxlen <= 16 ? 16 : maxlen <= 24 ? 24 : maxlen <= 32 ? 32 : 0;
    const double fill = W && s->n ? (double)W * s->n / std::max<int64_t>(1, rp[s->n]) : 99.0;
    if (W && fill <= 1.5 && !getenv("BD_NO_LAMBDA_ELL")) {
      int* bad = nullptr;
      if (dalloc(&s->ell_col, (int64_t)W * s->n) || dalloc(&s->ell_v1, (int64_t)W * s->n) ||
          dalloc(&s->ell_v2, (int64_t)W * s->m) || dalloc(&bad, 1) || cudaMemset(bad, 0, sizeof(int)))
        return fail(ctx, BD_ECUDA, "bd_system_create: ELL allocation failed");
      dev::k_build_lambda_ell<<<(int)((s->n + 255) / 256), 256>>>(
          S1->dev(), Si->dev(), (int)s->n, (int)s->m, W, s->ell_col, s->ell_v1, s->ell_v2, bad);
      int hb = 0;
      CK(ctx, cudaMemcpy(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost));
      cudaFree(bad);
      if (hb) {
        cudaFree(s->ell_col);
        cudaFree(s->ell_v1);
        cudaFree(s->ell_v2);
        s->ell_col = nullptr;
        s->ell_v1 = s->ell_v2 = nullptr;
      } else {
        s->ell_w = W;
      }
    }
  }
  // ΣM once, fixed order (bd/system.py:145 denominator)
  {
    Scope sc(ctx);
    bd_status st = launch_dot(ctx, s->mass, nullptr, s->n, s->ctl, dev::C_DOT, dev::FIN_STORE0,
                              dev::S_MSUM, -1, 1);
    if (st != BD_OK) return st;
  }
  *out = s;
  return BD_OK;
}

bd_status bd_system_destroy(bd_system* s) {
  if (!s) return BD_OK;
  cudaStreamSynchronize(s->ctx->stream);
  cudaFree(s->mass);
  cudaFree(s->mh);
  cudaFree(s->tmp);
  cudaFree(s->ell_col);
  cudaFree(s->ell_v1);
  cudaFree(s->ell_v2);
  cudaFree(s->track);
  ctl_free(&s->ctl);
  delete s;
  return BD_OK;
}

bd_status bd_system_apply(bd_system* s, const double* x, double* q) {
  if (!s || !x || !q) return BD_EINVAL;
  Scope sc(s->ctx);
  return launch_lambda(s, x, q, s->ctl, 0);
}

bd_status bd_system_normalize(bd_system* s, const double* x, double* y) {
  if (!s || !x || !y) return BD_EINVAL;
  bd_ctx* ctx = s->ctx;
  Scope sc(ctx);
  TRY(launch_dot(ctx, s->mass, x, s->n, s->ctl, dev::C_WMEAN, dev::FIN_WMEAN, 0, -1, 1));
  dev::k_normalize<<<grid_for(ctx, s->n + s->m, dev::TPB), dev::TPB, 0, ctx->stream>>>(
      x, y, s->n, s->n + s->m, s->ctl.sc, nullptr);
  LAUNCHED(ctx);
  return BD_OK;
}

bd_status bd_system_weighted_mean_u(bd_system* s, const double* u, double* out) {
  if (!s || !u || !out) return BD_EINVAL;
  bd_ctx* ctx = s->ctx;
  Scope sc(ctx);
  TRY(launch_dot(ctx, s->mass, u, s->n, s->ctl, dev::C_WMEAN, dev::FIN_WMEAN, 0, -1, 1));
  CK(ctx, cudaMemcpyAsync(ctx->h_pin, s->ctl.sc + dev::S_WMEAN, sizeof(double),
                          cudaMemcpyDeviceToHost, ctx->stream));
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  *out = ctx->h_pin[0];
  return BD_OK;
}

// ---- inner ------------------------------------------------------------------------
bd_status bd_inner_create(bd_ctx* ctx, int kind, int64_t n, const int64_t* indptr,
                          const int32_t* indices, const double* values, int max_restarts,
                          bd_inner** out, int* restarts_used) {
  return bd_inner_create_ex(ctx, kind, n, indptr, indices, values, max_restarts, nullptr, 0, out,
                            restarts_used);
}

bd_status bd_inner_create_ex(bd_ctx* ctx, int kind, int64_t n, const int64_t* indptr,
                             const int32_t* indices, const double* values, int max_restarts,
                             const double* coords, int dim, bd_inner** out, int* restarts_used) {
  if (!ctx || !out || n <= 0 || !indptr) return fail(ctx, BD_EINVAL, "bd_inner_create: bad arguments");
  if (kind != BD_INNER_EXACT && kind != BD_INNER_IC0 && kind != BD_INNER_JACOBI)
    return fail(ctx, BD_EINVAL, "unknown inner preconditioner kind");
  HostCsr a;
  a.n = n;
  a.indptr.assign(indptr, indptr + n + 1);
  a.indices.assign(indices, indices + indptr[n]);
  a.values.assign(values, values + indptr[n]);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = a.indptr[i]; p < a.indptr[i + 1]; ++p) {
      if (a.indices[p] < 0 || a.indices[p] >= n)
        return fail(ctx, BD_EINVAL, "bd_inner_create: column index out of range");
      if (p > a.indptr[i] && a.indices[p] <= a.indices[p - 1])
        return fail(ctx, BD_EINVAL, "bd_inner_create: CSR must be canonical (sorted, no duplicates)");
    }
  bd_inner* p = new bd_inner();
  p->ctx = ctx;
  p->kind = kind;
  p->n = n;
  if (ctl_alloc(&p->ctl, (int64_t)ctx->nsm * 8, 0, 0)) {
    delete p;
    return fail(ctx, BD_ECUDA, "bd_inner_create: allocation failed");
  }
  if (kind == BD_INNER_JACOBI) {
    // 1/diag, strictly positive diagonal required (bd/precond.py:224-232)
    std::vector<double> inv(n);
    for (int64_t i = 0; i < n; ++i) {
      double d = 0.0;
      for (int64_t q = a.indptr[i]; q < a.indptr[i + 1]; ++q)
        if (a.indices[q] == i) d = a.values[q];
      if (!(d > 0.0)) {
        bd_inner_destroy(p);
        return fail(ctx, BD_EPRECOND, "Jacobi requires a strictly positive diagonal");
      }
      inv[i] = 1.0 / d;
    }
    int64_t nnz = 0;
    for (int64_t i = 0; i < n; ++i) nnz += a.indptr[i + 1] - a.indptr[i];
    p->G = pick_g(n ? (double)nnz / n : 1.0);
    if (dalloc(&p->inv, n) || cudaMemcpy(p->inv, inv.data(), sizeof(double) * n, cudaMemcpyHostToDevice) ||
        dalloc(&p->x_int, n)) {
      bd_inner_destroy(p);
      return fail(ctx, BD_ECUDA, "bd_inner_create: allocation failed");
    }
    if (restarts_used) *restarts_used = 0;
    CK(ctx, cudaDeviceSynchronize());
    *out = p;
    return BD_OK;
  }
  std::string msg;
  HostCsr lower;
  if (kind == BD_INNER_IC0) {
    const double t_f = wall_s();
    const int rc = ic0_factor(a, max_restarts, &lower, &p->restarts, &msg);
    setup_log("ic0 factor", t_f);
    if (rc != 0) {
      bd_inner_destroy(p);
      return fail(ctx, BD_EPRECOND, msg);
    }
  } else {
    nested_dissection(a, &p->hperm);
    const int rc = cholesky(a, p->hperm, &lower, &msg);
    if (rc != 0) {
      bd_inner_destroy(p);
      return fail(ctx, BD_EPRECOND, "sparse Cholesky failed, matrix not positive definite: " + msg);
    }
    // relaxed supernodes (explicit zeros; measured on config 1's 263k-row bulk
    // factor, profiles/r02_cfg1_relax_sweep.txt: none 15.1 ms per time step,
    // frac 0.85 uncapped 13.7, frac 0.9 with blocks capped at 320 rows 12.5,
    // frac 1.0 uncapped 1188; nnz(L) +18 %)
    const double relax = getenv("BD_SUPER_RELAX") ? atof(getenv("BD_SUPER_RELAX")) : 0.9;
    const int relax_max = getenv("BD_SUPER_RELAX_MAX") ? atoi(getenv("BD_SUPER_RELAX_MAX")) : dev::SN_MAX;
    if (relax > 0.0) relax_supernodes(&lower, relax, std::min(relax_max, dev::SN_MAX));
  }
  HostCsr upper = transpose(lower);
  const double avg = lower.n ? (double)lower.nnz() / lower.n : 1.0;
  p->G = pick_g(avg - 1.0);
  bd_status st = upload_tri(ctx, lower, true, p->G, &p->L);
  if (st == BD_OK) st = upload_tri(ctx, upper, false, p->G, &p->U);
  // dense explicit inverse up to 8192 rows (config 0: 0.62 vs 3.9 ms per
  // step); above, the relaxed supernodal solves match it (config 1's 16k-row
  // Schur block: 13.63 vs 13.71 ms per step) without the n^2 buffers
  const int64_t dense_max = getenv("BD_EXACT_DENSE_MAX") ? atoll(getenv("BD_EXACT_DENSE_MAX")) : 8192;
  // the explicit inverse takes n^2 doubles on the host and on the device:
  // only when both have 4x that free (else the supernodal solves below)
  bool dense_fits = false;
  if (st == BD_OK && kind == BD_INNER_EXACT && n <= dense_max) {
    const double bytes = 8.0 * (double)n * (double)n;
    size_t dfree = 0, dtotal = 0;
    const double hfree = (double)sysconf(_SC_AVPHYS_PAGES) * (double)sysconf(_SC_PAGESIZE);
    dense_fits = cudaMemGetInfo(&dfree, &dtotal) == cudaSuccess && 4.0 * bytes <= (double)dfree &&
                 4.0 * bytes <= hfree;
  }
  if (st == BD_OK && kind == BD_INNER_EXACT && dense_fits) {
    // explicit inverse of P A P^T from the sparse factor, one column per host
    // thread (X^T = X up to rounding; row j of X holds the solve with e_j)
    std::vector<double> X((size_t)n * n);
    int bad = 0;
#pragma omp parallel reduction(| : bad)
    {
      std::vector<double> w(n);
#pragma omp for schedule(dynamic, 8)
      for (int64_t j = 0; j < n; ++j) {
        std::fill(w.begin(), w.end(), 0.0);
        w[j] = 1.0;
        for (int64_t i = j; i < n; ++i) {  // L w = e_j (diagonal last)
          double acc = w[i];
          const int64_t b = lower.indptr[i], e = lower.indptr[i + 1] - 1;
          for (int64_t q = b; q < e; ++q) acc -= lower.values[q] * w[lower.indices[q]];
          w[i] = acc / lower.values[e];
        }
        for (int64_t i = n - 1; i >= 0; --i) {  // L^T x = w (diagonal first)
          double acc = w[i];
          const int64_t b = upper.indptr[i], e = upper.indptr[i + 1];
          for (int64_t q = b + 1; q < e; ++q) acc -= upper.values[q] * w[upper.indices[q]];
          w[i] = acc / upper.values[b];
        }
        for (int64_t i = 0; i < n; ++i) {
          if (!std::isfinite(w[i])) bad = 1;
          X[(size_t)j * n + i] = w[i];
        }
      }
    }
    if (bad) {
      st = fail(ctx, BD_EPRECOND, "exact inner: non-finite explicit inverse");
    } else {
      CK(ctx, upload_vec(&p->dense, X));
    }
  } else if (st == BD_OK && kind == BD_INNER_EXACT) {
    const char* m = getenv("BD_EXACT_TRSV");
    if (!(m && std::string(m) == "rows")) {
      st = build_super(ctx, lower, &p->SL, &p->SU);
      if (st == BD_OK && (p->SL.task_kind || p->SU.task_kind) && dalloc(&p->rext, lower.n))
        st = fail(ctx, BD_ECUDA, "supernodal solve: allocation failed");
      if (st == BD_OK) p->super = true;
    }
  }
  if (st == BD_OK && kind == BD_INNER_IC0) {
    const char* mode = getenv("BD_TRSV");
    const std::string m = mode ? mode : "btile";
    if (m == "cluster") {
      st = setup_cluster(p, lower, upper, coords, dim);
    }
    if (m == "btile") {
      st = setup_btile(p, lower, upper, coords, dim);
    }
    if (m == "dtile" || (m == "btile" && st == BD_OK && !p->btile)) {
      st = setup_dtile(p, lower, upper, coords, dim);
    }
    if (m == "tiled" || m == "rows") {
      p->rows_mode = (m == "rows");
      st = setup_tiles(p, lower, upper, coords, dim);
    } else if (m == "persist" || (m == "cluster" && !p->cluster) || ((m == "dtile" || m == "btile") && !p->dtile && !p->btile)) {
      int64_t maxoff = 0;
      for (int64_t i = 0; i < n; ++i)
        maxoff = std::max<int64_t>(maxoff, lower.indptr[i + 1] - lower.indptr[i] - 1);
      for (int64_t i = 0; i < n; ++i)
        maxoff = std::max<int64_t>(maxoff, upper.indptr[i + 1] - upper.indptr[i] - 1);
      if (maxoff <= p->G) {
        st = build_ell(ctx, lower, true, p->G, &p->EL);
        if (st == BD_OK) st = build_ell(ctx, upper, false, p->G, &p->EU);
        if (st == BD_OK) p->persist = true;
      }
    }
  }
  if (st != BD_OK) {
    bd_inner_destroy(p);
    return st;
  }
  if (dalloc(&p->y_int, n) || dalloc(&p->x_int, n) ||
      cudaMemset(p->y_int, 0xFF, sizeof(double) * n)) {
    bd_inner_destroy(p);
    return fail(ctx, BD_ECUDA, "bd_inner_create: allocation failed");
  }
  // default 1: the forward pass resets the backward pass's output rows
  // (measured cfg2 1.433 -> 1.412 ms per PCG iteration); 2 also folds the
  // forward output's reset into the previous backward pass, which loses its
  // L2 residency and measured 1.82 ms per iteration
  p->fold_fill = getenv("BD_FOLD_FILL") ? atoi(getenv("BD_FOLD_FILL")) : 1;
  if (!p->hperm.empty()) {
    if (dalloc(&p->perm, n) ||
        cudaMemcpy(p->perm, p->hperm.data(), sizeof(int) * n, cudaMemcpyHostToDevice)) {
      bd_inner_destroy(p);
      return fail(ctx, BD_ECUDA, "bd_inner_create: allocation failed");
    }
  }
  p->hlower = std::move(lower);
  if (restarts_used) *restarts_used = p->restarts;
  CK(ctx, cudaDeviceSynchronize());
  *out = p;
  return BD_OK;
}

bd_status bd_inner_destroy(bd_inner* p) {
  if (!p) return BD_OK;
  cudaStreamSynchronize(p->ctx->stream);
  free_tri(&p->L);
  free_tri(&p->U);
  free_tile(&p->TL);
  free_tile(&p->TU);
  free_ell(&p->EL);
  free_ell(&p->EU);
  free_super(&p->SL);
  free_super(&p->SU);
  free_cluster(&p->CL);
  free_cluster(&p->CU);
  free_dtile(&p->DL);
  free_dtile(&p->DU);
  free_btile(&p->BL);
  free_btile(&p->BU);

  cudaFree(p->rtmp);
  cudaFree(p->rhs_pre);
  cudaFree(p->rext);
  cudaFree(p->dense);
  cudaFree(p->perm);
  cudaFree(p->inv);
  cudaFree(p->y_int);
  cudaFree(p->bt_f);
  cudaFree(p->bt_b);
  cudaFree(p->inbox);
  cudaFree(p->x_int);
  ctl_free(&p->ctl);
  delete p;
  return BD_OK;
}

bd_status bd_inner_apply(bd_inner* p, const double* y, double* z) {
  if (!p || !y || !z) return BD_EINVAL;
  Scope sc(p->ctx);
  dev::RhsVec rhs{y, (int)p->n, nullptr, p->perm};
  if (p->kind == BD_INNER_JACOBI) return inner_solve(p, rhs, z, nullptr, p->ctl, dev::C_JAC1);
  return inner_solve(p, rhs, p->x_int, z, p->ctl, dev::C_BULK1_S);
}

// Debug: enable the tiled-solve step trace (buffer of parts*steps*3 u64 on the
// device; NULL disables).  Not part of the public header.
bd_status bd_debug_tile_trace(void* dev_buf, int steps) {
  g_tile_trace_on = dev_buf != nullptr;
  cudaMemcpyToSymbol(dev::g_tile_trace, &dev_buf, sizeof(void*));
  cudaMemcpyToSymbol(dev::g_tile_trace_steps, &steps, sizeof(int));
  return cudaGetLastError() == cudaSuccess ? BD_OK : BD_ECUDA;
}

// Debug: first row of every blocked tile of one pass (0 forward, 1 backward)
// in task order; returns the tile count in *ntiles.  Not in the public header.
bd_status bd_debug_btile_rows(bd_inner* p, int pass, int32_t* first_row, int* ntiles) {
  if (!p || !p->btile) return BD_EINVAL;
  const DevBTile& b = pass ? p->BU : p->BL;
  *ntiles = b.ntiles;
  if (!first_row) return BD_OK;
  for (int t = 0; t < b.ntiles; ++t)
    cudaMemcpy(first_row + t, b.task_row + (size_t)t * b.rs, sizeof(int32_t), cudaMemcpyDeviceToHost);
  return cudaGetLastError() == cudaSuccess ? BD_OK : BD_ECUDA;
}

bd_status bd_inner_tile_info(bd_inner* p, int64_t* info) {
  // parts, threads, G, smem, max_part_rows, max_part_steps, L nsteps, U nsteps
  if (!p) return BD_EINVAL;
  info[0] = p->tiled ? p->tparts : 0;
  info[1] = p->tthreads;
  info[2] = p->TG;
  info[3] = (int64_t)p->tsmem;
  info[4] = p->TL.max_part_rows;
  info[5] = p->TL.max_part_steps;
  info[6] = p->TL.nsteps;
  info[7] = p->TU.nsteps;
  return BD_OK;
}

bd_status bd_inner_factor_info(bd_inner* p, int64_t* n, int64_t* nnz, int64_t* levels) {
  if (!p) return BD_EINVAL;
  if (n) *n = p->n;
  if (nnz) *nnz = p->kind == BD_INNER_JACOBI ? p->n : p->hlower.nnz();
  if (levels) *levels = p->kind == BD_INNER_JACOBI ? 1 : std::max(p->L.depth, p->U.depth);
  return BD_OK;
}

bd_status bd_inner_export_factor(bd_inner* p, int64_t* indptr, int32_t* indices, double* values,
                                 int32_t* perm) {
  if (!p) return BD_EINVAL;
  if (p->kind == BD_INNER_JACOBI) return fail(p->ctx, BD_EINVAL, "jacobi has no factor");
  const HostCsr& l = p->hlower;
  if (indptr) std::copy(l.indptr.begin(), l.indptr.end(), indptr);
  if (indices) std::copy(l.indices.begin(), l.indices.end(), indices);
  if (values) std::copy(l.values.begin(), l.values.end(), values);
  if (perm) {
    if (p->hperm.empty())
      for (int64_t i = 0; i < p->n; ++i) perm[i] = (int32_t)i;
    else
      std::copy(p->hperm.begin(), p->hperm.end(), perm);
  }
  return BD_OK;
}

// ---- block-LU ---------------------------------------------------------------------
bd_status bd_blocklu_create(bd_system* s, bd_inner* bulk, bd_inner* schur, double beta,
                            bd_prec** out) {
  if (!s || !bulk || !schur || !out) return BD_EINVAL;
  bd_ctx* ctx = s->ctx;
  if (bulk->n != s->n || schur->n != s->m)
    return fail(ctx, BD_EINVAL, "bd_blocklu_create: inner sizes do not match the system");
  if (!(beta > 0.0)) return fail(ctx, BD_EINVAL, "bd_blocklu_create: beta must be positive");
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  bd_prec* p = new bd_prec();
  p->sys = s;
  p->bulk = bulk;
  p->schur = schur;
  bulk->prof_cls = 2;
  schur->prof_cls = 3;
  p->beta = beta;
  const int64_t n = s->n, m = s->m, nm = n + m;
  int64_t parts = (int64_t)ctx->nsm * 8 * 2;
  parts = std::max<int64_t>(parts, std::max(bulk->U.nvb, schur->U.nvb));
  parts = std::max<int64_t>(parts, std::max(bulk->EU.nchunks, schur->EU.nchunks));
  p->hist_cap = 0;
  if (ctl_alloc(&p->ctl, parts, 0, 1) || dalloc(&p->traw, n) || dalloc(&p->z2raw, n) ||
      dalloc(&p->corr, m) || dalloc(&p->sbuf, m) || dalloc(&p->x, nm) || dalloc(&p->r, nm) ||
      dalloc(&p->z, nm) || dalloc(&p->d, nm) || dalloc(&p->q, nm) || dalloc(&p->zsc, dev::NSLOTS) ||
      cudaMemset(p->zsc, 0, sizeof(double) * dev::NSLOTS)) {
    bd_blocklu_destroy(p);
    return fail(ctx, BD_ECUDA, "bd_blocklu_create: allocation failed");
  }
  p->ctl_nf = p->ctl;
  p->ctl_nf.use_flags = 0;
  CK(ctx, cudaDeviceSynchronize());
  // beta and ΣM into the slots
  CK(ctx, cudaMemcpy(p->ctl.sc + dev::S_BULK_BETA, &beta, sizeof(double), cudaMemcpyHostToDevice));
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  CK(ctx, cudaMemcpy(p->ctl.sc + dev::S_MSUM, s->ctl.sc + dev::S_MSUM, sizeof(double),
                     cudaMemcpyDeviceToDevice));
  const char* env = getenv("BD_NO_GRAPH");
  p->use_graph = !(env && env[0] == '1');
  // The Schur solve's right-hand side r_v - S_i t: evaluated by one streaming kernel on
  // the ELL copy before the forward pass (BD_RHS_PRE=0: inside the pass's tiles)
  if (!(getenv("BD_RHS_PRE") && atoi(getenv("BD_RHS_PRE")) == 0) && schur->btile && schur->BL.rpipe &&
      !schur->rhs_pre && s->ell_w && !schur->perm)
    if (dalloc(&schur->rhs_pre, m)) return fail(ctx, BD_ECUDA, "bd_blocklu_create: out of device memory");
  *out = p;
  return BD_OK;
}

bd_status bd_blocklu_destroy(bd_prec* p) {
  if (!p) return BD_OK;
  cudaStreamSynchronize(p->sys->ctx->stream);
  if (p->gexec) cudaGraphExecDestroy(p->gexec);
  if (p->graph) cudaGraphDestroy(p->graph);
  ctl_free(&p->ctl);
  cudaFree(p->traw);
  cudaFree(p->zsc);
  cudaFree(p->z2raw);
  cudaFree(p->corr);
  cudaFree(p->sbuf);
  cudaFree(p->x);
  cudaFree(p->r);
  cudaFree(p->z);
  cudaFree(p->d);
  cudaFree(p->q);
  delete p;
  return BD_OK;
}

bd_status bd_blocklu_apply(bd_prec* p, const double* r, double* z) {
  if (!p || !r || !z) return BD_EINVAL;
  bd_system* s = p->sys;
  bd_ctx* ctx = s->ctx;
  Scope sc(ctx);
  const Ctl& c = p->ctl_nf;
  TRY(launch_dot(ctx, r, nullptr, s->n, c, dev::C_MEAN, dev::FIN_MEAN, dev::S_MU1, dev::S_C1, s->n));
  TRY(enqueue_pinv(p, r, z, p->sbuf, z + s->n, c, false));
  p->cnt[0] += 2;
  p->cnt[1] += 1;
  p->cnt[2] += 2;
  return BD_OK;
}

bd_status bd_blocklu_bulk_inverse(bd_prec* p, const double* y, double* z) {
  if (!p || !y || !z) return BD_EINVAL;
  bd_system* s = p->sys;
  bd_ctx* ctx = s->ctx;
  Scope sc(ctx);
  const Ctl& c = p->ctl_nf;
  const int64_t n = s->n;
  // mean, inner(y - mean), recentre, + mean/beta  (bd/precond.py:281-292)
  TRY(launch_dot(ctx, y, nullptr, n, c, dev::C_MEAN, dev::FIN_MEAN, dev::S_MU1, dev::S_C1, n));
  dev::RhsVec rhs{y, (int)n, c.sc + dev::S_MU1, p->bulk->perm};
  double* xi = p->bulk->perm ? p->bulk->x_int : p->traw;
  double* o = p->bulk->perm ? p->traw : nullptr;
  if (p->bulk->kind == BD_INNER_JACOBI) {
    xi = p->traw;
    o = nullptr;
  }
  TRY(inner_solve(p->bulk, rhs, xi, o, c, dev::C_BULK1_S, dev::FIN_MEAN, dev::S_MT, -1, n));
  // z = (traw - mt) + c1: k_combine with a zero second operand
  CK(ctx, cudaMemsetAsync(c.sc + dev::S_M2, 0, sizeof(double), ctx->stream));
  CK(ctx, cudaMemsetAsync(c.sc + dev::S_C2, 0, sizeof(double), ctx->stream));
  CK(ctx, cudaMemsetAsync(p->z2raw, 0, sizeof(double) * n, ctx->stream));
  dev::k_combine<<<grid_for(ctx, n, dev::TPB), dev::TPB, 0, ctx->stream>>>(p->traw, p->z2raw, z, n,
                                                                           c);
  LAUNCHED(ctx);
  p->cnt[0] += 1;
  return BD_OK;
}

bd_status bd_blocklu_schur_inverse(bd_prec* p, const double* y, double* z) {
  if (!p || !y || !z) return BD_EINVAL;
  Scope sc(p->sys->ctx);
  dev::RhsVec rhs{y, (int)p->sys->m, nullptr, p->schur->perm};
  bd_status st;
  if (p->schur->kind == BD_INNER_JACOBI)
    st = inner_solve(p->schur, rhs, z, nullptr, p->ctl_nf, dev::C_JAC2);
  else
    st = inner_solve(p->schur, rhs, p->schur->x_int, z, p->ctl_nf, dev::C_SCH_S);
  if (st == BD_OK) p->cnt[1] += 1;
  return st;
}

bd_status bd_blocklu_counters(bd_prec* p, int64_t* counters) {
  if (!p || !counters) return BD_EINVAL;
  std::copy(p->cnt, p->cnt + 3, counters);
  return BD_OK;
}

bd_status bd_blocklu_reset_counters(bd_prec* p) {
  if (!p) return BD_EINVAL;
  std::fill(p->cnt, p->cnt + 3, 0);
  return BD_OK;
}

// ---- PCG ----------------------------------------------------------------------------
bd_status bd_pcg_solve(bd_system* s, bd_prec* p, const double* b, const double* x0, double tol,
                       int64_t max_iter, double* x, bd_stats* stats, double* res_hist,
                       int64_t* n_res, double* prec_hist, int64_t* n_prec) {
  if (!s || !p || !b || !x || !stats) return BD_EINVAL;
  bd_ctx* ctx = s->ctx;
  std::memset(stats, 0, sizeof(*stats));
  stats->curvature = std::nan("");
  if (!(tol > 0.0)) return fail(ctx, BD_EINVAL, "tol must be strictly positive");
  if (max_iter < 0) return fail(ctx, BD_EINVAL, "max_iter must be non-negative");
  if (p->sys != s) return fail(ctx, BD_EINVAL, "preconditioner was built for another system");
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t n = s->n, nm = s->n + s->m;
  // history buffers (device), regrown on demand (invalidates the graph)
  const int need = (int)std::min<int64_t>(max_iter + 2, (int64_t)INT32_MAX);
  if (need > p->hist_cap) {
    CK(ctx, cudaStreamSynchronize(ctx->stream));
    cudaFree(p->ctl.res_hist);
    cudaFree(p->ctl.prec_hist);
    const int cap = std::max(need, 512);
    CK(ctx, dalloc(&p->ctl.res_hist, cap));
    CK(ctx, dalloc(&p->ctl.prec_hist, cap));
    p->hist_cap = cap;
    p->ctl.hist_cap = cap;
    p->ctl_nf = p->ctl;
    p->ctl_nf.use_flags = 0;
    if (p->gexec) {
      cudaGraphExecDestroy(p->gexec);
      cudaGraphDestroy(p->graph);
      p->gexec = nullptr;
      p->graph = nullptr;
    }
  }
  if (p->use_graph && !ctx->profile && !p->gexec) TRY(build_graph(p));
  Scope scope(ctx);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, ctx->stream);
  // control block init: flags, tol, max_iter
  {
    int* hf = (int*)ctx->h_pin;
    std::memset(hf, 0, sizeof(int) * dev::NFLAGS);
    hf[dev::F_FIRST] = 1;
    hf[dev::F_MAXITER] = (int)std::min<int64_t>(max_iter, INT32_MAX);
    CK(ctx, cudaMemcpyAsync(p->ctl.fl, hf, sizeof(int) * dev::NFLAGS, cudaMemcpyHostToDevice,
                            ctx->stream));
    double* hs = ctx->h_pin + 16;
    hs[0] = tol;
    CK(ctx, cudaMemcpyAsync(p->ctl.sc + dev::S_TOL, hs, sizeof(double), cudaMemcpyHostToDevice,
                            ctx->stream));
    // the pinned staging area is reused below only after a synchronise
  }
  const Ctl& c = p->ctl;
  prof_mark(ctx, 6);
  // ||b|| (and the zero-rhs exit)
  TRY(launch_dot(ctx, b, b, nm, c, dev::C_NORMB, dev::FIN_RHSNORM, 0, -1, 1));
  // x0 / r0
  if (x0) {
    dev::k_copy<<<grid_for(ctx, nm, dev::TPB), dev::TPB, 0, ctx->stream>>>(p->x, x0, nm, c);
    LAUNCHED(ctx);
    TRY(launch_lambda(s, p->x, p->q, c, 0));
    dev::k_init_res<<<grid_for(ctx, nm, dev::TPB), dev::TPB, 0, ctx->stream>>>(b, p->q, p->r, n,
                                                                               nm, c);
  } else {
    dev::k_fill<<<grid_for(ctx, nm, dev::TPB), dev::TPB, 0, ctx->stream>>>(p->x, nm, 0LL, c);
    LAUNCHED(ctx);
    dev::k_init_res<<<grid_for(ctx, nm, dev::TPB), dev::TPB, 0, ctx->stream>>>(b, nullptr, p->r, n,
                                                                               nm, c);
  }
  LAUNCHED(ctx);
  dev::k_fill<<<grid_for(ctx, nm, dev::TPB), dev::TPB, 0, ctx->stream>>>(p->d, nm, 0LL, c);
  LAUNCHED(ctx);
  prof_mark(ctx, 1);
  // z0 = deflate(P^{-1} r0); rho0; d0 = z0
  TRY(enqueue_pinv(p, p->r, p->z, p->z + n, nullptr, c, true));  // rho in its tail
  dev::k_dupdate<<<grid_for(ctx, nm, dev::TPB), dev::TPB, 0, ctx->stream>>>(p->z, p->d, n, nm, c);
  LAUNCHED(ctx);
  prof_mark(ctx, 5);
  int* hflag = (int*)(ctx->h_pin + 32);
  int64_t it_launch = 0;
  if (p->gexec && !ctx->profile) {
    CK(ctx, cudaGraphLaunch(p->gexec, ctx->stream));
    ctx->launches += 1;
    it_launch = -1;  // counted from the iteration count below
  } else {
    // (profile mode: one iteration per host round trip, so every profiled
    // iteration is a real one; the host gap before it goes to class 7)
    int batch = ctx->profile ? 1 : 2;
    for (;;) {
      prof_mark(ctx, 7);
      for (int i = 0; i < batch; ++i) TRY(enqueue_iteration(p));
      CK(ctx, cudaMemcpyAsync(hflag, c.fl, sizeof(int) * dev::NFLAGS, cudaMemcpyDeviceToHost,
                              ctx->stream));
      CK(ctx, cudaStreamSynchronize(ctx->stream));
      if (hflag[dev::F_DONE] || hflag[dev::F_STOP]) break;
      if (!ctx->profile) batch = std::min(batch * 2, 32);
    }
  }
  // x <- normalize(x) (bd/system.py:138-146), zero for a zero rhs
  TRY(launch_dot(ctx, s->mass, p->x, n, p->ctl_nf, dev::C_WMEAN, dev::FIN_WMEAN, 0, -1, 1));
  dev::k_normalize<<<grid_for(ctx, nm, dev::TPB), dev::TPB, 0, ctx->stream>>>(p->x, x, n, nm,
                                                                             c.sc, c.fl);
  LAUNCHED(ctx);
  prof_mark(ctx, 5);
  cudaEventRecord(e1, ctx->stream);
  // readback
  CK(ctx, cudaMemcpyAsync(hflag, c.fl, sizeof(int) * dev::NFLAGS, cudaMemcpyDeviceToHost,
                          ctx->stream));
  double* hsc = ctx->h_pin;
  CK(ctx, cudaMemcpyAsync(hsc, c.sc, sizeof(double) * 24, cudaMemcpyDeviceToHost, ctx->stream));
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  const int nres = std::min(hflag[dev::F_NRES], p->hist_cap);
  const int nprec = std::min(hflag[dev::F_NPREC], p->hist_cap);
  if (res_hist && nres)
    CK(ctx, cudaMemcpy(res_hist, c.res_hist, sizeof(double) * nres, cudaMemcpyDeviceToHost));
  if (prec_hist && nprec)
    CK(ctx, cudaMemcpy(prec_hist, c.prec_hist, sizeof(double) * nprec, cudaMemcpyDeviceToHost));
  if (n_res) *n_res = nres;
  if (n_prec) *n_prec = nprec;
  float dms = 0.f;
  cudaEventElapsedTime(&dms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  prof_collect(ctx);
  stats->iterations = hflag[dev::F_ITERS];
  stats->mv_count = hflag[dev::F_NMV];
  stats->p1_count = 2 * (int64_t)hflag[dev::F_NAPP];
  stats->pk_count = hflag[dev::F_NAPP];
  stats->converged = hflag[dev::F_CONV];
  stats->device_ms = dms;
  stats->final_residual = 0.0;
  if (nres)
    CK(ctx, cudaMemcpy(&stats->final_residual, c.res_hist + (nres - 1), sizeof(double),
                       cudaMemcpyDeviceToHost));
  p->cnt[0] += stats->p1_count;
  p->cnt[1] += stats->pk_count;
  p->cnt[2] += 2 * (int64_t)hflag[dev::F_NAPP];
  if (it_launch < 0)  // graph bodies run once per iteration (+1 for the exit test)
    ctx->launches += (iteration_launches(p) + 1) * (int64_t)std::max<int64_t>(stats->iterations, 1);
  bd_status st = BD_OK;
  if (hflag[dev::F_STATUS] == dev::ST_EBREAKDOWN) {
    st = BD_EBREAKDOWN;
    stats->curvature = hsc[dev::S_CURV];
    char buf[128];
    if (std::isnan(hsc[dev::S_CURV]) && stats->iterations > 0 && hsc[dev::S_DQ] > 0)
      std::snprintf(buf, sizeof buf, "non-finite residual");
    else
      std::snprintf(buf, sizeof buf, "conjugate gradient breakdown: curvature %g", hsc[dev::S_CURV]);
    tl_err = buf;
  } else if (!hflag[dev::F_CONV]) {
    st = BD_ENOCONV;
    char buf[160];
    std::snprintf(buf, sizeof buf, "PCG did not reach tol=%g within %lld iterations (residual %.3e)",
                  tol, (long long)max_iter, stats->final_residual);
    tl_err = buf;
  }
  stats->status = st;
  stats->wall_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return st;
}

// ---- membrane -------------------------------------------------------------------
bd_status bd_membrane_rhs(bd_system* s, const double* v, const double* w, const uint64_t* site_mask,
                          uint64_t active_sites, double amplitude, double chi, double v_rest,
                          double v_span, double tau_in, double tau_out, double c_m, double* rhs,
                          double* ion) {
  if (!s || !v || !w || !rhs) return BD_EINVAL;
  bd_ctx* ctx = s->ctx;
  Scope sc(ctx);
  dev::k_membrane_rhs<<<grid_for(ctx, s->n + s->m, dev::TPB), dev::TPB, 0, ctx->stream>>>(
      s->n, s->m, v, w, site_mask, active_sites, amplitude, chi, s->gamma, s->mh, v_rest, v_span,
      tau_in, tau_out, c_m, rhs, ion);
  LAUNCHED(ctx);
  return BD_OK;
}

bd_status bd_membrane_rhs_raw(bd_ctx* ctx, int64_t n, int64_t m, const double* heart_mass,
                              double gamma, const double* v, const double* w,
                              const uint64_t* site_mask, uint64_t active_sites, double amplitude,
                              double chi, double v_rest, double v_span, double tau_in,
                              double tau_out, double c_m, double* rhs, double* ion) {
  if (!ctx || !heart_mass || !v || !w || !rhs) return BD_EINVAL;
  Scope sc(ctx);
  dev::k_membrane_rhs<<<grid_for(ctx, n + m, dev::TPB), dev::TPB, 0, ctx->stream>>>(
      n, m, v, w, site_mask, active_sites, amplitude, chi, gamma, heart_mass, v_rest, v_span,
      tau_in, tau_out, c_m, rhs, ion);
  LAUNCHED(ctx);
  return BD_OK;
}

bd_status bd_step_track(bd_system* s, const double* v_prev, const double* v_new, double* phi,
                        double t_prev, double dt, double threshold, double band_lo, double band_hi,
                        const double* u, double* out) {
  if (!s || !v_prev || !v_new || !phi || !u || !out) return BD_EINVAL;
  bd_ctx* ctx = s->ctx;
  Scope sc(ctx);
  if (!s->track && dalloc(&s->track, 4)) return fail(ctx, BD_ECUDA, "bd_step_track: allocation failed");
  CK(ctx, cudaMemsetAsync(s->track, 0, 4 * sizeof(unsigned long long), ctx->stream));
  const int64_t len = std::max(s->n, s->m);
  dev::k_step_track<<<grid_for(ctx, len, dev::TPB), dev::TPB, 0, ctx->stream>>>(
      s->m, v_prev, v_new, phi, t_prev, dt, threshold, band_lo, band_hi, s->n, u, s->track);
  LAUNCHED(ctx);
  TRY(launch_dot(ctx, s->mass, u, s->n, s->ctl, dev::C_WMEAN, dev::FIN_WMEAN, 0, -1, 1));
  static_assert(sizeof(double) == sizeof(unsigned long long), "");
  CK(ctx, cudaMemcpyAsync(ctx->h_pin, s->track, 3 * sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->stream));
  CK(ctx, cudaMemcpyAsync(ctx->h_pin + 3, s->ctl.sc + dev::S_WMEAN, sizeof(double),
                          cudaMemcpyDeviceToHost, ctx->stream));
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  unsigned long long bits[3];
  std::memcpy(bits, ctx->h_pin, sizeof(bits));
  out[0] = bits[0] ? 1.0 : 0.0;
  out[1] = bits[1] ? 0.0 : 1.0;  // covered = no unset vertex left
  double umax;
  std::memcpy(&umax, &bits[2], sizeof(double));
  out[2] = umax;
  out[3] = ctx->h_pin[3];
  return BD_OK;
}

// ---- P1 assembly on the device (setup) -------------------------------------------
struct bd_asm {
  bd_ctx* ctx;
  int64_t nv = 0, nnz = 0;
  long long* rowptr = nullptr;
  int* col = nullptr;
  double* data = nullptr;
  double* mass = nullptr;
};

bd_status bd_assemble_destroy(bd_asm* a) {
  if (!a) return BD_OK;
  cudaFree(a->rowptr);
  cudaFree(a->col);
  cudaFree(a->data);
  cudaFree(a->mass);
  delete a;
  return BD_OK;
}

bd_status bd_assemble_p1(bd_ctx* ctx, int dim, int64_t nv, const double* vertices, int64_t ne,
                         const int64_t* elements, const double* sigma, const double* sigma2,
                         bd_asm** out, int64_t* nnz_out) {
  if (!ctx || !out || !vertices || (ne > 0 && (!elements || !sigma)) || nv <= 0 ||
      (dim != 2 && dim != 3))
    return fail(ctx, BD_EINVAL, "bd_assemble_p1: bad arguments");
  Scope sc(ctx);
  cudaStream_t st = ctx->stream;
  const int A = dim + 1;
  const int64_t np = ne * A * A;
  bd_asm* a = new bd_asm;
  a->ctx = ctx;
  a->nv = nv;
  asmk::DevScratch S;  // scratch, freed at scope exit
  auto bail = [&](const std::string& msg) {
    bd_assemble_destroy(a);
    return fail(ctx, BD_ECUDA, msg);
  };
  double *xv, *sa, *sb = nullptr, *local, *vol;
  int64_t* el;
  int* bad;
  unsigned long long *k0, *k1, *v0, *v1, *ukey;
  long long *head, *pos, *start;
  if (S.get(&xv, nv * dim) || S.get(&el, ne * A) || S.get(&sa, ne * dim * dim) ||
      (sigma2 && S.get(&sb, ne * dim * dim)) || S.get(&local, np) || S.get(&vol, ne) ||
      S.get(&bad, 1) || S.get(&k0, np) || S.get(&k1, np) || S.get(&v0, np) || S.get(&v1, np))
    return bail("bd_assemble_p1: device allocation failed");
  CK(ctx, cudaMemcpyAsync(xv, vertices, sizeof(double) * nv * dim, cudaMemcpyHostToDevice, st));
  if (ne > 0) {
    CK(ctx, cudaMemcpyAsync(el, elements, sizeof(int64_t) * ne * A, cudaMemcpyHostToDevice, st));
    CK(ctx, cudaMemcpyAsync(sa, sigma, sizeof(double) * ne * dim * dim, cudaMemcpyHostToDevice, st));
    if (sigma2)
      CK(ctx, cudaMemcpyAsync(sb, sigma2, sizeof(double) * ne * dim * dim, cudaMemcpyHostToDevice, st));
  }
  CK(ctx, cudaMemsetAsync(bad, 0, sizeof(int), st));
  const int gl = grid_for(ctx, std::max<int64_t>(ne, 1), 256);
  const int gp = grid_for(ctx, std::max<int64_t>(np, 1), 256);
  if (ne > 0) {
    if (dim == 2) {
      asmk::k_local<2><<<gl, 256, 0, st>>>(ne, xv, el, sa, sb, local, vol, bad);
      asmk::k_keys<2><<<gp, 256, 0, st>>>(ne, el, nv, k0, v0);
    } else {
      asmk::k_local<3><<<gl, 256, 0, st>>>(ne, xv, el, sa, sb, local, vol, bad);
      asmk::k_keys<3><<<gp, 256, 0, st>>>(ne, el, nv, k0, v0);
    }
    LAUNCHED(ctx);
  }
  int hbad = 0;
  CK(ctx, cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(ctx, cudaStreamSynchronize(st));
  if (hbad) {
    bd_assemble_destroy(a);
    return fail(ctx, BD_EINVAL, "degenerate element (non-positive volume)");
  }
  int end_bit = 1;
  while (end_bit < 64 && (((unsigned long long)nv * (unsigned long long)nv - 1ull) >> end_bit)) ++end_bit;
  // stable LSD radix sort: equal keys keep element order
  size_t tmp_bytes = 0;
  cub::DoubleBuffer<unsigned long long> dk(k0, k1), dv(v0, v1);
  CK(ctx, cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, dk, dv, np, 0, end_bit, st));
  void* tmp = nullptr;
  if (S.get((char**)&tmp, (int64_t)tmp_bytes)) return bail("bd_assemble_p1: sort scratch");
  if (np > 0) CK(ctx, cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, dk, dv, np, 0, end_bit, st));
  const unsigned long long* keys = dk.Current();
  const unsigned long long* vals = dv.Current();
  if (S.get(&head, np) || S.get(&pos, np)) return bail("bd_assemble_p1: allocation failed");
  int64_t nnz = 0;
  if (np > 0) {
    asmk::k_heads<<<gp, 256, 0, st>>>(np, keys, head);
    LAUNCHED(ctx);
    size_t sb_bytes = 0;
    CK(ctx, cub::DeviceScan::ExclusiveSum(nullptr, sb_bytes, head, pos, np, st));
    void* tmp2 = nullptr;
    if (S.get((char**)&tmp2, (int64_t)sb_bytes)) return bail("bd_assemble_p1: scan scratch");
    CK(ctx, cub::DeviceScan::ExclusiveSum(tmp2, sb_bytes, head, pos, np, st));
    long long last[2];
    CK(ctx, cudaMemcpyAsync(&last[0], pos + np - 1, sizeof(long long), cudaMemcpyDeviceToHost, st));
    CK(ctx, cudaMemcpyAsync(&last[1], head + np - 1, sizeof(long long), cudaMemcpyDeviceToHost, st));
    CK(ctx, cudaStreamSynchronize(st));
    nnz = last[0] + last[1];
  }
  if (S.get(&start, nnz) || S.get(&ukey, nnz) || dalloc(&a->col, std::max<int64_t>(nnz, 1)) ||
      dalloc(&a->data, std::max<int64_t>(nnz, 1)) || dalloc(&a->mass, nv) ||
      dalloc(&a->rowptr, nv + 1))
    return bail("bd_assemble_p1: allocation failed");
  CK(ctx, cudaMemsetAsync(a->mass, 0, sizeof(double) * nv, st));
  if (nnz > 0) {
    asmk::k_seg_start<<<gp, 256, 0, st>>>(np, head, pos, start);
    const int gu = grid_for(ctx, nnz, 256);
    if (dim == 2)
      asmk::k_segsum<2><<<gu, 256, 0, st>>>(nnz, np, nv, start, keys, vals, local, vol, a->col,
                                            a->data, ukey, a->mass);
    else
      asmk::k_segsum<3><<<gu, 256, 0, st>>>(nnz, np, nv, start, keys, vals, local, vol, a->col,
                                            a->data, ukey, a->mass);
    LAUNCHED(ctx);
  }
  asmk::k_rowptr<<<grid_for(ctx, nv + 1, 256), 256, 0, st>>>(nv, nnz, ukey, a->rowptr);
  LAUNCHED(ctx);
  CK(ctx, cudaStreamSynchronize(st));
  a->nnz = nnz;
  *nnz_out = nnz;
  *out = a;
  return BD_OK;
}

bd_status bd_tensors_transmural(bd_ctx* ctx, int64_t nv, const double* vertices, int64_t ne,
                                const int64_t* elements, const double* model, const double* gi,
                                const double* ge, int orthotropic, double* out_intra,
                                double* out_extra) {
  if (!ctx || !vertices || !model || !gi || !ge || !out_intra || !out_extra || ne < 0 || nv <= 0 ||
      (ne > 0 && !elements))
    return fail(ctx, BD_EINVAL, "bd_tensors_transmural: bad arguments");
  Scope sc(ctx);
  cudaStream_t st = ctx->stream;
  asmk::DevScratch S;
  double *xv, *oi, *oe;
  int64_t* el;
  if (S.get(&xv, nv * 3) || S.get(&el, ne * 4) || S.get(&oi, ne * 9) || S.get(&oe, ne * 9))
    return fail(ctx, BD_ECUDA, "bd_tensors_transmural: allocation failed");
  CK(ctx, cudaMemcpyAsync(xv, vertices, sizeof(double) * nv * 3, cudaMemcpyHostToDevice, st));
  if (ne > 0) {
    CK(ctx, cudaMemcpyAsync(el, elements, sizeof(int64_t) * ne * 4, cudaMemcpyHostToDevice, st));
    asmk::k_tensors_transmural<<<grid_for(ctx, ne, 256), 256, 0, st>>>(
        ne, xv, el, model[0], model[1], model[2], model[3], gi[0], gi[1], gi[2], ge[0], ge[1], ge[2],
        orthotropic, oi, oe);
    LAUNCHED(ctx);
    CK(ctx, cudaMemcpyAsync(out_intra, oi, sizeof(double) * ne * 9, cudaMemcpyDeviceToHost, st));
    CK(ctx, cudaMemcpyAsync(out_extra, oe, sizeof(double) * ne * 9, cudaMemcpyDeviceToHost, st));
  }
  CK(ctx, cudaStreamSynchronize(st));
  return BD_OK;
}

bd_status bd_assemble_export(bd_asm* a, int64_t* indptr, int32_t* indices, double* data,
                             double* mass) {
  if (!a) return BD_EINVAL;
  bd_ctx* ctx = a->ctx;
  Scope sc(ctx);
  cudaStream_t st = ctx->stream;
  static_assert(sizeof(long long) == sizeof(int64_t), "");
  if (indptr)
    CK(ctx, cudaMemcpyAsync(indptr, a->rowptr, sizeof(int64_t) * (a->nv + 1), cudaMemcpyDeviceToHost, st));
  if (indices && a->nnz)
    CK(ctx, cudaMemcpyAsync(indices, a->col, sizeof(int32_t) * a->nnz, cudaMemcpyDeviceToHost, st));
  if (data && a->nnz)
    CK(ctx, cudaMemcpyAsync(data, a->data, sizeof(double) * a->nnz, cudaMemcpyDeviceToHost, st));
  if (mass) CK(ctx, cudaMemcpyAsync(mass, a->mass, sizeof(double) * a->nv, cudaMemcpyDeviceToHost, st));
  CK(ctx, cudaStreamSynchronize(st));
  return BD_OK;
}

bd_status bd_membrane_gate(bd_ctx* ctx, int64_t m, const double* v, const double* w, double dt,
                           double v_rest, double v_span, double tau_open, double tau_close,
                           double u_gate, double* w_new) {
  if (!ctx || !v || !w || !w_new) return BD_EINVAL;
  if (!(dt > 0.0)) return fail(ctx, BD_EINVAL, "dt must be strictly positive");
  Scope sc(ctx);
  dev::k_membrane_gate<<<grid_for(ctx, m, dev::TPB), dev::TPB, 0, ctx->stream>>>(
      m, v, w, dt, v_rest, v_span, tau_open, tau_close, u_gate, w_new);
  LAUNCHED(ctx);
  return BD_OK;
}


}  // extern "C"

// ---- sharded PCG iteration (one rank of distributed.py; bd_shard.cuh) -------------
struct bd_shard {
  bd_ctx* ctx = nullptr;
  int64_t n = 0, m = 0, n_global = 0;
  bd_csr *S1 = nullptr, *Si = nullptr;
  bd_csr* Si_ext = nullptr;  // S_i with its ghost columns at n + j: reads [z1 | ghosts] in place
  double* z1ext = nullptr;    // caller-owned: z1 (n) followed by its heart ghosts
  double* zero_sc = nullptr;  // zero scalar slots (RhsSchur without recentring)
  bd_inner *bulk = nullptr, *schur = nullptr;
  double gamma = 0.0, msum = 1.0;
  double *x = nullptr, *r = nullptr, *d = nullptr, *q = nullptr, *z1 = nullptr, *z2 = nullptr,
         *s = nullptr, *rhs_s = nullptr, *corr = nullptr, *mh = nullptr, *mass = nullptr;
  double *sc = nullptr, *red = nullptr, *part = nullptr, *res_hist = nullptr, *prec_hist = nullptr;
  int *fl = nullptr, *si = nullptr;
  unsigned* ctr = nullptr;
  int hist_cap = 0;
  Ctl cb{}, cs{};  // the inners' control blocks with the shard's done flag
};

namespace {
__global__ void k_sh_begin(double* sc, int* fl, int* si, double tol, int64_t max_iter) {
  for (int i = 0; i < dev::SH_NSLOTS; ++i) sc[i] = 0.0;
  for (int i = 0; i < dev::NFLAGS; ++i) fl[i] = 0;
  for (int i = 0; i < dev::SHI_NINT; ++i) si[i] = 0;
  sc[dev::SH_TOL] = tol;
  si[dev::SHI_MAXITER] = (int)max_iter;
}

template <class Rhs>
bd_status shard_inner(bd_inner* p, const Rhs& rhs, double* z, const Ctl& c) {
  if (p->kind == BD_INNER_JACOBI) return inner_solve(p, rhs, z, nullptr, c, dev::C_JAC1);
  return inner_solve(p, rhs, p->x_int, z, c, dev::C_BULK1_S);
}
}  // namespace

extern "C" {

bd_status bd_shard_create(bd_ctx* ctx, int64_t n, int64_t m, int64_t n_global, bd_csr* S1,
                          bd_csr* Si, const double* mass, const double* heart_mass, double gamma,
                          bd_inner* bulk, bd_inner* schur, double msum, int64_t hist_cap,
                          double* red, bd_csr* Si_ext, double* z1ext, bd_shard** out) {
  if (!ctx || !S1 || !Si || !mass || !heart_mass || !bulk || !schur || !red || !out || n <= 0 || m < 0 ||
      m > n || S1->nrows != n || Si->nrows != m || bulk->n != n || schur->n != m)
    return fail(ctx, BD_EINVAL, "bd_shard_create: inconsistent arguments");
  auto* h = new bd_shard();
  h->ctx = ctx;
  h->n = n;
  h->m = m;
  h->n_global = n_global;
  h->S1 = S1;
  h->Si = Si;
  h->bulk = bulk;
  h->schur = schur;
  h->gamma = gamma;
  h->msum = msum;
  h->hist_cap = (int)std::max<int64_t>(hist_cap, 2);
  h->red = red;  // caller-owned (the host all-reduces slices of it in place)
  if (Si_ext && z1ext && Si_ext->nrows == m) {
    h->z1ext = z1ext;  // z1 and its halo stay contiguous either way
    // The Schur right-hand side r_v - S_i [z1 | ghosts]: with the TMA-ring tile kernel one
    // streaming split SpMV before the pass beats the product inside its tiles (as on one
    // GPU); BD_SHARD_RHS_PRE=0 keeps the in-tile RhsSchur on S_i's extended copy
    const bool pre = schur->btile && schur->BL.rpipe && Si->ell_w &&
                     !(getenv("BD_SHARD_RHS_PRE") && atoi(getenv("BD_SHARD_RHS_PRE")) == 0);
    if (!pre) h->Si_ext = Si_ext;
  }
  const int64_t nm = n + m;
  bool bad = dalloc(&h->x, nm) || dalloc(&h->r, nm) || dalloc(&h->d, nm) || dalloc(&h->q, nm) ||
             (!h->z1ext && dalloc(&h->z1, n)) || dalloc(&h->z2, n) ||
             dalloc(&h->zero_sc, dev::NSLOTS) || dalloc(&h->s, m) || dalloc(&h->rhs_s, m) ||
             dalloc(&h->corr, n) || dalloc(&h->mh, m) || dalloc(&h->mass, n) ||
             dalloc(&h->sc, dev::SH_NSLOTS) ||
             dalloc(&h->part, (int64_t)dev::SH_GRID * 4) || dalloc(&h->res_hist, h->hist_cap) ||
             dalloc(&h->prec_hist, h->hist_cap) || dalloc(&h->fl, dev::NFLAGS) ||
             dalloc(&h->si, dev::SHI_NINT) || dalloc(&h->ctr, 8);
  if (h->z1ext) h->z1 = h->z1ext;
  bad = bad || cudaMemset(h->corr, 0, sizeof(double) * n) ||
        cudaMemset(h->zero_sc, 0, sizeof(double) * dev::NSLOTS) || cudaMemset(h->d, 0, sizeof(double) * nm) ||
        cudaMemset(h->red, 0, sizeof(double) * dev::SH_RED) || cudaMemset(h->ctr, 0, sizeof(unsigned) * 8) ||
        cudaMemset(h->fl, 0, sizeof(int) * dev::NFLAGS) || cudaMemset(h->si, 0, sizeof(int) * dev::SHI_NINT) ||
        cudaMemcpy(h->mh, heart_mass, sizeof(double) * m, cudaMemcpyHostToDevice) ||
        cudaMemcpy(h->mass, mass, sizeof(double) * n, cudaMemcpyHostToDevice);
  if (bad) {
    bd_shard_destroy(h);
    return fail(ctx, BD_ECUDA, "bd_shard_create: device allocation failed");
  }
  h->cb = bulk->ctl;
  h->cb.fl = h->fl;
  h->cb.use_flags = 1;
  h->cs = schur->ctl;
  h->cs.fl = h->fl;
  h->cs.use_flags = 1;
  *out = h;
  return BD_OK;
}

bd_status bd_shard_destroy(bd_shard* h) {
  if (!h) return BD_OK;
  for (double* p : {h->x, h->r, h->d, h->q, h->z2, h->s, h->rhs_s, h->corr, h->mh, h->mass,
                    h->sc, h->part, h->res_hist, h->prec_hist, h->zero_sc})
    cudaFree(p);
  if (!h->z1ext) cudaFree(h->z1);
  cudaFree(h->fl);
  cudaFree(h->si);
  cudaFree(h->ctr);
  delete h;
  return BD_OK;
}

bd_status bd_shard_vectors(bd_shard* h, double** ptrs) {
  if (!h || !ptrs) return BD_EINVAL;
  double* v[9] = {h->x, h->r, h->d, h->q, h->z1, h->s, h->red, h->z2, h->corr};
  for (int i = 0; i < 9; ++i) ptrs[i] = v[i];
  return BD_OK;
}

bd_status bd_shard_begin(bd_shard* h, double tol, int64_t max_iter, const double* x0) {
  if (!h || !(tol > 0.0) || max_iter < 0) return BD_EINVAL;
  bd_ctx* ctx = h->ctx;
  if (max_iter + 2 > h->hist_cap) return fail(ctx, BD_EINVAL, "bd_shard_begin: max_iter exceeds the history capacity");
  Scope sc(ctx);
  k_sh_begin<<<1, 1, 0, ctx->stream>>>(h->sc, h->fl, h->si, tol, max_iter);
  LAUNCHED(ctx);
  if (x0)
    CK(ctx, cudaMemcpyAsync(h->x, x0, sizeof(double) * (h->n + h->m), cudaMemcpyDeviceToDevice, ctx->stream));
  else
    CK(ctx, cudaMemsetAsync(h->x, 0, sizeof(double) * (h->n + h->m), ctx->stream));
  return BD_OK;
}

// q = Λ_local v with v's halo (ug: all ghosts, vg: heart ghosts); red[0] = v·q
bd_status bd_shard_lambda(bd_shard* h, const double* v, const double* ug, const double* vg,
                          int use_flags) {
  if (!h || !v) return BD_EINVAL;
  bd_ctx* ctx = h->ctx;
  const int64_t n = h->n, m = h->m;
  if (h->S1->ell_w && (m == 0 || h->Si->ell_w) && !getenv("BD_SHARD_LAMBDA_SPLIT")) {
    Scope sc(ctx);  // one fused pass (k_sh_lambda_ell)
    dev::k_sh_lambda_ell<<<dev::SH_GRID, dev::TPB, 0, ctx->stream>>>(
        n, m, h->S1->ell_w, h->S1->ell_col, h->S1->ell_val, m ? h->Si->ell_w : 0,
        m ? h->Si->ell_col : nullptr, m ? h->Si->ell_val : nullptr, v, ug, vg, h->q, h->mh,
        h->gamma, h->part, h->ctr + 0, h->red + 0, h->fl, use_flags);
    LAUNCHED(ctx);
    return BD_OK;
  }
  TRY(bd_spmv_split(h->S1, v, n, ug, h->q, 1.0, 0.0));
  if (m > 0) {
    TRY(bd_spmv_split(h->Si, v + n, m, vg, h->q + n, 1.0, 0.0));  // S_i v
    Scope sc(ctx);
    dev::k_sh_lam_add<<<grid_for(ctx, m, dev::TPB), dev::TPB, 0, ctx->stream>>>(m, h->q, h->q + n,
                                                                             h->fl, use_flags);
    LAUNCHED(ctx);
  }
  if (m > 0) TRY(bd_spmv_split(h->Si, v, m, ug, h->q + n, 1.0, 1.0));  // S_i u_H + S_i v
  Scope sc(ctx);
  dev::k_sh_lam_fin<<<dev::SH_GRID, dev::TPB, 0, ctx->stream>>>(n, n + m, v, h->q, h->mh, h->gamma,
                                                                h->part, h->ctr + 0, h->red + 0,
                                                                h->fl, use_flags);
  LAUNCHED(ctx);
  return BD_OK;
}

// r = b − Λx0 (q from bd_shard_lambda on x0) or b; red[1], red[2], red[7]
bd_status bd_shard_init(bd_shard* h, const double* b, int has_x0) {
  if (!h || !b) return BD_EINVAL;
  bd_ctx* ctx = h->ctx;
  h->bulk->prefilled = h->schur->prefilled = false;  // a new solve starts with explicit fills
  Scope sc(ctx);
  dev::k_sh_init<<<dev::SH_GRID, dev::TPB, 0, ctx->stream>>>(h->n, h->n + h->m, b, has_x0 ? h->q : nullptr,
                                                             h->r, h->Si_ext ? nullptr : h->rhs_s,
                                                             h->part, h->ctr + 1,
                                                             h->red + 1);
  LAUNCHED(ctx);
  return BD_OK;
}

bd_status bd_shard_check(bd_shard* h, int initial) {
  if (!h) return BD_EINVAL;
  bd_ctx* ctx = h->ctx;
  Scope sc(ctx);
  if (initial) {  // k_sh_init wrote (‖r‖², Σr_u, ‖b‖²) to red[1..3]: move ‖b‖² to red[7]
    CK(ctx, cudaMemcpyAsync(h->red + 7, h->red + 3, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  }
  dev::k_sh_check<<<1, 1, 0, ctx->stream>>>(h->sc, h->fl, h->si, h->red, h->res_hist, h->hist_cap,
                                            h->n_global, initial);
  LAUNCHED(ctx);
  return BD_OK;
}

bd_status bd_shard_update(bd_shard* h) {
  if (!h) return BD_EINVAL;
  bd_ctx* ctx = h->ctx;
  Scope sc(ctx);
  dev::k_sh_alpha<<<1, 1, 0, ctx->stream>>>(h->sc, h->fl, h->si, h->red);
  LAUNCHED(ctx);
  // the first bulk solve (bd_shard_pinv1) follows: its polled forward output is reset here
  double* ft = fill_target(h->bulk);
  dev::k_sh_update<<<dev::SH_GRID, dev::TPB, 0, ctx->stream>>>(h->n, h->n + h->m, h->x, h->r, h->d, h->q,
                                                               h->Si_ext ? nullptr : h->rhs_s, h->sc,
                                                               h->part, h->ctr + 2,
                                                               h->red + 1, h->fl, ft, ft ? h->n : 0);
  LAUNCHED(ctx);
  if (ft) h->bulk->prefilled = true;
  return BD_OK;
}

// z1 = bulk^{-1}(r_u − μ1)
bd_status bd_shard_pinv1(bd_shard* h) {
  if (!h) return BD_EINVAL;
  Scope sc(h->ctx);
  dev::RhsVec rhs{h->r, (int)h->n, h->sc + dev::SH_MU1, h->bulk->perm};
  // the Schur solve follows (halo gathers in between do not touch its buffers): the bulk
  // solve's backward pass resets the Schur solve's polled forward output
  if (prefill_level() >= 2 && h->m > 0 && h->bulk != h->schur && h->bulk->btile && h->bulk->BU.rpipe) {
    if (double* ft = fill_target(h->schur)) {
      h->bulk->post_fill = ft;
      h->bulk->post_fill_n = h->m;
      h->bulk->post_fill_owner = h->schur;
    }
  }
  const bd_status st = shard_inner(h->bulk, rhs, h->z1, h->cb);
  h->bulk->post_fill = nullptr;
  h->bulk->post_fill_owner = nullptr;
  return st;
}

// s = K^{-1}(r_v − S_i [z1 | tg]); with S_i's ghost columns at n + j and the
// halo received into z1ext[n..), the product is formed inside the Schur
// forward pass (RhsSchur, as the single-GPU path) and tg is not read
bd_status bd_shard_pinv2(bd_shard* h, const double* tg) {
  if (!h) return BD_EINVAL;
  if (h->m == 0) return BD_OK;
  if (h->Si_ext) {
    Scope sc(h->ctx);
    dev::RhsSchur rhs{h->Si_ext->dev(), h->z1ext, h->zero_sc, h->r + h->n, h->schur->perm};
    return shard_inner(h->schur, rhs, h->s, h->cs);
  }
  TRY(bd_spmv_split(h->Si, h->z1, h->m, tg, h->rhs_s, -1.0, 1.0));
  Scope sc(h->ctx);
  dev::RhsVec rhs{h->rhs_s, (int)h->m, nullptr, h->schur->perm};
  return shard_inner(h->schur, rhs, h->s, h->cs);
}

// corr = pad(S_i [s | sg]); red[3] = Σ corr
bd_status bd_shard_pinv3(bd_shard* h, const double* sg) {
  if (!h) return BD_EINVAL;
  bd_ctx* ctx = h->ctx;
  if (h->m > 0 && h->Si->ell_w) {  // one pass: product and its sum
    Scope sc(ctx);
    double* ft = fill_target(h->bulk);  // the second bulk solve (bd_shard_pinv4) follows
    dev::k_sh_corr_ell<<<dev::SH_GRID, dev::TPB, 0, ctx->stream>>>(
        h->m, h->Si->ell_w, h->Si->ell_col, h->Si->ell_val, h->s, sg, h->corr, h->part, h->ctr + 3,
        h->red + 3, h->fl, ft, ft ? h->n : 0);
    LAUNCHED(ctx);
    if (ft) h->bulk->prefilled = true;
    return BD_OK;
  }
  if (h->m > 0) TRY(bd_spmv_split(h->Si, h->s, h->m, sg, h->corr, 1.0, 0.0));
  Scope sc(ctx);
  dev::k_sh_sum<<<dev::SH_GRID, dev::TPB, 0, ctx->stream>>>(h->m, h->corr, h->part, h->ctr + 3,
                                                            h->red + 3, h->fl);
  LAUNCHED(ctx);
  return BD_OK;
}

// z2 = bulk^{-1}(corr − μ2); w = z1 − z2; red[4..6] = Σw, r_u·w, r_v·s
bd_status bd_shard_pinv4(bd_shard* h) {
  if (!h) return BD_EINVAL;
  bd_ctx* ctx = h->ctx;
  Scope sc(ctx);
  dev::k_sh_mu2<<<1, 1, 0, ctx->stream>>>(h->sc, h->fl, h->red, h->n_global);
  LAUNCHED(ctx);
  dev::RhsVec rhs{h->corr, (int)h->n, h->sc + dev::SH_MU2, h->bulk->perm};
  TRY(shard_inner(h->bulk, rhs, h->z2, h->cb));
  dev::k_sh_combine<<<dev::SH_GRID, dev::TPB, 0, ctx->stream>>>(h->n, h->m, h->z1, h->z2, h->r, h->s,
                                                                h->part, h->ctr + 4, h->red + 4, h->fl);
  LAUNCHED(ctx);
  return BD_OK;
}

// ρ_next, β; d = z + βd (initial: d = z)
bd_status bd_shard_finish(bd_shard* h, int initial) {
  if (!h) return BD_EINVAL;
  bd_ctx* ctx = h->ctx;
  Scope sc(ctx);
  dev::k_sh_finish<<<1, 1, 0, ctx->stream>>>(h->sc, h->fl, h->si, h->red, h->prec_hist, h->hist_cap,
                                             h->n_global, initial);
  LAUNCHED(ctx);
  if (initial) CK(ctx, cudaMemsetAsync(h->d, 0, sizeof(double) * (h->n + h->m), ctx->stream));
  dev::k_sh_dupdate<<<grid_for(ctx, h->n + h->m, dev::TPB), dev::TPB, 0, ctx->stream>>>(
      h->n, h->m, h->z1, h->s, h->d, h->sc, h->fl);
  LAUNCHED(ctx);
  return BD_OK;
}

// red[8] = Σ mass ∘ x_u (the weighted mean's numerator, before its all-reduce)
bd_status bd_shard_wmean(bd_shard* h) {
  if (!h) return BD_EINVAL;
  bd_ctx* ctx = h->ctx;
  Scope sc(ctx);
  dev::k_sh_wmean<<<dev::SH_GRID, dev::TPB, 0, ctx->stream>>>(h->n, h->mass, h->x, h->part, h->ctr + 5,
                                                              h->red + 8);
  LAUNCHED(ctx);
  return BD_OK;
}

// out = normalize(x) with the all-reduced red[8] (zero for a zero rhs)
bd_status bd_shard_normalize(bd_shard* h, double* out) {
  if (!h || !out) return BD_EINVAL;
  bd_ctx* ctx = h->ctx;
  Scope sc(ctx);
  dev::k_sh_normalize<<<grid_for(ctx, h->n + h->m, dev::TPB), dev::TPB, 0, ctx->stream>>>(
      h->n, h->n + h->m, h->x, out, h->red, h->msum, h->si);
  LAUNCHED(ctx);
  return BD_OK;
}

// done flag only (the host's periodic loop test); synchronising
bd_status bd_shard_done(bd_shard* h, int* done) {
  if (!h || !done) return BD_EINVAL;
  bd_ctx* ctx = h->ctx;
  Scope sc(ctx);
  int* hp = (int*)(ctx->h_pin + 40);
  CK(ctx, cudaMemcpyAsync(hp, h->fl + dev::F_DONE, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  *done = hp[0];
  return BD_OK;
}

// info = {iterations, converged, breakdown, zero_rhs, max_iter_hit, n_res, n_prec};
// scal = {last relative residual, curvature at a breakdown}; histories: host
// arrays of capacity cap (may be NULL).  Synchronising.
bd_status bd_shard_read(bd_shard* h, int64_t* info, double* scal, double* res_hist,
                        double* prec_hist, int64_t cap) {
  if (!h || !info) return BD_EINVAL;
  bd_ctx* ctx = h->ctx;
  Scope sc(ctx);
  int si[dev::SHI_NINT];
  double s[dev::SH_NSLOTS];
  CK(ctx, cudaStreamSynchronize(ctx->stream));
  CK(ctx, cudaMemcpy(si, h->si, sizeof(si), cudaMemcpyDeviceToHost));
  CK(ctx, cudaMemcpy(s, h->sc, sizeof(s), cudaMemcpyDeviceToHost));
  info[0] = si[dev::SHI_ITERS];
  info[1] = si[dev::SHI_CONV];
  info[2] = si[dev::SHI_BAD];
  info[3] = si[dev::SHI_ZERO];
  info[4] = si[dev::SHI_MAXIT];
  info[5] = std::min(si[dev::SHI_NRES], h->hist_cap);
  info[6] = std::min(si[dev::SHI_NPREC], h->hist_cap);
  if (scal) {
    scal[0] = s[dev::SH_REL];
    scal[1] = s[dev::SH_CURV];
  }
  if (res_hist && info[5])
    CK(ctx, cudaMemcpy(res_hist, h->res_hist, sizeof(double) * std::min<int64_t>(info[5], cap),
                       cudaMemcpyDeviceToHost));
  if (prec_hist && info[6])
    CK(ctx, cudaMemcpy(prec_hist, h->prec_hist, sizeof(double) * std::min<int64_t>(info[6], cap),
                       cudaMemcpyDeviceToHost));
  return BD_OK;
}

// dst[i] = src[idx[i]] (device; halo packing)
bd_status bd_gather(bd_ctx* ctx, int64_t k, const int64_t* idx, const double* src, double* dst) {
  if (!ctx || k < 0 || (k && (!idx || !src || !dst))) return BD_EINVAL;
  if (k == 0) return BD_OK;
  Scope sc(ctx);
  dev::k_sh_gather<<<grid_for(ctx, k, dev::TPB), dev::TPB, 0, ctx->stream>>>(k, idx, src, dst);
  LAUNCHED(ctx);
  return BD_OK;
}

}  // extern "C"
