// Device kernels of the bidomain PCG hot path (sm_100a, fp64, HBM-bound).
//
// Every reduction is deterministic: per-block partials land in a fixed slot
// and the last block to finish sums them in a fixed order (no fp64 atomics),
// so two identical runs are bitwise identical (tests/test_simulate.py:147-151
// in the reference).  Kernels that belong to the PCG loop first check the
// control flags and return when the solve is finished, so an iteration can be
// enqueued (or replayed from a CUDA graph) without a host round trip.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace bd {
namespace dev {

constexpr int TPB = 256;               // threads per block everywhere
constexpr long long SENTINEL = -1LL;   // all-ones NaN: "not yet solved"

// Scalar slots of one PCG / preconditioner context (device doubles).
enum Slot {
  S_RHSNORM = 0, S_RR, S_REL, S_RHO, S_DQ, S_ALPHA, S_BETA,
  S_MU1, S_C1, S_MT, S_MU2, S_C2, S_M2, S_MZ, S_TOL, S_BULK_BETA,
  S_MSUM, S_WMEAN, S_TMP0, S_TMP1, S_CURV, NSLOTS = 32
};
// Integer flags.
enum Flag {
  F_DONE = 0, F_STOP, F_STATUS, F_ITERS, F_NAPP, F_NMV, F_FIRST, F_MAXITER,
  F_ZERO, F_CONV, F_NRES, F_NPREC, NFLAGS = 16
};
// Reduction finalisers (what the last block does with the totals).
enum Fin {
  FIN_STORE0 = 0,   // sc[slot] = tot0
  FIN_RHSNORM,      // ||b||, zero-rhs early exit (bd/krylov.py:68-72)
  FIN_INIT_RES,     // rel0, history[0], warm-start exit (:85-93); mu1
  FIN_MEAN,         // sc[slot] = tot0 / n; sc[slot2] = sc[slot] / beta (if slot2>=0)
  FIN_DQ,           // curvature / breakdown / alpha (:101-109)
  FIN_UPDATE,       // iterations, rel, history, convergence (:114-123); mu1
  FIN_RHO,          // rho, beta, history, max_iter stop (:95-97, :125-131)
  FIN_WMEAN         // mass-weighted mean (bd/system.py:145)
};
enum Status { ST_OK = 0, ST_ENOCONV = 3, ST_EBREAKDOWN = 4 };

struct Ctl {
  double* sc;          // NSLOTS
  int* fl;             // NFLAGS
  double* res_hist;    // max_iter + 2
  double* prec_hist;   // max_iter + 2
  double* partials;    // scratch for block partials
  unsigned* ctr;       // last-block counters, one per kernel class
  int hist_cap;
  int use_flags;       // 0: always active (standalone calls)
};

// Counter indices (one per kernel class so a kernel never shares its counter
// with the next one on the stream).
enum Ctr {
  C_NORMB = 0, C_INITR, C_LAMBDA, C_UPDATE, C_BULK1_S, C_BULK1_D, C_BULK1B_S, C_BULK1B_D,
  C_SCH_S, C_SCH_D, C_SCHB_S, C_SCHB_D, C_CORR, C_BULK2_S, C_BULK2_D, C_BULK2B_S,
  C_BULK2B_D, C_COMBINE, C_RHO, C_WMEAN, C_DOT, C_MEAN, C_JAC1, C_JAC2, C_JAC3, NCTR = 32
};

__device__ __forceinline__ bool inactive(const Ctl& c, bool allow_stop = false) {
  if (!c.use_flags) return false;
  const volatile int* f = c.fl;
  return f[F_DONE] || (!allow_stop && f[F_STOP]);
}

// ---- polled loads / stores for the sync-free triangular solves ----------
__device__ __forceinline__ double spin_load(const double* p) {
  long long b;
  do {
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(b) : "l"(p) : "memory");
  } while (b == SENTINEL);
  return __longlong_as_double(b);
}
__device__ __forceinline__ void publish(double* p, double v) {
  long long b = __double_as_longlong(v);
  if (b == SENTINEL) b = 0x7FF8000000000000LL;  // never publish the sentinel
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(b) : "memory");
}

// ---- reductions ----------------------------------------------------------
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) { return group_sum<32>(v); }

// Fixed-tree block sum; result valid in thread 0.  Uses sm[32].
__device__ __forceinline__ double block_sum(double v, double* sm) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sm[w] = v;
  __syncthreads();
  v = (threadIdx.x < (blockDim.x >> 5)) ? sm[threadIdx.x] : 0.0;
  if (w == 0) v = warp_sum(v);
  return v;
}

// Commit NV block partials (thread 0 holds them) and tell whether this block
// is the last one; partial layout [NV][nblocks].
template <int NV>
__device__ __forceinline__ bool commit(const double (&v)[NV], double* partials, int nblocks,
                                       int pidx, unsigned* ctr) {
  __shared__ int last;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) partials[k * nblocks + pidx] = v[k];
    __threadfence();
    const unsigned t = atomicAdd(ctr, 1u);
    last = (t == (unsigned)nblocks - 1u);
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}
// Whole-block fixed-order sum of partials[k*nblocks ...]; result in thread 0.
__device__ __forceinline__ double sum_partials(const double* partials, int nblocks, int k,
                                               double* sm) {
  double s = 0.0;
  for (int i = threadIdx.x; i < nblocks; i += blockDim.x) s += __ldcg(&partials[k * nblocks + i]);
  return block_sum(s, sm);
}

// Finaliser, run by thread 0 of the last block.
__device__ void finalize(const Ctl& c, int fin, int slot, int slot2, const double* tot, int64_t n) {
  double* sc = c.sc;
  int* fl = c.fl;
  switch (fin) {
    case FIN_STORE0:
      sc[slot] = tot[0];
      break;
    case FIN_RHSNORM: {
      const double nb = sqrt(tot[0]);
      sc[S_RHSNORM] = nb;
      if (nb == 0.0) {
        fl[F_ZERO] = 1;
        fl[F_CONV] = 1;
        fl[F_DONE] = 1;
        c.res_hist[0] = 0.0;
        fl[F_NRES] = 1;
      }
      break;
    }
    case FIN_INIT_RES: {
      const double rel = sqrt(tot[0]) / sc[S_RHSNORM];
      sc[S_REL] = rel;
      c.res_hist[0] = rel;
      fl[F_NRES] = 1;
      fl[F_NMV] = 1;
      if (rel <= sc[S_TOL]) {
        fl[F_CONV] = 1;
        fl[F_DONE] = 1;
      }
      sc[S_MU1] = tot[1] / (double)n;
      sc[S_C1] = sc[S_MU1] / sc[S_BULK_BETA];
      break;
    }
    case FIN_MEAN:
      sc[slot] = tot[0] / (double)n;
      if (slot2 >= 0) sc[slot2] = sc[slot] / sc[S_BULK_BETA];
      break;
    case FIN_DQ: {
      const double dq = tot[0];
      sc[S_DQ] = dq;
      fl[F_NMV] += 1;
      if (!isfinite(dq) || dq <= 0.0) {
        fl[F_STATUS] = ST_EBREAKDOWN;
        sc[S_CURV] = dq;
        fl[F_DONE] = 1;
      } else {
        sc[S_ALPHA] = sc[S_RHO] / dq;
      }
      break;
    }
    case FIN_UPDATE: {
      fl[F_ITERS] += 1;
      const double rel = sqrt(tot[0]) / sc[S_RHSNORM];
      sc[S_REL] = rel;
      if (!isfinite(rel)) {
        fl[F_STATUS] = ST_EBREAKDOWN;
        sc[S_CURV] = __longlong_as_double(0x7FF8000000000000LL);
        fl[F_DONE] = 1;
        break;
      }
      const int k = fl[F_NRES];
      if (k < c.hist_cap) c.res_hist[k] = rel;
      fl[F_NRES] = k + 1;
      if (rel <= sc[S_TOL]) {
        fl[F_CONV] = 1;
        fl[F_DONE] = 1;
      }
      sc[S_MU1] = tot[1] / (double)n;
      sc[S_C1] = sc[S_MU1] / sc[S_BULK_BETA];
      break;
    }
    case FIN_RHO: {
      const double rho_next = tot[0];
      const int k = fl[F_NPREC];
      if (k < c.hist_cap) c.prec_hist[k] = rho_next;
      fl[F_NPREC] = k + 1;
      fl[F_NAPP] += 1;
      if (fl[F_FIRST]) {
        sc[S_BETA] = 0.0;
        fl[F_FIRST] = 0;
      } else {
        sc[S_BETA] = rho_next / sc[S_RHO];
      }
      sc[S_RHO] = rho_next;
      if (fl[F_ITERS] >= fl[F_MAXITER]) fl[F_STOP] = 1;
      break;
    }
    case FIN_WMEAN:
      sc[S_WMEAN] = tot[0] / sc[S_MSUM];
      break;
  }
}

// Reduction tail shared by every kernel: thread 0 holds v[NV]; commits and,
// in the last block, sums and finalises, then resets the counter.
template <int NV>
__device__ __forceinline__ void reduce_tail(const Ctl& c, double (&v)[NV], int nblocks, int pidx,
                                            int ctr, int fin, int slot, int slot2, int64_t n,
                                            double* sm) {
  if (commit<NV>(v, c.partials, nblocks, pidx, &c.ctr[ctr])) {
    double tot[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      tot[k] = sum_partials(c.partials, nblocks, k, sm);
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      finalize(c, fin, slot, slot2, tot, n);
      c.ctr[ctr] = 0u;
      __threadfence();
    }
  }
}

// ---- device CSR -----------------------------------------------------------
struct Csr {
  int nrows;
  const int* rowptr;
  const int* col;
  const double* val;
};

// Group dot of row `row` with x; `ok == false` gives 0 but still joins the
// group shuffle (every lane of a warp must reach it).
template <int G>
__device__ __forceinline__ double row_dot(const Csr& a, int row, bool ok, int lane,
                                          const double* __restrict__ x) {
  int b = 0, e = 0;
  if (ok) {
    b = a.rowptr[row];
    e = a.rowptr[row + 1];
  }
  double s = 0.0;
  for (int k = b + lane; k < e; k += G) s = fma(a.val[k], __ldg(&x[a.col[k]]), s);
  return group_sum<G>(s);
}

// ---- generic kernels ------------------------------------------------------
__global__ void k_fill(double* p, int64_t n, long long bits, Ctl c) {
  if (inactive(c)) return;
  const double v = __longlong_as_double(bits);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
__global__ void k_copy(double* dst, const double* src, int64_t n, Ctl c) {
  if (inactive(c)) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// sum_i x_i*y_i (y null: sum x_i) with finaliser; grid-stride, fixed grid.
__global__ void __launch_bounds__(TPB) k_dot(const double* x, const double* y, int64_t n, Ctl c,
                                             int ctr, int fin, int slot, int slot2, int64_t nmean) {
  if (inactive(c, true)) return;
  __shared__ double sm[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s = y ? fma(x[i], y[i], s) : s + x[i];
  double v[1] = {block_sum(s, sm)};
  reduce_tail<1>(c, v, gridDim.x, blockIdx.x, ctr, fin, slot, slot2, nmean, sm);
}

// y = alpha*A*x + beta*y
template <int G>
__global__ void __launch_bounds__(TPB) k_spmv(Csr a, const double* __restrict__ x, double* y,
                                              double alpha, double beta) {
  const int lane = threadIdx.x % G;
  const int rpb = TPB / G;
  for (int64_t base = (int64_t)blockIdx.x * rpb; base < a.nrows; base += (int64_t)gridDim.x * rpb) {
    const int64_t row = base + threadIdx.x / G;
    const bool ok = row < a.nrows;
    const double s = row_dot<G>(a, (int)row, ok, lane, x);
    if (ok && lane == 0) y[row] = (beta == 0.0) ? alpha * s : fma(beta, y[row], alpha * s);
  }
}

// q = Λ x (bd/system.py:106-116) with optional x·q (the PCG curvature d·q):
//   top    = S_1 u ; top[:m] += S_i v
//   bottom = (S_i u[:m] + S_i v) + γ (M_H ∘ v)
template <int G>
__global__ void __launch_bounds__(TPB) k_lambda(Csr s1, Csr si, const double* __restrict__ x,
                                                double* __restrict__ q, const double* __restrict__ mh,
                                                double gamma, int n, int m, Ctl c, int with_dot) {
  if (inactive(c)) return;
  __shared__ double sm[32];
  const int lane = threadIdx.x % G;
  const int rpb = TPB / G;
  const double* u = x;
  const double* v = x + n;
  double acc = 0.0;
  for (int64_t base = (int64_t)blockIdx.x * rpb; base < n; base += (int64_t)gridDim.x * rpb) {
    const int row = (int)(base + threadIdx.x / G);
    const bool ok = row < n;
    double top = row_dot<G>(s1, row, ok, lane, u);
    if (base < m) {  // block-uniform: some row of this chunk is a heart row
      const bool okh = row < m;
      int b = 0, e = 0;
      if (okh) {
        b = si.rowptr[row];
        e = si.rowptr[row + 1];
      }
      double su = 0.0, sv = 0.0;
      for (int k = b + lane; k < e; k += G) {
        const double a = si.val[k];
        const int j = si.col[k];
        su = fma(a, __ldg(&u[j]), su);
        sv = fma(a, __ldg(&v[j]), sv);
      }
      su = group_sum<G>(su);
      sv = group_sum<G>(sv);
      if (okh) {
        top = __dadd_rn(top, sv);
        const double vi = v[row];
        const double bot = __dadd_rn(__dadd_rn(su, sv), __dmul_rn(gamma, __dmul_rn(mh[row], vi)));
        if (lane == 0) {
          q[n + row] = bot;
          acc = fma(vi, bot, acc);
        }
      }
    }
    if (ok && lane == 0) {
      q[row] = top;
      acc = fma(u[row], top, acc);
    }
  }
  if (with_dot) {
    double vv[1] = {block_sum(acc, sm)};
    reduce_tail<1>(c, vv, gridDim.x, blockIdx.x, C_LAMBDA, FIN_DQ, 0, -1, 0, sm);
  }
}

// r = b - q (warm start) or r = b; ||r||^2 and sum(r_u) (bd/krylov.py:74-85)
__global__ void __launch_bounds__(TPB) k_init_res(const double* b, const double* q, double* r,
                                                  int64_t n, int64_t nm, Ctl c) {
  if (inactive(c)) return;
  __shared__ double sm[32];
  double rr = 0.0, su = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nm;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double ri = q ? __dsub_rn(b[i], q[i]) : b[i];
    r[i] = ri;
    rr = fma(ri, ri, rr);
    if (i < n) su += ri;
  }
  double v[2] = {block_sum(rr, sm), 0.0};
  v[1] = block_sum(su, sm);
  reduce_tail<2>(c, v, gridDim.x, blockIdx.x, C_INITR, FIN_INIT_RES, 0, -1, n, sm);
}

// x += αd ; r -= αq ; ||r||^2 ; sum(r_u)   (bd/krylov.py:109-123)
__global__ void __launch_bounds__(TPB) k_update(double* x, double* r, const double* d,
                                                const double* q, int64_t n, int64_t nm, Ctl c) {
  if (inactive(c)) return;
  __shared__ double sm[32];
  const double alpha = c.sc[S_ALPHA];
  double rr = 0.0, su = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nm;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, d[i]));
    const double ri = __dsub_rn(r[i], __dmul_rn(alpha, q[i]));
    r[i] = ri;
    rr = fma(ri, ri, rr);
    if (i < n) su += ri;
  }
  double v[2] = {block_sum(rr, sm), 0.0};
  v[1] = block_sum(su, sm);
  reduce_tail<2>(c, v, gridDim.x, blockIdx.x, C_UPDATE, FIN_UPDATE, 0, -1, n, sm);
}

// ---- right-hand sides of the inner solves --------------------------------
// (src[i] or 0 past src_len) - shift: the mean-projected bulk input
// `y - y.mean()` of _bulk_inverse (bd/precond.py:289-290); perm for the
// fill-reducing ordering of the exact factor.
struct RhsVec {
  const double* src;
  int src_len;
  const double* shift;
  const int* perm;
  template <int G>
  __device__ __forceinline__ double eval(int row, int) const {
    if (row < 0) return 0.0;
    const int i = perm ? perm[row] : row;
    const double v = i < src_len ? src[i] : 0.0;
    return shift ? __dsub_rn(v, *shift) : v;
  }
};
// w_i = r_v[i] - (S_i t)[i] with t = (t_raw - mt) + mu1/beta formed on the
// fly: `rhs.v - stiff_intra @ t[:nh]` (bd/precond.py:307) fused with the
// recentring of the first bulk solve (:291-292).
struct RhsSchur {
  Csr si;
  const double* traw;
  const double* sc;
  const double* rv;
  const int* perm;
  template <int G>
  __device__ __forceinline__ double eval(int row, int lane) const {
    const int i = row < 0 ? -1 : (perm ? perm[row] : row);
    const double mt = sc[S_MT], c1 = sc[S_C1];
    int b = 0, e = 0;
    if (i >= 0) {
      b = si.rowptr[i];
      e = si.rowptr[i + 1];
    }
    double s = 0.0;
    for (int k = b + lane; k < e; k += G) {
      const double t = __dadd_rn(__dsub_rn(__ldg(&traw[si.col[k]]), mt), c1);
      s = fma(si.val[k], t, s);
    }
    s = group_sum<G>(s);
    return i >= 0 ? __dsub_rn(rv[i], s) : 0.0;
  }
};

// ---- sync-free triangular solves -----------------------------------------
// Rows are processed in a level-sorted task order; a group of G lanes owns a
// row and polls the entries it depends on until they stop reading as the
// sentinel.  Block ids are taken from an atomic counter so that any block
// that runs has all lower tasks already owned by running blocks (no
// deadlock).  LOWER: diagonal last in the row; else diagonal first.
struct Tri {
  int n;
  const int* rowptr;
  const int* col;
  const double* val;
  const int* tasks;
  int ntasks;
};

template <int G, bool LOWER, class Rhs>
__global__ void __launch_bounds__(TPB) k_trsv_fwd(Tri t, Rhs rhs, double* __restrict__ y, Ctl c,
                                                  int ctr_start, int ctr_done, int nvb) {
  if (inactive(c)) return;
  __shared__ int vb;
  if (threadIdx.x == 0) vb = (int)atomicAdd(&c.ctr[ctr_start], 1u);
  __syncthreads();
  const int lane = threadIdx.x % G;
  const int task = vb * (TPB / G) + threadIdx.x / G;
  const int row = task < t.ntasks ? t.tasks[task] : -1;
  int kb = 0, ke = 0;
  double diag = 1.0;
  if (row >= 0) {
    const int b = t.rowptr[row], e = t.rowptr[row + 1];
    kb = LOWER ? b : b + 1;
    ke = LOWER ? e - 1 : e;
    diag = LOWER ? t.val[e - 1] : t.val[b];
  }
  // the rhs first: its loads overlap the polling below
  const double bi = rhs.template eval<G>(row, lane);
  double s = 0.0;
  for (int k = kb + lane; k < ke; k += G) s = fma(t.val[k], spin_load(&y[t.col[k]]), s);
  s = group_sum<G>(s);
  if (row >= 0 && lane == 0) publish(&y[row], __ddiv_rn(__dsub_rn(bi, s), diag));
  // the last block resets the start counter for the next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned d = atomicAdd(&c.ctr[ctr_done], 1u);
    if (d == (unsigned)nvb - 1u) {
      c.ctr[ctr_start] = 0u;
      c.ctr[ctr_done] = 0u;
      __threadfence();
    }
  }
}

// Backward solve reading its right-hand side from the forward output yin
// (and resetting it to the sentinel: the forward buffer has no other
// reader), publishing into x (polled), optionally scattering through perm
// into out, and optionally reducing sum(out) for the mean that follows.
template <int G, bool LOWER>
__global__ void __launch_bounds__(TPB) k_trsv_bwd(Tri t, double* __restrict__ yin,
                                                  double* __restrict__ x, double* __restrict__ out,
                                                  const int* __restrict__ perm, Ctl c, int ctr_start,
                                                  int ctr_done, int nvb, int fin, int slot, int slot2,
                                                  int64_t nmean) {
  if (inactive(c)) return;
  __shared__ int vb;
  __shared__ double sm[32];
  if (threadIdx.x == 0) vb = (int)atomicAdd(&c.ctr[ctr_start], 1u);
  __syncthreads();
  const int lane = threadIdx.x % G;
  const int task = vb * (TPB / G) + threadIdx.x / G;
  const int row = task < t.ntasks ? t.tasks[task] : -1;
  int kb = 0, ke = 0;
  double diag = 1.0, bi = 0.0;
  if (row >= 0) {
    const int b = t.rowptr[row], e = t.rowptr[row + 1];
    kb = LOWER ? b : b + 1;
    ke = LOWER ? e - 1 : e;
    diag = LOWER ? t.val[e - 1] : t.val[b];
    if (lane == 0) bi = yin[row];  // only lane 0 reads: it also resets it
  }
  double s = 0.0;
  for (int k = kb + lane; k < ke; k += G) s = fma(t.val[k], spin_load(&x[t.col[k]]), s);
  s = group_sum<G>(s);
  double val = 0.0;
  if (row >= 0) {
    val = __ddiv_rn(__dsub_rn(bi, s), diag);
    if (lane == 0) {
      publish(&x[row], val);
      yin[row] = __longlong_as_double(SENTINEL);
      if (out) out[perm ? perm[row] : row] = val;
    }
  }
  if (fin >= 0) {
    double v[1] = {block_sum(lane == 0 ? val : 0.0, sm)};
    __shared__ int last_s;
    if (threadIdx.x == 0) {
      // the done-counter doubles as the reduction counter
      c.partials[vb] = v[0];
      __threadfence();
      const unsigned d = atomicAdd(&c.ctr[ctr_done], 1u);
      last_s = (d == (unsigned)nvb - 1u);
    }
    __syncthreads();
    const bool last = last_s != 0;
    if (last) {
      __threadfence();
      double tot[1];
      tot[0] = sum_partials(c.partials, nvb, 0, sm);
      if (threadIdx.x == 0) {
        finalize(c, fin, slot, slot2, tot, nmean);
        c.ctr[ctr_start] = 0u;
        c.ctr[ctr_done] = 0u;
        __threadfence();
      }
    }
  } else {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned d = atomicAdd(&c.ctr[ctr_done], 1u);
      if (d == (unsigned)nvb - 1u) {
        c.ctr[ctr_start] = 0u;
        c.ctr[ctr_done] = 0u;
        __threadfence();
      }
    }
  }
}

// Jacobi "solve": out_i = inv_i * rhs_i (bd/precond.py:231-232), with the
// same rhs functors and the optional mean reduction.
template <int G, class Rhs>
__global__ void __launch_bounds__(TPB) k_jacobi(int n, const double* __restrict__ inv, Rhs rhs,
                                                double* __restrict__ out, Ctl c, int ctr, int fin,
                                                int slot, int slot2, int64_t nmean) {
  if (inactive(c)) return;
  __shared__ double sm[32];
  const int lane = threadIdx.x % G;
  const int rpb = TPB / G;
  double acc = 0.0;
  for (int64_t base = (int64_t)blockIdx.x * rpb; base < n; base += (int64_t)gridDim.x * rpb) {
    const int64_t r = base + threadIdx.x / G;
    const bool ok = r < n;
    const double bi = rhs.template eval<G>(ok ? (int)r : -1, lane);
    if (ok && lane == 0) {
      const double z = __dmul_rn(inv[r], bi);
      out[r] = z;
      acc += z;
    }
  }
  if (fin >= 0) {
    double v[1] = {block_sum(acc, sm)};
    reduce_tail<1>(c, v, gridDim.x, blockIdx.x, ctr, fin, slot, slot2, nmean, sm);
  }
}

// corr = S_i s, sum(corr) -> mu2 (bd/precond.py:308-311: `correction[:nh] =
// stiff_intra @ s` then its mean inside _bulk_inverse).
template <int G>
__global__ void __launch_bounds__(TPB) k_corr(Csr si, const double* __restrict__ s,
                                              double* __restrict__ corr, Ctl c, int64_t n) {
  if (inactive(c)) return;
  __shared__ double sm[32];
  const int lane = threadIdx.x % G;
  const int rpb = TPB / G;
  double acc = 0.0;
  for (int64_t base = (int64_t)blockIdx.x * rpb; base < si.nrows; base += (int64_t)gridDim.x * rpb) {
    const int64_t r = base + threadIdx.x / G;
    const bool ok = r < si.nrows;
    const double v = row_dot<G>(si, (int)r, ok, lane, s);
    if (ok && lane == 0) {
      corr[r] = v;
      acc += v;
    }
  }
  double v[1] = {block_sum(acc, sm)};
  reduce_tail<1>(c, v, gridDim.x, blockIdx.x, C_CORR, FIN_MEAN, S_MU2, S_C2, n, sm);
}

// z_u = t - bulk(corr) with both recentrings applied on the fly
// (bd/precond.py:291-292, 311); optional sum(z_u) for the deflation mean.
__global__ void __launch_bounds__(TPB) k_combine(const double* __restrict__ traw,
                                                 const double* __restrict__ z2raw,
                                                 double* __restrict__ zu, int64_t n, Ctl c,
                                                 int with_sum) {
  if (inactive(c)) return;
  __shared__ double sm[32];
  const double* sc = c.sc;
  const double mt = sc[S_MT], c1 = sc[S_C1], m2 = sc[S_M2], c2 = sc[S_C2];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double t = __dadd_rn(__dsub_rn(traw[i], mt), c1);
    const double b = __dadd_rn(__dsub_rn(z2raw[i], m2), c2);
    const double z = __dsub_rn(t, b);
    zu[i] = z;
    acc += z;
  }
  if (with_sum) {
    double v[1] = {block_sum(acc, sm)};
    reduce_tail<1>(c, v, gridDim.x, blockIdx.x, C_COMBINE, FIN_MEAN, S_MZ, -1, n, sm);
  }
}

// rho = r·z with z_u deflated on the fly (`_deflate`, bd/krylov.py:41-43;
// `r.dot(z)`, :96 / :126)
__global__ void __launch_bounds__(TPB) k_rho(const double* __restrict__ r, const double* __restrict__ z,
                                             int64_t n, int64_t nm, Ctl c) {
  if (inactive(c)) return;
  __shared__ double sm[32];
  const double mz = c.sc[S_MZ];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nm;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double zi = i < n ? __dsub_rn(z[i], mz) : z[i];
    acc = fma(r[i], zi, acc);
  }
  double v[1] = {block_sum(acc, sm)};
  reduce_tail<1>(c, v, gridDim.x, blockIdx.x, C_RHO, FIN_RHO, 0, -1, 0, sm);
}

// d = z_deflated + beta d (bd/krylov.py:98, 130-131); runs after the
// max_iter stop so the last preconditioned direction is formed as in the
// reference loop.
__global__ void __launch_bounds__(TPB) k_dupdate(const double* __restrict__ z, double* __restrict__ d,
                                                 int64_t n, int64_t nm, Ctl c) {
  if (inactive(c, true)) return;
  const double mz = c.sc[S_MZ], beta = c.sc[S_BETA];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nm;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double zi = i < n ? __dsub_rn(z[i], mz) : z[i];
    d[i] = __dadd_rn(zi, __dmul_rn(beta, d[i]));
  }
}

// y = x with u shifted by the mass-weighted mean (bd/system.py:138-146);
// zero when the rhs was zero.
__global__ void k_normalize(const double* __restrict__ x, double* __restrict__ y, int64_t n,
                            int64_t nm, const double* sc, const int* fl) {
  const bool zero = fl && fl[F_ZERO];
  const double a = sc[S_WMEAN];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nm;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = zero ? 0.0 : (i < n ? __dsub_rn(x[i], a) : x[i]);
}

// ---- membrane (bd/ionic.py:45-68, 124-134; bd/system.py:118-136) -------
__global__ void k_membrane_rhs(int64_t n, int64_t m, const double* __restrict__ v,
                               const double* __restrict__ w, const uint64_t* __restrict__ mask,
                               uint64_t active, double amp, double chi, double gamma,
                               const double* __restrict__ mh, double v_rest, double v_span,
                               double tau_in, double tau_out, double c_m, double* __restrict__ rhs,
                               double* __restrict__ ion_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n + m;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n) {
      rhs[i] = 0.0;
      continue;
    }
    const int64_t k = i - n;
    const double vk = v[k];
    const double u = __ddiv_rn(__dsub_rn(vk, v_rest), v_span);
    // rate = w*u*u*(1-u)/tau_in - u/tau_out ; ion = -c_m*v_span*rate
    const double a = __dmul_rn(__dmul_rn(__dmul_rn(w[k], u), u), __dsub_rn(1.0, u));
    const double rate = __dsub_rn(__ddiv_rn(a, tau_in), __ddiv_rn(u, tau_out));
    const double ion = __dmul_rn(__dmul_rn(-c_m, v_span), rate);
    const double stim = (mask && (mask[k] & active)) ? amp : 0.0;
    // load = gamma*v - chi*(ion - stim) ; rhs_v = mh*load
    const double load = __dsub_rn(__dmul_rn(gamma, vk), __dmul_rn(chi, __dsub_rn(ion, stim)));
    rhs[i] = __dmul_rn(mh[k], load);
    if (ion_out) ion_out[k] = ion;
  }
}

__global__ void k_membrane_gate(int64_t m, const double* __restrict__ v, const double* __restrict__ w,
                                double dt, double v_rest, double v_span, double tau_open,
                                double tau_close, double u_gate, double* __restrict__ w_new) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double u = __ddiv_rn(__dsub_rn(v[k], v_rest), v_span);
    const double wk = w[k];
    const double rate = (u < u_gate) ? __ddiv_rn(__dsub_rn(1.0, wk), tau_open)
                                     : __ddiv_rn(-wk, tau_close);
    double out = __dadd_rn(wk, __dmul_rn(dt, rate));
    out = out < 0.0 ? 0.0 : (out > 1.0 ? 1.0 : out);
    w_new[k] = out;
  }
}

}  // namespace dev
}  // namespace bd
