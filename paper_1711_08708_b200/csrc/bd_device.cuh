// Device kernels of the bidomain PCG hot path (sm_100a, fp64, HBM-bound).
//
// Every reduction is deterministic: per-block partials land in a fixed slot
// and the last block to finish sums them in a fixed order (no fp64 atomics),
// so two identical runs are bitwise identical (tests/test_simulate.py:147-151
// in the reference).  Kernels that belong to the PCG loop first check the
// control flags and return when the solve is finished, so an iteration can be
// enqueued (or replayed from a CUDA graph) without a host round trip.
#pragma once
#include <cooperative_groups.h>
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
  FIN_RHO3,         // rho of the deflated z from (Σz_u, r_u·z_u, r_v·z_v); beta, history,
                    // max_iter stop (bd/krylov.py:95-97, :125-131)
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
    case FIN_RHO3: {
      // r·(z − mean(z_u) on u) = r_u·z_u − mean(z_u) Σr_u + r_v·z_v, with
      // Σr_u = n mu1 from the update's tail; the deflation shift goes to S_MZ
      const double mz = tot[0] / (double)n;
      sc[S_MZ] = mz;
      const double rho_next = tot[1] - mz * (sc[S_MU1] * (double)n) + tot[2];
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

// Generic SpMV on the entry-major ELL copy of a CSR matrix with short,
// near-uniform rows (P1 stencils): one thread per row, W entries in chunks of
// 8 with all loads of a chunk issued before the FMAs; padding entries have
// column -1.  Row sums run in column order, like the CSR kernels.
// x split in two arrays (sharded ranks: owned entries, then the ghost halo):
// column c reads x[c] for c < nsplit and x2[c - nsplit] otherwise.
template <int W>
__global__ void __launch_bounds__(TPB) k_spmv_ell(int64_t nrows, const int* __restrict__ col,
                                                  const double* __restrict__ val,
                                                  const double* __restrict__ x, double* y,
                                                  double alpha, double beta,
                                                  const double* __restrict__ x2 = nullptr,
                                                  int nsplit = 0x7fffffff) {
  for (int64_t r = blockIdx.x * (int64_t)TPB + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * TPB) {
    double s = 0.0;
#pragma unroll
    for (int e0 = 0; e0 < W; e0 += 8) {
      int cl[8];
      double a[8], xv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        cl[e] = __ldg(&col[(int64_t)(e0 + e) * nrows + r]);
        a[e] = __ldg(&val[(int64_t)(e0 + e) * nrows + r]);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e)
        xv[e] = cl[e] < 0 ? 0.0 : (cl[e] < nsplit ? __ldg(&x[cl[e]]) : __ldg(&x2[cl[e] - nsplit]));
#pragma unroll
      for (int e = 0; e < 8; ++e) s = fma(a[e], xv[e], s);
    }
    y[r] = (beta == 0.0) ? alpha * s : fma(beta, y[r], alpha * s);
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

// Λ with K entries per lane: the S_1 and S_i entries of a row are loaded, and
// their operands gathered, before any reduction (two memory round trips per
// row instead of four).  Rows longer than G*K fall back to a loop.
// ---- Λ on an entry-major ELL copy of the blocks ------------------------------
// One thread per row; S_1 and S_i share the column array (pattern(S_i) is a
// subset of the heart rows of pattern(S_1); absent / padding entries are 0).
// Entry e of row r sits at [e * rows + r], so every load of a warp is one
// contiguous 128/256-byte request, and all of a row's loads are independent.
struct LamEll {
  const int* col;     // [W][n]  (padding: the row itself)
  const double* v1;   // [W][n]  S_1
  const double* v2;   // [W][m]  S_i on heart rows
};

__global__ void k_build_lambda_ell(Csr s1, Csr si, int n, int m, int W, int* __restrict__ col,
                                   double* __restrict__ v1, double* __restrict__ v2,
                                   int* __restrict__ bad) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  const int b1 = s1.rowptr[row], e1 = s1.rowptr[row + 1];
  if (e1 - b1 > W) {
    atomicExch(bad, 1);
    return;
  }
  int b2 = 0, e2 = 0;
  if (row < m) {
    b2 = si.rowptr[row];
    e2 = si.rowptr[row + 1];
  }
  int j = b2;
  for (int e = 0; e < W; ++e) {
    const int k = b1 + e;
    const int cc = k < e1 ? s1.col[k] : row;
    col[(size_t)e * n + row] = cc;
    v1[(size_t)e * n + row] = k < e1 ? s1.val[k] : 0.0;
    if (row < m) {
      double a = 0.0;
      if (k < e1 && j < e2 && si.col[j] == cc) a = si.val[j++];
      v2[(size_t)e * m + row] = a;
    }
  }
  if (j != e2) atomicExch(bad, 1);  // an S_i entry outside the S_1 pattern (or unsorted)
}

template <int W>
__global__ void __launch_bounds__(TPB) k_lambda_ell(LamEll L, const double* __restrict__ x,
                                                    double* __restrict__ q,
                                                    const double* __restrict__ mh, double gamma,
                                                    int n, int m, Ctl c, int with_dot) {
  if (inactive(c)) return;
  __shared__ double sm[32];
  const double* __restrict__ u = x;
  const double* __restrict__ v = x + n;
  double acc = 0.0;
  for (int row = blockIdx.x * TPB + threadIdx.x; row < n; row += gridDim.x * TPB) {
    const bool h = row < m;
    double s_top = 0.0, su = 0.0, sv = 0.0;
#pragma unroll
    for (int e0 = 0; e0 < W; e0 += 8) {
      int cl[8];
      double a1[8], a2[8], xu[8], xv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        // matrix entries are read once per apply: streaming (evict-first) loads keep the
        // vectors of the neighbouring kernels in L2
        cl[e] = __ldcs(&L.col[(size_t)(e0 + e) * n + row]);
        a1[e] = __ldcs(&L.v1[(size_t)(e0 + e) * n + row]);
        a2[e] = h ? __ldcs(&L.v2[(size_t)(e0 + e) * m + row]) : 0.0;
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        xu[e] = __ldg(&u[cl[e]]);
        xv[e] = (h && cl[e] < m) ? __ldg(&v[cl[e]]) : 0.0;
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        s_top = fma(a1[e], xu[e], s_top);
        su = fma(a2[e], xu[e], su);
        sv = fma(a2[e], xv[e], sv);
      }
    }
    double top = s_top;
    if (h) {
      top = __dadd_rn(top, sv);
      const double vi = v[row];
      const double bot = __dadd_rn(__dadd_rn(su, sv), __dmul_rn(gamma, __dmul_rn(mh[row], vi)));
      q[n + row] = bot;
      acc = fma(vi, bot, acc);
    }
    q[row] = top;
    acc = fma(u[row], top, acc);
  }
  if (with_dot) {
    double vv[1] = {block_sum(acc, sm)};
    reduce_tail<1>(c, vv, gridDim.x, blockIdx.x, C_LAMBDA, FIN_DQ, 0, -1, 0, sm);
  }
}

template <int G, int K>
__global__ void __launch_bounds__(TPB) k_lambda2(Csr s1, Csr si, const double* __restrict__ x,
                                                 double* __restrict__ q,
                                                 const double* __restrict__ mh, double gamma,
                                                 int n, int m, Ctl c, int with_dot) {
  if (inactive(c)) return;
  __shared__ double sm[32];
  const int lane = threadIdx.x % G;
  const int rpb = TPB / G;
  const double* __restrict__ u = x;
  const double* __restrict__ v = x + n;
  double acc = 0.0;
  for (int64_t base = (int64_t)blockIdx.x * rpb; base < n; base += (int64_t)gridDim.x * rpb) {
    const int row = (int)(base + threadIdx.x / G);
    const bool ok = row < n, okh = row < m;
    int b1 = 0, e1 = 0, b2 = 0, e2 = 0;
    if (ok) {
      b1 = s1.rowptr[row];
      e1 = s1.rowptr[row + 1];
    }
    if (okh) {
      b2 = si.rowptr[row];
      e2 = si.rowptr[row + 1];
    }
    double a1[K], a2[K], x1[K], x2u[K], x2v[K];
    int c1[K], c2[K];
#pragma unroll
    for (int t = 0; t < K; ++t) {
      const int k1 = b1 + lane + t * G, k2 = b2 + lane + t * G;
      c1[t] = k1 < e1 ? s1.col[k1] : -1;
      a1[t] = k1 < e1 ? s1.val[k1] : 0.0;
      c2[t] = k2 < e2 ? si.col[k2] : -1;
      a2[t] = k2 < e2 ? si.val[k2] : 0.0;
    }
#pragma unroll
    for (int t = 0; t < K; ++t) {
      x1[t] = c1[t] >= 0 ? __ldg(&u[c1[t]]) : 0.0;
      x2u[t] = c2[t] >= 0 ? __ldg(&u[c2[t]]) : 0.0;
      x2v[t] = c2[t] >= 0 ? __ldg(&v[c2[t]]) : 0.0;
    }
    double s_top = 0.0, su = 0.0, sv = 0.0;
#pragma unroll
    for (int t = 0; t < K; ++t) {
      s_top = fma(a1[t], x1[t], s_top);
      su = fma(a2[t], x2u[t], su);
      sv = fma(a2[t], x2v[t], sv);
    }
    for (int k1 = b1 + lane + K * G; k1 < e1; k1 += G) s_top = fma(s1.val[k1], __ldg(&u[s1.col[k1]]), s_top);
    for (int k2 = b2 + lane + K * G; k2 < e2; k2 += G) {
      const double a = si.val[k2];
      const int j = si.col[k2];
      su = fma(a, __ldg(&u[j]), su);
      sv = fma(a, __ldg(&v[j]), sv);
    }
    s_top = group_sum<G>(s_top);
    if (base < m) {  // block-uniform
      su = group_sum<G>(su);
      sv = group_sum<G>(sv);
    }
    if (lane == 0 && ok) {
      double top = s_top;
      if (okh) {
        top = __dadd_rn(top, sv);
        const double vi = v[row];
        const double bot = __dadd_rn(__dadd_rn(su, sv), __dmul_rn(gamma, __dmul_rn(mh[row], vi)));
        q[n + row] = bot;
        acc = fma(vi, bot, acc);
      }
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
// `fill` (optional): the polled forward output of the bulk inner solve that
// follows, reset to the sentinel in the same pass (saves that solve's k_fill
// launch; the lines are still L2-resident when the pass polls them).
__global__ void __launch_bounds__(TPB) k_update(double* x, double* r, const double* d,
                                                const double* q, int64_t n, int64_t nm, Ctl c,
                                                double* __restrict__ fill = nullptr,
                                                int64_t nfill = 0) {
  if (inactive(c)) return;
  __shared__ double sm[32];
  const double alpha = c.sc[S_ALPHA];
  double rr = 0.0, su = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nm;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nfill) fill[i] = __longlong_as_double(SENTINEL);
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
  static constexpr bool kScalar = true;
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
  // two-phase form (k_trsv_rpipe): the load goes out early and nothing uses it
  // until the tile's inputs have landed, so the in-order warp does not stall on it
  __device__ __forceinline__ double pass_const() const { return shift ? *shift : 0.0; }
  __device__ __forceinline__ double load(int row) const {
    if (row < 0) return 0.0;
    const int i = perm ? perm[row] : row;
    return i < src_len ? src[i] : 0.0;
  }
  __device__ __forceinline__ double finish(double v, double sh) const {
    return shift ? __dsub_rn(v, sh) : v;
  }
};
// w_i = r_v[i] - (S_i t)[i] with t = (t_raw - mt) + mu1/beta formed on the
// fly: `rhs.v - stiff_intra @ t[:nh]` (bd/precond.py:307) fused with the
// recentring of the first bulk solve (:291-292).
struct RhsSchur {
  static constexpr bool kScalar = false;
  Csr si;
  const double* traw;
  const double* sc;
  const double* rv;
  const int* perm;
  // optional: the entry-major ELL copy of S_i (LamEll::col / v2), for the streaming
  // pre-evaluation k_schur_rhs_ell (ell_w = 0: none)
  const int* ell_col = nullptr;
  const double* ell_v2 = nullptr;
  int ell_w = 0, ell_n = 0;
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
#pragma unroll 4
    for (int k = b + lane; k < e; k += G) {
      const double t = __dadd_rn(__dsub_rn(__ldg(&traw[si.col[k]]), mt), c1);
      s = fma(si.val[k], t, s);
    }
    s = group_sum<G>(s);
    return i >= 0 ? __dsub_rn(rv[i], s) : 0.0;
  }
};


}  // namespace dev
}  // namespace bd

#include "bd_trsv.cuh"
#include "bd_vec.cuh"
#include "bd_shard.cuh"
