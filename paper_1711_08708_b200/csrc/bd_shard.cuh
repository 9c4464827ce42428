// ---- sharded (multi-GPU) PCG iteration: the vector work of one rank --------------
// The deflated PCG of bd/krylov.py:46-140 with the block-LU preconditioner of
// bd/precond.py:281-312 on a rank's owned rows; the host (distributed.py)
// interleaves these kernels with the halo exchanges and the four all-reduces
// of an iteration (<= 4 packed reductions):
//   red[0]        d·q                                   (after Λ)
//   red[1], red[2] ‖r‖², Σ r_u                          (after the x/r update)
//   red[3]        Σ (S_i s)                             (mean of the S_i correction)
//   red[4..6]     Σ w, r_u·w, r_v·s with w = z1 − z2     (r·z of the deflated z)
// The recentrings of _bulk_inverse (mean of each inner output, precond.py:
// 289-291) and the deflation (krylov.py:41-43) collapse: with t = z1 −
// mean(z1) + μ1/β and u = t − (z2 − mean(z2) + μ2/β), the deflated
// z_u = u − mean(u) = w − mean(w), and S_i t = S_i z1 because S_i 𝟙 = 0.
// Every partial sum is deterministic (fixed-order block partials, last block
// sums them in block order); every scalar lives in device memory; after
// convergence / breakdown the F_DONE flag turns every kernel (the inner
// triangular passes included) into a no-op, so a captured iteration can be
// replayed past the end.
#pragma once

namespace bd {
namespace dev {

// shard scalar slots
enum ShSlot {
  SH_RHO = 0, SH_ALPHA, SH_NB, SH_MU1, SH_MU2, SH_BETA, SH_MEANW, SH_TOL, SH_CURV, SH_REL,
  SH_NSLOTS = 16
};
// shard integer slots (beside the dev::Ctl flags F_DONE / F_STOP used by the
// inner solves)
enum ShInt { SHI_ITERS = 0, SHI_NRES, SHI_NPREC, SHI_CONV, SHI_BAD, SHI_ZERO, SHI_MAXIT,
             SHI_MAXITER, SHI_NINT = 8 };
constexpr int SH_RED = 16;       // reduction slots
constexpr int SH_GRID = 592;     // blocks of the partial-sum kernels (4 per SM)

// K simultaneous block sums (fixed tree), then the last block adds the
// per-block partials in block order.  part: SH_GRID*K doubles; ctr: counter.
template <int K>
__device__ __forceinline__ void sh_reduce(double (&v)[K], double* part, unsigned* ctr,
                                          double* out) {
  __shared__ double sm[K][TPB / 32];
  __shared__ bool last;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double x = warp_sum(v[k]);
    if (l == 0) sm[k][w] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = 0.0;
      for (int q = 0; q < TPB / 32; ++q) s += sm[k][q];
      part[(size_t)blockIdx.x * K + k] = s;
    }
    __threadfence();
    last = atomicAdd(ctr, 1u) == gridDim.x - 1u;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = 0.0;
      for (unsigned b = 0; b < gridDim.x; ++b) s += part[(size_t)b * K + k];
      out[k] = s;
    }
    *ctr = 0u;
  }
}

__device__ __forceinline__ bool sh_done(const int* fl) {
  return *(const volatile int*)(fl + F_DONE) != 0;
}

// q_u[:m] += q_v  (the S_i v term of the top block, bd/system.py:112)
__global__ void __launch_bounds__(TPB) k_sh_lam_add(int64_t m, double* qu, const double* qv,
                                                    const int* fl, int use_flags) {
  if (use_flags && sh_done(fl)) return;
  for (int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x; i < m; i += (int64_t)gridDim.x * TPB)
    qu[i] += qv[i];
}

// q_v += γ (M_H ∘ v_v); red = v·q over the whole local block vector
__global__ void __launch_bounds__(TPB) k_sh_lam_fin(int64_t n, int64_t nm, const double* v,
                                                    double* q, const double* mh, double gamma,
                                                    double* part, unsigned* ctr, double* red,
                                                    const int* fl, int use_flags) {
  if (use_flags && sh_done(fl)) return;
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x; i < nm; i += (int64_t)gridDim.x * TPB) {
    double qi = q[i];
    if (i >= n) {
      qi += gamma * (mh[i - n] * v[i]);
      q[i] = qi;
    }
    acc[0] = fma(v[i], qi, acc[0]);
  }
  sh_reduce<1>(acc, part, ctr, red);
}

// The whole local Λ in one pass over the ELL copies of S1 (n rows, columns
// [owned | ghosts]) and S_i (m rows, columns [owned heart | heart ghosts]),
// with the reference's association (bd/system.py:111-115):
//   q_u = S1 u (+ S_i v on heart rows),  q_v = (S_i u_H + S_i v) + γ (M_H ∘ v);
// red = v·q (d·q of the iteration).  u = x[0..n), v = x[n..n+m); ug: all
// ghosts of u (the heart ones first), vg: heart ghosts of v.
__global__ void __launch_bounds__(TPB) k_sh_lambda_ell(
    int64_t n, int64_t m, int w1, const int* __restrict__ c1, const double* __restrict__ a1,
    int w2, const int* __restrict__ c2, const double* __restrict__ a2, const double* __restrict__ x,
    const double* __restrict__ ug, const double* __restrict__ vg, double* __restrict__ q,
    const double* __restrict__ mh, double gamma, double* part, unsigned* ctr, double* red,
    const int* fl, int use_flags) {
  if (use_flags && sh_done(fl)) return;
  const double* v = x + n;
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TPB) {
    double su = 0.0;
    for (int e0 = 0; e0 < w1; e0 += 8) {  // 8 entries in flight (as k_spmv_ell)
      int cl[8];
      double a[8], xv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        cl[e] = __ldcs(&c1[(int64_t)(e0 + e) * n + i]);  // matrix entries: streaming loads
        a[e] = __ldcs(&a1[(int64_t)(e0 + e) * n + i]);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) xv[e] = cl[e] < 0 ? 0.0 : (cl[e] < n ? __ldg(&x[cl[e]]) : __ldg(&ug[cl[e] - n]));
#pragma unroll
      for (int e = 0; e < 8; ++e) su = fma(a[e], xv[e], su);
    }
    if (i < m) {
      double sv = 0.0, sh = 0.0;
      for (int e0 = 0; e0 < w2; e0 += 8) {
        int cl[8];
        double a[8], xv[8], xu[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          cl[e] = __ldcs(&c2[(int64_t)(e0 + e) * m + i]);
          a[e] = __ldcs(&a2[(int64_t)(e0 + e) * m + i]);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int c = cl[e];
          xv[e] = c < 0 ? 0.0 : (c < m ? __ldg(&v[c]) : __ldg(&vg[c - m]));
          xu[e] = c < 0 ? 0.0 : (c < m ? __ldg(&x[c]) : __ldg(&ug[c - m]));
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          sv = fma(a[e], xv[e], sv);
          sh = fma(a[e], xu[e], sh);
        }
      }
      const double qu = su + sv;
      const double qv = (sh + sv) + gamma * (mh[i] * v[i]);
      q[i] = qu;
      q[n + i] = qv;
      acc[0] = fma(x[i], qu, acc[0]);
      acc[0] = fma(v[i], qv, acc[0]);
    } else {
      q[i] = su;
      acc[0] = fma(x[i], su, acc[0]);
    }
  }
  sh_reduce<1>(acc, part, ctr, red);
}

// corr[0..m) = S_i [s | sg] (ELL, 8 entries in flight) and red = Σ corr
__global__ void __launch_bounds__(TPB) k_sh_corr_ell(int64_t m, int w, const int* __restrict__ c2,
                                                     const double* __restrict__ a2,
                                                     const double* __restrict__ s,
                                                     const double* __restrict__ sg,
                                                     double* __restrict__ corr, double* part,
                                                     unsigned* ctr, double* red, const int* fl,
                                                     double* __restrict__ fill = nullptr,
                                                     int64_t nfill = 0) {
  if (sh_done(fl)) return;
  // optional: sentinel reset of the polled forward output of the bulk solve that follows
  for (int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x; i < nfill; i += (int64_t)gridDim.x * TPB)
    fill[i] = __longlong_as_double(SENTINEL);
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x; i < m; i += (int64_t)gridDim.x * TPB) {
    double v = 0.0;
    for (int e0 = 0; e0 < w; e0 += 8) {
      int cl[8];
      double a[8], xv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        cl[e] = __ldcs(&c2[(int64_t)(e0 + e) * m + i]);
        a[e] = __ldcs(&a2[(int64_t)(e0 + e) * m + i]);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) xv[e] = cl[e] < 0 ? 0.0 : (cl[e] < m ? __ldg(&s[cl[e]]) : __ldg(&sg[cl[e] - m]));
#pragma unroll
      for (int e = 0; e < 8; ++e) v = fma(a[e], xv[e], v);
    }
    corr[i] = v;
    acc[0] += v;
  }
  sh_reduce<1>(acc, part, ctr, red);
}

// r = b − q (x0 given) or r = b; red[1] = ‖r‖², red[2] = Σ r_u, red[7] = ‖b‖²;
// rhs_s = r_v (the Schur right-hand side buffer starts as r_v)
__global__ void __launch_bounds__(TPB) k_sh_init(int64_t n, int64_t nm, const double* b,
                                                 const double* q, double* r, double* rhs_s,
                                                 double* part, unsigned* ctr, double* red3) {
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x; i < nm; i += (int64_t)gridDim.x * TPB) {
    const double bi = b[i];
    const double ri = q ? bi - q[i] : bi;
    r[i] = ri;
    if (rhs_s && i >= n) rhs_s[i - n] = ri;
    acc[0] = fma(ri, ri, acc[0]);
    if (i < n) acc[1] += ri;
    acc[2] = fma(bi, bi, acc[2]);
  }
  sh_reduce<3>(acc, part, ctr, red3);
}

// α = ρ / d·q, breakdown on d·q <= 0 or non-finite (bd/krylov.py:101-108)
__global__ void k_sh_alpha(double* sc, int* fl, int* si, const double* red) {
  if (sh_done(fl)) return;
  const double dq = red[0];
  if (!(isfinite(dq) && dq > 0.0)) {
    si[SHI_BAD] = 1;
    sc[SH_CURV] = dq;
    sc[SH_ALPHA] = 0.0;
    fl[F_DONE] = 1;
    return;
  }
  sc[SH_ALPHA] = sc[SH_RHO] / dq;
  si[SHI_ITERS] += 1;
}

// x += α d, r −= α q; red[1] = ‖r‖², red[2] = Σ r_u; rhs_s = r_v
__global__ void __launch_bounds__(TPB) k_sh_update(int64_t n, int64_t nm, double* x, double* r,
                                                   const double* d, const double* q,
                                                   double* rhs_s, const double* sc, double* part,
                                                   unsigned* ctr, double* red2, const int* fl,
                                                   double* __restrict__ fill = nullptr,
                                                   int64_t nfill = 0) {
  if (sh_done(fl)) return;
  const double a = sc[SH_ALPHA];
  double acc[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x; i < nm; i += (int64_t)gridDim.x * TPB) {
    if (i < nfill) fill[i] = __longlong_as_double(SENTINEL);  // the next bulk solve's polled output
    x[i] = fma(a, d[i], x[i]);
    const double ri = fma(-a, q[i], r[i]);
    r[i] = ri;
    if (rhs_s && i >= n) rhs_s[i - n] = ri;
    acc[0] = fma(ri, ri, acc[0]);
    if (i < n) acc[1] += ri;
  }
  sh_reduce<2>(acc, part, ctr, red2);
}

// convergence test on the recursive residual (bd/krylov.py:112-123) and μ1;
// initial != 0: the residual of the starting guess (‖b‖ from red[7])
__global__ void k_sh_check(double* sc, int* fl, int* si, const double* red, double* res_hist,
                           int hist_cap, int64_t n_global, int initial) {
  if (sh_done(fl)) return;
  if (initial) {
    const double nb = sqrt(red[7]);
    sc[SH_NB] = nb;
    if (nb == 0.0) {  // zero right-hand side: x = 0, no iteration (krylov.py:69-72)
      si[SHI_ZERO] = 1;
      si[SHI_CONV] = 1;
      res_hist[0] = 0.0;
      si[SHI_NRES] = 1;
      fl[F_DONE] = 1;
      return;
    }
  }
  const double rel = sqrt(red[1]) / sc[SH_NB];
  sc[SH_REL] = rel;
  const int k = si[SHI_NRES];
  if (k < hist_cap) res_hist[k] = rel;
  si[SHI_NRES] = k + 1;
  if (!isfinite(rel)) {
    si[SHI_BAD] = 1;
    sc[SH_CURV] = rel;
    fl[F_DONE] = 1;
    return;
  }
  if (rel <= sc[SH_TOL]) {
    si[SHI_CONV] = 1;
    fl[F_DONE] = 1;
    return;
  }
  if (!initial && si[SHI_ITERS] >= si[SHI_MAXITER]) {
    si[SHI_MAXIT] = 1;
    fl[F_DONE] = 1;
    return;
  }
  sc[SH_MU1] = red[2] / (double)n_global;
}

// μ2 = Σ(S_i s) / n_global (the mean of pad(S_i s), precond.py:289)
__global__ void k_sh_mu2(double* sc, const int* fl, const double* red, int64_t n_global) {
  if (sh_done(fl)) return;
  sc[SH_MU2] = red[3] / (double)n_global;
}

// red = Σ x[0..m)
__global__ void __launch_bounds__(TPB) k_sh_sum(int64_t m, const double* x, double* part,
                                                unsigned* ctr, double* red, const int* fl) {
  if (sh_done(fl)) return;
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x; i < m; i += (int64_t)gridDim.x * TPB)
    acc[0] += x[i];
  sh_reduce<1>(acc, part, ctr, red);
}

// w = z1 − z2 (in z1); red[4..6] = Σ w, r_u·w, r_v·s
__global__ void __launch_bounds__(TPB) k_sh_combine(int64_t n, int64_t m, double* z1,
                                                    const double* z2, const double* r,
                                                    const double* s, double* part, unsigned* ctr,
                                                    double* red3, const int* fl) {
  if (sh_done(fl)) return;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x; i < n + m;
       i += (int64_t)gridDim.x * TPB) {
    if (i < n) {
      const double w = z1[i] - z2[i];
      z1[i] = w;
      acc[0] += w;
      acc[1] = fma(r[i], w, acc[1]);
    } else {
      acc[2] = fma(r[i], s[i - n], acc[2]);
    }
  }
  sh_reduce<3>(acc, part, ctr, red3);
}

// ρ_next = r·z with z_u = w − mean(w): r_u·w − mean(w) Σr_u + r_v·s; β
__global__ void k_sh_finish(double* sc, const int* fl, int* si, const double* red,
                            double* prec_hist, int hist_cap, int64_t n_global, int initial) {
  if (sh_done(fl)) return;
  const double mw = red[4] / (double)n_global;
  const double rho = red[5] - mw * red[2] + red[6];
  sc[SH_MEANW] = mw;
  const int k = si[SHI_NPREC];
  if (k < hist_cap) prec_hist[k] = rho;
  si[SHI_NPREC] = k + 1;
  sc[SH_BETA] = initial ? 0.0 : rho / sc[SH_RHO];
  sc[SH_RHO] = rho;
}

// d_u = (w − mean w) + β d_u ; d_v = s + β d_v
__global__ void __launch_bounds__(TPB) k_sh_dupdate(int64_t n, int64_t m, const double* w,
                                                    const double* s, double* d, const double* sc,
                                                    const int* fl) {
  if (sh_done(fl)) return;
  const double be = sc[SH_BETA], mw = sc[SH_MEANW];
  for (int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x; i < n + m;
       i += (int64_t)gridDim.x * TPB) {
    const double z = i < n ? w[i] - mw : s[i - n];
    d[i] = fma(be, d[i], z);
  }
}

// y = alpha * A [x ; x2] + beta * y on the CSR arrays, one thread per row
// (bd_spmv_split for blocks without an ELL copy: small or irregular local
// blocks of a partition)
__global__ void __launch_bounds__(TPB) k_spmv_csr_split(int64_t nrows, const int* __restrict__ rp,
                                                        const int* __restrict__ col,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ x,
                                                        const double* __restrict__ x2, int nsplit,
                                                        double* y, double alpha, double beta) {
  for (int64_t r = blockIdx.x * (int64_t)TPB + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * TPB) {
    double s = 0.0;
    for (int q = rp[r]; q < rp[r + 1]; ++q) {
      const int c = col[q];
      s = fma(val[q], c < nsplit ? x[c] : x2[c - nsplit], s);
    }
    y[r] = (beta == 0.0) ? alpha * s : fma(beta, y[r], alpha * s);
  }
}

// dst[i] = src[idx[i]] (halo packing)
__global__ void __launch_bounds__(TPB) k_sh_gather(int64_t k, const int64_t* idx, const double* src,
                                                   double* dst) {
  for (int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x; i < k; i += (int64_t)gridDim.x * TPB)
    dst[i] = src[idx[i]];
}

// out = x with u − alpha, alpha = red[8] / msum (normalize, bd/system.py:138-146)
__global__ void __launch_bounds__(TPB) k_sh_normalize(int64_t n, int64_t nm, const double* x,
                                                      double* out, const double* red, double msum,
                                                      const int* si) {
  const double a = si[SHI_ZERO] ? 0.0 : red[8] / msum;
  for (int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x; i < nm; i += (int64_t)gridDim.x * TPB)
    out[i] = si[SHI_ZERO] ? 0.0 : (i < n ? x[i] - a : x[i]);
}

// red[8] = Σ mass ∘ x_u
__global__ void __launch_bounds__(TPB) k_sh_wmean(int64_t n, const double* mass, const double* x,
                                                  double* part, unsigned* ctr, double* red) {
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * TPB)
    acc[0] = fma(mass[i], x[i], acc[0]);
  sh_reduce<1>(acc, part, ctr, red);
}

}  // namespace dev
}  // namespace bd
