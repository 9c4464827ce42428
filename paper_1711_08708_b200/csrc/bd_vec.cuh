// Inner Jacobi application, P^-1 combination, PCG vector kernels, membrane
// and time-loop bookkeeping kernels.  Included by bd_device.cuh.
#pragma once

namespace bd {
namespace dev {

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

// Dense explicit inverse of a small exact inner (n <= BD_EXACT_DENSE_MAX):
// the right-hand side is evaluated into y (the inner's permuted order, as the
// Rhs functors index it), then z = X y with X = (P A P^T)^{-1} row-major, one
// warp per row, lane-strided dot + fixed butterfly (deterministic).  HBM/L2
// streaming instead of the latency-bound supernodal passes of a tiny factor.
template <int G, class Rhs>
__global__ void __launch_bounds__(TPB) k_rhs_eval(int n, Rhs rhs, double* __restrict__ y, Ctl c) {
  if (inactive(c)) return;
  const int lane = threadIdx.x % G;
  const int rpb = TPB / G;
  for (int64_t base = (int64_t)blockIdx.x * rpb; base < n; base += (int64_t)gridDim.x * rpb) {
    const int64_t r = base + threadIdx.x / G;
    const bool ok = r < n;
    const double b = rhs.template eval<G>(ok ? (int)r : -1, lane);
    if (ok && lane == 0) y[r] = b;
  }
}

__global__ void __launch_bounds__(256) k_dense_gemv(int64_t n, const double* __restrict__ X,
                                                    const double* __restrict__ y,
                                                    double* __restrict__ x, double* __restrict__ out,
                                                    const int* __restrict__ perm, Ctl c) {
  if (inactive(c)) return;
  const int lane = threadIdx.x & 31;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const double* row = X + r * n;
    double s0 = 0.0, s1 = 0.0;
    int64_t q = lane;
    for (; q + 32 < n; q += 64) {
      s0 = fma(__ldcs(&row[q]), __ldg(&y[q]), s0);
      s1 = fma(__ldcs(&row[q + 32]), __ldg(&y[q + 32]), s1);
    }
    if (q < n) s0 = fma(__ldcs(&row[q]), __ldg(&y[q]), s0);
    const double z = warp_sum(s0 + s1);
    if (lane == 0) {
      x[r] = z;
      if (out) out[perm ? perm[r] : r] = z;
    }
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

// k_corr with K entries per lane, loads issued before the reduction.
template <int G, int K>
__global__ void __launch_bounds__(TPB) k_corr2(Csr si, const double* __restrict__ s,
                                               double* __restrict__ corr, Ctl c, int64_t n) {
  if (inactive(c)) return;
  __shared__ double sm[32];
  const int lane = threadIdx.x % G;
  const int rpb = TPB / G;
  double acc = 0.0;
  for (int64_t base = (int64_t)blockIdx.x * rpb; base < si.nrows; base += (int64_t)gridDim.x * rpb) {
    const int64_t r = base + threadIdx.x / G;
    const bool ok = r < si.nrows;
    int b = 0, e = 0;
    if (ok) {
      b = si.rowptr[r];
      e = si.rowptr[r + 1];
    }
    double a[K], xv[K];
    int cc[K];
#pragma unroll
    for (int t = 0; t < K; ++t) {
      const int k = b + lane + t * G;
      cc[t] = k < e ? si.col[k] : -1;
      a[t] = k < e ? si.val[k] : 0.0;
    }
#pragma unroll
    for (int t = 0; t < K; ++t) xv[t] = cc[t] >= 0 ? __ldg(&s[cc[t]]) : 0.0;
    double v = 0.0;
#pragma unroll
    for (int t = 0; t < K; ++t) v = fma(a[t], xv[t], v);
    for (int k = b + lane + K * G; k < e; k += G) v = fma(si.val[k], __ldg(&s[si.col[k]]), v);
    v = group_sum<G>(v);
    if (ok && lane == 0) {
      corr[r] = v;
      acc += v;
    }
  }
  double vv[1] = {block_sum(acc, sm)};
  reduce_tail<1>(c, vv, gridDim.x, blockIdx.x, C_CORR, FIN_MEAN, S_MU2, S_C2, n, sm);
}

// corr = S_i s on the ELL copy (thread per heart row), + its sum for mu2.
template <int W>
__global__ void __launch_bounds__(TPB) k_corr_ell(LamEll L, int n, int m, const double* __restrict__ s,
                                                  double* __restrict__ corr, Ctl c, int64_t nmean,
                                                  double* __restrict__ fill = nullptr,
                                                  int64_t nfill = 0) {
  if (inactive(c)) return;
  __shared__ double sm[32];
  // optional: reset the polled forward output of the bulk solve that follows (see k_update)
  for (int64_t i = blockIdx.x * (int64_t)TPB + threadIdx.x; i < nfill; i += (int64_t)gridDim.x * TPB)
    fill[i] = __longlong_as_double(SENTINEL);
  double acc = 0.0;
  for (int r = blockIdx.x * TPB + threadIdx.x; r < m; r += gridDim.x * TPB) {
    double v = 0.0;
#pragma unroll
    for (int e0 = 0; e0 < W; e0 += 8) {
      int cl[8];
      double a[8], xv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        cl[e] = __ldcs(&L.col[(size_t)(e0 + e) * n + r]);
        a[e] = __ldcs(&L.v2[(size_t)(e0 + e) * m + r]);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) xv[e] = cl[e] < m ? __ldg(&s[cl[e]]) : 0.0;
#pragma unroll
      for (int e = 0; e < 8; ++e) v = fma(a[e], xv[e], v);
    }
    corr[r] = v;
    acc += v;
  }
  double vv[1] = {block_sum(acc, sm)};
  reduce_tail<1>(c, vv, gridDim.x, blockIdx.x, C_CORR, FIN_MEAN, S_MU2, S_C2, nmean, sm);
}

// w = r_v - S_i t on the ELL copy (thread per heart row), t = (t_raw - mt) + c1 as in
// RhsSchur: the Schur solve's right-hand side evaluated by one streaming kernel before
// the forward pass, which then reads a plain vector (bd/precond.py:307).
template <int W>
__global__ void __launch_bounds__(TPB) k_schur_rhs_ell(const int* __restrict__ col,
                                                       const double* __restrict__ v2, int n, int m,
                                                       const double* __restrict__ traw,
                                                       const double* __restrict__ sc,
                                                       const double* __restrict__ rv,
                                                       double* __restrict__ y, Ctl c) {
  if (inactive(c)) return;
  const double mt = sc[S_MT], c1 = sc[S_C1];
  for (int r = blockIdx.x * TPB + threadIdx.x; r < m; r += gridDim.x * TPB) {
    double v = 0.0;
#pragma unroll
    for (int e0 = 0; e0 < W; e0 += 8) {
      int cl[8];
      double a[8], xv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        cl[e] = __ldcs(&col[(size_t)(e0 + e) * n + r]);
        a[e] = __ldcs(&v2[(size_t)(e0 + e) * m + r]);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e)
        xv[e] = cl[e] < m ? __dadd_rn(__dsub_rn(__ldg(&traw[cl[e]]), mt), c1) : 0.0;
#pragma unroll
      for (int e = 0; e < 8; ++e) v = fma(a[e], xv[e], v);
    }
    y[r] = __dsub_rn(rv[r], v);
  }
}

// z_u = t - bulk(corr) with both recentrings applied on the fly
// (bd/precond.py:291-292, 311): the standalone P^{-1} (bd_blocklu_apply)
__global__ void __launch_bounds__(TPB) k_combine(const double* __restrict__ traw,
                                                 const double* __restrict__ z2raw,
                                                 double* __restrict__ zu, int64_t n, Ctl c) {
  if (inactive(c)) return;
  const double* sc = c.sc;
  const double mt = sc[S_MT], c1 = sc[S_C1], m2 = sc[S_M2], c2 = sc[S_C2];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double t = __dadd_rn(__dsub_rn(traw[i], mt), c1);
    const double b = __dadd_rn(__dsub_rn(z2raw[i], m2), c2);
    const double z = __dsub_rn(t, b);
    zu[i] = z;
  }
}

// PCG-internal P^{-1} tail: z_u = t_raw − z2_raw (the recentrings of the two
// bulk solves are constants and fall out under the deflation), and the
// partials of Σz_u, r_u·z_u, r_v·z_v for rho (FIN_RHO3) in the same pass
__global__ void __launch_bounds__(TPB) k_combine_rho(const double* __restrict__ traw,
                                                     const double* __restrict__ z2raw,
                                                     double* __restrict__ zu,
                                                     const double* __restrict__ zv,
                                                     const double* __restrict__ r, int64_t n,
                                                     int64_t nm, Ctl c) {
  if (inactive(c)) return;
  __shared__ double sm[32];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nm;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n) {
      const double z = __dsub_rn(traw[i], z2raw[i]);
      zu[i] = z;
      a0 += z;
      a1 = fma(r[i], z, a1);
    } else {
      a2 = fma(r[i], zv[i - n], a2);
    }
  }
  double v[3];
  v[0] = block_sum(a0, sm);
  v[1] = block_sum(a1, sm);
  v[2] = block_sum(a2, sm);
  reduce_tail<3>(c, v, gridDim.x, blockIdx.x, C_RHO, FIN_RHO3, 0, -1, n, sm);
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

// Time-loop bookkeeping of one step (bd/simulate.py:67-89, 229-245): the
// running first-crossing activation map with sub-step interpolation, the
// depolarisation-band / full-coverage flags and max|u|.  flags[0] |= any
// v_new in [lo, hi]; flags[1] |= any phi still unset after the update;
// flags[2] = max over |u| as ordered bits (non-negative doubles order like
// their bit patterns, so the integer max is exact and deterministic).
__global__ void __launch_bounds__(TPB) k_step_track(int64_t m, const double* __restrict__ v_prev,
                                                    const double* __restrict__ v_new,
                                                    double* __restrict__ phi, double t_prev,
                                                    double dt, double thr, double lo, double hi,
                                                    int64_t n, const double* __restrict__ u,
                                                    unsigned long long* __restrict__ flags) {
  int band = 0, unset = 0;
  unsigned long long umax = 0ull;
  const int64_t len = m > n ? m : n;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < len;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (k < m) {
      const double vn = v_new[k];
      double ph = phi[k];
      if (!isfinite(ph) && vn >= thr) {
        const double vp = v_prev[k];
        // frac = (thr - v_prev) / (v_new - v_prev); phi = t_prev + dt * frac
        ph = vp < thr ? __dadd_rn(t_prev, __dmul_rn(dt, __ddiv_rn(__dsub_rn(thr, vp), __dsub_rn(vn, vp))))
                      : t_prev;
        phi[k] = ph;
      }
      band |= (vn >= lo) && (vn <= hi);
      unset |= !isfinite(ph);
    }
    if (k < n) {
      const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(u[k]));
      umax = b > umax ? b : umax;
    }
  }
  band = __syncthreads_or(band);
  unset = __syncthreads_or(unset);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long q = __shfl_xor_sync(0xffffffffu, umax, o);
    umax = q > umax ? q : umax;
  }
  if (threadIdx.x == 0) {
    if (band) atomicOr(&flags[0], 1ull);
    if (unset) atomicOr(&flags[1], 1ull);
  }
  if ((threadIdx.x & 31) == 0 && umax) atomicMax(&flags[2], umax);
}


}  // namespace dev
}  // namespace bd
