// Triangular-solve kernels (IncompleteCholesky0.apply_inverse,
// bd/precond.py:191-194, and the exact factor solves, :117-120).  Included by
// bd_device.cuh after the shared helpers, CSR/ELL types and right-hand sides.
#pragma once

namespace bd {
namespace dev {

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

// ---- tiled cooperative triangular solve -----------------------------------
// One CTA per row part (graph partition of the factor's pattern); the part's
// rows are processed in level order, one level chunk ("step") per
// __syncthreads.  Dependencies inside the part are read from shared memory
// (xs holds the right-hand side, overwritten in place by the solution);
// dependencies on other parts are polled in global memory (sentinel).  The
// ELL entries of upcoming steps stream into a D-stage shared-memory ring with
// cp.async, issued D-1 steps ahead, so the step loop never waits on HBM.
struct TileDev {
  const int* part_task_ptr;
  const int* part_step_ptr;
  const int* step_task_ptr;
  const int* task_row;
  const double* task_diag;
  const int* ell_col;
  const double* ell_val;
  int max_part_rows;
  int max_part_steps;
};

struct RhsGather {  // backward pass: the forward output
  static constexpr bool kScalar = true;
  const double* src;
  template <int G>
  __device__ __forceinline__ double eval(int row, int) const {
    return row < 0 ? 0.0 : src[row];
  }
  __device__ __forceinline__ double pass_const() const { return 0.0; }
  __device__ __forceinline__ double load(int row) const { return row < 0 ? 0.0 : src[row]; }
  __device__ __forceinline__ double finish(double v, double) const { return v; }
};

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

constexpr int TILE_INVALID = (int)0x80000000;

// Optional step trace (debug): per CTA and step, [globaltimer at step top,
// spin-poll iterations in the step, globaltimer after the barrier].
__device__ unsigned long long* g_tile_trace = nullptr;
__device__ int g_tile_trace_steps = 0;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}  // ring slot of a group with no row this step

__host__ __device__ constexpr size_t tile_ring_offset(int max_rows, int max_steps) {
  return (((size_t)(max_rows + 1) * 8 + (size_t)(max_steps + 1) * 4) + 15) & ~(size_t)15;
}
__host__ __device__ constexpr size_t tile_smem_bytes(int max_rows, int max_steps, int threads,
                                                     int G, int D) {
  return tile_ring_offset(max_rows, max_steps) + (size_t)D * threads * 12 +
         (size_t)D * (threads / G) * 12;
}

__device__ __forceinline__ double ld_relaxed(const double* p) {
  long long b;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(b) : "l"(p) : "memory");
  return __longlong_as_double(b);
}

template <int G, int D, class Rhs>
__global__ void __launch_bounds__(1024, 1) k_trsv_tiled(TileDev T, Rhs rhs, double* __restrict__ xg,
                                                        Ctl c, int ctr, int fin, int slot,
                                                        int slot2, int64_t nmean) {
  static_assert(D >= 3, "ring needs >= 3 stages");
  if (inactive(c)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double sm[32];
  const int R = blockDim.x / G;
  const int p = blockIdx.x;
  const int t0 = T.part_task_ptr[p], t1 = T.part_task_ptr[p + 1];
  const int nrows = t1 - t0;
  const int s0 = T.part_step_ptr[p], nst = T.part_step_ptr[p + 1] - s0;
  double* xs = reinterpret_cast<double*>(smem_raw);
  int* steps = reinterpret_cast<int*>(xs + T.max_part_rows + 1);
  double* rv = reinterpret_cast<double*>(smem_raw + tile_ring_offset(T.max_part_rows, T.max_part_steps));
  int* rc = reinterpret_cast<int*>(rv + (size_t)D * blockDim.x);
  double* rd = reinterpret_cast<double*>(rc + (size_t)D * blockDim.x);
  int* rr = reinterpret_cast<int*>(rd + (size_t)D * R);
  const int grp = threadIdx.x / G, lane = threadIdx.x % G;

  // prologue: step table, right-hand side of the own rows into xs, sentinel into xg
  for (int k = threadIdx.x; k <= nst; k += blockDim.x) steps[k] = T.step_task_ptr[s0 + k];
  if constexpr (Rhs::kScalar) {
    // thread per row, 4 independent rows in flight per thread
    constexpr int U = 4;
    for (int base = 0; base < nrows; base += U * blockDim.x) {
      int row[U];
      double b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = base + u * blockDim.x + threadIdx.x;
        row[u] = s < nrows ? T.task_row[t0 + s] : -1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) b[u] = rhs.template eval<1>(row[u], 0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = base + u * blockDim.x + threadIdx.x;
        if (row[u] >= 0) {
          xs[s] = b[u];
          xg[row[u]] = __longlong_as_double(SENTINEL);
        }
      }
    }
  } else {
    for (int base = 0; base < nrows; base += 2 * R) {
      const int s0 = base + grp, s1 = base + R + grp;
      const int r0 = s0 < nrows ? T.task_row[t0 + s0] : -1;
      const int r1 = s1 < nrows ? T.task_row[t0 + s1] : -1;
      const double b0 = rhs.template eval<G>(r0, lane);
      const double b1 = rhs.template eval<G>(r1, lane);
      if (lane == 0) {
        if (r0 >= 0) {
          xs[s0] = b0;
          xg[r0] = __longlong_as_double(SENTINEL);
        }
        if (r1 >= 0) {
          xs[s1] = b1;
          xg[r1] = __longlong_as_double(SENTINEL);
        }
      }
    }
  }
  if (threadIdx.x == 0) xs[nrows] = 0.0;  // zero cell for ELL padding
  __threadfence();
  cooperative_groups::this_grid().sync();

  // each thread copies exactly the ring entries it will consume
  auto issue = [&](int k) {
    if (k < nst) {
      const int st = k % D;
      const int t = steps[k] + grp;
      if (t < steps[k + 1]) {
        cp_async8(&rv[st * blockDim.x + threadIdx.x], &T.ell_val[(int64_t)t * G + lane]);
        cp_async4(&rc[st * blockDim.x + threadIdx.x], &T.ell_col[(int64_t)t * G + lane]);
        if (lane == 0) {
          cp_async8(&rd[st * R + grp], &T.task_diag[t]);
          cp_async4(&rr[st * R + grp], &T.task_row[t]);
        }
      } else {
        rc[st * blockDim.x + threadIdx.x] = TILE_INVALID;
      }
    }
    cp_async_commit();
  };
  // external-dependency lookahead: poll value for the next step, issued one step early
  auto lookahead = [&](int k, int& col, double& pre) {
    col = TILE_INVALID;
    pre = 0.0;
    if (k < nst) {
      col = rc[(k % D) * blockDim.x + threadIdx.x];
      if (col >= 0) pre = ld_relaxed(&xg[col]);
    }
  };
  __syncthreads();  // steps[] visible
#pragma unroll
  for (int k = 0; k < D - 1; ++k) issue(k);
  cp_async_wait<D - 2>();
  int col;
  double pre;
  lookahead(0, col, pre);
  __shared__ unsigned spins_s;
  __shared__ unsigned long long tmax_wait, tmax_done;
  unsigned long long* trace = g_tile_trace;
  if (threadIdx.x == 0) {
    spins_s = 0;
    tmax_wait = 0;
    tmax_done = 0;
  }
  __syncthreads();
  for (int k = 0; k < nst; ++k) {
    unsigned long long t_top = 0;
    if (trace && threadIdx.x == 0) t_top = gtimer();
    issue(k + D - 1);
    cp_async_wait<D - 2>();  // own copies of step k+1 landed
    if (trace && lane == 0) atomicMax(&tmax_wait, gtimer());
    int col_n;
    double pre_n;
    lookahead(k + 1, col_n, pre_n);
    const int st = k % D;
    const bool ok = col != TILE_INVALID;
    double acc = 0.0;
    if (ok) {
      double dep;
      if (col < 0) {
        dep = xs[-col - 1];
      } else if (__double_as_longlong(pre) != SENTINEL) {
        dep = pre;
      } else {
        if (trace) atomicAdd(&spins_s, 1u);
        dep = spin_load(&xg[col]);
      }
      acc = rv[st * blockDim.x + threadIdx.x] * dep;
    }
    acc = group_sum<G>(acc);
    if (ok && lane == 0) {
      const int sl = steps[k] + grp - t0;
      const double val = __ddiv_rn(__dsub_rn(xs[sl], acc), rd[st * R + grp]);
      xs[sl] = val;
      publish(&xg[rr[st * R + grp]], val);
    }
    if (trace && lane == 0) atomicMax(&tmax_done, gtimer());
    __syncthreads();
    if (trace && threadIdx.x == 0 && k < g_tile_trace_steps) {
      unsigned long long* tr = trace + ((size_t)blockIdx.x * g_tile_trace_steps + k) * 5;
      tr[0] = t_top;
      tr[1] = spins_s;
      tr[2] = gtimer();
      tr[3] = tmax_wait;
      tr[4] = tmax_done;
      spins_s = 0;
      tmax_wait = 0;
      tmax_done = 0;
    }
    col = col_n;
    pre = pre_n;
  }
  cp_async_wait<0>();
  if (fin >= 0) {
    double acc = 0.0;
    for (int s = threadIdx.x; s < nrows; s += blockDim.x) acc += xs[s];
    double v[1] = {block_sum(acc, sm)};
    reduce_tail<1>(c, v, gridDim.x, blockIdx.x, ctr, fin, slot, slot2, nmean, sm);
  }
}

// ---- tiled solve, thread per row ------------------------------------------------
// Same schedule as k_trsv_tiled (ELL width E, one CTA per part, level steps of
// at most R rows) but one THREAD per row: the step loop runs on R/32 warps
// synchronised with a named barrier, so a step costs a few hundred issued
// instructions instead of thousands; the other warps of the CTA only help
// with the prologue (right-hand side gather) and the epilogue.
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async16_zfill(void* dst, const void* src, int bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async8_zfill(void* dst, const void* src, int bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async4_zfill(void* dst, const void* src, int bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(s), "l"(src), "r"(bytes)
               : "memory");
}
// relaxed gpu-scope load executed only when `pred` (else 0.0), without a branch
__device__ __forceinline__ double ld_relaxed_if(const double* p, bool pred) {
  long long b = 0;
  asm volatile(
      "{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.relaxed.gpu.global.b64 %0, [%1]; }"
      : "+l"(b)
      : "l"(p), "r"((int)pred)
      : "memory");
  return __longlong_as_double(b);
}

__host__ __device__ constexpr size_t tile2_ring_offset(int max_rows, int max_steps) {
  return (((size_t)(max_rows + 1) * 8 + (size_t)(max_steps + 1) * 4) + 15) & ~(size_t)15;
}
__host__ __device__ constexpr size_t tile2_smem_bytes(int max_rows, int max_steps, int R, int E,
                                                      int D) {
  return tile2_ring_offset(max_rows, max_steps) + (size_t)D * R * (E * 12 + 16);
}

template <int E, int D, class Rhs>
__global__ void __launch_bounds__(512, 1) k_trsv_rows(TileDev T, Rhs rhs, double* __restrict__ xg,
                                                       Ctl c, int ctr, int fin, int slot, int slot2,
                                                       int64_t nmean, int R) {
  static_assert(D >= 3, "ring needs >= 3 stages");
  if (inactive(c)) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double sm[32];
  const int p = blockIdx.x;
  const int t0 = T.part_task_ptr[p], t1 = T.part_task_ptr[p + 1];
  const int nrows = t1 - t0;
  const int s0 = T.part_step_ptr[p], nst = T.part_step_ptr[p + 1] - s0;
  double* xs = reinterpret_cast<double*>(smem_raw);
  int* steps = reinterpret_cast<int*>(xs + T.max_part_rows + 1);
  unsigned char* ring = smem_raw + tile2_ring_offset(T.max_part_rows, T.max_part_steps);
  // stage layout: vals [R][E] f64 | cols [R][E] i32 | diag [R] f64 | row [R] i32 (+pad)
  const size_t stage_bytes = (size_t)R * (E * 12 + 16);
  // prologue (all threads): step table, rhs into xs, sentinel into xg
  for (int k = threadIdx.x; k <= nst; k += blockDim.x) steps[k] = T.step_task_ptr[s0 + k];
  if constexpr (Rhs::kScalar) {
    constexpr int U = 4;
    for (int base = 0; base < nrows; base += U * blockDim.x) {
      int row[U];
      double b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = base + u * blockDim.x + threadIdx.x;
        row[u] = s < nrows ? T.task_row[t0 + s] : -1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) b[u] = rhs.template eval<1>(row[u], 0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = base + u * blockDim.x + threadIdx.x;
        if (row[u] >= 0) {
          xs[s] = b[u];
          xg[row[u]] = __longlong_as_double(SENTINEL);
        }
      }
    }
  } else {
    constexpr int GG = 8;  // lanes per row for the SpMV-shaped right-hand side
    const int grp = threadIdx.x / GG, lane = threadIdx.x % GG, ngrp = blockDim.x / GG;
    for (int base = 0; base < nrows; base += 2 * ngrp) {
      const int sa = base + grp, sb = base + ngrp + grp;
      const int ra = sa < nrows ? T.task_row[t0 + sa] : -1;
      const int rb = sb < nrows ? T.task_row[t0 + sb] : -1;
      const double ba = rhs.template eval<GG>(ra, lane);
      const double bb = rhs.template eval<GG>(rb, lane);
      if (lane == 0) {
        if (ra >= 0) {
          xs[sa] = ba;
          xg[ra] = __longlong_as_double(SENTINEL);
        }
        if (rb >= 0) {
          xs[sb] = bb;
          xg[rb] = __longlong_as_double(SENTINEL);
        }
      }
    }
  }
  if (threadIdx.x == 0) xs[nrows] = 0.0;  // zero cell for ELL padding
  __threadfence();
  cooperative_groups::this_grid().sync();

  if ((int)threadIdx.x < R) {
    const int tid = threadIdx.x;
    const int zero_slot = nrows;
    // stage layout (entry-major per step): vals [E][ns] f64 | cols [E][ns] i32 |
    // diag [ns] f64 | row [ns] i32, each sub-array sized for ns = R
    auto stage_vals = [&](int st) { return reinterpret_cast<double*>(ring + st * stage_bytes); };
    auto stage_cols = [&](int st) {
      return reinterpret_cast<int*>(ring + st * stage_bytes + (size_t)R * E * 8);
    };
    auto stage_diag = [&](int st) {
      return reinterpret_cast<double*>(ring + st * stage_bytes + (size_t)R * E * 12);
    };
    auto stage_row = [&](int st) {
      return reinterpret_cast<int*>(ring + st * stage_bytes + (size_t)R * E * 12 + (size_t)R * 8);
    };
    // branch-free, zero-filling copies of step k's block (E*ns is a multiple of 4)
    auto issue = [&](int k) {
      if (k < nst) {
        const int st = k % D;
        const int a = steps[k], ns = steps[k + 1] - a;
        const double* gv = T.ell_val + (int64_t)a * E;
        const int* gc = T.ell_col + (int64_t)a * E;
        double* sv = stage_vals(st);
        int* sc = stage_cols(st);
        const int nv2 = (E * ns) >> 1, nc4 = (E * ns) >> 2;
#pragma unroll
        for (int u = 0; u < E / 2; ++u) {
          const int q = tid + u * R;
          const bool ok = q < nv2;
          cp_async16_zfill(sv + 2 * q, ok ? gv + 2 * q : gv, ok ? 16 : 0);
        }
#pragma unroll
        for (int u = 0; u < E / 4; ++u) {
          const int q = tid + u * R;
          const bool ok = q < nc4;
          cp_async16_zfill(sc + 4 * q, ok ? gc + 4 * q : gc, ok ? 16 : 0);
        }
        const bool okr = tid < ns;
        cp_async8_zfill(stage_diag(st) + tid, okr ? T.task_diag + a + tid : T.task_diag, okr ? 8 : 0);
        cp_async4_zfill(stage_row(st) + tid, okr ? T.task_row + a + tid : T.task_row, okr ? 4 : 0);
      }
      cp_async_commit();
    };
    double pre[E];
    // predicated (branch-free) polls of the external dependencies of step k
    auto lookahead = [&](int k) {
      if (k < nst) {
        const int ns = steps[k + 1] - steps[k];
        const bool valid = tid < ns;
        const int* sc = stage_cols(k % D);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int col = valid ? sc[e * ns + tid] : -1;
          pre[e] = ld_relaxed_if(&xg[col < 0 ? 0 : col], col >= 0);
        }
      }
    };
#pragma unroll
    for (int k = 0; k < D - 1; ++k) issue(k);
    cp_async_wait<D - 3>();  // own copies of steps 0, 1 landed
    named_bar(1, R);
    lookahead(0);
    unsigned long long* trace = g_tile_trace;
    const bool tr_on = trace && blockIdx.x == 0 && tid == 0;
    for (int k = 0; k < nst; ++k) {
      long long c0 = 0, c1 = 0, c2 = 0, c3 = 0;
      if (tr_on) c0 = clock64();
      issue(k + D - 1);
      const int st = k % D;
      double cur[E];
#pragma unroll
      for (int e = 0; e < E; ++e) cur[e] = pre[e];
      if (tr_on) c1 = clock64();
      cp_async_wait<D - 3>();  // own copies of step k+2 landed (visible after this step's barrier)
      if (tr_on) c2 = clock64();
      lookahead(k + 1);
      if (tr_on) c3 = clock64();
      const int a = steps[k], ns = steps[k + 1] - a;
      if (tid < ns) {
        const double* sv = stage_vals(st);
        const int* sc = stage_cols(st);
        int col[E];
        double val[E], xv[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          col[e] = sc[e * ns + tid];
          val[e] = sv[e * ns + tid];
        }
#pragma unroll
        for (int e = 0; e < E; ++e) xv[e] = xs[col[e] < 0 ? -col[e] - 1 : zero_slot];
        bool late = false;
#pragma unroll
        for (int e = 0; e < E; ++e)
          late |= (col[e] >= 0) && (__double_as_longlong(cur[e]) == SENTINEL);
        double acc = 0.0;
        if (!late) {
#pragma unroll
          for (int e = 0; e < E; ++e) acc = fma(val[e], col[e] < 0 ? xv[e] : cur[e], acc);
        } else {
          for (int e = 0; e < E; ++e) {
            double dep = xv[e];
            if (col[e] >= 0)
              dep = __double_as_longlong(cur[e]) != SENTINEL ? cur[e] : spin_load(&xg[col[e]]);
            acc = fma(val[e], dep, acc);
          }
        }
        const int sl = a + tid - t0;
        const double v = __ddiv_rn(__dsub_rn(xs[sl], acc), stage_diag(st)[tid]);
        xs[sl] = v;
        publish(&xg[stage_row(st)[tid]], v);
      }
      long long c4 = 0, c5 = 0;
      if (tr_on) c4 = clock64();
      named_bar(1, R);
      if (tr_on) {
        c5 = clock64();
        if (k < g_tile_trace_steps) {
          unsigned long long* q = trace + (size_t)k * 5;
          q[0] = c1 - c0;
          q[1] = c2 - c1;
          q[2] = c3 - c2;
          q[3] = c4 - c3;
          q[4] = c5 - c4;
        }
      }
    }
    cp_async_wait<0>();
  }
  __syncthreads();
  if (fin >= 0) {
    double acc = 0.0;
    for (int s = threadIdx.x; s < nrows; s += blockDim.x) acc += xs[s];
    double v[1] = {block_sum(acc, sm)};
    reduce_tail<1>(c, v, gridDim.x, blockIdx.x, ctr, fin, slot, slot2, nmean, sm);
  }
}

// ---- cluster-wavefront triangular solve ----------------------------------------
// One thread-block cluster (P CTAs, one part each) steps through the global
// levels in lockstep: per level, every CTA solves its own rows (thread per
// row) reading dependencies from a ring of W level windows in shared memory,
// pushes the values its neighbours import into THEIR windows through
// distributed shared memory, and the cluster barrier publishes everything.
// The per-level ELL block (values, int16 window codes, diagonal, right-hand
// side, row ids, export list) streams through a D-stage cp.async ring.
struct ClusterDev {
  const int* lvl_ptr;     // parts*(nlevels+1)
  const int* task_row;
  const double* task_diag;
  const double* ell_val;  // ntasks*E
  const short* ell_code;  // ntasks*E
  const int* exp_ptr;     // parts*(nlevels+1)
  const int* exp_src;
  const int* exp_dst;
  int nlevels, W, wmax, rmax, emax;
};

__host__ __device__ constexpr size_t cl_stage_bytes(int rmax, int emax, int E) {
  return (size_t)rmax * (E * 10 + 20) + (size_t)emax * 8;
}
__host__ __device__ constexpr size_t cl_ring_offset(int wmax, int W) {
  return ((size_t)W * wmax * 8 + 15) & ~(size_t)15;
}
__host__ __device__ constexpr size_t cl_smem_bytes(int rmax, int emax, int wmax, int W, int E,
                                                   int D, int nlevels) {
  return cl_ring_offset(wmax, W) + (size_t)D * cl_stage_bytes(rmax, emax, E) +
         (size_t)(nlevels + 1) * 8 + 16;
}

template <int E, int D, class Rhs>
__global__ void __launch_bounds__(1024, 1) k_trsv_cluster(ClusterDev S, Rhs rhs, double* __restrict__ xg,
                                                          double* __restrict__ rtmp, Ctl c) {
  namespace cg = cooperative_groups;
  if (inactive(c)) return;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int p = (int)cluster.block_rank();
  const int NL = S.nlevels;
  double* win = reinterpret_cast<double*>(smem_raw);
  unsigned char* ring = smem_raw + cl_ring_offset(S.wmax, S.W);
  const size_t sb = cl_stage_bytes(S.rmax, S.emax, E);
  const int tid = threadIdx.x, nth = blockDim.x;
  // per-level row / export offsets of this part, in shared memory
  int* lp = reinterpret_cast<int*>(ring + (size_t)D * sb);
  int* ep = lp + (NL + 1);
  for (int k = tid; k <= NL; k += nth) {
    lp[k] = S.lvl_ptr[(size_t)p * (NL + 1) + k];
    ep[k] = S.exp_ptr[(size_t)p * (NL + 1) + k];
  }
  __syncthreads();
  // prologue: right-hand side of every own row (task order), zero windows
  {
    const int t0 = lp[0], t1 = lp[NL];
    constexpr int U = 4;
    for (int base = t0; base < t1; base += U * nth) {
      int row[U];
      double b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = base + u * nth + tid;
        row[u] = k < t1 ? S.task_row[k] : -1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) b[u] = rhs.template eval<1>(row[u], 0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = base + u * nth + tid;
        if (k < t1) rtmp[k] = b[u];
      }
    }
    for (int k = tid; k < S.W * S.wmax; k += nth) win[k] = 0.0;
  }
  __threadfence();
  __syncthreads();
  auto issue = [&](int L) {
    if (L < NL) {
      unsigned char* st = ring + (size_t)(L % D) * sb;
      const int a = lp[L], n = lp[L + 1] - a;  // n is a multiple of 8
      const int ea = ep[L], ne = ep[L + 1] - ea;  // multiple of 4
      double* sv = reinterpret_cast<double*>(st);
      short* sc = reinterpret_cast<short*>(st + (size_t)S.rmax * E * 8);
      double* sd = reinterpret_cast<double*>(st + (size_t)S.rmax * E * 10);
      double* sr = sd + S.rmax;
      int* srow = reinterpret_cast<int*>(sr + S.rmax);
      int* ssrc = srow + S.rmax;
      int* sdst = ssrc + S.emax;
      for (int q = tid; q < n * E / 2; q += nth) cp_async16(sv + 2 * q, S.ell_val + (size_t)a * E + 2 * q);
      for (int q = tid; q < n * E / 8; q += nth) cp_async16(sc + 8 * q, S.ell_code + (size_t)a * E + 8 * q);
      for (int q = tid; q < n / 2; q += nth) {
        cp_async16(sd + 2 * q, S.task_diag + a + 2 * q);
        cp_async16(sr + 2 * q, rtmp + a + 2 * q);
      }
      for (int q = tid; q < n / 4; q += nth) cp_async16(srow + 4 * q, S.task_row + a + 4 * q);
      for (int q = tid; q < ne / 4; q += nth) {
        cp_async16(ssrc + 4 * q, S.exp_src + ea + 4 * q);
        cp_async16(sdst + 4 * q, S.exp_dst + ea + 4 * q);
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int L = 0; L < D - 1; ++L) issue(L);
  cp_async_wait<D - 2>();  // own copies of level 0 landed
  cluster.sync();           // every CTA resident and initialised; level-0 data visible
  unsigned long long* trace = g_tile_trace;
  const bool tr_on = trace && p == 0 && tid == 0;
  for (int L = 0; L < NL; ++L) {
    long long c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0, c5 = 0;
    if (tr_on) c0 = clock64();
    issue(L + D - 1);
    if (tr_on) c1 = clock64();
    const unsigned char* st = ring + (size_t)(L % D) * sb;
    const double* sv = reinterpret_cast<const double*>(st);
    const short* sc = reinterpret_cast<const short*>(st + (size_t)S.rmax * E * 8);
    const double* sd = reinterpret_cast<const double*>(st + (size_t)S.rmax * E * 10);
    const double* sr = sd + S.rmax;
    const int* srow = reinterpret_cast<const int*>(sr + S.rmax);
    const int* ssrc = srow + S.rmax;
    const int* sdst = ssrc + S.emax;
    const int n = lp[L + 1] - lp[L];
    double* wl = win + (size_t)(L % S.W) * S.wmax;
    for (int r = tid; r < n; r += nth) {
      const int row = srow[r];
      if (row < 0) continue;
      double acc = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int code = sc[r * E + e];
        const double d = code >= 0 ? win[code] : 0.0;
        acc = fma(sv[r * E + e], d, acc);
      }
      const double v = __ddiv_rn(__dsub_rn(sr[r], acc), sd[r]);
      wl[r] = v;
      xg[row] = v;
    }
    if (tr_on) c2 = clock64();
    __syncthreads();
    if (tr_on) c3 = clock64();
    const int ne = ep[L + 1] - ep[L];
    for (int e = tid; e < ne; e += nth) {
      const int src = ssrc[e];
      if (src < 0) continue;
      const int dst = sdst[e];
      double* remote = cluster.map_shared_rank(win, dst >> 16);
      remote[dst & 0xffff] = wl[src];
    }
    if (tr_on) c4 = clock64();
    cp_async_wait<D - 2>();  // own copies of level L+1 landed
    if (tr_on) c5 = clock64();
    cluster.sync();           // exports + next level's data visible
    if (tr_on && L < g_tile_trace_steps) {
      const long long c6 = clock64();
      unsigned long long* q = trace + (size_t)L * 6;
      q[0] = c1 - c0; q[1] = c2 - c1; q[2] = c3 - c2; q[3] = c4 - c3; q[4] = c5 - c4; q[5] = c6 - c5;
    }
  }
  cp_async_wait<0>();
}

// ---- dynamic-tile triangular solve --------------------------------------------------
// Rows are grouped into small tiles (~64 rows, a 4x4x4 box on the Kuhn grid)
// listed in a topological order of the tile DAG.  A persistent grid grabs
// tiles in that order (a tile only waits on earlier tiles, all owned by
// running blocks); inside a tile one thread owns one row and the tile steps
// through its own few levels with a block barrier, reading same-tile
// dependencies from shared memory and polling only cross-tile ones.
struct DTileDev {
  const int* tile_row_ptr;
  const int* tile_step_ptr;
  const int* step_row;
  const int* task_row;
  const double* task_diag;
  const int* ell_col;
  const double* ell_val;
  int ntiles;
  int tmax;
};
constexpr int DT_MAX_ROWS = 256;
constexpr int DT_MAX_STEPS = 96;

template <int E, class Rhs, int H = 1>
__global__ void __launch_bounds__(256) k_trsv_dtile(DTileDev T, Rhs rhs, double* __restrict__ xg,
                                                    Ctl c, int ctr_task, int ctr_done) {
  if (inactive(c)) return;
  __shared__ double xs[DT_MAX_ROWS + 1];
  __shared__ int steps_s[DT_MAX_STEPS + 1];
  __shared__ int task_s;
  __shared__ int last_s;
  const int tid = threadIdx.x, nth = blockDim.x;
  for (;;) {
    if (tid == 0) task_s = (int)atomicAdd(&c.ctr[ctr_task], 1u);
    __syncthreads();
    const int t = task_s;
    if (t >= T.ntiles) break;
    const int r0 = T.tile_row_ptr[t], nr = T.tile_row_ptr[t + 1] - r0;
    const int s0 = T.tile_step_ptr[t], ns = T.tile_step_ptr[t + 1] - s0;
    for (int k = tid; k < ns; k += nth) steps_s[k] = T.step_row[s0 + k];
    if (tid == 0) {
      steps_s[ns] = nr;
      xs[T.tmax] = 0.0;
    }
    // this thread's rows (tiles of up to H*nth rows: k = tid, tid + nth, ...)
    int row[H], cl[H][E];
    double dg[H], vl[H][E], b[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int k = tid + h * nth;
      const bool ok = k < nr;
      row[h] = ok ? T.task_row[r0 + k] : -1;
      dg[h] = ok ? T.task_diag[r0 + k] : 1.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        cl[h][e] = ok ? T.ell_col[(int64_t)(r0 + k) * E + e] : -(T.tmax + 1);
        vl[h][e] = ok ? T.ell_val[(int64_t)(r0 + k) * E + e] : 0.0;
      }
      b[h] = rhs.template eval<1>(row[h], 0);
    }
    __syncthreads();
    for (int st = 0; st < ns; ++st) {
      const int a = steps_s[st], e_ = steps_s[st + 1];
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const int k = tid + h * nth;
        if (k >= a && k < e_) {
          double xv[E];
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int code = cl[h][e];
            xv[e] = code < 0 ? xs[-code - 1] : ld_relaxed_if(&xg[code < 0 ? 0 : code], code >= 0);
          }
          bool late = false;
#pragma unroll
          for (int e = 0; e < E; ++e)
            late |= (cl[h][e] >= 0) && (__double_as_longlong(xv[e]) == SENTINEL);
          if (late) {
#pragma unroll
            for (int e = 0; e < E; ++e)
              if (cl[h][e] >= 0 && __double_as_longlong(xv[e]) == SENTINEL)
                xv[e] = spin_load(&xg[cl[h][e]]);
          }
          double acc = 0.0;
#pragma unroll
          for (int e = 0; e < E; ++e) acc = fma(vl[h][e], xv[e], acc);
          const double v = __ddiv_rn(__dsub_rn(b[h], acc), dg[h]);
          xs[k] = v;
          publish(&xg[row[h]], v);
        }
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    __threadfence();
    const unsigned d = atomicAdd(&c.ctr[ctr_done], 1u);
    last_s = (d == gridDim.x - 1u);
  }
  __syncthreads();
  if (last_s && tid == 0) {
    c.ctr[ctr_task] = 0u;
    c.ctr[ctr_done] = 0u;
    __threadfence();
  }
}

// ---- blocked-tile triangular solve ------------------------------------------
// Same tiles and priority-topological tile order as k_trsv_dtile, but a tile
// no longer walks its ~10 internal levels: it gathers b_T - L_T,ext x_ext once
// (one thread per row, polling only the entries that reach other tiles), then
// applies the precomputed dense inverse of its diagonal block from shared
// memory (4 lanes per row + shuffles).  The inverse is copied in with cp.async
// as soon as the tile is grabbed, i.e. while its inputs are still in flight,
// so a pass costs ~(tile-DAG depth) x (one cross-SM hop + a short dense step).
struct BTileDev {
  // fixed per-tile strides: every load of a tile depends on the tile id only
  const int* tile_nr;               // rows of each tile
  const int* task_row;              // [tile][rs] (-1 padding)
  const unsigned short* ent_rp;     // [tile][rps]: per-row ranges into the tile's external entries
  const unsigned short* ent_slot;   // [tile][es]: slot in the tile's input list
  const double* ent_val;            // [tile][es]
  const int* in_col;                // [tile][xs] (-1 padding)
  const double* inv;                // [tile][is] packed lower triangle (slot order)
  int ntiles;
  int rs, xs, is, es, rps;          // strides (doubles / elements); 16-byte multiples
  int sleep_ns;                     // cap of the polling back-off (0: spin)
  int prefetch;                     // L2 bulk prefetch of the tile one grid-width ahead
  int poll_depth;                   // k_trsv_rtile: polls kept in flight per input (1..3)
  // inbox mode (k_trsv_rtile): producers push each value into the input slots
  // of its consumer tiles (inbox[c*xs + j]); a tile polls its own contiguous
  // inbox instead of scattered rows of the output vector
  double* inbox;                    // nullptr: poll the output vector
  const int* dst;                   // [tile][rs][dmax] inbox slots fed by each row (-1 pad)
  int dmax;                         // <= 8
  int exw;                          // max external entries of a row (k_trsv_rtile: <= 16)
  // k_trsv_rpipe: one packed record per tile (see rp_layout), fetched with a
  // single 1D TMA bulk copy into a ring of `depth` shared-memory slots
  const unsigned char* rec;
  int recb;                         // record stride in bytes (16-byte multiple)
  int depth;                        // ring slots per CTA (>= 2)
  int reset1_n;                     // rows below this bound are reset through `reset1` (launch-time)
};
constexpr int BT_LANES = 4;  // lanes per row in the dense step

__host__ __device__ constexpr int bt_even(int v) { return (v + 1) & ~1; }
__host__ __device__ constexpr int bt_round8(int v) { return (v + 7) & ~7; }
// shared-memory layout (bytes) of one tile:
// partials[256] | ys | xin | inv | ent_val | ent_slot | ent_rp
constexpr int BT_PART = 256;
__host__ __device__ constexpr size_t bt_smem(int rs, int xs, int is, int es, int rps) {
  return sizeof(double) * ((size_t)BT_PART + rs + xs + 2 + is + 2 + es) +
         sizeof(unsigned short) * ((size_t)es + rps);
}

template <class Rhs>
__global__ void __launch_bounds__(256) k_trsv_btile(BTileDev T, Rhs rhs, double* __restrict__ xg,
                                                    Ctl c, int ctr_task, int ctr_done,
                                                    double* __restrict__ reset) {
  if (inactive(c)) return;
  extern __shared__ __align__(16) double bt_sm[];
  double* part = bt_sm;              // dense partials [G][R], G*R <= BT_PART
  double* ys = part + BT_PART;       // rs
  double* xin = ys + T.rs;           // xs external inputs
  double* is = xin + T.xs + 2;       // inverse, packed column-major: column l = rows l..nr-1
  double* ev = is + T.is + 2;        // external entries (is[T.is] = 0: zero slot)
  unsigned short* esl = reinterpret_cast<unsigned short*>(ev + T.es);
  unsigned short* erp = esl + T.es;
  __shared__ int task_s;
  __shared__ int last_s;
  const int tid = threadIdx.x, nth = blockDim.x;
  // dense step mapping: G column groups x R rows (R = rs rounded to 32)
  const int R = (T.rs + 31) & ~31;
  const int G = max(1, nth / R);
  const int kk = tid % R, gg = tid / R;
  if (tid == 0) {  // zero slots (never overwritten: copies stop short of them)
    is[T.is] = 0.0;
    xin[T.xs] = 0.0;
  }
  for (;;) {
    if (tid == 0) task_s = (int)atomicAdd(&c.ctr[ctr_task], 1u);
    __syncthreads();
    const int t = task_s;
    if (t >= T.ntiles) break;
    unsigned long long* trace = g_tile_trace;
    if (trace && tid == 0) trace[8 * t] = gtimer();
    if (tid == 0 && T.prefetch && t + (int)gridDim.x < T.ntiles) {
      const int u = t + (int)gridDim.x;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(T.inv + (int64_t)u * T.is),
                   "r"((unsigned)(T.is * 8)) : "memory");
    }
    // everything below up to the polls depends on t only (one round trip)
    const int nr = T.tile_nr[t];
    const int row = tid < T.rs ? T.task_row[(int64_t)t * T.rs + tid] : -1;
    int icol[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = tid + h * nth;
      icol[h] = j < T.xs ? T.in_col[(int64_t)t * T.xs + j] : -1;
    }
    {  // group 1: external entries (small); group 2: the inverse
      const double* vb = T.ent_val + (int64_t)t * T.es;
      for (int q = tid; 2 * q < T.es; q += nth) cp_async16(ev + 2 * q, vb + 2 * q);
      const unsigned short* sb = T.ent_slot + (int64_t)t * T.es;
      for (int q = tid; 8 * q < T.es; q += nth) cp_async16(esl + 8 * q, sb + 8 * q);
      const unsigned short* rb = T.ent_rp + (int64_t)t * T.rps;
      for (int q = tid; 8 * q < T.rps; q += nth) cp_async16(erp + 8 * q, rb + 8 * q);
      cp_async_commit();
      const int ninv = bt_even(nr * (nr + 1) / 2);
      const double* ib = T.inv + (int64_t)t * T.is;
      for (int q = tid; 2 * q < ninv; q += nth) cp_async16(is + 2 * q, ib + 2 * q);
      cp_async_commit();
    }
    double b;
    if constexpr (Rhs::kScalar) {
      b = rhs.template eval<1>(row, 0);
    } else {
      // gather-heavy right-hand side (e.g. the fused S_i product of the Schur
      // solve): BT_LANES lanes per row, staged through ys
      for (int k0 = 0; k0 < T.rs; k0 += nth / BT_LANES) {
        const int k = k0 + tid / BT_LANES;
        const int rk = k < T.rs ? T.task_row[(int64_t)t * T.rs + k] : -1;
        const double v = rhs.template eval<BT_LANES>(rk, tid & (BT_LANES - 1));
        if ((tid & (BT_LANES - 1)) == 0 && k < T.rs) ys[k] = v;
      }
      __syncthreads();
      b = tid < T.rs ? ys[tid] : 0.0;
    }
    if (reset && row >= 0) reset[row] = __longlong_as_double(SENTINEL);  // optional row reset
    if (trace) {
      __syncthreads();
      if (tid == 0) trace[8 * t + 5] = gtimer();
    }
    // the tile's distinct inputs: one poller each
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (icol[h] < 0) continue;
      const double* pj = &xg[icol[h]];
      long long v;
      asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(pj) : "memory");
      unsigned nap = 16;
      while (v == SENTINEL) {
        if (T.sleep_ns) {
          __nanosleep(nap);
          nap = min(2u * nap, (unsigned)T.sleep_ns);
        }
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(pj) : "memory");
      }
      xin[tid + h * nth] = __longlong_as_double(v);
    }
    cp_async_wait<0>();
    __syncthreads();
    if (trace && tid == 0) trace[8 * t + 4] = gtimer();
    // y_k = b_k - sum_ext: branch-free (padding entries read the zero input
    // slot xin[xs] with a zero-padded value)
    if (tid < T.rs) {
      const int e0 = erp[tid], e1 = erp[tid + 1];
      int sl[8];
      double vl[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const bool ok = e0 + e < e1;
        const int ei = ok ? e0 + e : 0;
        sl[e] = ok ? (int)esl[ei] : T.xs;
        vl[e] = ev[ei];
      }
      double acc = 0.0;
#pragma unroll
      for (int e = 0; e < 8; ++e) acc = fma(vl[e], xin[sl[e]], acc);
      ys[tid] = row >= 0 ? __dsub_rn(b, acc) : 0.0;
    }
    if (trace && tid == 0) trace[8 * t + 6] = gtimer();
    __syncthreads();
    if (trace && tid == 0) trace[8 * t + 1] = gtimer();
    // x_k = sum_g sum_{l in group g, l <= k} inv[k][l] y_l ; column l of the
    // packed column-major inverse starts at l*nr - l*(l-1)/2
    {
      const int L = (nr + G - 1) / G;
      const int l0 = gg * L;
      double s4[4] = {0.0, 0.0, 0.0, 0.0};
      if (gg < G && kk < nr) {
        // no conditional loads (they compile to branches that serialise the
        // shared-memory pipeline): out-of-range lanes read the zero slot
        // is[T.is] and a valid y; column offsets advance incrementally,
        // idx(l+1) = idx(l) + nr - l - 1
        const int zero = T.is;
        int l = l0;
        int idx = l * nr - ((l * (l - 1)) >> 1) + (kk - l);
        const int lend = min(l0 + L, kk + 1);
        for (int u0 = l0; u0 < lend; u0 += 16) {
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const bool ok = l < lend;
            const double av = is[ok ? idx : zero];
            const double yy = ys[ok ? l : 0];
            s4[u & 3] = fma(av, yy, s4[u & 3]);
            idx += nr - l - 1;
            ++l;
          }
        }
      }
      const double sp = (s4[0] + s4[1]) + (s4[2] + s4[3]);
      if (gg < G) part[gg * R + kk] = sp;
    }
    __syncthreads();
    if (tid < nr) {
      double x = part[tid];
      for (int g = 1; g < G; ++g) x += part[g * R + tid];
      publish(&xg[row], x);
    }
    if (trace && tid == 0) trace[8 * t + 7] = gtimer();
    __syncthreads();  // smem reuse by the next tile
    if (trace && tid == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      trace[8 * t + 2] = gtimer();
      trace[8 * t + 3] = ((unsigned long long)smid << 32) | blockIdx.x;
    }
  }
  if (tid == 0) {
    __threadfence();
    const unsigned d = atomicAdd(&c.ctr[ctr_done], 1u);
    last_s = (d == gridDim.x - 1u);
  }
  __syncthreads();
  if (last_s && tid == 0) {
    c.ctr[ctr_task] = 0u;
    c.ctr[ctr_done] = 0u;
    __threadfence();
  }
}

// ---- register-tile triangular solve -------------------------------------------
// Same schedule and data as k_trsv_btile (tiles of <= 64 rows), but the dense
// inverse never touches shared memory: during the tile's preparation (before
// its inputs arrive) each thread loads its 16 entries of inv(L_TT) straight
// into registers.  Thread mapping: row slot k = 8*warp + lane/4 and column
// group g = lane%4 (columns g, g+4, ..., g+60), so the 4 partial sums of a row
// sit in one warp and are combined with two shuffles.  Critical path of a tile
// after its inputs land: one barrier (inputs -> shared), the external sum
// (2 entries per lane + 2 shuffles), one barrier (y -> shared), 16 broadcast
// loads + FMAs, 2 shuffles, publish.  k_trsv_btile had a third barrier and a
// dense step bound by shared-memory bandwidth (the inverse read from smem).
constexpr int RT_ROWS = 64;

// Rolling poll: keep three relaxed loads of the word in flight, re-issuing
// each as soon as it returns the sentinel, so the word is sampled about every
// third of an L2 round trip instead of once per round trip.
__device__ __forceinline__ long long poll_rolling3(const double* p) {
  long long v0, v1, v2;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v0) : "l"(p) : "memory");
  if (v0 != SENTINEL) return v0;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v1) : "l"(p) : "memory");
  __nanosleep(100);
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v2) : "l"(p) : "memory");
  for (;;) {
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v0) : "l"(p) : "memory");
    if (v1 != SENTINEL) return v1;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v1) : "l"(p) : "memory");
    if (v2 != SENTINEL) return v2;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v2) : "l"(p) : "memory");
    if (v0 != SENTINEL) return v0;
  }
}
// shared memory: ys | xin (+zero slot) | ent_val | ent_slot | ent_rp | [inverse (+zero slot)]
__host__ __device__ constexpr size_t rt_smem(int xs, int es, int rps, int is) {
  return sizeof(double) * ((size_t)RT_ROWS + xs + 2 + es) + sizeof(unsigned short) * ((size_t)es + rps) +
         (is > 0 ? sizeof(double) * ((size_t)is + 2) : 0);
}

// kSmemInv: the inverse is copied to shared memory with cp.async instead of
// held in registers (fewer registers -> more tiles in flight per SM).
// kTileRhs: the right-hand side comes pre-gathered in tile order (bt, slot
// t*rs + k, see k_tile_rhs) instead of through the Rhs functor, so the tile's
// preparation is a single round of independent loads; with bt_next set the
// pass also writes its output into the next pass's tile order through opos.
template <bool kSmemInv, bool kTileRhs, class Rhs>
__global__ void __launch_bounds__(256, kSmemInv ? 8 : 4)
    k_trsv_rtile(BTileDev T, Rhs rhs, double* __restrict__ xg, Ctl c, int ctr_task, int ctr_done,
                 const double* __restrict__ bt, const int* __restrict__ opos,
                 double* __restrict__ bt_next, double* reset0 = nullptr,
                 double* reset1 = nullptr) {
  if (inactive(c)) return;
  extern __shared__ __align__(16) double rt_sm[];
  double* ys = rt_sm;                 // RT_ROWS
  double* xin = ys + RT_ROWS;         // xs external inputs, xin[xs] = 0 (zero slot)
  double* ev = xin + T.xs + 2;        // external entries
  unsigned short* esl = reinterpret_cast<unsigned short*>(ev + T.es);
  unsigned short* erp = esl + T.es;
  double* is_s = reinterpret_cast<double*>(erp + T.rps);  // kSmemInv only
  __shared__ int task_s;
  __shared__ int last_s;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int k = warp * 8 + (lane >> 2);  // row slot
  const int g = lane & 3;                // column group
  const int jmax = (8 * warp + 7) >> 2;  // warp-uniform: columns g + 4j beyond the warp's rows are zero
  if (tid == 0) {
    xin[T.xs] = 0.0;
    if constexpr (kSmemInv) is_s[T.is] = 0.0;
  }
  for (;;) {
    if (tid == 0) task_s = (int)atomicAdd(&c.ctr[ctr_task], 1u);
    __syncthreads();
    const int t = task_s;
    if (t >= T.ntiles) break;
    unsigned long long* trace = g_tile_trace;
    if (trace && tid == 0) trace[8 * t] = gtimer();
    if (tid < (T.prefetch >= 2 ? 5 : T.prefetch) && t + (int)gridDim.x < T.ntiles) {
      // the tile one grid-width ahead: inverse (prefetch 1); + rows, inputs, entries (2) -> L2
      const int64_t u = t + (int)gridDim.x;
      const void* src;
      unsigned bytes;
      switch (tid) {
        case 0: src = T.inv + u * T.is; bytes = T.is * 8; break;
        case 1: src = T.task_row + u * T.rs; bytes = T.rs * 4; break;
        case 2: src = T.in_col + u * T.xs; bytes = T.xs * 4; break;
        case 3: src = T.ent_val + u * T.es; bytes = T.es * 8; break;
        default: src = T.ent_slot + u * T.es; bytes = T.es * 2; break;
      }
      const uintptr_t lo = reinterpret_cast<uintptr_t>(src) & ~(uintptr_t)15;
      const uintptr_t hi = (reinterpret_cast<uintptr_t>(src) + bytes) & ~(uintptr_t)15;
      if (hi > lo)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((unsigned)(hi - lo))
                     : "memory");
    }
    // preparation: everything up to the polls depends on t only
    const int nr = T.tile_nr[t];
    const int row = k < nr ? T.task_row[(int64_t)t * T.rs + k] : -1;
    int icol[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = tid + h * nth;
      icol[h] = j < T.xs ? T.in_col[(int64_t)t * T.xs + j] : -1;
    }
    {
      const double* vb = T.ent_val + (int64_t)t * T.es;
      for (int q = tid; 2 * q < T.es; q += nth) cp_async16(ev + 2 * q, vb + 2 * q);
      const unsigned short* sb = T.ent_slot + (int64_t)t * T.es;
      for (int q = tid; 8 * q < T.es; q += nth) cp_async16(esl + 8 * q, sb + 8 * q);
      const unsigned short* rb = T.ent_rp + (int64_t)t * T.rps;
      for (int q = tid; 8 * q < T.rps; q += nth) cp_async16(erp + 8 * q, rb + 8 * q);
      cp_async_commit();
    }
    // inverse entries inv[k][g+4j] (packed column-major: column l = rows l..nr-1
    // at l*nr - l(l-1)/2); idx(j+1) = idx(j) + 4nr - 4l - 10 with l = g + 4j
    double a[kSmemInv ? 1 : 16];
    if constexpr (kSmemInv) {
      const int ninv = bt_even(nr * (nr + 1) / 2);
      const double* ib = T.inv + (int64_t)t * T.is;
      for (int q = tid; 2 * q < ninv; q += nth) cp_async16(is_s + 2 * q, ib + 2 * q);
      cp_async_commit();
    } else {
      const double* ib = T.inv + (int64_t)t * T.is;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int l = g + 4 * j;
        const bool ok = (j <= jmax) && l <= k && k < nr;
        const int idx = ok ? l * nr - ((l * (l - 1)) >> 1) + (k - l) : 0;
        const double v = __ldcs(ib + idx);
        a[j] = ok ? v : 0.0;
      }
    }
    int dsl[2] = {-1, -1};  // inbox slots this lane feeds (lanes g: entries 2g, 2g+1)
    if (T.inbox && k < nr) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (2 * g + h < T.dmax) dsl[h] = T.dst[((int64_t)t * T.rs + k) * T.dmax + 2 * g + h];
    }
    double b;
    int op = -1;
    if constexpr (kTileRhs) {
      b = bt[(int64_t)t * T.rs + k];  // k < rs: padding slots hold 0
      if (bt_next && k < nr) op = opos[(int64_t)t * T.rs + k];
    } else if constexpr (Rhs::kScalar) {
      b = rhs.template eval<1>(row, 0);
    } else {
      b = rhs.template eval<4>(row, g);  // 4 consecutive lanes per row; valid in all four
    }
    // sentinel resets folded into the pass (BD_FOLD_FILL): reset0 = the next
    // pass's polled output, reset1 = this pass's gathered right-hand side
    // (the forward output, read above) for the inner's next forward pass
    if (g == 0 && row >= 0) {
      if (reset0) reset0[row] = __longlong_as_double(SENTINEL);
      if (reset1 && row < T.reset1_n) reset1[row] = __longlong_as_double(SENTINEL);
    }
    if (trace) {
      __syncthreads();
      if (tid == 0) trace[8 * t + 5] = gtimer();
    }
    // the tile's distinct inputs: one poller each
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (icol[h] < 0) continue;
      const double* pj = T.inbox ? &T.inbox[(int64_t)t * T.xs + tid + h * nth] : &xg[icol[h]];
      long long v;
      if (T.poll_depth >= 3) {
        v = poll_rolling3(pj);
      } else {
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(pj) : "memory");
        while (v == SENTINEL) {
          if (T.sleep_ns) __nanosleep(T.sleep_ns);
          asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(pj) : "memory");
        }
      }
      xin[tid + h * nth] = __longlong_as_double(v);
    }
    cp_async_wait<0>();
    __syncthreads();
    if (trace && tid == 0) trace[8 * t + 4] = gtimer();
    // y_k = b_k - sum_ext: entries e0+g and e0+g+4 of row k (<= 8 per row),
    // padding lanes read the zero input slot
    {
      const int kc = k < nr ? k : 0;
      const int e0 = erp[kc], e1 = k < nr ? erp[kc + 1] : e0;
      double acc = 0.0;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        if (h >= 2 && 4 * h >= T.exw) break;  // rows with > 8 entries: heart-first torso rows
        const int e = e0 + g + 4 * h;
        const bool ok = e < e1;
        const int ei = ok ? e : 0;
        const int sl = ok ? (int)esl[ei] : T.xs;
        acc = fma(ev[ei], xin[sl], acc);
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if (g == 0) ys[k] = row >= 0 ? __dsub_rn(b, acc) : 0.0;
    }
    if (trace && tid == 0) trace[8 * t + 6] = gtimer();
    __syncthreads();
    if (trace && tid == 0) trace[8 * t + 1] = gtimer();
    // x_k = sum_l inv[k][l] y_l: 4 column groups per row, in-warp combine
    {
      double s[4] = {0.0, 0.0, 0.0, 0.0};
      int idx = g * nr - ((g * (g - 1)) >> 1) + (k - g);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j <= jmax) {
          double av;
          if constexpr (kSmemInv) {
            const int l = g + 4 * j;
            av = is_s[(l <= k && k < nr) ? idx : T.is];  // branch-free: zero slot
            idx += 4 * nr - 4 * l - 10;
          } else {
            av = a[j];
          }
          s[j & 3] = fma(av, ys[g + 4 * j], s[j & 3]);
        }
      }
      double x = (s[0] + s[1]) + (s[2] + s[3]);
      x += __shfl_xor_sync(0xffffffffu, x, 1);
      x += __shfl_xor_sync(0xffffffffu, x, 2);
      if (T.inbox) {
        // push into the consumers' inboxes first (critical), then the output
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (dsl[h] >= 0) publish(&T.inbox[dsl[h]], x);
        if (g == 0 && row >= 0) {
          xg[row] = x;
          if (kTileRhs && op >= 0) bt_next[op] = x;
        }
      } else if (g == 0 && row >= 0) {
        publish(&xg[row], x);
        if (kTileRhs && op >= 0) bt_next[op] = x;
      }
    }
    if (trace && tid == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      trace[8 * t + 7] = gtimer();
      trace[8 * t + 2] = gtimer();
      trace[8 * t + 3] = ((unsigned long long)smid << 32) | blockIdx.x;
    }
  }
  if (tid == 0) {
    __threadfence();
    const unsigned d = atomicAdd(&c.ctr[ctr_done], 1u);
    last_s = (d == gridDim.x - 1u);
  }
  __syncthreads();
  if (last_s && tid == 0) {
    c.ctr[ctr_task] = 0u;
    c.ctr[ctr_done] = 0u;
    __threadfence();
  }
}

// ---- register tiles fed by a TMA ring -----------------------------------------
// k_trsv_rtile's arithmetic (same thread mapping, same sums in the same order,
// so the results are bit-identical) with the tile's preparation taken off the
// CTA's serial path.  Every array of a tile is packed into ONE record
// (rp_layout: header, rows, inputs, entry ranges / slots / values, inverse), so
// a tile is fetched by a single cp.async.bulk into a shared-memory ring slot,
// completion signalled on the slot's mbarrier.  The CTA holds `depth` tiles:
// it works on the oldest while the others' records are in flight.  Thread 0
// fires the atomic grab for the slot's refill at the top of an iteration and
// consumes it after the tile's second barrier, when the slot is free again, so
// neither the grab's round trip nor the record's DRAM latency sits between two
// tiles.  When a record has landed the inverse goes smem -> registers while the
// first poll loads are already in flight.  Deadlock-free like the other
// in-order grabbers: a CTA finishes its tiles in grab order, so the smallest
// unfinished tile is always some CTA's current one.
// The record's inverse is stored in the threads' own order: block j (columns
// l = g + 4j of every row slot k) holds the entries of threads tid >= 16j at
// RP_INV_BASE(j) + tid - 16j, zeros where l > k or k >= rows, so a thread's 16
// loads are conflict-free shared-memory reads at compile-time offsets.
__host__ __device__ constexpr int rp_inv_base(int j) { return 256 * j - 8 * j * (j - 1); }
constexpr int RP_INV = rp_inv_base(16);  // 2176 doubles
struct RpLayout {
  int o_row, o_in, o_rp, o_slot, o_val, o_inv, bytes;
};
__host__ __device__ inline RpLayout rp_layout(int rs, int xs, int is, int es, int rps) {
  RpLayout l;
  l.o_row = 16;                 // header: int nr, 3 x pad
  l.o_in = l.o_row + 4 * rs;
  l.o_rp = l.o_in + 4 * xs;
  l.o_slot = l.o_rp + 2 * rps;
  l.o_val = l.o_slot + 2 * es;
  l.o_inv = l.o_val + 8 * es;
  l.bytes = (l.o_inv + 8 * is + 15) & ~15;
  return l;
}
// shared memory: ring [depth][recb] | ys | xin (+zero slot) | mbarriers | tile ids
__host__ __device__ inline size_t rp_smem(int recb, int depth, int xs) {
  return (size_t)depth * recb + sizeof(double) * ((size_t)RT_ROWS + xs + 2) + 8 * (size_t)depth +
         4 * (size_t)((depth + 3) & ~3);
}
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(void* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(void* bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
  unsigned ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
// one elected thread: arm the slot's barrier with the byte count and start the copy
// The records are read once per pass and never again before 400 MB more have gone by:
// fetched with an evict-first L2 policy so they do not push out the vectors the tiles poll.
__device__ __forceinline__ void tma_fetch(void* dst, const void* src, unsigned bytes, void* bar) {
  const unsigned b = smem_u32(bar);
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
      "[%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(b), "l"(pol)
      : "memory");
}

// kWide: tiles with more than 256 inputs (two per thread); kTrace: per-tile
// timestamps for tools/btile_trace.py (launched only while a trace buffer is set)
template <bool kWide, bool kTrace, class Rhs>
__global__ void __launch_bounds__(256, 4)
    k_trsv_rpipe(BTileDev T, Rhs rhs, double* __restrict__ xg, Ctl c, int ctr_task, int ctr_done,
                 double* reset0 = nullptr, double* reset1 = nullptr) {
  if (inactive(c)) return;
  extern __shared__ __align__(128) unsigned char rp_sm[];
  constexpr int D = 2;  // ring slots (three measured no gain and cost a CTA per SM)
  const RpLayout lay = rp_layout(T.rs, T.xs, RP_INV, T.es, T.rps);
  double* ys = reinterpret_cast<double*>(rp_sm + (size_t)D * T.recb);  // RT_ROWS
  double* xin = ys + RT_ROWS;                                          // xs inputs, xin[xs] = 0
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(xin + T.xs + 2);
  int* ids = reinterpret_cast<int*>(mbar + D);
  __shared__ int last_s;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int k = warp * 8 + (lane >> 2);  // row slot
  const int g = lane & 3;                // column group
  const int jmax = (8 * warp + 7) >> 2;  // warp-uniform: columns beyond the warp's rows are zero
  // trace selector (bd_debug_tile_trace steps): 1 = backward passes only, 2 = forward only
  constexpr bool kBackward = Rhs::kScalar && sizeof(Rhs) == sizeof(RhsGather);
  unsigned long long* trace = nullptr;
  if constexpr (kTrace)
    trace = (g_tile_trace_steps == 1 && !kBackward) || (g_tile_trace_steps == 2 && kBackward) ? nullptr
                                                                                            : g_tile_trace;
  (void)kBackward;
  if (tid == 0) {
    xin[T.xs] = 0.0;
    for (int s = 0; s < D; ++s) mbar_init(&mbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int s = 0; s < D; ++s) {
      const int t = (int)atomicAdd(&c.ctr[ctr_task], 1u);
      ids[s] = t;
      if (t < T.ntiles) {
        tma_fetch(rp_sm + (size_t)s * T.recb, T.rec + (size_t)t * T.recb, (unsigned)T.recb, &mbar[s]);
        if (trace) trace[8 * t] = gtimer();
      }
    }
  }
  __syncthreads();
  double rhs_c = 0.0;  // per-pass constant of a scalar right-hand side (the mean shift)
  if constexpr (Rhs::kScalar) rhs_c = rhs.pass_const();
  for (int it = 0;; ++it) {
    const int s = it % D;
    const int t = ids[s];
    if (t >= T.ntiles) break;
    unsigned nxt = 0;
    if (tid == 0) nxt = atomicAdd(&c.ctr[ctr_task], 1u);  // the slot's refill; used after barrier 2
    const unsigned char* buf = rp_sm + (size_t)s * T.recb;
    if (trace && tid == 0) trace[8 * t + 7] = gtimer();  // rpipe: [7] = became the CTA's current tile
    mbar_wait(&mbar[s], (unsigned)(it / D) & 1u);
    if (trace && tid == 0) trace[8 * t + 6] = gtimer();  // rpipe: [6] = record landed
    const int nr = *reinterpret_cast<const int*>(buf);
    const int* rowa = reinterpret_cast<const int*>(buf + lay.o_row);
    const int* ina = reinterpret_cast<const int*>(buf + lay.o_in);
    const unsigned short* erp = reinterpret_cast<const unsigned short*>(buf + lay.o_rp);
    const unsigned short* esl = reinterpret_cast<const unsigned short*>(buf + lay.o_slot);
    const double* ev = reinterpret_cast<const double*>(buf + lay.o_val);
    const double* ib = reinterpret_cast<const double*>(buf + lay.o_inv);
    const int row = k < nr ? rowa[k] : -1;
    // the tile's distinct inputs, one poller each: first loads go out now
    constexpr int NH = kWide ? 2 : 1;
    int icol[NH];
    long long pv[NH] = {};
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      const int j = tid + h * nth;
      icol[h] = j < T.xs ? ina[j] : -1;
      if (icol[h] >= 0)
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(pv[h]) : "l"(&xg[icol[h]]) : "memory");
    }
    double b;
    if constexpr (Rhs::kScalar) {
      b = rhs.load(row);  // finished (mean shift) after the inputs have landed
    } else {
      b = rhs.template eval<4>(row, g);  // 4 consecutive lanes per row; valid in all four
    }
    // inverse entries inv[k][g+4j] from the ring slot into registers
    double a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = tid >= 16 * j ? ib[rp_inv_base(j) - 16 * j + tid] : 0.0;
    if (g == 0 && row >= 0) {  // sentinel resets folded into the pass (BD_FOLD_FILL)
      if (reset0) reset0[row] = __longlong_as_double(SENTINEL);
      if (reset1 && row < T.reset1_n) reset1[row] = __longlong_as_double(SENTINEL);
    }
    if (trace && tid == 0) trace[8 * t + 5] = gtimer();
#pragma unroll
    for (int h = 0; h < NH; ++h) {
      if (icol[h] < 0) continue;
      const double* pj = &xg[icol[h]];
      long long v = pv[h];
      while (v == SENTINEL)
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(pj) : "memory");
      xin[tid + h * nth] = __longlong_as_double(v);
    }
    __syncthreads();  // barrier 1: inputs in shared memory
    if (trace && tid == 0) trace[8 * t + 4] = gtimer();
    {
      const int kc = k < nr ? k : 0;
      const int e0 = erp[kc], e1 = k < nr ? erp[kc + 1] : e0;
      double acc = 0.0;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        if (h >= 2 && 4 * h >= T.exw) break;  // rows with > 8 entries: heart-first torso rows
        const int e = e0 + g + 4 * h;
        const bool ok = e < e1;
        const int ei = ok ? e : 0;
        const int sl = ok ? (int)esl[ei] : T.xs;
        acc = fma(ev[ei], xin[sl], acc);
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if constexpr (Rhs::kScalar) b = rhs.finish(b, rhs_c);
      if (g == 0) ys[k] = row >= 0 ? __dsub_rn(b, acc) : 0.0;
    }
    __syncthreads();  // barrier 2: y in shared memory; the ring slot is free
    if (trace && tid == 0) trace[8 * t + 1] = gtimer();
    {
      double sm[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j <= jmax) sm[j & 3] = fma(a[j], ys[g + 4 * j], sm[j & 3]);
      double x = (sm[0] + sm[1]) + (sm[2] + sm[3]);
      x += __shfl_xor_sync(0xffffffffu, x, 1);
      x += __shfl_xor_sync(0xffffffffu, x, 2);
      if (g == 0 && row >= 0) publish(&xg[row], x);
    }
    // refill the slot (free since barrier 2) once this thread's rows are published, so the
    // copy's set-up does not delay them
    if (tid == 0) {
      ids[s] = (int)nxt;  // read at the top of iteration it + D (D >= 2: a barrier in between)
      if ((int)nxt < T.ntiles) {
        tma_fetch(rp_sm + (size_t)s * T.recb, T.rec + (size_t)nxt * T.recb, (unsigned)T.recb, &mbar[s]);
        if (trace) trace[8 * (size_t)nxt] = gtimer();
      }
    }
    if (trace && tid == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      trace[8 * t + 2] = gtimer();
      trace[8 * t + 3] = ((unsigned long long)smid << 32) | blockIdx.x;
    }
  }
  if (tid == 0) {
    __threadfence();
    const unsigned d = atomicAdd(&c.ctr[ctr_done], 1u);
    last_s = (d == gridDim.x - 1u);
  }
  __syncthreads();
  if (last_s && tid == 0) {
    c.ctr[ctr_task] = 0u;
    c.ctr[ctr_done] = 0u;
    __threadfence();
  }
}

// ---- pipelined register-tile triangular solve ---------------------------------
// k_trsv_rtile with the tile's preparation taken off its critical path: every
// array a tile needs (inverse, right-hand side in tile order, rows, inputs,
// external entries) sits at a fixed per-tile stride, so the whole preparation
// is ONE group of cp.async copies into a shared-memory buffer.  A CTA grabs
// its next tile as soon as it starts on the current one and streams the next
// tile's group into the second buffer while it polls and computes (two tiles
// in flight per CTA; deadlock-free because a CTA finishes its tiles in grab
// order and the smallest unfinished tile is always being worked on).  The
// right-hand side is gathered into tile order by k_tile_rhs before the
// forward pass; the forward pass writes its output both to the polled buffer
// and, through `opos`, into the backward pass's tile-ordered right-hand side.
struct PBuf {
  double* inv;
  double* b;
  double* ev;
  int* row;
  int* icol;
  int* opos;
  unsigned short* esl;
  unsigned short* erp;
};
__host__ __device__ constexpr size_t pt_buf_bytes(int rs, int xs, int is, int es, int rps) {
  return 8 * ((size_t)is + 2) + 8 * (size_t)rs + 8 * (size_t)es + 4 * (size_t)rs + 4 * (size_t)xs +
         4 * (size_t)rs + 2 * (size_t)es + 2 * (size_t)rps;
}
__host__ __device__ constexpr size_t pt_smem(int rs, int xs, int is, int es, int rps) {
  return 8 * ((size_t)RT_ROWS + xs + 2) + 2 * pt_buf_bytes(rs, xs, is, es, rps);
}
__device__ __forceinline__ PBuf pt_view(char* p, const BTileDev& T) {
  PBuf B;
  B.inv = reinterpret_cast<double*>(p);
  p += 8 * ((size_t)T.is + 2);
  B.b = reinterpret_cast<double*>(p);
  p += 8 * (size_t)T.rs;
  B.ev = reinterpret_cast<double*>(p);
  p += 8 * (size_t)T.es;
  B.row = reinterpret_cast<int*>(p);
  p += 4 * (size_t)T.rs;
  B.icol = reinterpret_cast<int*>(p);
  p += 4 * (size_t)T.xs;
  B.opos = reinterpret_cast<int*>(p);
  p += 4 * (size_t)T.rs;
  B.esl = reinterpret_cast<unsigned short*>(p);
  p += 2 * (size_t)T.es;
  B.erp = reinterpret_cast<unsigned short*>(p);
  return B;
}
// one commit group: everything tile t needs (strides are 16-byte multiples)
template <bool kOut>
__device__ __forceinline__ void pt_issue(const BTileDev& T, const int* __restrict__ opos_g,
                                         const double* __restrict__ bt, const PBuf& B, int t) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int64_t tt = t;
  for (int q = tid; 2 * q < T.is; q += nth) cp_async16(B.inv + 2 * q, T.inv + tt * T.is + 2 * q);
  for (int q = tid; 2 * q < T.rs; q += nth) cp_async16(B.b + 2 * q, bt + tt * T.rs + 2 * q);
  for (int q = tid; 2 * q < T.es; q += nth) cp_async16(B.ev + 2 * q, T.ent_val + tt * T.es + 2 * q);
  for (int q = tid; 4 * q < T.rs; q += nth) cp_async16(B.row + 4 * q, T.task_row + tt * T.rs + 4 * q);
  for (int q = tid; 4 * q < T.xs; q += nth) cp_async16(B.icol + 4 * q, T.in_col + tt * T.xs + 4 * q);
  if constexpr (kOut)
    for (int q = tid; 4 * q < T.rs; q += nth) cp_async16(B.opos + 4 * q, opos_g + tt * T.rs + 4 * q);
  for (int q = tid; 8 * q < T.es; q += nth) cp_async16(B.esl + 8 * q, T.ent_slot + tt * T.es + 8 * q);
  for (int q = tid; 8 * q < T.rps; q += nth) cp_async16(B.erp + 8 * q, T.ent_rp + tt * T.rps + 8 * q);
  cp_async_commit();
}

template <bool kOut>
__global__ void __launch_bounds__(256, 4) k_trsv_ptile(BTileDev T, const int* __restrict__ opos_g,
                                                       const double* __restrict__ bt,
                                                       double* __restrict__ xg,
                                                       double* __restrict__ bt_next, Ctl c,
                                                       int ctr_task, int ctr_done) {
  if (inactive(c)) return;
  extern __shared__ __align__(16) double pt_sm[];
  double* ys = pt_sm;          // RT_ROWS
  double* xin = ys + RT_ROWS;  // xs inputs + zero slot
  char* bufs = reinterpret_cast<char*>(xin + T.xs + 2);
  const size_t bufb = pt_buf_bytes(T.rs, T.xs, T.is, T.es, T.rps);
  __shared__ int task_s;
  __shared__ int last_s;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int k = warp * 8 + (lane >> 2);
  const int g = lane & 3;
  const int jmax = (8 * warp + 7) >> 2;
  if (tid == 0) {
    xin[T.xs] = 0.0;
    reinterpret_cast<double*>(bufs)[T.is] = 0.0;  // zero slots after each inverse
    reinterpret_cast<double*>(bufs + bufb)[T.is] = 0.0;
    task_s = (int)atomicAdd(&c.ctr[ctr_task], 1u);
  }
  __syncthreads();
  int t = task_s;
  int nr = 0;
  if (t < T.ntiles) {
    pt_issue<kOut>(T, opos_g, bt, pt_view(bufs, T), t);
    nr = T.tile_nr[t];
  }
  int cur = 0;
  while (t < T.ntiles) {
    __syncthreads();  // everyone has read task_s / finished the previous tile
    if (tid == 0) task_s = (int)atomicAdd(&c.ctr[ctr_task], 1u);
    __syncthreads();
    const int tn = task_s;
    int nr_n = 0;
    if (tn < T.ntiles) {
      pt_issue<kOut>(T, opos_g, bt, pt_view(bufs + (cur ^ 1) * bufb, T), tn);
      nr_n = T.tile_nr[tn];
    } else {
      cp_async_commit();  // empty group: keeps wait_group<1> meaning "the current tile"
    }
    unsigned long long* trace = g_tile_trace;
    if (trace && tid == 0) trace[8 * t] = gtimer();
    cp_async_wait<1>();
    __syncthreads();
    const PBuf Bc = pt_view(bufs + cur * bufb, T);
    if (trace && tid == 0) trace[8 * t + 5] = gtimer();
    const int row = k < nr ? Bc.row[k] : -1;
    const int op = kOut && k < nr ? Bc.opos[k] : -1;
    // inverse entries inv[k][g+4j] into registers (branch-free: zero slot)
    double a[16];
    {
      int idx = g * nr - ((g * (g - 1)) >> 1) + (k - g);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int l = g + 4 * j;
        a[j] = (j <= jmax) ? Bc.inv[(l <= k && k < nr) ? idx : T.is] : 0.0;
        idx += 4 * nr - 4 * l - 10;
      }
    }
    // the tile's distinct inputs: one poller each
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = tid + h * nth;
      if (j >= T.xs) continue;
      const int col = Bc.icol[j];
      if (col < 0) continue;
      const double* pj = &xg[col];
      long long v;
      asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(pj) : "memory");
      while (v == SENTINEL)
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(pj) : "memory");
      xin[j] = __longlong_as_double(v);
    }
    __syncthreads();
    if (trace && tid == 0) trace[8 * t + 4] = gtimer();
    {
      const int kc = k < nr ? k : 0;
      const int e0 = Bc.erp[kc], e1 = k < nr ? Bc.erp[kc + 1] : e0;
      double acc = 0.0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = e0 + g + 4 * h;
        const bool ok = e < e1;
        const int ei = ok ? e : 0;
        const int sl = ok ? (int)Bc.esl[ei] : T.xs;
        acc = fma(Bc.ev[ei], xin[sl], acc);
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      if (g == 0) ys[k] = row >= 0 ? __dsub_rn(Bc.b[k], acc) : 0.0;
    }
    if (trace && tid == 0) trace[8 * t + 6] = gtimer();
    __syncthreads();
    if (trace && tid == 0) trace[8 * t + 1] = gtimer();
    {
      double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j <= jmax) s[j & 3] = fma(a[j], ys[g + 4 * j], s[j & 3]);
      double x = (s[0] + s[1]) + (s[2] + s[3]);
      x += __shfl_xor_sync(0xffffffffu, x, 1);
      x += __shfl_xor_sync(0xffffffffu, x, 2);
      if (g == 0 && row >= 0) {
        publish(&xg[row], x);
        if constexpr (kOut) bt_next[op] = x;
      }
    }
    if (trace && tid == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      trace[8 * t + 7] = gtimer();
      trace[8 * t + 2] = gtimer();
      trace[8 * t + 3] = ((unsigned long long)smid << 32) | blockIdx.x;
    }
    t = tn;
    nr = nr_n;
    cur ^= 1;
  }
  cp_async_wait<0>();
  if (tid == 0) {
    __threadfence();
    const unsigned d = atomicAdd(&c.ctr[ctr_done], 1u);
    last_s = (d == gridDim.x - 1u);
  }
  __syncthreads();
  if (last_s && tid == 0) {
    c.ctr[ctr_task] = 0u;
    c.ctr[ctr_done] = 0u;
    __threadfence();
  }
}

// Right-hand side of a tile pass gathered into tile order (slot t*rs + k),
// plus the sentinel fill of the pass's polled output.  Gather right-hand
// sides (the fused Schur product) use 4 lanes per slot.
template <class Rhs>
__global__ void __launch_bounds__(256) k_tile_rhs(const int* __restrict__ task_row, int64_t nslots,
                                                  Rhs rhs, double* __restrict__ bt,
                                                  double* __restrict__ fill, int64_t nfill, Ctl c) {
  if (inactive(c)) return;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < nfill; i += nthr) fill[i] = __longlong_as_double(SENTINEL);
  if constexpr (Rhs::kScalar) {
    for (int64_t s = tid; s < nslots; s += nthr) bt[s] = rhs.template eval<1>(task_row[s], 0);
  } else {
    // whole warps per iteration (the gather shuffles within groups of 4 lanes)
    const int64_t nq = (nslots + 7) / 8 * 32;  // lanes needed, rounded to warps
    for (int64_t q = tid - (threadIdx.x & 31); q < nq; q += nthr) {
      const int64_t s = (q + (threadIdx.x & 31)) / 4;
      const int row = s < nslots ? task_row[s] : -1;
      const double v = rhs.template eval<4>(row, threadIdx.x & 3);
      if ((threadIdx.x & 3) == 0 && s < nslots) bt[s] = v;
    }
  }
}

// ---- persistent sync-free triangular solve ----------------------------------
// Tasks (rows) in level order, ELL entries (G per row, column -1 = padding)
// stored in task order so a chunk of rows is one contiguous, coalesced read.
// A persistent grid sized to keep only ~3 levels of rows in flight grabs
// chunks in order with an atomic counter (a chunk only depends on lower
// chunks, all owned by running blocks => no deadlock) and polls its
// dependencies with a short nanosleep backoff, keeping L2 poll traffic low.
struct EllTri {
  const int* task_row;
  const double* task_diag;
  const int* ell_col;
  const double* ell_val;
  int ntasks;
};

// Staggered polling: keep several polls of the same word in flight, issued
// ~STAGGER ns apart, so a value that lands is seen about one one-way L2
// latency later instead of up to a full round trip.
__device__ __forceinline__ long long ld_relaxed_bits(const double* p) {
  long long b;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(b) : "l"(p) : "memory");
  return b;
}
__device__ __forceinline__ double spin_load_staggered(const double* p) {
  long long b0 = ld_relaxed_bits(p);
  if (b0 != SENTINEL) return __longlong_as_double(b0);
  for (;;) {
    __nanosleep(60);
    const long long b1 = ld_relaxed_bits(p);
    __nanosleep(60);
    const long long b2 = ld_relaxed_bits(p);
    __nanosleep(60);
    const long long b3 = ld_relaxed_bits(p);
    if (b1 != SENTINEL) return __longlong_as_double(b1);
    if (b2 != SENTINEL) return __longlong_as_double(b2);
    if (b3 != SENTINEL) return __longlong_as_double(b3);
  }
}

__device__ __forceinline__ double spin_load_backoff(const double* p) {
  long long b;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(b) : "l"(p) : "memory");
  while (b == SENTINEL) {
    __nanosleep(32);
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(b) : "l"(p) : "memory");
  }
  return __longlong_as_double(b);
}

template <int G, class Rhs>
__global__ void __launch_bounds__(TPB) k_trsv_persist(EllTri t, Rhs rhs, double* __restrict__ y,
                                                      Ctl c, int ctr_chunk, int ctr_done,
                                                      int nchunks, int fin, int slot, int slot2,
                                                      int64_t nmean) {
  if (inactive(c)) return;
  __shared__ int chunk_s[2];
  __shared__ int last_s;
  __shared__ double sm[32];
  const int rpc = TPB / G;
  const int grp = threadIdx.x / G, lane = threadIdx.x % G;
  // a chunk's inputs, loaded one chunk ahead of its processing
  struct Pre {
    int task, row, col;
    double val, diag, b;
  };
  auto load = [&](int chunk, Pre& p) {
    p.task = chunk * rpc + grp;
    p.row = (chunk < nchunks && p.task < t.ntasks) ? t.task_row[p.task] : -1;
    p.b = rhs.template eval<G>(p.row, lane);
    p.col = p.row >= 0 ? t.ell_col[(int64_t)p.task * G + lane] : -1;
    p.val = p.row >= 0 ? t.ell_val[(int64_t)p.task * G + lane] : 0.0;
    p.diag = p.row >= 0 ? t.task_diag[p.task] : 1.0;
  };
  if (threadIdx.x == 0) chunk_s[0] = (int)atomicAdd(&c.ctr[ctr_chunk], 1u);
  __syncthreads();
  int chunk = chunk_s[0];
  Pre cur;
  load(chunk, cur);
  int par = 0;
  while (chunk < nchunks) {
    // grab and prefetch the next chunk before waiting on this one
    if (threadIdx.x == 0) chunk_s[par ^ 1] = (int)atomicAdd(&c.ctr[ctr_chunk], 1u);
    __syncthreads();
    const int next = chunk_s[par ^ 1];
    Pre nx;
    load(next, nx);
    double a = 0.0;
#ifdef BD_STAGGER
    if (cur.col >= 0) a = cur.val * spin_load_staggered(&y[cur.col]);
#else
    if (cur.col >= 0) a = cur.val * spin_load(&y[cur.col]);
#endif
    a = group_sum<G>(a);  // every lane of the warp reaches the shuffle
    double val = 0.0;
    if (cur.row >= 0) {
      val = __ddiv_rn(__dsub_rn(cur.b, a), cur.diag);
      if (lane == 0) publish(&y[cur.row], val);
    }
    if (fin >= 0) {
      const double v = block_sum(lane == 0 && cur.row >= 0 ? val : 0.0, sm);
      if (threadIdx.x == 0) c.partials[chunk] = v;
    }
    cur = nx;
    chunk = next;
    par ^= 1;
  }
  // completion: the last block finalises the (optional) mean and resets counters
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned d = atomicAdd(&c.ctr[ctr_done], 1u);
    last_s = (d == gridDim.x - 1u);
  }
  __syncthreads();
  if (last_s) {
    __threadfence();
    if (fin >= 0) {
      double tot[1];
      tot[0] = sum_partials(c.partials, nchunks, 0, sm);
      if (threadIdx.x == 0) finalize(c, fin, slot, slot2, tot, nmean);
    }
    if (threadIdx.x == 0) {
      c.ctr[ctr_chunk] = 0u;
      c.ctr[ctr_done] = 0u;
      __threadfence();
    }
  }
}

// ---- supernodal triangular solve (exact / Cholesky factors) -----------------------
// A supernode is a run of consecutive rows [c0, c0+ns) whose mutual
// dependencies form a dense triangle (the separators of a nested-dissection
// factor).  One CTA owns a supernode task: (1) the external sparse dots of all
// its rows in parallel (warp per row, polling only other supernodes), then
// (2) the dense diagonal block in 32-row panels: one warp solves a panel with
// shuffles, all warps update the remaining rows.  Tasks (supernodes in DAG
// level order) are taken in order by a persistent grid, so the row-level
// chain through a separator no longer costs one cross-SM round trip per row.
struct SuperTri {
  int n;
  const int* rowptr;
  const int* col;
  const double* val;
  const int* sn_start;  // per supernode (level order): first row
  const int* sn_size;   // per supernode: rows
  const int* task_sn;   // per task: first supernode; tasks = [task_sn[t], task_sn[t+1])
  int ntasks;           // a task is either ONE big supernode (> 32 rows) or up to
                        // 16 small independent ones (same level), one per warp
  const int* perm;      // nullable: scatter of the output (original order)
  // split external phase of big forward supernodes (nullable): task_kind 1 =
  // chunk of SN_CHUNK rows (first row task_arg) whose b - L_ext x_ext goes to
  // rext; task_kind 2 = the supernode's dense phase, waiting for task_arg
  // chunks on sn_cnt[supernode]
  const int* task_kind;
  const int* task_arg;
  int* sn_cnt;
  double* rext;
  // dense phase of big supernodes (nullable): inverses of the 32x32 diagonal
  // blocks of every panel, in solve order, pinv[(panel*32 + l)*32 + m], the
  // supernode's first panel at sn_pan[supernode]
  const double* pinv;
  const int* sn_pan;
  const int* task_w;  // small-supernode tasks: lanes per supernode (nullable: 32)
  // dense phase of the largest supernodes (nullable): the whole diagonal
  // block's inverse in solve order, packed lower rows (row l at l(l+1)/2),
  // starting at sn_inv[supernode] (-1: panels)
  const double* sinv;
  const long long* sn_inv;
  int dchunk;  // rows per dense-phase slice (kind-3 tasks)
};

constexpr int SN_MAX = 1024;
constexpr int SN_CHUNK = 64;  // rows per external-phase chunk (16 warps x RW 4)

// One warp solves one small supernode (<= 32 rows): external dots RW rows at
// a time, then the dense triangle with the coefficients in registers.
// W: lanes per supernode (4, 8, 16 or 32; 32/W supernodes share a warp, all
// lanes take part in the shuffles, ns = 0 marks an idle group).
template <bool LOWER, class Rhs>
__device__ __forceinline__ void super_small_warp(const SuperTri& t, const Rhs& rhs,
                                                 double* __restrict__ x,
                                                 double* __restrict__ out, int c0, int ns,
                                                 int lane, int W = 32) {
  const int c1 = c0 + ns;
  // lane l owns the l-th row in solve order: its right-hand side minus its
  // external part, entries walked sequentially, 4 loads in flight
  double ri = 0.0;
  {
    const int k = LOWER ? lane : ns - 1 - lane;
    const bool ok = lane < ns;
    const int i = ok ? c0 + k : -1;
    int eb = 0, ee = 0;
    if (ok) {
      const int b = t.rowptr[i], e = t.rowptr[i + 1];
      eb = LOWER ? b : b + (c1 - i);
      ee = LOWER ? e - 1 - k : e;
    }
    double acc = 0.0;
    for (int q = eb; q < ee; q += 4) {
      int cl[4];
      double vl[4], xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool in = q + u < ee;
        cl[u] = in ? t.col[q + u] : -1;
        vl[u] = in ? t.val[q + u] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) xv[u] = ld_relaxed_if(&x[cl[u] < 0 ? 0 : cl[u]], cl[u] >= 0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        double d = xv[u];
        if (cl[u] >= 0 && __double_as_longlong(d) == SENTINEL) d = spin_load(&x[cl[u]]);
        acc = fma(vl[u], d, acc);
      }
    }
    const double bi = rhs.template eval<1>(i, 0);
    if (ok) ri = __dsub_rn(bi, acc);
  }
  // dense triangle: lane l owns the l-th row in solve order
  const bool ok = lane < ns;
  const int k = LOWER ? lane : ns - 1 - lane;
  const int i = ok ? c0 + k : c0;
  double diag = 1.0;
  int base = 0;
  if (ok) {
    const int b = t.rowptr[i], e = t.rowptr[i + 1];
    diag = LOWER ? t.val[e - 1] : t.val[b];
    base = LOWER ? (e - 1 - k) : b;
  }
  // the pivot's reciprocal, formed by every lane at once off the chain: each
  // step of the chain then multiplies instead of dividing (DDIV ~68 cycles vs
  // DMUL 8; the result moves by at most an ulp)
  const double dinv = 1.0 / diag;
  // coefficients fetched 8 steps ahead instead of held in 32 registers (keeps
  // the kernel at 2 CTAs/SM); the loads are off the shuffle chain
  auto coef = [&](int jj) -> double {
    if (!(ok && jj < lane)) return 0.0;
    const int kj = LOWER ? jj : ns - 1 - jj;
    const int j = c0 + kj;
    return __ldg(&t.val[LOWER ? base + (j - c0) : base + (j - i)]);
  };
  double win[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) win[u] = coef(u);
  // loop bound uniform over the warp (W); groups with fewer rows idle through
  // the tail (the shuffles need every lane)
  const int nsw = __reduce_max_sync(0xffffffffu, ns);
  for (int j0 = 0; j0 < nsw; j0 += 8) {
    double nxt[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) nxt[u] = coef(j0 + 8 + u);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int jj = j0 + u;
      if (jj >= nsw) break;
      const double rj = __shfl_sync(0xffffffffu, ri, jj, W);
      const double dj = __shfl_sync(0xffffffffu, dinv, jj, W);
      if (jj < ns) {
        const double xj = __dmul_rn(rj, dj);
        if (lane == jj) ri = xj;
        if (ok && lane > jj) ri = __dsub_rn(ri, __dmul_rn(win[u], xj));
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) win[u] = nxt[u];
  }
  if (ok) {
    publish(&x[i], ri);
    if (out) out[t.perm ? t.perm[i] : i] = ri;
  }
}

// External phase of a big supernode: r[k] = b_k - L_k,ext x_ext for rows
// [kbeg, kend) of the supernode (c0, c1), RW rows per warp in flight, each
// row's entries lane-strided and combined with a warp sum.  dst is indexed by
// the row offset k (shared r, or rext + c0 for a chunk task).
template <bool LOWER, int RW, class Rhs>
__device__ __forceinline__ void super_ext_rows(const SuperTri& t, const Rhs& rhs,
                                               double* __restrict__ x, int c0, int c1, int kbeg,
                                               int kend, double* dst) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int k0 = kbeg + warp * RW; k0 < kend; k0 += nw * RW) {
    int eb[RW], ee[RW];
    double sacc[RW];
#pragma unroll
    for (int u = 0; u < RW; ++u) {
      const int k = k0 + u;
      sacc[u] = 0.0;
      eb[u] = ee[u] = 0;
      if (k < kend) {
        const int i = c0 + k;
        const int b = t.rowptr[i], e = t.rowptr[i + 1];
        eb[u] = LOWER ? b : b + (c1 - i);
        ee[u] = LOWER ? e - 1 - k : e;
      }
    }
    int len = 0;
#pragma unroll
    for (int u = 0; u < RW; ++u) len = max(len, ee[u] - eb[u]);
    for (int q = lane; q < len; q += 32) {
      int cl[RW];
      double vl[RW], xv[RW];
#pragma unroll
      for (int u = 0; u < RW; ++u) {
        const bool ok = eb[u] + q < ee[u];
        cl[u] = ok ? t.col[eb[u] + q] : -1;
        vl[u] = ok ? t.val[eb[u] + q] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < RW; ++u) xv[u] = ld_relaxed_if(&x[cl[u] < 0 ? 0 : cl[u]], cl[u] >= 0);
#pragma unroll
      for (int u = 0; u < RW; ++u) {
        double d = xv[u];
        if (cl[u] >= 0 && __double_as_longlong(d) == SENTINEL) d = spin_load(&x[cl[u]]);
        sacc[u] = fma(vl[u], d, sacc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < RW; ++u) {
      const double sum = group_sum<32>(sacc[u]);
      const int k = k0 + u;
      const double bi = rhs.template eval<32>(k < kend ? c0 + k : -1, lane);
      if (lane == 0 && k < kend) dst[k] = __dsub_rn(bi, sum);
    }
  }
}

template <bool LOWER, class Rhs>
__global__ void __launch_bounds__(512, 2) k_trsv_super(SuperTri t, Rhs rhs, double* __restrict__ x,
                                                    double* __restrict__ out, Ctl c, int ctr_task,
                                                    int ctr_done) {
  if (inactive(c)) return;
  constexpr int RW = 4;  // rows per warp in flight
  __shared__ double r[SN_MAX];
  __shared__ double panel[32][33];
  __shared__ int task_s;
  __shared__ int last_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (;;) {
    if (threadIdx.x == 0) task_s = (int)atomicAdd(&c.ctr[ctr_task], 1u);
    __syncthreads();
    const int task = task_s;
    __syncthreads();
    if (task >= t.ntasks) break;
    const int s0 = t.task_sn[task], s1 = t.task_sn[task + 1];
    const int kind = t.task_kind ? t.task_kind[task] : 0;
    if (kind == 1) {  // external-phase chunk of a big supernode
      const int c0 = t.sn_start[s0], ns = t.sn_size[s0];
      const int kb = t.task_arg[task], ke = min(ns, kb + SN_CHUNK);
      super_ext_rows<LOWER, RW>(t, rhs, x, c0, c0 + ns, kb, ke, t.rext + c0);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(t.sn_cnt + s0, 1);
      }
      continue;
    }
    if (kind == 3) {
      // one slice of a big supernode's dense phase through its whole-block
      // inverse: wait for the supernode's external-phase chunks (y in rext),
      // then rows [l0, l1) of x = X y, published as they complete
      const int a = t.task_arg[task], nch = a & 0xff, part = (a >> 8) & 0xff, nparts = a >> 16;
      const int c0 = t.sn_start[s0], ns = t.sn_size[s0];
      if (threadIdx.x == 0) {
        const volatile int* cnt = t.sn_cnt + s0;
        while (*cnt < nch) __nanosleep(64);
      }
      __syncthreads();
      for (int k = threadIdx.x; k < ns; k += blockDim.x) r[k] = ld_relaxed_if(&t.rext[c0 + k], true);
      __syncthreads();
      const double* X = t.sinv + t.sn_inv[s0];
      const int l0 = part * t.dchunk, l1 = min(ns, l0 + t.dchunk);
      for (int l = l0 + warp; l < l1; l += nw) {
        const double* xr = X + (long long)l * (l + 1) / 2;
        double acc = 0.0;
        for (int m = lane; m <= l; m += 32) acc = fma(__ldg(&xr[m]), r[LOWER ? m : ns - 1 - m], acc);
        const double v = group_sum<32>(acc);
        if (lane == 0) {
          const int i = c0 + (LOWER ? l : ns - 1 - l);
          publish(&x[i], v);
          if (out) out[t.perm ? t.perm[i] : i] = v;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        // the last slice resets the counter for the next pass (every slice
        // has passed its wait once all of them have counted in)
        if (atomicAdd(t.sn_cnt + s0, 1) == nch + nparts - 1) t.sn_cnt[s0] = 0;
      }
      continue;
    }
    unsigned long long t_beg = 0;
    // trace (debug): steps > 0 traces the backward passes, < 0 the forward ones
    const int tsteps = g_tile_trace_steps < 0 ? -g_tile_trace_steps : g_tile_trace_steps;
    unsigned long long* trace = ((g_tile_trace_steps < 0) == LOWER) ? g_tile_trace : nullptr;
    if (trace && threadIdx.x == 0) t_beg = gtimer();
    if (s1 - s0 > 1 || t.sn_size[s0] <= 32) {
      // group of small independent supernodes: W lanes each (32/W per warp),
      // no CTA barrier
      const int W = t.task_w ? t.task_w[task] : 32;
      const int sidx = s0 + warp * (32 / W) + lane / W;
      const bool has = sidx < s1;
      if (warp * (32 / W) < s1 - s0)
        super_small_warp<LOWER>(t, rhs, x, out, has ? t.sn_start[sidx] : 0,
                                has ? t.sn_size[sidx] : 0, lane % W, W);
      if (trace) {
        __syncthreads();
        if (threadIdx.x == 0 && task < tsteps) {
          trace[task * 4 + 0] = t_beg;
          trace[task * 4 + 1] = gtimer();
          trace[task * 4 + 2] = blockIdx.x;
          trace[task * 4 + 3] = (unsigned long long)(s1 - s0);
        }
      }
      continue;
    }
    const int c0 = t.sn_start[s0], ns = t.sn_size[s0], c1 = c0 + ns;
    if (kind == 2) {
      // (1) precomputed by the chunk tasks: wait for them, then stage r
      if (threadIdx.x == 0) {
        const volatile int* cnt = t.sn_cnt + s0;
        while (*cnt < t.task_arg[task]) __nanosleep(64);
        t.sn_cnt[s0] = 0;  // ready for the next pass
        __threadfence();
      }
      __syncthreads();
      for (int k = threadIdx.x; k < ns; k += blockDim.x)
        r[k] = ld_relaxed_if(&t.rext[c0 + k], true);
    } else {
      // (1) right-hand side minus the external part, RW rows per warp in flight
      super_ext_rows<LOWER, RW>(t, rhs, x, c0, c1, 0, ns, r);
    }
    __syncthreads();
    unsigned long long t_ext = 0;
    if (trace && threadIdx.x == 0) t_ext = gtimer();
    const long long inv_off = t.sn_inv ? t.sn_inv[s0] : -1;
    if (inv_off >= 0) {
      // (2') dense block through its precomputed inverse: x_l = sum_{m<=l}
      //      X[l][m] r_m, two rows per warp in flight, lane-strided rows
      const double* X = t.sinv + inv_off;
      for (int l0 = warp; l0 < ns; l0 += 2 * nw) {
        double acc[2] = {0.0, 0.0};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int l = l0 + h * nw;
          if (l < ns) {
            const double* xr = X + (long long)l * (l + 1) / 2;
            for (int m = lane; m <= l; m += 32)
              acc[h] = fma(__ldg(&xr[m]), r[LOWER ? m : ns - 1 - m], acc[h]);
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int l = l0 + h * nw;
          const double v = group_sum<32>(acc[h]);
          if (lane == 0 && l < ns) {
            const int i = c0 + (LOWER ? l : ns - 1 - l);
            publish(&x[i], v);
            if (out) out[t.perm ? t.perm[i] : i] = v;
          }
        }
      }
    } else
    // (2) dense block, left-looking 32-row panels (solve order: ascending rows
    //     for L, descending for U).  r[k] holds row k's rhs, then its solution.
    for (int p0 = 0; p0 < ns; p0 += 32) {
      const int pn = min(32, ns - p0);
      // panel inverse rows of this warp (rows warp, warp + nw), loaded before
      // the update so their latency hides behind it
      double pv[2] = {0.0, 0.0};
      const double* pinv = t.pinv ? t.pinv + ((int64_t)t.sn_pan[s0] + p0 / 32) * 1024 : nullptr;
      if (pinv) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int l = warp + h * nw;
          if (l < pn && lane <= l) pv[h] = __ldg(&pinv[l * 32 + lane]);
        }
      }
      // (a) panel rows minus the already solved rows [0, p0) of the block
      if (p0 > 0) {
        for (int w = warp; w < pn; w += nw) {
          const int k = LOWER ? p0 + w : ns - 1 - (p0 + w);
          const int i = c0 + k;
          const int b = t.rowptr[i], e = t.rowptr[i + 1];
          double s = 0.0;
          for (int jj = lane; jj < p0; jj += 32) {
            const int kj = LOWER ? jj : ns - 1 - jj;
            const int j = c0 + kj;
            const int pos = LOWER ? (e - 1 - k) + (j - c0) : b + (j - i);
            s = fma(t.val[pos], r[kj], s);
          }
          s = group_sum<32>(s);
          if (lane == 0) r[k] = __dsub_rn(r[k], s);
        }
        __syncthreads();
      }
      // (b) the panel triangle
      if (pinv) {
        // precomputed block inverse: x_l = sum_{m<=l} inv[l][m] r_m, one warp per row
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int l = warp + h * nw;
          if (l < pn) {
            const int km = LOWER ? p0 + lane : ns - 1 - (p0 + lane);
            double v = (lane <= l) ? pv[h] * r[km] : 0.0;
            v = group_sum<32>(v);
            if (lane == 0) panel[0][l] = v;
          }
        }
        __syncthreads();
        if (threadIdx.x < pn) {
          const int k = LOWER ? p0 + threadIdx.x : ns - 1 - (p0 + threadIdx.x);
          const int i = c0 + k;
          const double xi = panel[0][threadIdx.x];
          r[k] = xi;
          publish(&x[i], xi);
          if (out) out[t.perm ? t.perm[i] : i] = xi;
        }
      } else if (warp == 0) {
        // one warp, coefficients in shared memory
        const int k = LOWER ? p0 + lane : ns - 1 - (p0 + lane);
        const bool ok = lane < pn;
        const int i = ok ? c0 + k : c0;
        double diag = 1.0;
        if (ok) {
          const int b = t.rowptr[i], e = t.rowptr[i + 1];
          diag = LOWER ? t.val[e - 1] : t.val[b];
          const int base = LOWER ? (e - 1 - k) : b;
#pragma unroll 8
          for (int jj = 0; jj < 32; ++jj) {
            double a = 0.0;
            if (jj < lane) {
              const int kj = LOWER ? p0 + jj : ns - 1 - (p0 + jj);
              const int j = c0 + kj;
              a = LOWER ? t.val[base + (j - c0)] : t.val[base + (j - i)];
            }
            panel[lane][jj] = a;
          }
        }
        double ri = ok ? r[k] : 0.0;
        const double dinv = 1.0 / diag;  // (reciprocal off the chain, as above)
        __syncwarp();
        for (int jj = 0; jj < pn; ++jj) {
          const double rj = __shfl_sync(0xffffffffu, ri, jj);
          const double dj = __shfl_sync(0xffffffffu, dinv, jj);
          const double xj = __dmul_rn(rj, dj);
          if (lane == jj) ri = xj;
          if (ok && lane > jj) ri = __dsub_rn(ri, __dmul_rn(panel[lane][jj], xj));
        }
        if (ok) {
          r[k] = ri;
          publish(&x[i], ri);
          if (out) out[t.perm ? t.perm[i] : i] = ri;
        }
      }
      __syncthreads();
    }
    if (trace && threadIdx.x == 0 && task < tsteps) {
      trace[task * 4 + 0] = t_beg;
      trace[task * 4 + 1] = gtimer();
      trace[task * 4 + 2] = blockIdx.x;
      trace[task * 4 + 3] = ((t_ext - t_beg) << 20) | (1u << 19) | (unsigned)ns;
    }
  }
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned d = atomicAdd(&c.ctr[ctr_done], 1u);
    last_s = (d == gridDim.x - 1u);
  }
  __syncthreads();
  if (last_s && threadIdx.x == 0) {
    c.ctr[ctr_task] = 0u;
    c.ctr[ctr_done] = 0u;
    __threadfence();
  }
}


}  // namespace dev
}  // namespace bd
