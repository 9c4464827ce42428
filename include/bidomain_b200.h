/*
 * bidomain_b200.h — C ABI of the B200-native bidomain PCG hot path.
 *
 * The reference (arxiv/paper_1711_08708, /root/reference/pkg/src/bidomain) is a
 * pure-Python package; its "FFI" is the set of Python objects that the time
 * loop and the tests call.  Each entry point below replaces one of those
 * calls (file:line cites the reference symbol it stands in for).  The Python
 * mirror (paper_1711_08708_b200/) binds this header with ctypes; see
 * INTEGRATION.md for the binding a maintainer of the reference would add.
 *
 * Conventions
 *  - All arithmetic is fp64.  Vectors live in DEVICE memory and are passed as
 *    raw pointers owned by the caller; a block vector (u ∈ R^n, v ∈ R^m) is ONE
 *    contiguous buffer of n+m doubles, u first (bd/system.py:29-47).
 *  - Matrices are passed once, as HOST CSR arrays (int64 indptr, int32
 *    indices, double values, sorted column indices); the library copies them
 *    to the device and owns the copy.
 *  - Every call is asynchronous on the handle's context stream except the ones
 *    documented as synchronising (they return host-visible results).
 *  - Every function returns a bd_status; on failure bd_last_error(ctx) holds
 *    the message of the calling thread's last failing call.  Handles are
 *    thread-compatible, not thread-safe; different handles may be set up on
 *    different threads at once.
 */
#ifndef BIDOMAIN_B200_H
#define BIDOMAIN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the Python layer maps them onto the reference exception types
 * (bd/errors.py:4-44): EINVAL→ValueError, EPRECOND→PreconditionerError,
 * ENOCONV→NonConvergenceError, EBREAKDOWN→NumericalBreakdownError. */
typedef enum {
  BD_OK = 0,
  BD_EINVAL = 1,
  BD_EPRECOND = 2,
  BD_ENOCONV = 3,
  BD_EBREAKDOWN = 4,
  BD_ECUDA = 5,
  BD_ENOMEM = 6
} bd_status;

/* Inner preconditioner kinds; names as INNER_NAMES (bd/precond.py:31). */
typedef enum { BD_INNER_EXACT = 0, BD_INNER_IC0 = 1, BD_INNER_JACOBI = 2 } bd_inner_kind;

typedef struct bd_ctx bd_ctx;         /* device + stream + scratch */
typedef struct bd_csr bd_csr;         /* device CSR matrix */
typedef struct bd_system bd_system;   /* Λ = [[S_1, Π^T S_i],[S_i Π, γ M_H + S_i]] */
typedef struct bd_inner bd_inner;     /* exact / ic0 / jacobi inner solve */
typedef struct bd_prec bd_prec;       /* block-LU preconditioner P_Λ */
typedef struct bd_shard bd_shard;     /* one rank of the mesh-partitioned PCG */

/* Solve statistics (bd/krylov.py:23-38).  Filled even on error. */
typedef struct {
  int64_t iterations;
  int64_t mv_count;
  int64_t p1_count;
  int64_t pk_count;
  int32_t converged;
  int32_t status;          /* bd_status of the solve */
  double wall_ms;          /* host wall time of the call */
  double device_ms;        /* CUDA-event time of the solve on the stream */
  double final_residual;   /* last entry of the residual history */
  double curvature;        /* d·q at a breakdown (NaN otherwise) */
} bd_stats;

/* ---- context ---------------------------------------------------------- */
bd_status bd_ctx_create(int device, void* stream, bd_ctx** out);
bd_status bd_ctx_destroy(bd_ctx* ctx);
bd_status bd_ctx_set_stream(bd_ctx* ctx, void* stream);
bd_status bd_ctx_synchronize(bd_ctx* ctx);
const char* bd_last_error(bd_ctx* ctx);
/* Library version / build tag (sm_100a). */
const char* bd_version(void);

/* ---- sparse matrices (scipy CSR `@`, bd/system.py:111-113) ------------- */
bd_status bd_csr_create(bd_ctx* ctx, int64_t nrows, int64_t ncols, int64_t nnz,
                        const int64_t* indptr, const int32_t* indices,
                        const double* values, bd_csr** out);
bd_status bd_csr_destroy(bd_csr* a);
/* y = alpha*A*x + beta*y (device pointers). */
bd_status bd_spmv(bd_csr* a, const double* x, double* y, double alpha, double beta);
/* y = alpha * A [x ; x_ghost] + beta * y with the input split in two device
 * arrays: column c < nsplit reads x[c], column c >= nsplit reads
 * x_ghost[c - nsplit] (a sharded rank's owned entries and its halo, without
 * concatenating them).  Uses the ELL copy bd_csr_create builds for short,
 * near-uniform rows (P1 stencils), else the CSR rows. */
bd_status bd_spmv_split(bd_csr* a, const double* x, int64_t nsplit, const double* x_ghost,
                        double* y, double alpha, double beta);

/* ---- vector primitives (BlockVector.dot/norm, bd/system.py:39-43) ------ */
/* Deterministic fixed-order dot product; synchronising (result on host). */
bd_status bd_dot(bd_ctx* ctx, int64_t n, const double* x, const double* y, double* out);
/* Euclidean mean (numpy .mean(), bd/krylov.py:42); synchronising. */
bd_status bd_mean(bd_ctx* ctx, int64_t n, const double* x, double* out);

/* ---- coupled operator (BidomainSystem, bd/system.py:50-150) ----------- */
/* S1: n×n bulk stiffness (stiff_total), Si: m×m intra stiffness; mass: host
 * diag(M) (n), heart_mass: host diag(M_H) (m); gamma = χ c_m / dt. */
bd_status bd_system_create(bd_ctx* ctx, bd_csr* S1, bd_csr* Si, const double* mass,
                           const double* heart_mass, double gamma, bd_system** out);
bd_status bd_system_destroy(bd_system* s);
/* q = Λ x (bd/system.py:106-116); x, q: device (n+m). */
bd_status bd_system_apply(bd_system* s, const double* x, double* q);
/* y = normalize(x): u − (M·u)/ΣM, v copied (bd/system.py:138-146). */
bd_status bd_system_normalize(bd_system* s, const double* x, double* y);
/* (M·u)/ΣM on the host (bd/system.py:148-150); synchronising. */
bd_status bd_system_weighted_mean_u(bd_system* s, const double* u, double* out);

/* ---- inner preconditioners (bd/precond.py:84-243) ---------------------- */
/* Factor/prepare an SPD matrix given as host CSR (duplicates summed, sorted).
 * IC0 reproduces IncompleteCholesky0._try_factor bit for bit, including the
 * (1+1e-3)^k diagonal restarts (bd/precond.py:136-189); EXACT is a sparse
 * Cholesky LL^T with a fill-reducing ordering (stands in for CHOLMOD,
 * bd/precond.py:96-120); JACOBI is 1/diag (bd/precond.py:219-232).
 * restarts_used may be NULL. */
bd_status bd_inner_create(bd_ctx* ctx, int kind, int64_t n, const int64_t* indptr,
                          const int32_t* indices, const double* values, int max_restarts,
                          bd_inner** out, int* restarts_used);
/* As bd_inner_create, with optional vertex coordinates (row-major n×dim,
 * host) used only to partition the rows of the tiled triangular-solve
 * schedule (coordinate bisection); NULL falls back to a graph bisection.
 * The factor itself does not depend on them. */
bd_status bd_inner_create_ex(bd_ctx* ctx, int kind, int64_t n, const int64_t* indptr,
                             const int32_t* indices, const double* values, int max_restarts,
                             const double* coords, int dim, bd_inner** out, int* restarts_used);
bd_status bd_inner_destroy(bd_inner* p);
/* z = P^{-1} y (device pointers, length n). */
bd_status bd_inner_apply(bd_inner* p, const double* y, double* z);
/* Factor export for tests (IncompleteCholesky0.lower_factor, bd/precond.py:196-198):
 * call with NULL arrays to get nnz; arrays are host. For EXACT the factor is of
 * the permuted matrix and perm (length n, may be NULL) receives the ordering. */
bd_status bd_inner_factor_info(bd_inner* p, int64_t* n, int64_t* nnz, int64_t* levels);
bd_status bd_inner_export_factor(bd_inner* p, int64_t* indptr, int32_t* indices,
                                 double* values, int32_t* perm);

/* ---- block-LU preconditioner (BlockLUPreconditioner, bd/precond.py:246-312) */
bd_status bd_blocklu_create(bd_system* s, bd_inner* bulk, bd_inner* schur, double beta,
                            bd_prec** out);
bd_status bd_blocklu_destroy(bd_prec* p);
/* z = P_Λ^{-1} r (apply_inverse, :298-312); r, z device (n+m). */
bd_status bd_blocklu_apply(bd_prec* p, const double* r, double* z);
/* z = regularised bulk inverse of y (_bulk_inverse, :281-292); device (n). */
bd_status bd_blocklu_bulk_inverse(bd_prec* p, const double* y, double* z);
/* z = inner_schur^{-1} y (_schur_inverse, :294-296); device (m). */
bd_status bd_blocklu_schur_inverse(bd_prec* p, const double* y, double* z);
/* counters[3] = {p1_count, pk_count, si_count}; reset zeroes them. */
bd_status bd_blocklu_counters(bd_prec* p, int64_t* counters);
bd_status bd_blocklu_reset_counters(bd_prec* p);

/* ---- deflated PCG (pcg_solve, bd/krylov.py:46-140) --------------------- */
/* b, x0 (nullable), x: device (n+m). res_hist / prec_hist: HOST arrays of
 * capacity max_iter+2 (may be NULL); *n_res / *n_prec receive their lengths.
 * Synchronising.  Returns BD_ENOCONV / BD_EBREAKDOWN with stats filled; x then
 * holds the last iterate (not normalised), as the reference raises before
 * normalising. */
bd_status bd_pcg_solve(bd_system* s, bd_prec* p, const double* b, const double* x0,
                       double tol, int64_t max_iter, double* x, bd_stats* stats,
                       double* res_hist, int64_t* n_res, double* prec_hist,
                       int64_t* n_prec);
/* Optional per-stage device timing of subsequent solves (CUDA events between
 * kernel classes on the context stream).  times_ms receives, per stage
 * class, the accumulated milliseconds since the last enable:
 *   0 Λ apply, 1 x/r update, 2 bulk triangular solves, 3 Schur triangular
 *   solves, 4 S_i SpMVs in P^{-1}, 5 vector kernels (combine/deflate/d-update),
 *   6 sentinel/reset memsets; launches[7] the launch count per class. */
bd_status bd_profile_enable(bd_ctx* ctx, int enable);
bd_status bd_profile_read(bd_ctx* ctx, double* times_ms, int64_t* launches, int cap);
/* Total kernel launches issued by this context since creation (for bench). */
int64_t bd_launch_count(bd_ctx* ctx);

/* ---- membrane model (bd/ionic.py:45-68,124-134; bd/system.py:118-136) -- */
/* rhs (device n+m) = (0^n, M_H ∘ (γ v − χ (I_ion(v,w) − stim))), where
 * stim_k = max over active sites s with (site_mask[k] >> s) & 1 of amplitude,
 * active_sites a bitmask evaluated by the caller from the time window
 * (half-open [start, start+duration), bd/ionic.py:130). ion (device m,
 * nullable) receives the ionic current.  Ionic params: v_rest, v_span,
 * tau_in, tau_out, c_m.  Bitwise equal to the numpy evaluation order. */
bd_status bd_membrane_rhs(bd_system* s, const double* v, const double* w,
                          const uint64_t* site_mask, uint64_t active_sites,
                          double amplitude, double chi, double v_rest, double v_span,
                          double tau_in, double tau_out, double c_m, double* rhs,
                          double* ion);
/* Same without a bd_system (sharded ranks): n, m, heart_mass (device, m) and
 * gamma given explicitly. */
bd_status bd_membrane_rhs_raw(bd_ctx* ctx, int64_t n, int64_t m, const double* heart_mass,
                              double gamma, const double* v, const double* w,
                              const uint64_t* site_mask, uint64_t active_sites, double amplitude,
                              double chi, double v_rest, double v_span, double tau_in,
                              double tau_out, double c_m, double* rhs, double* ion);
/* w_new = clip(w + dt * (u < u_gate ? (1-w)/tau_open : -w/tau_close), 0, 1)
 * with u = (v - v_rest)/v_span (update_gate, bd/ionic.py:55-68); device m. */
bd_status bd_membrane_gate(bd_ctx* ctx, int64_t m, const double* v, const double* w,
                           double dt, double v_rest, double v_span, double tau_open,
                           double tau_close, double u_gate, double* w_new);

/* ---- P1 assembly on the device (setup; bd/assembly.py:36-97) ---------- */
/* Stiffness K = sum_e vol_e * sym(G_e sigma_e G_e^T) and the row-sum lumped
 * mass m_v = sum_e vol_e/(dim+1), assembled on the device.  Host inputs:
 * vertices (nv x dim, fp64 row-major; the space's vertices are 0..nv-1),
 * elements (ne x (dim+1) int64), sigma (ne x dim x dim).  If sigma2 is given
 * the element tensor is the harmonic mean sym(inv(inv(sigma)+inv(sigma2)))
 * (the monodomain tensor of build_monodomain_matrix, bd/precond.py:34-47).
 * Result: sorted CSR with duplicates summed in element order (deterministic),
 * explicit zeros kept like the reference's COO -> CSR.  BD_EINVAL on a
 * non-positive element volume (AssemblyError in the reference). */
typedef struct bd_asm bd_asm;
bd_status bd_assemble_p1(bd_ctx* ctx, int dim, int64_t nv, const double* vertices, int64_t ne,
                         const int64_t* elements, const double* sigma, const double* sigma2,
                         bd_asm** out, int64_t* nnz);
/* Heart conductivity tensors of the transmural-rotation fibre model on the
 * device (3D; centroid, fibre angle linear in z, frame (f, s, e_z)):
 * model = {z0, z1, angle0_deg, angle1_deg}; gi / ge = the three intra / extra
 * gains (fibre, sheet, normal; orthotropic != 0) or (longitudinal,
 * transverse, -) for the transversely isotropic form.  Host in, host out
 * (ne x 3 x 3 each). */
bd_status bd_tensors_transmural(bd_ctx* ctx, int64_t nv, const double* vertices, int64_t ne,
                                const int64_t* elements, const double* model, const double* gi,
                                const double* ge, int orthotropic, double* out_intra,
                                double* out_extra);
/* Copy the result to host arrays (indptr nv+1, indices nnz, data nnz,
 * mass nv); any pointer may be NULL. */
bd_status bd_assemble_export(bd_asm* a, int64_t* indptr, int32_t* indices, double* data,
                             double* mass);
bd_status bd_assemble_destroy(bd_asm* a);

/* ---- time-loop bookkeeping (bd/simulate.py:67-89, 190-268) ------------- */
/* One step's bookkeeping on the device, replacing the host-side passes of
 * run_simulation over v and u (ActivationTracker.record, bd/simulate.py:74-89;
 * the depolarisation-band test :229-233; max|u| and weighted_mean_u :240-244):
 *  phi (device m, NaN = not yet activated) is updated in place: a pending
 *  vertex with v_new >= threshold gets t_prev + dt*(threshold - v_prev) /
 *  (v_new - v_prev) if v_prev < threshold, else t_prev (bitwise equal to numpy).
 * out (HOST double[4]): [0] 1.0 if any v_new lies in [band_lo, band_hi],
 * [1] 1.0 if every phi is finite after the update, [2] max |u|, [3] the
 * mass-weighted mean of u (bd/system.py:145).  Synchronises once. */
bd_status bd_step_track(bd_system* s, const double* v_prev, const double* v_new, double* phi,
                        double t_prev, double dt, double threshold, double band_lo,
                        double band_hi, const double* u, double* out);

/* ---- mesh-partitioned PCG, one rank (distributed.py) -------
 * The deflated PCG (bd/krylov.py:46-140) with the block-LU preconditioner
 * (bd/precond.py:281-312) on a rank's owned rows [u_own (n) | v_own (m)],
 * block-Jacobi inners (the owned diagonal blocks), all vector work and
 * scalars on the device.  The caller interleaves the calls with the halo
 * exchanges and four all-reduces of the device buffer red (see vectors):
 *   begin; [halo x0] lambda(x, use_flags=0) (if x0); init; ALLREDUCE red[1..3];
 *   check(initial=1); pinv1; [halo z1_H] pinv2; [halo s] pinv3;
 *   ALLREDUCE red[3]; pinv4; ALLREDUCE red[4..6]; finish(initial=1);
 *   per iteration: [halo d] lambda(d, 1); ALLREDUCE red[0]; update;
 *   ALLREDUCE red[1..2]; check(0); pinv1; [halo] pinv2; [halo] pinv3;
 *   ALLREDUCE red[3]; pinv4; ALLREDUCE red[4..6]; finish(0);
 *   then wmean; ALLREDUCE red[8]; normalize; read.
 * After convergence / breakdown / max_iter every call is a device no-op, so
 * a captured iteration may be replayed past the end (done() tells).
 * S1: n x (n + ghosts), Si: m x (m + heart ghosts); mass / heart_mass
 * host; msum = global sum of mass;
 * red: caller-owned device buffer of >= 16 doubles (the reduction slots the
 * caller all-reduces in place).  Optional (both or neither): Si_ext = S_i
 * with ghost column j renumbered n + j, and z1ext = a caller-owned device
 * buffer of n + heart-ghost doubles that holds z1 followed by its halo (the
 * caller receives the halo there); then pinv2 forms r_v − S_i t inside the
 * Schur forward pass and ignores its tg argument. */
bd_status bd_shard_create(bd_ctx* ctx, int64_t n, int64_t m, int64_t n_global, bd_csr* S1,
                          bd_csr* Si, const double* mass, const double* heart_mass, double gamma,
                          bd_inner* bulk, bd_inner* schur, double msum, int64_t hist_cap,
                          double* red, bd_csr* Si_ext, double* z1ext, bd_shard** out);
bd_status bd_shard_destroy(bd_shard* h);
/* device pointers: {x, r, d, q, z1, s, red, z2, corr} (red: the caller's) */
bd_status bd_shard_vectors(bd_shard* h, double** ptrs);
bd_status bd_shard_begin(bd_shard* h, double tol, int64_t max_iter, const double* x0);
bd_status bd_shard_lambda(bd_shard* h, const double* v, const double* ug, const double* vg,
                          int use_flags);
bd_status bd_shard_init(bd_shard* h, const double* b, int has_x0);
bd_status bd_shard_check(bd_shard* h, int initial);
bd_status bd_shard_update(bd_shard* h);
bd_status bd_shard_pinv1(bd_shard* h);
bd_status bd_shard_pinv2(bd_shard* h, const double* tg);
bd_status bd_shard_pinv3(bd_shard* h, const double* sg);
bd_status bd_shard_pinv4(bd_shard* h);
bd_status bd_shard_finish(bd_shard* h, int initial);
bd_status bd_shard_wmean(bd_shard* h);
bd_status bd_shard_normalize(bd_shard* h, double* out);
bd_status bd_shard_done(bd_shard* h, int* done);
/* info = {iterations, converged, breakdown, zero_rhs, max_iter_hit, n_res,
 * n_prec}; scal = {last relative residual, curvature}; histories host. */
bd_status bd_shard_read(bd_shard* h, int64_t* info, double* scal, double* res_hist,
                        double* prec_hist, int64_t cap);
/* dst[i] = src[idx[i]] (device; halo packing) */
bd_status bd_gather(bd_ctx* ctx, int64_t k, const int64_t* idx, const double* src, double* dst);

#ifdef __cplusplus
}
#endif
#endif /* BIDOMAIN_B200_H */
