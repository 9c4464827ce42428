// Host-side setup for the inner preconditioners: factorisations and the
// solve schedules consumed by the sync-free triangular-solve kernels.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace bd {

// Host CSR (int64 indptr for the ABI, int32 indices).
struct HostCsr {
  int64_t n = 0;
  std::vector<int64_t> indptr;
  std::vector<int32_t> indices;
  std::vector<double> values;
  int64_t nnz() const { return indptr.empty() ? 0 : indptr.back(); }
};

// IncompleteCholesky0.setup (bd/precond.py:136-152): zero-fill IC on tril(A)
// with multiplicative diagonal restarts.  Returns 0 on success, 1 on a missing
// diagonal (msg set), 2 when all restarts broke down.  Bit-exact restatement of
// _try_factor (:155-189) — compile with -ffp-contract=off.
int ic0_factor(const HostCsr& a, int max_restarts, HostCsr* lower, int* restarts_used,
               std::string* msg);

// CSR transpose (scipy `.T.tocsr()`: sorted columns per row).
HostCsr transpose(const HostCsr& a);

// Level of each row of a triangular CSR factor: 1 + max level of the rows it
// depends on (lower: columns < row; upper: columns > row).  Returns depth.
int64_t row_levels(const HostCsr& t, bool lower, std::vector<int32_t>* level);

// Solve order: rows sorted by level (stable), each level padded with -1 to a
// multiple of `pad` so that the row groups of one warp never depend on each
// other.  level_start receives the task offset of each level.
void build_schedule(const std::vector<int32_t>& level, int64_t depth, int pad,
                    std::vector<int32_t>* tasks);

// Nested-dissection fill-reducing ordering of the symmetric pattern of a
// (BFS level-structure bisection; separators numbered last).  perm[k] = old
// index of new row k.
void nested_dissection(const HostCsr& a, std::vector<int32_t>* perm);

// Sparse Cholesky LL^T of P A P^T (up-looking, row by row).  Returns 0 on
// success, 2 on a non-positive pivot (msg set).  L returned as CSR with the
// diagonal last in each row.
int cholesky(const HostCsr& a, const std::vector<int32_t>& perm, HostCsr* lower,
             std::string* msg);

// Relaxed supernodes: explicit zeros completing near-dense triangles of
// consecutive rows (see bd_host.cpp); frac = tolerated missing fraction.
void relax_supernodes(HostCsr* L, double frac, int smax);

}  // namespace bd

namespace bd {

// Balanced partition of the rows of a symmetric pattern into `parts` pieces
// by recursive BFS-distance bisection (RCB-like slabs on mesh graphs).
void partition_rows(const HostCsr& a, int parts, std::vector<int32_t>* part);

// Recursive coordinate bisection of n points (row-major n×dim) into `parts`
// axis-aligned boxes (split along the widest extent at the proportional
// quantile).  On structured meshes numbered lexicographically the lower-
// triangular dependencies point to smaller coordinates, so the part DAG of a
// triangular solve is acyclic with chains of length ~ the box grid diameter.
// Lattice-aligned tiles: bin every axis into slabs of ~k = target^(1/dim)
// coordinate layers (by the rank of the distinct coordinate value when the
// axis has few distinct values, i.e. a structured grid; by equal-width bins
// otherwise) and split by `cls` (e.g. heart / torso) so that the tile DAG of a
// natural ordering stays acyclic and its depth is ~sum of bins per axis.
// Returns the number of (non-empty) tiles.
int partition_grid(int64_t n, int dim, const double* coords, int target,
                   const std::vector<int32_t>* cls, std::vector<int32_t>* tile);
void partition_coords(int64_t n, int dim, const double* coords, int parts,
                      std::vector<int32_t>* part);

// Tiled triangular-solve schedule: rows grouped by part (one CTA each), each
// part's rows sorted by DAG level and cut into steps of at most R rows (a step
// never spans two levels).  Off-diagonal entries in ELL form (G per row):
// col >= 0 is a row of another part (polled), col < 0 is -(slot+1) of a row of
// the same part (shared memory); padding points at the part's zero cell.
struct TileSchedule {
  int parts = 0, G = 0, R = 0;
  int max_part_rows = 0;
  int max_part_steps = 0;
  int64_t depth = 0;
  std::vector<int32_t> part_task_ptr;  // parts+1
  std::vector<int32_t> part_step_ptr;  // parts+1
  std::vector<int32_t> step_task_ptr;  // nsteps+1
  std::vector<int32_t> task_row;       // ntasks
  std::vector<double> task_diag;       // ntasks
  std::vector<int32_t> ell_col;        // ntasks*G
  std::vector<double> ell_val;         // ntasks*G
};
// Returns false if some row has more than G off-diagonal entries.
// entry_major: within each step the ELL block is stored [G][rows_in_step]
// (entry-major) instead of [rows][G], for lane-contiguous shared-memory reads.
bool build_tile_schedule(const HostCsr& t, bool lower, const std::vector<int32_t>& part,
                         int parts, int G, int R, TileSchedule* out, bool entry_major = false);

}  // namespace bd

namespace bd {

// Cluster-wavefront schedule: P parts (one CTA each, one thread-block cluster),
// all parts step through the global levels together.  Dependencies are read
// from a ring of W level windows in shared memory: a part's own rows of a
// level plus the rows of other parts it imports (pushed by their owners via
// distributed shared memory).  Valid only if every dependency is at most W-1
// levels back.
struct ClusterSchedule {
  int parts = 0, E = 0, W = 4;
  int nlevels = 0;
  int wmax = 0;        // window slots per level (own + imported), max over parts/levels
  int rmax = 0;        // own rows per level, max over parts/levels
  int emax = 0;        // export entries per level, max
  std::vector<int32_t> lvl_ptr;   // parts*(nlevels+1): row offsets (task order, part-major)
  std::vector<int32_t> task_row;  // ntasks
  std::vector<double> task_diag;  // ntasks
  std::vector<double> ell_val;    // ntasks*E
  std::vector<int16_t> ell_code;  // ntasks*E: window index ((lvl%W)*wmax + slot), -1 padding
  std::vector<int32_t> exp_ptr;   // parts*(nlevels+1)
  std::vector<int32_t> exp_src;   // own slot (within the level window)
  std::vector<int32_t> exp_dst;   // (dest part << 16) | dest window index
};
// Returns false if a dependency reaches further back than W-1 levels or the
// windows/rows exceed the given caps.
bool build_cluster_schedule(const HostCsr& t, bool lower, const std::vector<int32_t>& part,
                            int parts, int E, int W, int cap_rows, int cap_slots,
                            ClusterSchedule* out, std::string* why);

}  // namespace bd

namespace bd {

// Dynamic-tile schedule: rows grouped into small tiles (coordinate or graph
// bisection, ~tile_rows each), tiles listed in a priority topological order of
// the tile DAG (priority = lowest row level), each tile's rows sorted by level
// into steps.  ELL entries: col >= 0 row of another tile (polled), col < 0 is
// -(slot+1) of a row of the same tile, padding = zero slot.
struct DTileSchedule {
  int E = 0, tmax = 0, smax = 0;
  std::vector<int32_t> tile_row_ptr;   // ntiles+1 (task order)
  std::vector<int32_t> tile_step_ptr;  // ntiles+1 into step_row
  std::vector<int32_t> step_row;       // per step: first row offset within its tile
  std::vector<int32_t> task_row;
  std::vector<double> task_diag;
  std::vector<int32_t> ell_col;        // ntasks*E
  std::vector<double> ell_val;
};
bool build_dtile_schedule(const HostCsr& t, bool lower, const std::vector<int32_t>& tile,
                          int ntiles, int E, DTileSchedule* out, std::string* why);

// Blocked-tile schedule derived from a DTileSchedule (same tiles, same task
// order): per tile the dense inverse of its diagonal block (lower triangular
// in slot order, packed row-major, each block padded to an even length so it
// is 16-byte aligned) and per row only the entries that reach other tiles.
// A pass is then y_T = b_T - L_T,ext x_ext ; x_T = inv(L_TT) y_T.
struct BTileSchedule {
  int Ex = 0, tmax = 0, xmax = 0;
  std::vector<int32_t> tile_row_ptr;  // ntiles+1 (task order)
  std::vector<int64_t> tile_inv_ptr;  // ntiles+1 (doubles)
  std::vector<int32_t> task_row;
  std::vector<int32_t> ext_col;       // ntasks*Ex: slot in the tile's input list, -1 = padding
  std::vector<double> ext_val;
  std::vector<int32_t> tile_in_ptr;   // ntiles+1: distinct external inputs of each tile
  std::vector<int32_t> in_col;        // their global rows
  std::vector<double> inv;
};
bool build_btile_schedule(const DTileSchedule& ds, BTileSchedule* out, std::string* why);

}  // namespace bd
