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

}  // namespace bd
