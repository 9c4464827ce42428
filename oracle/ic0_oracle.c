/* TEST INFRASTRUCTURE ONLY (oracle): C restatement of the reference IC(0)
 * factorisation, IncompleteCholesky0.setup/_try_factor/_sparse_row_dot
 * (/root/reference/pkg/src/bidomain/precond.py:136-216), used by the oracle
 * for configurations where the reference's pure-Python loop takes minutes.
 * Input: tril(A) in CSR with the diagonal last in each row.  Compile with
 * -ffp-contract=off so every product/sum rounds like numpy scalars.
 * Returns the attempt index that succeeded (>= 0) or -1 after all restarts. */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static double row_merge(const int32_t* ca, const double* va, int64_t na,
                        const int32_t* cb, const double* vb, int64_t nb) {
  /* precond.py:201-216 */
  int64_t ia = 0, ib = 0;
  double acc = 0.0;
  while (ia < na && ib < nb) {
    if (ca[ia] == cb[ib]) {
      double prod = va[ia] * vb[ib];
      acc = acc + prod;
      ia++;
      ib++;
    } else if (ca[ia] < cb[ib]) {
      ia++;
    } else {
      ib++;
    }
  }
  return acc;
}

static int sweep(int64_t n, const int64_t* ip, const int32_t* ci, double* v) {
  /* precond.py:170-189 */
  for (int64_t i = 0; i < n; i++) {
    int64_t rs = ip[i], re = ip[i + 1];
    for (int64_t k = rs; k < re; k++) {
      int32_t j = ci[k];
      int64_t js = ip[j], je = ip[j + 1];
      double s = row_merge(ci + rs, v + rs, k - rs, ci + js, v + js, (je - 1) - js);
      if (j == i) {
        double piv = v[k] - s;
        if (piv <= 0.0) return 0;
        v[k] = sqrt(piv);
      } else {
        v[k] = (v[k] - s) / v[ip[j + 1] - 1];
      }
    }
  }
  return 1;
}

int oracle_ic0(int64_t n, const int64_t* ip, const int32_t* ci, const double* data,
               int max_restarts, double* out) {
  /* precond.py:136-152: shift *= 1 + 1e-3 per failed attempt */
  double shift = 1.0;
  int64_t nnz = ip[n];
  for (int attempt = 0; attempt <= max_restarts; attempt++) {
    memcpy(out, data, sizeof(double) * (size_t)nnz);
    if (shift != 1.0)
      for (int64_t i = 0; i < n; i++) out[ip[i + 1] - 1] = out[ip[i + 1] - 1] * shift;
    if (sweep(n, ip, ci, out)) return attempt;
    shift = shift * (1.0 + 1e-3);
  }
  return -1;
}

/* IC(0) apply, IncompleteCholesky0.apply_inverse (precond.py:191-194):
 * scipy.sparse.linalg.spsolve_triangular(L, y, lower=True) then
 * spsolve_triangular(L^T, z, lower=False), restated in the arithmetic order of
 * scipy 1.18 (linsolve.py spsolve_triangular -> SuperLU gstrs, trans='T'):
 *
 * lower (CSR L, diagonal last in each row): the strictly lower entries are
 * scaled by the inverse diagonal of their column, a unit-lower solve runs in
 * column order with each row's products subtracted one by one, and the result
 * is multiplied by the inverse diagonal:
 *   y_i = b_i - sum_{j<i} (L_ij * (1/L_jj)) * y_j (ascending j),  x = y * (1/L_ii).
 * upper (CSR U = L^T, diagonal first): the right-hand side is first divided by
 * the scaled diagonal U_ii * (1/U_ii), then a unit-upper back substitution,
 * then the multiplication by the inverse diagonal.
 * Output is bit-identical to the scipy calls (tests/test_oracle_golden.py). */
void oracle_trsv_lower(int64_t n, const int64_t* ip, const int32_t* ci, const double* val,
                       const double* b, double* x, double* work) {
  double* inv = work;
  for (int64_t i = 0; i < n; i++) inv[i] = 1.0 / val[ip[i + 1] - 1];
  for (int64_t i = 0; i < n; i++) {
    double s = b[i];
    for (int64_t k = ip[i]; k < ip[i + 1] - 1; k++) {
      int32_t j = ci[k];
      s = s - x[j] * (val[k] * inv[j]);
    }
    x[i] = s;
  }
  for (int64_t i = 0; i < n; i++) x[i] = x[i] * inv[i];
}

void oracle_trsv_upper(int64_t n, const int64_t* ip, const int32_t* ci, const double* val,
                       const double* b, double* x, double* work) {
  double* inv = work;
  for (int64_t i = 0; i < n; i++) inv[i] = 1.0 / val[ip[i]];
  for (int64_t i = 0; i < n; i++) x[i] = b[i] / (val[ip[i]] * inv[i]);
  for (int64_t i = n - 1; i >= 0; i--) {
    double s = x[i];
    for (int64_t k = ip[i] + 1; k < ip[i + 1]; k++) {
      int32_t j = ci[k];
      s = s - x[j] * (val[k] * inv[j]);
    }
    x[i] = s;
  }
  for (int64_t i = 0; i < n; i++) x[i] = x[i] * inv[i];
}
