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
