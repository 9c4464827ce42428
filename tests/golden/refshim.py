"""Import shim for the read-only reference package (golden-vector generation only).

The reference (`/root/reference/pkg/src/bidomain`) imports `cvxopt` at module
level (`bd/precond.py:23`) and `matplotlib` through `bd/plots.py:11-15`;
neither is installed in this image.  This shim installs minimal stand-ins in
`sys.modules` before the import:

* `cvxopt.spmatrix/matrix` build scipy CSC matrices / float columns;
* `cvxopt.cholmod.symbolic/numeric/solve` factor with scipy SuperLU in
  symmetric mode (`diag_pivot_thresh=0`), raise ArithmeticError on a
  non-positive pivot and write the solution in place, like CHOLMOD.

For `inner="ic0"` and `inner="jacobi"` the shim is never called, so the
reference runs bit-for-bit.  Used ONLY by tests/golden/make_golden.py and the
optional CPU cross-check tests, in the container where /root/reference exists.
"""
from __future__ import annotations

import sys
import types

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

REFERENCE_SRC = "/root/reference/pkg/src"


class _Col:
    def __init__(self, a):
        self.a = np.array(a, dtype=float).reshape(-1, 1)

    def __array__(self, dtype=None, copy=None):
        return self.a if dtype is None else self.a.astype(dtype)


class _Factor:
    def __init__(self, mat):
        self.mat = mat
        self.lu = None


def _spmatrix(data, rows, cols, size):
    return sp.csc_matrix((np.asarray(data, float), (np.asarray(rows), np.asarray(cols))),
                         shape=size)


def _symbolic(mat):
    return _Factor(mat)


def _numeric(mat, factor):
    lu = spla.splu(sp.csc_matrix(mat), permc_spec="MMD_AT_PLUS_A",
                   diag_pivot_thresh=0.0, options={"SymmetricMode": True})
    if (lu.U.diagonal() <= 0).any():
        raise ArithmeticError("non-positive pivot")
    factor.lu = lu


def _solve(factor, rhs):
    rhs.a[:, 0] = factor.lu.solve(rhs.a[:, 0])


def install() -> None:
    if "cvxopt" not in sys.modules:
        cvx = types.ModuleType("cvxopt")
        chol = types.ModuleType("cvxopt.cholmod")
        cvx.spmatrix = _spmatrix
        cvx.matrix = _Col
        chol.symbolic = _symbolic
        chol.numeric = _numeric
        chol.solve = _solve
        cvx.cholmod = chol
        sys.modules["cvxopt"] = cvx
        sys.modules["cvxopt.cholmod"] = chol
    if "matplotlib" not in sys.modules:
        mpl = types.ModuleType("matplotlib")
        plt = types.ModuleType("matplotlib.pyplot")
        mpl.use = lambda *a, **k: None
        plt.subplots = lambda *a, **k: (None, None)
        plt.savefig = lambda *a, **k: None
        plt.close = lambda *a, **k: None
        mpl.pyplot = plt
        sys.modules["matplotlib"] = mpl
        sys.modules["matplotlib.pyplot"] = plt
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)


def import_reference():
    """Return the reference `bidomain` package (raises ImportError if absent)."""
    install()
    import bidomain  # noqa: F401
    return bidomain
