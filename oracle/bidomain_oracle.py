"""TEST INFRASTRUCTURE ONLY — numpy/scipy restatement of the reference hot path.

Each function follows the reference file:line it cites
(/root/reference/pkg/src/bidomain/...).  Operates on scipy CSR matrices and
numpy vectors; block vectors are (u, v) tuples.  Nothing here imports the
product package.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

_HERE = os.path.dirname(os.path.abspath(__file__))


class OracleBreakdown(Exception):
    def __init__(self, msg, stats):
        super().__init__(msg)
        self.stats = stats


class OracleNoConvergence(Exception):
    def __init__(self, msg, stats):
        super().__init__(msg)
        self.stats = stats


class OraclePrecondError(Exception):
    pass


# ---- operator (system.py:22-150) ------------------------------------------
def gamma(chi, c_m, dt):
    """system.py:22-26"""
    return chi * c_m / dt


def lambda_apply(S1, Si, mh, gam, u, v):
    """system.py:106-116 — top = S1 u; top[:m] += Si v; bottom = Si u_H + Si v + γ M_H v."""
    m = Si.shape[0]
    iv = Si @ v
    iu = Si @ u[:m]
    top = S1 @ u
    top[:m] += iv
    bottom = iu + iv + gam * (mh * v)
    return top, bottom


def bdot(a, b):
    """BlockVector.dot (system.py:39-40)."""
    return float(a[0] @ b[0] + a[1] @ b[1])


def bnorm(a):
    return float(np.sqrt(bdot(a, a)))


def build_rhs(n, mh, gam, v_prev, ion, stim, chi):
    """system.py:118-136"""
    load = gam * v_prev - chi * (ion - stim)
    return np.zeros(n), mh * load


def normalize(mass, u, v):
    """system.py:138-146"""
    alpha = float(mass @ u) / float(mass.sum())
    return u - alpha, v.copy()


# ---- membrane (ionic.py:45-68, 124-134) --------------------------------------
def ionic_current(v, w, v_rest=-90.0, v_peak=50.0, tau_in=0.3, tau_out=6.0, c_m=1.0):
    span = v_peak - v_rest
    u = (np.asarray(v, dtype=float) - v_rest) / span
    rate = np.asarray(w) * u * u * (1.0 - u) / tau_in - u / tau_out
    return -c_m * span * rate


def update_gate(w, v, dt, v_rest=-90.0, v_peak=50.0, tau_open=120.0, tau_close=150.0,
                u_gate=0.13):
    u = (np.asarray(v, dtype=float) - v_rest) / (v_peak - v_rest)
    w = np.asarray(w, dtype=float)
    rate = np.where(u < u_gate, (1.0 - w) / tau_open, -w / tau_close)
    return np.clip(w + dt * rate, 0.0, 1.0)


# ---- preconditioner setup (precond.py:34-81) -----------------------------------
def regularize(S1):
    """precond.py:50-81: beta = mean diag; grounded = S1 + beta e0 e0^T (CSR add)."""
    S1 = sp.csr_matrix(S1)
    beta = float(S1.diagonal().mean())
    bump = sp.csr_matrix(([beta], ([0], [0])), shape=S1.shape)
    g = (S1 + bump).tocsr()
    g.sort_indices()
    return beta, g


def monodomain(stiff_mono, mh, gam):
    """precond.py:34-47: K_m = S_m + γ diag(M_H), duplicates summed, sorted."""
    out = (stiff_mono + gam * sp.diags(mh)).tocsr()
    out.sum_duplicates()
    out.sort_indices()
    return out


# ---- IC(0) (precond.py:123-198) -------------------------------------------------
def _tril_checked(a):
    a = sp.csr_matrix(a, dtype=float)
    a.sum_duplicates()
    a.sort_indices()
    low = sp.tril(a, format="csr")
    ip, ix = low.indptr, low.indices
    for i in range(a.shape[0]):
        last = ip[i + 1] - 1
        if last < ip[i] or ix[last] != i:
            raise OraclePrecondError(f"missing diagonal entry in row {i}")
    return low


def ic0_factor_py(a, max_restarts=20):
    """Pure-Python restatement of _try_factor with restarts (precond.py:136-189);
    small matrices only."""
    low = _tril_checked(a)
    n = low.shape[0]
    ip, ix = low.indptr, low.indices
    shift = 1.0
    for attempt in range(max_restarts + 1):
        vals = low.data.copy()
        if shift != 1.0:
            for i in range(n):
                vals[ip[i + 1] - 1] *= shift
        ok = True
        for i in range(n):
            rs, re = ip[i], ip[i + 1]
            for k in range(rs, re):
                j = ix[k]
                js, je = ip[j], ip[j + 1]
                s = _merge(ix[rs:k], vals[rs:k], ix[js:je - 1], vals[js:je - 1])
                if j == i:
                    piv = vals[k] - s
                    if piv <= 0.0:
                        ok = False
                        break
                    vals[k] = np.sqrt(piv)
                else:
                    vals[k] = (vals[k] - s) / vals[ip[j + 1] - 1]
            if not ok:
                break
        if ok:
            return sp.csr_matrix((vals, ix.copy(), ip.copy()), shape=(n, n)), attempt
        shift *= 1.0 + 1e-3
    raise OraclePrecondError(f"incomplete Cholesky failed after {max_restarts} diagonal "
                             "shift restarts")


def _merge(ca, va, cb, vb):
    """precond.py:201-216"""
    ia = ib = 0
    out = 0.0
    while ia < len(ca) and ib < len(cb):
        if ca[ia] == cb[ib]:
            out += va[ia] * vb[ib]
            ia += 1
            ib += 1
        elif ca[ia] < cb[ib]:
            ia += 1
        else:
            ib += 1
    return out


_clib = None


def _c_lib():
    global _clib
    if _clib is None:
        path = os.path.join(_HERE, "_build", "libic0_oracle.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-C", _HERE], check=True, capture_output=True)
        lib = ctypes.CDLL(path)
        lib.oracle_ic0.restype = ctypes.c_int
        lib.oracle_ic0.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 3 + [ctypes.c_int,
                                                                               ctypes.c_void_p]
        for f in (lib.oracle_trsv_lower, lib.oracle_trsv_upper):
            f.restype = None
            f.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 6
        _clib = lib
    return _clib


def ic0_factor(a, max_restarts=20):
    """C restatement of the same sweep (bit-identical to ic0_factor_py)."""
    low = _tril_checked(a)
    n = low.shape[0]
    ip = np.ascontiguousarray(low.indptr, dtype=np.int64)
    ix = np.ascontiguousarray(low.indices, dtype=np.int32)
    data = np.ascontiguousarray(low.data, dtype=np.float64)
    out = np.empty_like(data)
    got = _c_lib().oracle_ic0(n, ip.ctypes.data, ix.ctypes.data, data.ctypes.data,
                              max_restarts, out.ctypes.data)
    if got < 0:
        raise OraclePrecondError(f"incomplete Cholesky failed after {max_restarts} diagonal "
                                 "shift restarts")
    return sp.csr_matrix((out, low.indices.copy(), low.indptr.copy()), shape=(n, n)), got


def _trsv_c(fn, a, y):
    """C restatement of one spsolve_triangular call (bit-identical; ic0_oracle.c)."""
    n = a.shape[0]
    ip = np.ascontiguousarray(a.indptr, dtype=np.int64)
    ci = np.ascontiguousarray(a.indices, dtype=np.int32)
    val = np.ascontiguousarray(a.data, dtype=np.float64)
    b = np.ascontiguousarray(y, dtype=np.float64)
    x = np.empty(n)
    work = np.empty(n)
    fn(n, ip.ctypes.data, ci.ctypes.data, val.ctypes.data, b.ctypes.data, x.ctypes.data,
       work.ctypes.data)
    return x


class InnerIC0:
    """precond.py:123-198 (apply: spsolve_triangular lower then upper).

    ``fast_apply=True`` runs the two triangular solves through the C
    restatement of scipy's spsolve_triangular arithmetic (``oracle_trsv_*``,
    bit-identical, ~10x faster); the default keeps the scipy calls the
    reference makes, so timing the oracle times the reference's own cost."""

    def __init__(self, a, max_restarts=20, python=False, fast_apply=False):
        f = ic0_factor_py if python else ic0_factor
        self.lower, self.restarts_used = f(a, max_restarts)
        self.upper = self.lower.T.tocsr()
        self.fast_apply = fast_apply

    def apply(self, y):
        if self.fast_apply:
            lib = _c_lib()
            z = _trsv_c(lib.oracle_trsv_lower, self.lower, y)
            return _trsv_c(lib.oracle_trsv_upper, self.upper, z)
        z = spla.spsolve_triangular(self.lower, np.asarray(y, dtype=float), lower=True)
        return spla.spsolve_triangular(self.upper, z, lower=False)


class InnerJacobi:
    """precond.py:219-232"""

    def __init__(self, a):
        d = np.asarray(sp.csr_matrix(a).diagonal())
        if (d <= 0).any():
            raise OraclePrecondError("Jacobi requires a strictly positive diagonal")
        self.inv = 1.0 / d

    def apply(self, y):
        return self.inv * y


class InnerExact:
    """CHOLMOD boundary (precond.py:96-120) restated with SuperLU in symmetric
    mode, as the survey's shim does; machine-precision, not bitwise CHOLMOD."""

    def __init__(self, a):
        self.lu = spla.splu(sp.csc_matrix(a), permc_spec="MMD_AT_PLUS_A", diag_pivot_thresh=0.0,
                            options={"SymmetricMode": True})
        if (self.lu.U.diagonal() <= 0).any():
            raise OraclePrecondError("sparse Cholesky failed, matrix not positive definite")

    def apply(self, y):
        return self.lu.solve(np.asarray(y, dtype=float))


def make_inner(name, a, fast_apply=False):
    if name == "ic0":
        return InnerIC0(a, fast_apply=fast_apply)
    if name == "jacobi":
        return InnerJacobi(a)
    if name == "exact":
        return InnerExact(a)
    raise ValueError(name)


class BlockLU:
    """precond.py:246-312 (P_Λ with the monodomain K_m)."""

    def __init__(self, S1, Si, Km, inner="exact", fast_apply=False):
        self.Si = sp.csr_matrix(Si)
        self.n, self.m = S1.shape[0], Si.shape[0]
        self.beta, grounded = regularize(S1)
        self.bulk = make_inner(inner, grounded, fast_apply)
        self.schur = make_inner(inner, Km, fast_apply)
        self.p1 = self.pk = self.si = 0

    def bulk_inverse(self, y):
        """precond.py:281-292"""
        self.p1 += 1
        mean = y.mean()
        z = self.bulk.apply(y - mean)
        z -= z.mean()
        return z + mean / self.beta

    def schur_inverse(self, y):
        self.pk += 1
        return self.schur.apply(y)

    def apply(self, ru, rv):
        """precond.py:298-312"""
        m = self.m
        t = self.bulk_inverse(ru)
        self.si += 1
        s = self.schur_inverse(rv - self.Si @ t[:m])
        self.si += 1
        corr = np.zeros(self.n)
        corr[:m] = self.Si @ s
        return t - self.bulk_inverse(corr), s


# ---- PCG (krylov.py:46-146) ----------------------------------------------------------
def pcg(S1, Si, mh, mass, gam, prec: BlockLU, bu, bv, tol=1e-6, max_iter=500, x0=None):
    """Returns ((u, v) normalised, stats dict).  Raises OracleBreakdown /
    OracleNoConvergence with stats, like the reference."""
    if tol <= 0:
        raise ValueError("tol must be strictly positive")
    st = {"iterations": 0, "residual_history": [], "preconditioned_history": [],
          "mv_count": 0, "p1_count": 0, "pk_count": 0, "converged": False}
    p1s, pks = prec.p1, prec.pk
    t0 = time.perf_counter()
    b = (np.asarray(bu, float), np.asarray(bv, float))
    nb = bnorm(b)
    n, m = S1.shape[0], Si.shape[0]

    def fin():
        st["p1_count"] = prec.p1 - p1s
        st["pk_count"] = prec.pk - pks
        st["wall_time_ms"] = (time.perf_counter() - t0) * 1e3

    if nb == 0.0:
        st["residual_history"].append(0.0)
        st["converged"] = True
        return (np.zeros(n), np.zeros(m)), st
    if x0 is None:
        xu, xv = np.zeros(n), np.zeros(m)
        ru, rv = b[0].copy(), b[1].copy()
    else:
        xu, xv = np.array(x0[0], float), np.array(x0[1], float)
        au, av = lambda_apply(S1, Si, mh, gam, xu, xv)
        ru, rv = b[0] - au, b[1] - av
    st["mv_count"] += 1
    rel = bnorm((ru, rv)) / nb
    st["residual_history"].append(rel)
    if rel <= tol:
        st["converged"] = True
        fin()
        return normalize(mass, xu, xv), st
    zu, zv = prec.apply(ru, rv)
    zu = zu - zu.mean()  # _deflate (krylov.py:41-43)
    rho = bdot((ru, rv), (zu, zv))
    st["preconditioned_history"].append(rho)
    du, dv = zu.copy(), zv.copy()
    for _ in range(max_iter):
        qu, qv = lambda_apply(S1, Si, mh, gam, du, dv)
        st["mv_count"] += 1
        dq = bdot((du, dv), (qu, qv))
        if not np.isfinite(dq) or dq <= 0.0:
            fin()
            raise OracleBreakdown(f"conjugate gradient breakdown: curvature {dq}", st)
        alpha = rho / dq
        xu += alpha * du
        xv += alpha * dv
        ru -= alpha * qu
        rv -= alpha * qv
        st["iterations"] += 1
        rel = bnorm((ru, rv)) / nb
        if not np.isfinite(rel):
            fin()
            raise OracleBreakdown("non-finite residual", st)
        st["residual_history"].append(rel)
        if rel <= tol:
            st["converged"] = True
            break
        zu, zv = prec.apply(ru, rv)
        zu = zu - zu.mean()
        rho_next = bdot((ru, rv), (zu, zv))
        st["preconditioned_history"].append(rho_next)
        beta = rho_next / rho
        rho = rho_next
        du = zu + beta * du
        dv = zv + beta * dv
    fin()
    if not st["converged"]:
        # the normalised iterate after max_iter iterations (iteration-level
        # parity at sizes where a full solve is out of reach on the CPU)
        st["iterate"] = normalize(mass, xu, xv)
        raise OracleNoConvergence(f"PCG did not reach tol={tol} within {max_iter} iterations", st)
    return normalize(mass, xu, xv), st


# ---- time step (simulate.py:134-170) --------------------------------------------------
def time_step(state, S1, Si, mh, mass, gam, prec, chi, c_m, stim, dt, tol=1e-6, max_iter=500,
              ionic=None):
    """state = (u, v, w); stim = stimulus current vector at state time (m)."""
    ionic = ionic or {}
    u, v, w = state
    ion = ionic_current(v, w, c_m=c_m, **{k: ionic[k] for k in ("v_rest", "v_peak", "tau_in",
                                                                  "tau_out") if k in ionic})
    bu, bv = build_rhs(S1.shape[0], mh, gam, v, ion, stim, chi)
    (un, vn), st = pcg(S1, Si, mh, mass, gam, prec, bu, bv, tol=tol, max_iter=max_iter,
                       x0=(u, v))
    wn = update_gate(w, vn, dt, **{k: ionic[k] for k in ("v_rest", "v_peak", "tau_open",
                                                          "tau_close", "u_gate") if k in ionic})
    return (un, vn, wn), st
