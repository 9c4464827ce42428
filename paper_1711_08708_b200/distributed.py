"""Mesh-partitioned (multi-GPU) coupled solve: partition, halo plan, distributed PCG.

One process per GPU.  The vertices are split by recursive coordinate
bisection (RCB); each rank owns a box of vertices and keeps a one-layer ghost
halo (P1 stencils only couple mesh neighbours).  Local numbering keeps the
reference's heart-first property per rank: owned heart vertices, owned torso
vertices, then ghost heart, ghost torso.  So the local v block is a prefix of
the local u block, as `bd/mesh.py:252-263` guarantees globally.

The distributed iteration is `pcg_solve` (bd/krylov.py:46-140) with the
block-LU preconditioner (bd/precond.py:281-312), with two changes:
* dots and means are global, via all_reduce; Λ and the two S_i products
  exchange halos;
* the inner solves become block-Jacobi: the owned diagonal block of the
  grounded S_1 / K_m.  Jacobi shards exactly; IC(0) and exact change the
  preconditioner, so their iteration counts are reported next to the
  1-GPU counts.

The rank-local iteration is native: ``NativeShard`` holds the rank's PCG
state and runs every vector operation, the local Λ and the block-Jacobi inner
solves as sm_100a kernels (bd_shard_*, csrc/bd_shard.cuh) with all scalars on
the device.  ``ShardSolver`` interleaves them with three halo all-gathers and
four all-reduces per iteration (torch.distributed: NCCL over NVLink on the
box) and captures one iteration, collectives included, in a CUDA graph.
``TorchShard`` restates the same kernels on CPU tensors so the CPU tests run
the identical orchestration with gloo at world size 2.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp


# ---- partition (host) ----------------------------------------------------------
def rcb_partition(coords: np.ndarray, parts: int) -> np.ndarray:
    """Recursive coordinate bisection: split along the widest extent at the
    proportional quantile; returns the part id of every point."""
    coords = np.asarray(coords, dtype=float)
    out = np.zeros(coords.shape[0], dtype=np.int64)

    def rec(ids, p, first):
        if p <= 1 or ids.size <= 1:
            out[ids] = first
            return
        x = coords[ids]
        axis = int(np.argmax(x.max(axis=0) - x.min(axis=0)))
        pa = p // 2
        cut = int(round(ids.size * pa / p))
        order = np.lexsort((ids, x[:, axis]))
        rec(ids[order[:cut]], pa, first)
        rec(ids[order[cut:]], p - pa, first + pa)

    rec(np.arange(coords.shape[0]), parts, 0)
    return out


@dataclass
class LocalProblem:
    """Rank-local blocks in local numbering (owned heart, owned torso, ghost
    heart, ghost torso) and the halo plan."""

    rank: int
    nprocs: int
    n_global: int
    m_global: int
    owned: np.ndarray          # global ids of owned vertices, local order
    ghosts: np.ndarray         # global ids of ghost vertices, local order
    n_own: int
    m_own: int                 # owned heart vertices (prefix of owned)
    m_ghost: int               # ghost heart vertices (prefix of ghosts)
    S1: sp.csr_matrix          # n_own × (n_own + n_ghost)
    Si: sp.csr_matrix          # m_own × (m_own + m_ghost)
    mass: np.ndarray           # n_own
    heart_mass: np.ndarray     # m_own
    gamma: float
    bulk_block: sp.csr_matrix  # owned diagonal block of the grounded S_1
    schur_block: sp.csr_matrix  # owned diagonal block of K_m
    # halo plan: per neighbour, local indices to send / ghost slots to fill
    send: dict = field(default_factory=dict)
    recv: dict = field(default_factory=dict)
    send_heart: dict = field(default_factory=dict)
    recv_heart: dict = field(default_factory=dict)


def build_local(S1, Si, mass, heart_mass, gamma, grounded, Km, part: np.ndarray,
                rank: int, nprocs: int) -> LocalProblem:
    """Rank `rank`'s local problem from the global CSR blocks (every rank can
    compute every rank's plan: the halo lists are consistent by construction)."""
    S1 = sp.csr_matrix(S1)
    Si = sp.csr_matrix(Si)
    n, m = S1.shape[0], Si.shape[0]
    part = np.asarray(part)

    def layout(r):
        own = np.flatnonzero(part == r)
        own = np.concatenate([own[own < m], own[own >= m]])
        rows = S1[own]
        cols = np.unique(rows.indices)
        gh = order_ghosts(cols[part[cols] != r], m, part)
        return own, gh

    lay = [layout(r) for r in range(nprocs)]
    owned, ghosts = lay[rank]
    n_own, m_own = owned.size, int((owned < m).sum())
    m_ghost = int((ghosts < m).sum())
    ext = np.concatenate([owned, ghosts])
    g2l = -np.ones(n, dtype=np.int64)
    g2l[ext] = np.arange(ext.size)
    s1 = S1[owned][:, ext]
    # heart extended numbering: owned heart, ghost heart
    hext = np.concatenate([owned[:m_own], ghosts[:m_ghost]])
    si = Si[owned[:m_own]][:, hext]
    for a in (s1, si):
        a.sort_indices()
    gb = sp.csr_matrix(grounded)[owned][:, owned]
    kb = sp.csr_matrix(Km)[owned[:m_own]][:, owned[:m_own]]
    lp = LocalProblem(rank, nprocs, n, m, owned, ghosts, n_own, m_own, m_ghost, s1.tocsr(),
                      si.tocsr(), np.asarray(mass)[owned], np.asarray(heart_mass)[owned[:m_own]],
                      float(gamma), gb.tocsr(), kb.tocsr())
    # halo: my ghosts owned by q are received from q in q's send order
    for q in range(nprocs):
        if q == rank:
            continue
        q_own, q_gh = lay[q]
        # what q needs from me: q's ghosts that I own, in q's ghost order
        need_from_me = q_gh[part[q_gh] == rank]
        if need_from_me.size:
            lp.send[q] = g2l[need_from_me]
            hm = need_from_me < m
            if hm.any():
                lp.send_heart[q] = g2l[need_from_me[hm]]
        mine = ghosts[part[ghosts] == q]
        if mine.size:
            lp.recv[q] = g2l[mine] - n_own  # ghost slots
            hm = mine < m
            if hm.any():
                # heart ghosts are the prefix of ghosts: slot = ghost index
                lp.recv_heart[q] = g2l[mine[hm]] - n_own
    return lp


# ---- communication -------------------------------------------------------------------
class Comm:
    """torch.distributed wrapper: in-place global sums of device tensors and
    point-to-point halo messages (NCCL on the box, gloo in the CPU tests).
    Nothing here reads a value back to the host."""

    def __init__(self, dist, device):
        self.dist = dist
        self.device = device
        # one rank: every sum is already global (no collective in the loop)
        self.single = dist.get_world_size() == 1

    def allreduce(self, vals):
        """Host list -> host list (setup only: synchronises)."""
        if self.single:
            return [float(v) for v in vals]
        torch = _torch()
        t = torch.tensor(vals, dtype=torch.float64, device=self.device)
        self.dist.all_reduce(t)
        return t.tolist()

    def allreduce_(self, t):
        """In-place global sum of a device tensor (no host round trip)."""
        if not self.single:
            self.dist.all_reduce(t)
        return t

    def allgather(self, send, out):
        """out (P x len(send), flat) <- every rank's send buffer, rank order
        (one collective: capturable in a CUDA graph with NCCL)."""
        if self.single:
            out.copy_(send)
            return out
        if hasattr(self.dist, "all_gather_into_tensor") and send.is_cuda:
            self.dist.all_gather_into_tensor(out, send)
        else:
            self.dist.all_gather(list(out.view(-1, send.numel()).unbind(0)), send)
        return out

    def allgather_object(self, obj):
        """Setup only (host objects)."""
        if self.single:
            return [obj]
        res = [None] * self.dist.get_world_size()
        self.dist.all_gather_object(res, obj)
        return res


def _torch():
    import torch

    return torch


def order_ghosts(g: np.ndarray, m: int, part: np.ndarray) -> np.ndarray:
    """Ghost order of a rank: heart ghosts, then torso ghosts, each grouped by
    owning rank (ascending) and ascending within a group, so every
    neighbour's ghosts are one contiguous heart range and one contiguous
    torso range (halos land in place, no scatter)."""
    g = np.asarray(g, dtype=np.int64)
    out = []
    for blk in (g[g < m], g[g >= m]):
        out.append(blk[np.lexsort((blk, part[blk]))])
    return np.concatenate(out)


class HaloPlan:
    """The three halos of an iteration -- the search direction d = [u | v]
    (every ghost of u, the heart ghosts of v) before Λ, and the heart ghosts
    of z1 (for S_i t) and of s (for S_i s) in P^{-1} -- as ONE all-gather
    each: every rank publishes the values of its boundary vertices (the
    owned vertices some other rank holds as ghosts), packed by one gather
    kernel into a buffer of the common maximal size, and unpacks its ghosts
    from the gathered buffer with a second gather.  A collective instead of
    point-to-point messages: capturable in the iteration's CUDA graph with
    NCCL, and identical under gloo in the CPU tests."""

    def __init__(self, lp: "LocalProblem", comm: Comm, device, gather):
        torch = _torch()
        self.gather = gather
        self.comm = comm
        self.n_ghost, self.m_ghost = lp.ghosts.size, lp.m_ghost
        f64 = dict(dtype=torch.float64, device=device)
        self.ug = torch.zeros(max(self.n_ghost, 1), **f64)
        self.vg = torch.zeros(max(self.m_ghost, 1), **f64)
        self.tg = torch.zeros(max(self.m_ghost, 1), **f64)
        self.sg = torch.zeros(max(self.m_ghost, 1), **f64)
        self.active = not comm.single and (lp.ghosts.size > 0 or any(len(v) for v in lp.send.values()))
        m_glob = lp.m_global
        snd = [np.asarray(v, dtype=np.int64) for v in lp.send.values()]
        loc = np.unique(np.concatenate(snd)) if snd else np.zeros(0, np.int64)
        b_glob = lp.owned[loc]
        order = np.argsort(b_glob)
        b_glob, loc = b_glob[order], loc[order]
        allb = comm.allgather_object(b_glob)
        self.active = not comm.single
        if not self.active:
            return
        bh = [b[b < m_glob] for b in allb]
        self.maxb = max(1, max(b.size for b in allb))
        self.maxbh = max(1, max(b.size for b in bh))
        hm = b_glob < m_glob
        # pack: [u(B_r) | pad][v(Bh_r) | pad] from d = [u | v]; heart-only halos
        # from a heart vector: [x(Bh_r) | pad]
        pd = np.zeros(self.maxb + self.maxbh, dtype=np.int64)
        pd[: loc.size] = loc
        pd[self.maxb: self.maxb + int(hm.sum())] = lp.n_own + loc[hm]  # heart rows lead the owned
        ph = np.zeros(self.maxbh, dtype=np.int64)
        ph[: int(hm.sum())] = loc[hm]
        # unpack: ghost g owned by rank q
        gh = lp.ghosts
        owner = np.empty(gh.size, dtype=np.int64)
        pos = np.empty(gh.size, dtype=np.int64)
        posh = np.zeros(gh.size, dtype=np.int64)
        part = getattr(lp, "ghost_owner", None)
        for q in range(len(allb)):
            if q == lp.rank:
                continue
            sel = np.isin(gh, allb[q]) if part is None else (part == q)
            if not sel.any():
                continue
            owner[sel] = q
            pos[sel] = np.searchsorted(allb[q], gh[sel])
            hsel = sel & (gh < m_glob)
            posh[hsel] = np.searchsorted(bh[q], gh[hsel])
        w = self.maxb + self.maxbh
        ud = owner * w + pos
        vd = owner[: lp.m_ghost] * w + self.maxb + posh[: lp.m_ghost]
        hh = owner[: lp.m_ghost] * self.maxbh + posh[: lp.m_ghost]
        T = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.int64), device=device)  # noqa: E731
        self.pack_d, self.pack_h = T(pd), T(ph)
        self.unpack_u, self.unpack_v, self.unpack_h = T(ud), T(vd), T(hh)
        P = len(allb)
        self.send_d = torch.zeros(w, **f64)
        self.recv_d = torch.zeros(P * w, **f64)
        self.send_h = torch.zeros(self.maxbh, **f64)
        self.recv_h = torch.zeros(P * self.maxbh, **f64)

    def halo_d(self, comm, src):
        """ug, vg <- ghosts of u and heart ghosts of v of the block vector src."""
        if not self.active:
            return
        self.gather(self.pack_d, src, self.send_d)
        comm.allgather(self.send_d, self.recv_d)
        self.gather(self.unpack_u, self.recv_d, self.ug)
        if self.m_ghost:
            self.gather(self.unpack_v, self.recv_d, self.vg)

    def halo_h(self, comm, src, dst):
        """dst <- heart ghosts of the heart-block vector src."""
        if not self.active:
            return
        self.gather(self.pack_h, src, self.send_h)
        comm.allgather(self.send_h, self.recv_h)
        if self.m_ghost:
            self.gather(self.unpack_h, self.recv_h, dst)


# ---- the rank-local iteration: native (sm_100a) and a CPU restatement ----------------
class NativeShard:
    """One rank's PCG state and vector kernels in the sm_100a library
    (bd_shard_*, csrc/bd_shard.cuh): Λ on the local rows, the x/r update, the
    block-Jacobi P^{-1} with the collapsed recentrings, r·z, d; every scalar
    on the device, partial sums in the caller-visible buffer `red`."""

    def __init__(self, lp: "LocalProblem", inner: str, ctx=None):
        import ctypes as C

        from . import _lib
        from .precond import make_inner
        from .system import NativeCsr

        torch = _torch()
        self._lib, self.C = _lib, C
        self.ctx = ctx or _lib.Context.default()
        self.device = self.ctx.device
        self.lp = lp
        self.n, self.m = lp.n_own, lp.m_own
        self.S1 = NativeCsr(self.ctx, sp.csr_matrix(lp.S1))
        self.Si = NativeCsr(self.ctx, sp.csr_matrix(lp.Si))
        # S_i with ghost column j at n + j: reads [z1 (n) | heart ghosts] in place,
        # so r_v − S_i t is formed inside the Schur forward pass (RhsSchur)
        si = sp.csr_matrix(lp.Si)
        col = si.indices.astype(np.int64)
        col = np.where(col >= lp.m_own, col + (lp.n_own - lp.m_own), col)
        self.Si_ext = NativeCsr(self.ctx, sp.csr_matrix((si.data, col, si.indptr),
                                                        shape=(lp.m_own, lp.n_own + lp.m_ghost)))
        self.z1ext = torch.zeros(lp.n_own + max(lp.m_ghost, 1), dtype=torch.float64,
                                 device=self.device)
        xyz = getattr(lp, "coords", None)
        self.bulk = make_inner(inner)
        self.schur = make_inner(inner)
        if inner == "ic0" and xyz is not None:
            self.bulk.setup(lp.bulk_block, coords=xyz)
            self.schur.setup(lp.schur_block, coords=xyz[: lp.m_own])
        else:
            self.bulk.setup(lp.bulk_block)
            self.schur.setup(lp.schur_block)
        self.red = torch.zeros(16, dtype=torch.float64, device=self.device)
        self.hist_cap = 0
        self.h = None
        self.msum = None

    def create(self, msum: float, hist_cap: int):
        C, L = self.C, self._lib
        if self.h is not None and hist_cap <= self.hist_cap:
            return
        self.destroy()
        h = C.c_void_p()
        mass = np.ascontiguousarray(self.lp.mass, dtype=np.float64)
        mh = np.ascontiguousarray(self.lp.heart_mass, dtype=np.float64)
        L.check(L.lib().bd_shard_create(
            self.ctx.handle, self.n, self.m, self.lp.n_global, self.S1.handle, self.Si.handle,
            mass.ctypes.data, mh.ctypes.data, float(self.lp.gamma), self.bulk.handle,
            self.schur.handle, float(msum), int(hist_cap), L.ptr(self.red), self.Si_ext.handle,
            L.ptr(self.z1ext), C.byref(h)),
            self.ctx.handle)
        self.h, self.hist_cap, self.msum = h, hist_cap, msum
        ptrs = (C.c_void_p * 9)()
        L.check(L.lib().bd_shard_vectors(h, ptrs), self.ctx.handle)
        self.ptr = {k: C.c_void_p(ptrs[i]) for i, k in enumerate(
            ("x", "r", "d", "q", "z1", "s", "red", "z2", "corr"))}

    def destroy(self):
        if self.h is not None and self._lib._lib is not None:
            self._lib._lib.bd_shard_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def _c(self, st):
        self._lib.check(st, self.ctx.handle)

    def sync(self):
        """Run on torch's current stream (graph capture, torch ordering)."""
        self.ctx.sync_stream()

    # the kernels (see include/bidomain_b200.h, bd_shard_*)
    def gather(self, idx, src, dst):
        L = self._lib
        self._c(L.lib().bd_gather(self.ctx.handle, int(idx.numel()), L.ptr(idx),
                                  src if isinstance(src, self.C.c_void_p) else L.ptr(src),
                                  L.ptr(dst)))

    def begin(self, tol, max_iter, x0):
        self._c(self._lib.lib().bd_shard_begin(self.h, float(tol), int(max_iter),
                                               self._lib.ptr(x0)))

    def lambda_(self, which, ug, vg, use_flags):
        L = self._lib
        self._c(L.lib().bd_shard_lambda(self.h, self.ptr[which], L.ptr(ug), L.ptr(vg),
                                        int(use_flags)))

    def init(self, b, has_x0):
        self._c(self._lib.lib().bd_shard_init(self.h, self._lib.ptr(b), int(has_x0)))

    def check(self, initial):
        self._c(self._lib.lib().bd_shard_check(self.h, int(initial)))

    def update(self):
        self._c(self._lib.lib().bd_shard_update(self.h))

    def pinv1(self):
        self._c(self._lib.lib().bd_shard_pinv1(self.h))

    def pinv2(self, tg):
        self._c(self._lib.lib().bd_shard_pinv2(self.h, self._lib.ptr(tg)))

    def pinv3(self, sg):
        self._c(self._lib.lib().bd_shard_pinv3(self.h, self._lib.ptr(sg)))

    def pinv4(self):
        self._c(self._lib.lib().bd_shard_pinv4(self.h))

    def finish(self, initial):
        self._c(self._lib.lib().bd_shard_finish(self.h, int(initial)))

    def wmean(self):
        self._c(self._lib.lib().bd_shard_wmean(self.h))

    def normalize(self, out):
        self._c(self._lib.lib().bd_shard_normalize(self.h, self._lib.ptr(out)))

    def done(self):
        d = self.C.c_int()
        self._c(self._lib.lib().bd_shard_done(self.h, self.C.byref(d)))
        return bool(d.value)

    def read(self, cap):
        C = self.C
        info = (C.c_int64 * 7)()
        scal = (C.c_double * 2)()
        res = np.zeros(cap)
        pre = np.zeros(cap)
        self._c(self._lib.lib().bd_shard_read(self.h, info, scal, res.ctypes.data,
                                              pre.ctypes.data, cap))
        return {"iterations": int(info[0]), "converged": bool(info[1]), "breakdown": bool(info[2]),
                "zero_rhs": bool(info[3]), "max_iter": bool(info[4]),
                "residual_history": res[: info[5]].tolist(),
                "preconditioned_history": pre[: info[6]].tolist(), "curvature": float(scal[1])}

    def tg_buffer(self, plan):
        """Where the halo of z1 lands: right after z1 in z1ext."""
        return self.z1ext[self.n: self.n + max(plan.m_ghost, 1)]

    def factor_nnz(self):
        try:
            return int(self.bulk.factor_info()["nnz"]), int(self.schur.factor_info()["nnz"])
        except Exception:  # jacobi
            return 0, 0


class TorchShard:
    """CPU restatement of NativeShard's kernels (same arithmetic order, same
    reduction slots, the same done-flag semantics) on torch CPU tensors with
    caller-supplied inner solves: it lets the CPU tests run the sharded
    orchestration (ShardSolver: halo plan, the four all-reduces, the loop)
    with gloo at world size > 1.  Test infrastructure, not a product path."""

    def __init__(self, lp: "LocalProblem", inner_factory):
        torch = _torch()
        self.lp = lp
        self.n, self.m = lp.n_own, lp.m_own
        self.S1, self.Si = sp.csr_matrix(lp.S1), sp.csr_matrix(lp.Si)
        self.bulk = inner_factory(lp.bulk_block)
        self.schur = inner_factory(lp.schur_block)
        nm = self.n + self.m
        f64 = torch.float64
        self.v = {k: torch.zeros(nm, dtype=f64) for k in ("x", "r", "d", "q")}
        self.v.update({k: torch.zeros(self.n, dtype=f64) for k in ("z1", "z2", "corr")})
        self.v.update({k: torch.zeros(self.m, dtype=f64) for k in ("s", "rhs_s")})
        self.red = torch.zeros(16, dtype=f64)
        self.device = torch.device("cpu")
        self.msum = None

    def create(self, msum, hist_cap):
        self.msum = msum

    def sync(self):
        pass

    def gather(self, idx, src, dst):
        s = self.v[src] if isinstance(src, str) else src
        dst[: idx.numel()] = s.index_select(0, idx)

    def begin(self, tol, max_iter, x0):
        self.tol, self.max_iter = tol, max_iter
        self.sc = {"rho": 0.0, "alpha": 0.0, "nb": 0.0, "mu1": 0.0, "mu2": 0.0, "beta": 0.0,
                   "meanw": 0.0, "curv": float("nan")}
        self.fl = {"done": False, "iters": 0, "conv": False, "bad": False, "zero": False,
                   "maxit": False}
        self.res, self.pre = [], []
        self.v["x"].copy_(x0 if x0 is not None else self.v["x"] * 0.0)

    def _split(self, a, x, nsplit, ghost):
        import torch
        return torch.as_tensor(a @ np.concatenate([x[:nsplit].numpy(), ghost.numpy()]))

    def lambda_(self, which, ug, vg, use_flags):
        if use_flags and self.fl["done"]:
            return
        n, m = self.n, self.m
        v = self.v[which]
        q = self.v["q"]
        q[:n] = self._split(self.S1, v, n, ug[: self.lp.ghosts.size])
        iv = self._split(self.Si, v[n:], m, vg[: self.lp.m_ghost])
        q[:m] += iv
        q[n:] = self._split(self.Si, v, m, ug[: self.lp.m_ghost]) + iv
        q[n:] += self.lp.gamma * (_torch().as_tensor(self.lp.heart_mass) * v[n:])
        self.red[0] = float((v * q).sum())

    def init(self, b, has_x0):
        n = self.n
        r = self.v["r"]
        r.copy_(b - self.v["q"] if has_x0 else b)
        self.v["rhs_s"].copy_(r[n:])
        self.red[1], self.red[2], self.red[3] = float((r * r).sum()), float(r[:n].sum()), float(
            (b * b).sum())

    def check(self, initial):
        if self.fl["done"]:
            return
        if initial:
            self.red[7] = self.red[3]
            self.sc["nb"] = float(self.red[7]) ** 0.5
            if self.sc["nb"] == 0.0:
                self.fl.update(zero=True, conv=True, done=True)
                self.res.append(0.0)
                return
        rel = float(self.red[1]) ** 0.5 / self.sc["nb"]
        self.res.append(rel)
        if not np.isfinite(rel):
            self.fl.update(bad=True, done=True)
        elif rel <= self.tol:
            self.fl.update(conv=True, done=True)
        elif not initial and self.fl["iters"] >= self.max_iter:
            self.fl.update(maxit=True, done=True)
        else:
            self.sc["mu1"] = float(self.red[2]) / self.lp.n_global

    def update(self):
        if self.fl["done"]:
            return
        dq = float(self.red[0])
        if not (np.isfinite(dq) and dq > 0.0):
            self.fl.update(bad=True, done=True)
            self.sc["curv"] = dq
            return
        a = self.sc["rho"] / dq
        self.fl["iters"] += 1
        x, r, d, q = (self.v[k] for k in ("x", "r", "d", "q"))
        x += a * d
        r -= a * q
        self.v["rhs_s"].copy_(r[self.n:])
        self.red[1], self.red[2] = float((r * r).sum()), float(r[: self.n].sum())

    def pinv1(self):
        if self.fl["done"]:
            return
        y = (self.v["r"][: self.n] - self.sc["mu1"]).numpy()
        self.v["z1"].copy_(_torch().as_tensor(self.bulk.apply(y)))

    def pinv2(self, tg):
        if self.fl["done"] or self.m == 0:
            return
        rhs = self.v["rhs_s"] - self._split(self.Si, self.v["z1"], self.m, tg[: self.lp.m_ghost])
        self.v["s"].copy_(_torch().as_tensor(self.schur.apply(rhs.numpy())))

    def pinv3(self, sg):
        if self.fl["done"]:
            return
        c = self.v["corr"]
        if self.m:
            c[: self.m] = self._split(self.Si, self.v["s"], self.m, sg[: self.lp.m_ghost])
        self.red[3] = float(c[: self.m].sum())

    def pinv4(self):
        if self.fl["done"]:
            return
        self.sc["mu2"] = float(self.red[3]) / self.lp.n_global
        y = (self.v["corr"] - self.sc["mu2"]).numpy()
        z2 = _torch().as_tensor(self.bulk.apply(y))
        w = self.v["z1"] - z2
        self.v["z1"].copy_(w)
        n = self.n
        self.red[4], self.red[5] = float(w.sum()), float((self.v["r"][:n] * w).sum())
        self.red[6] = float((self.v["r"][n:] * self.v["s"]).sum())

    def finish(self, initial):
        if self.fl["done"]:
            return
        mw = float(self.red[4]) / self.lp.n_global
        rho = float(self.red[5]) - mw * float(self.red[2]) + float(self.red[6])
        self.pre.append(rho)
        beta = 0.0 if initial else rho / self.sc["rho"]
        self.sc.update(meanw=mw, rho=rho, beta=beta)
        d = self.v["d"]
        if initial:
            d.zero_()
        d[: self.n] = (self.v["z1"] - mw) + beta * d[: self.n]
        d[self.n:] = self.v["s"] + beta * d[self.n:]

    def tg_buffer(self, plan):
        return plan.tg

    def wmean(self):
        self.red[8] = float((_torch().as_tensor(self.lp.mass) * self.v["x"][: self.n]).sum())

    def normalize(self, out):
        if self.fl["zero"]:
            out.zero_()
            return
        out.copy_(self.v["x"])
        out[: self.n] -= float(self.red[8]) / self.msum

    def done(self):
        return self.fl["done"]

    def read(self, cap):
        f = self.fl
        return {"iterations": f["iters"], "converged": f["conv"], "breakdown": f["bad"],
                "zero_rhs": f["zero"], "max_iter": f["maxit"], "residual_history": list(self.res),
                "preconditioned_history": list(self.pre), "curvature": self.sc["curv"]}


class ShardSolver:
    """The sharded deflated PCG (bd/krylov.py:46-140, block-Jacobi block-LU
    preconditioner bd/precond.py:281-312) of one rank: halo all-gathers and the
    four all-reduces per iteration around the rank-local kernels of `ops`
    (NativeShard on the box, TorchShard in the CPU tests).  On a CUDA device
    one iteration, collectives included, is captured into a CUDA graph and
    replayed; the host reads the done flag every `check_every` iterations
    (replays past the end are device no-ops)."""

    def __init__(self, lp: "LocalProblem", comm: Comm, ops):
        self.lp, self.comm, self.ops = lp, comm, ops
        self.plan = HaloPlan(lp, comm, ops.device, ops.gather)
        self.msum = comm.allreduce([float(np.sum(lp.mass))])[0]
        self.graph = None
        self._graph_key = None
        self.graph_error = None
        self.body_launches = 0      # native kernels in one captured iteration
        self.replayed_launches = 0  # launched by graph replays (not seen by ctx.launches)

    def _pinv(self, initial):
        ops, plan, comm = self.ops, self.plan, self.comm
        ops.pinv1()
        tg = ops.tg_buffer(plan)
        plan.halo_h(comm, ops.ptr["z1"] if hasattr(ops, "ptr") else "z1", tg)
        ops.pinv2(tg)
        plan.halo_h(comm, ops.ptr["s"] if hasattr(ops, "ptr") else "s", plan.sg)
        ops.pinv3(plan.sg)
        comm.allreduce_(ops.red[3:4])
        ops.pinv4()
        comm.allreduce_(ops.red[4:7])
        ops.finish(initial)

    def _body(self):
        ops, plan, comm = self.ops, self.plan, self.comm
        plan.halo_d(comm, ops.ptr["d"] if hasattr(ops, "ptr") else "d")
        ops.lambda_("d", plan.ug, plan.vg, 1)
        comm.allreduce_(ops.red[0:1])
        ops.update()
        comm.allreduce_(ops.red[1:3])
        ops.check(0)
        self._pinv(0)

    def solve(self, b, x0=None, tol=1e-6, max_iter=500, check_every=16, graph=None):
        """b, x0: this rank's [u_own | v_own] (device tensors).  Returns
        (normalised x, stats dict); raises NonConvergenceError /
        NumericalBreakdownError with the stats (bd/krylov.py:103-108, 133-139)."""
        torch = _torch()
        if tol <= 0:
            raise ValueError("tol must be strictly positive")
        ops, plan, comm = self.ops, self.plan, self.comm
        h_before = getattr(ops, "h", None)
        ops.create(self.msum, max(max_iter + 2, 20002))
        if getattr(ops, "h", None) is not h_before:
            self.graph, self._graph_key = None, None  # new device buffers: recapture
        ops.sync()
        ops.begin(tol, max_iter, x0)
        if x0 is not None:
            plan.halo_d(comm, ops.ptr["x"] if hasattr(ops, "ptr") else "x")
            ops.lambda_("x", plan.ug, plan.vg, 0)
        ops.init(b, x0 is not None)
        comm.allreduce_(ops.red[1:4])
        ops.check(1)
        self._pinv(1)
        dev = b.device
        use_graph = (graph if graph is not None else
                     (dev.type == "cuda" and getattr(comm, "capturable", True)
                      and os.environ.get("BD_SHARDED_GRAPH", "1") != "0"))
        k = 0
        if not ops.done():
            if use_graph and self.graph is None and self._graph_key != id(ops):
                self._graph_key = id(ops)
                self._capture()
            g = self.graph if use_graph else None
            while k < max_iter:
                if g is not None:
                    g.replay()
                    self.replayed_launches += self.body_launches
                else:
                    self._body()
                k += 1
                if (k % check_every == 0 or k == max_iter) and ops.done():
                    break
            if not ops.done() and k >= max_iter:
                pass  # the device already flagged max_iter on the last check
        ops.wmean()
        comm.allreduce_(ops.red[8:9])
        out = torch.empty_like(b)
        ops.normalize(out)
        st = ops.read(max_iter + 2)
        st["graph"] = self.graph is not None and use_graph
        if self.graph_error:
            st["graph_error"] = self.graph_error
        st["mv_count"] = st["iterations"] + 1 + (1 if st["breakdown"] else 0)
        from .errors import NonConvergenceError, NumericalBreakdownError
        from .krylov import SolveStats
        stats = SolveStats(iterations=st["iterations"], residual_history=st["residual_history"],
                           preconditioned_history=st["preconditioned_history"],
                           mv_count=st["mv_count"], p1_count=2 * st["iterations"],
                           pk_count=st["iterations"], converged=st["converged"])
        if st["breakdown"]:
            raise NumericalBreakdownError(
                f"conjugate gradient breakdown: curvature {st['curvature']}", stats=stats)
        if not st["converged"]:
            raise NonConvergenceError(f"PCG did not reach tol={tol} within {max_iter} iterations",
                                      stats=stats)
        return out, st

    def _capture(self):
        """One iteration (kernels, halos, all-reduces) into a CUDA graph."""
        torch = _torch()
        dev = self.ops.device
        from . import _lib
        ctx = self.ops.ctx
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        try:
            g = torch.cuda.CUDAGraph()
            l0 = ctx.launches()
            with torch.cuda.graph(g, stream=side):
                ctx.sync_stream()
                self._body()
            self.body_launches = ctx.launches() - l0
            self.graph = g
        except Exception as e:  # capture unsupported here (e.g. P2P in capture): eager body
            self.graph = None
            self.graph_error = f"{type(e).__name__}: {e}"[:300]
        torch.cuda.current_stream(dev).wait_stream(side)
        ctx.sync_stream()
        _ = _lib


class HostStagedComm(Comm):
    """Comm whose partial sums and halos travel through host memory over a
    gloo process group.  For running several ranks on ONE GPU (tests and the
    iteration-count study, tools/sharded_iters.py): no kernel ever waits on
    another rank's kernels, the host does.  Not graph-capturable; not a
    product path (NCCL over NVLink is)."""

    capturable = False

    def allreduce_(self, t):
        if self.single:
            return t
        c = t.detach().cpu()
        self.dist.all_reduce(c)
        t.copy_(c)
        return t

    def allgather(self, send, out):
        if self.single:
            out.copy_(send)
            return out
        c = send.detach().cpu()
        parts = [_torch().empty_like(c) for _ in range(self.dist.get_world_size())]
        self.dist.all_gather(parts, c)
        out.copy_(_torch().cat(parts))
        return out


def _cpu_inner(kind):
    """Oracle inner solves for TorchShard (CPU tests only)."""
    def make(a):
        from oracle import bidomain_oracle as orc
        return orc.make_inner(kind, a)
    return make


# ---- per-rank setup without global matrices (large meshes) --------------------------
def _rows_csr(mesh, field, space, owned_rows, n_cols):
    """CSR (len(owned_rows) × n_cols, global column ids) of the stiffness rows
    of `owned_rows`, assembled from the elements that touch them only
    (same element matrices as assembly.assemble_stiffness)."""
    from .assembly import _grads_volumes, _select
    elements, tags, n = _select(mesh, space)
    pos = -np.ones(n, dtype=np.int64)
    pos[owned_rows] = np.arange(owned_rows.size)
    touch = (pos[elements] >= 0).any(axis=1)
    el, tg = elements[touch], tags[touch]
    if el.shape[0] == 0:
        return sp.csr_matrix((owned_rows.size, n_cols))
    grads, vols = _grads_volumes(mesh.vertices, el, mesh.dim)
    sigma = field.evaluate_batch(mesh.vertices[el].mean(axis=1), tg)
    local = np.einsum("eid,edk,ejk->eij", grads, sigma, grads)
    local = 0.5 * (local + local.transpose(0, 2, 1))
    local *= vols[:, None, None]
    arity = mesh.dim + 1
    rows = np.repeat(el, arity, axis=1).ravel()
    cols = np.tile(el, (1, arity)).ravel()
    keep = pos[rows] >= 0
    out = sp.coo_matrix((local.ravel()[keep], (pos[rows[keep]], cols[keep])),
                        shape=(owned_rows.size, n_cols)).tocsr()
    out.sum_duplicates()
    out.sort_indices()
    return out


def _rows_mass(mesh, space, owned_rows):
    from .assembly import _select
    import math
    elements, _, n = _select(mesh, space)
    pos = -np.ones(n, dtype=np.int64)
    pos[owned_rows] = np.arange(owned_rows.size)
    touch = (pos[elements] >= 0).any(axis=1)
    el = elements[touch]
    coords = mesh.vertices[el]
    det = np.linalg.det(coords[:, 1:, :] - coords[:, :1, :])
    share = det / math.factorial(mesh.dim) / (mesh.dim + 1)
    out = np.zeros(owned_rows.size)
    for k in range(mesh.dim + 1):
        p = pos[el[:, k]]
        ok = p >= 0
        np.add.at(out, p[ok], share[ok])
    return out


def ghost_sets(mesh, part: np.ndarray, nprocs: int):
    """Ghost vertices of every rank from the element connectivity: vertices
    of other ranks sharing an element with an owned vertex, in the order
    build_local uses (order_ghosts: heart then torso, grouped by owner)."""
    el = mesh.elements
    m = mesh.heart_vertex_count
    pe = part[el]
    out = []
    for r in range(nprocs):
        touch = (pe == r).any(axis=1)
        v = np.unique(el[touch])
        out.append(order_ghosts(v[part[v] != r], m, part))
    return out


def _rows_device(mesh, params, fibers, owned, m_own):
    """(S1, Si, Sm, mass, mh) of the owned rows, global columns, like
    `_rows_csr` / `_rows_mass` but assembled on the GPU: the elements touching
    owned vertices form a local mesh (owned + one ghost layer, renumbered
    heart-first), `DeviceAssembler` assembles it, and the owned rows are mapped
    back to global columns.  Owned rows are complete (every element touching
    an owned vertex is in the local mesh); ghost rows are discarded."""
    from .assembly import DeviceAssembler, Space
    from .mesh import Mesh

    n, m = mesh.vertex_count, mesh.heart_vertex_count
    pos = np.zeros(n, dtype=bool)
    pos[owned] = True
    touch = pos[mesh.elements].any(axis=1)
    el = mesh.elements[touch]
    verts = np.unique(el)                               # ascending global ids
    lv = np.concatenate([verts[verts < m], verts[verts >= m]])  # heart-first (already sorted)
    g2L = -np.ones(n, dtype=np.int64)
    g2L[lv] = np.arange(lv.size)
    hv = int((lv < m).sum())
    local = Mesh(mesh.dim, np.ascontiguousarray(mesh.vertices[lv]), g2L[el],
                 np.asarray(mesh.tags)[touch], hv)
    da = DeviceAssembler(local, params, fibers)

    def back(a, rows, cols_global, nglob):
        a = a[g2L[rows]].tocsr()
        out = sp.csr_matrix((a.data, cols_global[a.indices], a.indptr), shape=(rows.size, nglob))
        out.sort_indices()
        return out

    S1 = back(da.stiffness("bar1"), owned, lv, n)
    Si = back(da.stiffness("intra"), owned[:m_own], lv[:hv], m)
    Sm = back(da.stiffness("mono"), owned[:m_own], lv[:hv], m)
    mass = da.lumped_mass(Space.FULL)[g2L[owned]]
    mh = da.lumped_mass(Space.HEART_ONLY)[g2L[owned[:m_own]]]
    return S1, Si, Sm, mass, mh


def build_local_from_mesh(mesh, params, fibers, dt, part: np.ndarray, rank: int, nprocs: int,
                          comm_allreduce=None, assembly: str = "host") -> "LocalProblem":
    """The rank-local problem assembled from the elements touching the owned
    vertices only (assembly="device": on the GPU, `_rows_device`).  beta (mean
    diagonal of S_1, bd/precond.py:79-81) needs a global sum:
    comm_allreduce(list) -> list (None: single process)."""
    from .assembly import Space
    from .conductivity import TensorField
    from .system import gamma as gamma_fn
    n, m, d = mesh.vertex_count, mesh.heart_vertex_count, mesh.dim
    gam = gamma_fn(params.chi, params.c_m, dt)
    own = np.flatnonzero(part == rank)
    owned = np.concatenate([own[own < m], own[own >= m]])
    ghosts_all = ghost_sets(mesh, part, nprocs)
    ghosts = ghosts_all[rank]
    m_own, m_ghost = int((owned < m).sum()), int((ghosts < m).sum())
    if assembly == "device":
        S1, Si, Sm, mass, mh = _rows_device(mesh, params, fibers, owned, m_own)
    else:
        S1 = _rows_csr(mesh, TensorField(params, d, "bar1", fibers), Space.FULL, owned, n)
        Si = _rows_csr(mesh, TensorField(params, d, "intra", fibers), Space.HEART_ONLY,
                       owned[:m_own], m)
        Sm = _rows_csr(mesh, TensorField(params, d, "mono", fibers), Space.HEART_ONLY,
                       owned[:m_own], m)
        mass = _rows_mass(mesh, Space.FULL, owned)
        mh = _rows_mass(mesh, Space.HEART_ONLY, owned[:m_own])
    diag_sum = float(S1[np.arange(owned.size), owned].sum())
    tot = comm_allreduce([diag_sum]) if comm_allreduce else [diag_sum]
    beta = tot[0] / n
    ext = np.concatenate([owned, ghosts])
    g2l = -np.ones(n, dtype=np.int64)
    g2l[ext] = np.arange(ext.size)
    s1 = S1[:, ext].tocsr()
    hext = np.concatenate([owned[:m_own], ghosts[:m_ghost]])
    hmap = -np.ones(m, dtype=np.int64)
    hmap[hext] = np.arange(hext.size)
    si = Si[:, hext].tocsr()
    # block-Jacobi diagonal blocks: grounded S_1 (beta on global vertex 0) and K_m
    gb = S1[:, owned].tocsr()
    if part[0] == rank:
        k0 = int(np.flatnonzero(owned == 0)[0])
        bump = sp.csr_matrix(([beta], ([k0], [k0])), shape=gb.shape)
        gb = (gb + bump).tocsr()
    km = (Sm[:, owned[:m_own]] + gam * sp.diags(mh)).tocsr()
    for a in (s1, si, gb, km):
        a.sum_duplicates()
        a.sort_indices()
    lp = LocalProblem(rank, nprocs, n, m, owned, ghosts, owned.size, m_own, m_ghost, s1, si,
                      mass, mh, float(gam), gb, km)
    for q in range(nprocs):
        if q == rank:
            continue
        need = ghosts_all[q][part[ghosts_all[q]] == rank]
        if need.size:
            lp.send[q] = g2l[need]
            hm = need < m
            if hm.any():
                lp.send_heart[q] = g2l[need[hm]]
        mine = ghosts[part[ghosts] == q]
        if mine.size:
            lp.recv[q] = g2l[mine] - owned.size
            hm = mine < m
            if hm.any():
                lp.recv_heart[q] = g2l[mine[hm]] - owned.size
    lp.beta = beta
    lp.coords = np.ascontiguousarray(mesh.vertices[owned], dtype=float)
    return lp


class DistributedSimulation:
    """Sharded time loop: membrane RHS and gate on the owned heart vertices
    (sm_100a kernels), the coupled solve by ShardSolver over NativeShard."""

    def __init__(self, wl, part: np.ndarray, rank: int, nprocs: int, dist, device, inner=None,
                 comm=None):
        import torch

        from . import _lib
        from .ionic import site_masks

        self.wl = wl
        self.comm = comm or Comm(dist, device)
        self.lp = build_local_from_mesh(wl.mesh, wl.params, wl.fibers, wl.dt, part, rank, nprocs,
                                        comm_allreduce=self.comm.allreduce,
                                        assembly=os.environ.get("BD_ASSEMBLY", "device"))
        self.ctx = _lib.Context.default()
        self.shard = NativeShard(self.lp, inner or wl.inner, self.ctx)
        self.solver = ShardSolver(self.lp, self.comm, self.shard)
        lp = self.lp
        pts = wl.mesh.vertices[lp.owned[: lp.m_own]]
        masks = site_masks(pts, wl.protocol) if wl.protocol.sites else None
        self.mask = (torch.as_tensor(masks.view(np.int64)).to(device) if masks is not None
                     else None)
        self.mh = torch.as_tensor(lp.heart_mass, device=device)
        self._lib = _lib
        self.device = device

    def resting(self):
        import torch
        lp, ion = self.lp, self.wl.ionic
        return (torch.zeros(lp.n_own, dtype=torch.float64, device=self.device),
                torch.full((lp.m_own,), ion.v_rest, dtype=torch.float64, device=self.device),
                torch.ones(lp.m_own, dtype=torch.float64, device=self.device), 0.0)

    def step(self, state):
        """(u, v, w, t) -> new state, stats (bd/simulate.py:134-170, sharded)."""
        import torch
        from .ionic import active_sites
        u, v, w, t = state
        lp, wl, L = self.lp, self.wl, self._lib
        ion = wl.ionic
        self.ctx.sync_stream()
        rhs = torch.empty(lp.n_own + lp.m_own, dtype=torch.float64, device=self.device)
        L.check(L.lib().bd_membrane_rhs_raw(
            self.ctx.handle, lp.n_own, lp.m_own, L.ptr(self.mh), lp.gamma, L.ptr(v), L.ptr(w),
            L.ptr(self.mask), int(active_sites(t, wl.protocol)), float(wl.protocol.amplitude),
            float(wl.params.chi), float(ion.v_rest), float(ion.v_span), float(ion.tau_in),
            float(ion.tau_out), float(wl.params.c_m), L.ptr(rhs), None), self.ctx.handle)
        x, st = self.solver.solve(rhs, x0=torch.cat([u, v]), tol=wl.tol, max_iter=20000)
        v_new = x[lp.n_own:].contiguous()
        w_new = torch.empty_like(w)
        L.check(L.lib().bd_membrane_gate(
            self.ctx.handle, lp.m_own, L.ptr(v_new), L.ptr(w), float(wl.dt), float(ion.v_rest),
            float(ion.v_span), float(ion.tau_open), float(ion.tau_close), float(ion.u_gate),
            L.ptr(w_new)), self.ctx.handle)
        return (x[: lp.n_own].contiguous(), v_new, w_new, t + wl.dt), st
