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

Local compute goes through a backend object.  ``NativeBackend`` runs SpMV and
the inner solves in the sm_100a library.  The CPU tests inject a scipy backend
(tests/test_distributed.py) to check the partition / halo / collective logic
with gloo at world size 2.  Vectors are torch tensors on the rank's device;
collectives are torch.distributed (NCCL over NVLink on the box).
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
        gh = cols[part[cols] != r]
        gh = np.concatenate([gh[gh < m], gh[gh >= m]])
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
    """torch.distributed wrapper: halo exchange and global sums.

    Nothing here reads a value back to the host: sums are all-reduced in place
    on device tensors (NCCL on the box, gloo in the CPU tests) and the halo
    index lists are uploaded once."""

    def __init__(self, dist, device):
        self.dist = dist
        self.device = device
        self._idx = {}
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

    def _index(self, key, idx):
        torch = _torch()
        t = self._idx.get(key)
        if t is None:
            t = torch.as_tensor(np.asarray(idx, dtype=np.int64), device=self.device)
            self._idx[key] = t
        return t

    def halo(self, x_own, send: dict, recv: dict, nslots: int, tag: str = ""):
        """Ghost values of x from the owning neighbours (one layer)."""
        torch = _torch()
        out = torch.zeros(nslots, dtype=x_own.dtype, device=x_own.device)
        ops, bufs = [], {}
        for q, idx in send.items():
            buf = x_own.index_select(0, self._index((tag, "s", q), idx))
            ops.append(self.dist.P2POp(self.dist.isend, buf, q))
        for q, slots in recv.items():
            bufs[q] = torch.empty(len(slots), dtype=x_own.dtype, device=x_own.device)
            ops.append(self.dist.P2POp(self.dist.irecv, bufs[q], q))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        for q, slots in recv.items():
            out.index_copy_(0, self._index((tag, "r", q), slots), bufs[q])
        return out


def _torch():
    import torch

    return torch


# ---- distributed operator and solver ----------------------------------------------------
class DistributedSystem:
    """Λ on the rank's owned rows (block vector = [u_own | v_own])."""

    def __init__(self, lp: LocalProblem, comm: Comm, backend):
        self.lp, self.comm, self.be = lp, comm, backend
        self.S1 = backend.matrix(lp.S1)
        self.Si = backend.matrix(lp.Si)
        torch = _torch()
        self.mh = torch.as_tensor(lp.heart_mass, device=comm.device)
        self.mass = torch.as_tensor(lp.mass, device=comm.device)
        self.msum = comm.allreduce([float(lp.mass.sum())])[0]

    @property
    def n(self):
        return self.lp.n_own

    @property
    def m(self):
        return self.lp.m_own

    def heart_ghosts(self, v):
        lp = self.lp
        return self.comm.halo(v, lp.send_heart, lp.recv_heart, lp.m_ghost, "h")

    def spmv_split(self, a, x, nsplit, x_ghost, out=None):
        """a @ [x[:nsplit] ; x_ghost] without concatenating (native backend:
        bd_spmv_split); backends without it (the CPU test double) concatenate."""
        f = getattr(self.be, "spmv_split", None)
        if f is not None:
            return f(a, x, nsplit, x_ghost, out)
        y = self.be.spmv(a, _torch().cat([x[:nsplit], x_ghost]))
        if out is None:
            return y
        out.copy_(y)
        return out

    def apply(self, x):
        """q = Λ x (bd/system.py:106-116) with halo exchanges of u and v.
        Local columns are [owned | ghosts] for S_1 and [owned heart | ghost
        heart] for S_i; heart vertices lead both the owned and the ghost lists,
        so the S_i products read u and v with a split at m_own."""
        lp = self.lp
        n, m = lp.n_own, lp.m_own
        u, v = x[:n], x[n:]
        ug = self.comm.halo(u, lp.send, lp.recv, lp.ghosts.size, "u")
        vg = self.heart_ghosts(v)
        q = _torch().empty_like(x)
        iv = self.spmv_split(self.Si, v, m, vg)
        self.spmv_split(self.S1, u, n, ug, out=q[:n])
        q[:m] += iv
        qv = q[n:]
        self.spmv_split(self.Si, u, m, ug, out=qv)
        qv += iv
        qv += lp.gamma * (self.mh * v)
        return q

    def dot_t(self, a, b):
        """Global a·b as a device 0-d tensor (one fused dot per rank)."""
        return self.comm.allreduce_(_torch().dot(a, b).reshape(1))[0]

    def mean_u_t(self, u):
        return self.comm.allreduce_(u.sum().reshape(1))[0] / self.lp.n_global

    def dot(self, a, b):
        return float(self.dot_t(a, b))

    def mean_u(self, u):
        return float(self.mean_u_t(u))

    def normalize(self, x):
        lp = self.lp
        alpha = self.comm.allreduce_((self.mass * x[: lp.n_own]).sum().reshape(1))[0] / self.msum
        out = x.clone()
        out[: lp.n_own] -= alpha
        return out


class DistributedBlockLU:
    """Block-LU P_Λ (bd/precond.py:281-312) with block-Jacobi inner solves."""

    def __init__(self, dsys: DistributedSystem, inner: str, beta: float):
        self.s, self.beta = dsys, beta
        be = dsys.be
        lp = dsys.lp
        xyz = getattr(lp, "coords", None)  # owned-vertex coordinates: lattice tiles for IC(0)
        self.bulk = be.inner(inner, lp.bulk_block, None if xyz is None else xyz)
        self.schur = be.inner(inner, lp.schur_block, None if xyz is None else xyz[: lp.m_own])
        self.p1 = self.pk = self.si = 0
        self._corr = None  # pad(S_i s): torso rows stay zero, heart rows rewritten per apply

    def bulk_inverse(self, y, mean=None):
        """`mean` (device 0-d): mean(y) when the caller already reduced it."""
        self.p1 += 1
        s = self.s
        if mean is None:
            mean = s.mean_u_t(y)
        z = s.be.inner_apply(self.bulk, y - mean)
        z = z - s.mean_u_t(z)
        return z + mean / self.beta

    def apply(self, r, mean_ru=None):
        s, lp = self.s, self.s.lp
        ru, rv = r[: lp.n_own], r[lp.n_own:]
        t = self.bulk_inverse(ru, mean_ru)
        tg = s.heart_ghosts(t[: lp.m_own])  # collective on all ranks
        self.si += 1
        self.pk += 1
        sv = s.be.inner_apply(self.schur, rv - s.spmv_split(s.Si, t, lp.m_own, tg))
        sg = s.heart_ghosts(sv)
        self.si += 1
        if self._corr is None or self._corr.shape != ru.shape or self._corr.device != ru.device:
            self._corr = _torch().zeros_like(ru)
        corr = self._corr
        s.spmv_split(s.Si, sv, lp.m_own, sg, out=corr[: lp.m_own])
        u = t - self.bulk_inverse(corr)
        return _torch().cat([u, sv])


def distributed_pcg(dsys: DistributedSystem, prec: DistributedBlockLU, b, tol=1e-6,
                    max_iter=500, x0=None, check_every=16, graph=None):
    """The reference iteration (bd/krylov.py:46-140) on the sharded system,
    device-resident: every scalar (α, β, ρ, the means, the residual) stays a
    device tensor, reductions are in-place all-reduces, and the host reads the
    convergence / breakdown flags only every `check_every` iterations.
    Iterations after convergence are masked to exact no-ops (α = 0, ρ and d
    kept), so iterates, histories and counts equal those of the per-iteration
    test.  On a CUDA device one iteration is captured into a CUDA graph (NCCL
    collectives included) and replayed; `graph=False` (or a failed capture)
    runs the same body eagerly.  Returns (x_local, stats dict); raises
    RuntimeError past max_iter / on breakdown (bd/krylov.py:103-108, 133-135)."""
    torch = _torch()
    st = {"iterations": 0, "residual_history": [], "preconditioned_history": [],
          "mv_count": 0, "converged": False}
    n = dsys.n
    nb = float(dsys.dot_t(b, b)) ** 0.5
    if nb == 0.0:
        st["residual_history"].append(0.0)
        st["converged"] = True
        return torch.zeros_like(b), st
    if x0 is None:
        x = torch.zeros_like(b)
        r = b.clone()
    else:
        x = x0.clone()
        r = b - dsys.apply(x)
    st["mv_count"] += 1
    rel = float(dsys.dot_t(r, r)) ** 0.5 / nb
    st["residual_history"].append(rel)
    if rel <= tol:
        st["converged"] = True
        return dsys.normalize(x), st

    def precond(r, mean_ru=None):
        z = prec.apply(r, mean_ru)
        z[:n] -= dsys.mean_u_t(z[:n])  # _deflate
        return z

    dev, f64 = b.device, torch.float64
    cnt = [prec.p1, prec.pk, prec.si]
    z = precond(r)
    S = {  # static state of the loop (graph-safe: only updated in place)
        "x": x, "r": r, "d": z.clone(),
        "rho": dsys.dot_t(r, z).reshape(()).clone(),
        "active": torch.ones((), dtype=torch.bool, device=dev),
        "bad": torch.zeros((), dtype=torch.bool, device=dev),
        "iters": torch.zeros((), dtype=torch.int64, device=dev),
        "k": torch.zeros((), dtype=torch.int64, device=dev),
        "res": torch.full((max_iter + 1,), -1.0, dtype=f64, device=dev),
        "pre": torch.full((max_iter + 1,), float("nan"), dtype=f64, device=dev),
    }
    S["pre"][0] = S["rho"]
    zero = torch.zeros((), dtype=f64, device=dev)

    def body():
        d, rho, active = S["d"], S["rho"], S["active"]
        q = dsys.apply(d)
        dq = dsys.dot_t(d, q)
        brk = active & ~(torch.isfinite(dq) & (dq > 0))
        S["bad"].logical_or_(brk)
        go = active & ~brk
        alpha = torch.where(go, rho / dq, zero)
        S["x"].addcmul_(d, alpha)
        S["r"].addcmul_(q, alpha, value=-1.0)
        S["iters"].add_(go.to(torch.int64))
        # ‖r‖² and Σ r_u (the first bulk solve's mean) in one all-reduce
        pair = torch.stack([torch.dot(S["r"], S["r"]), S["r"][:n].sum()])
        dsys.comm.allreduce_(pair)
        relk = torch.sqrt(pair[0]) / nb
        S["k"].add_(1)
        S["res"].index_put_((S["k"],), torch.where(go, relk, torch.full_like(relk, -1.0)))
        act = go & ~(relk <= tol)
        zz = precond(S["r"], pair[1] / dsys.lp.n_global)
        rho_next = dsys.dot_t(S["r"], zz)
        S["pre"].index_put_((S["k"],), torch.where(act, rho_next, torch.full_like(rho_next, float("nan"))))
        beta = torch.where(act, rho_next / rho, zero)
        d.copy_(torch.where(act, zz + beta * d, d))
        rho.copy_(torch.where(act, rho_next, rho))
        active.copy_(act)

    use_graph = graph if graph is not None else (dev.type == "cuda" and os.environ.get("BD_SHARDED_GRAPH", "1") != "0")
    g = None
    k_done = 0
    if use_graph:
        from . import _lib
        ctx = _lib.Context.default()
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):  # first iteration eagerly: warms the allocator pools
            ctx.sync_stream()
            body()
        torch.cuda.current_stream(dev).wait_stream(side)
        k_done = 1
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                ctx.sync_stream()
                body()
        except Exception as e:  # capture unsupported here (e.g. P2P in capture): eager body
            g = None
            st["graph_error"] = f"{type(e).__name__}: {e}"[:300]
        ctx.sync_stream()
    while k_done < max_iter:
        if g is not None:
            g.replay()
        else:
            body()
        k_done += 1
        if k_done % check_every == 0 or k_done == max_iter:
            if not bool(S["active"]) or bool(S["bad"]):
                break
    n_it = int(S["iters"])
    # the reference applies P^-1 once before the loop and once per
    # non-final iteration (bd/krylov.py:95, 125): p1 += 2, pk += 1, si += 2 each
    prec.p1, prec.pk, prec.si = cnt[0] + 2 * n_it, cnt[1] + n_it, cnt[2] + 2 * n_it
    bad = bool(S["bad"])
    res = S["res"][1: k_done + 1].tolist()
    st["residual_history"].extend(h for h in res if h >= 0)
    pre = S["pre"][: k_done + 1].tolist()
    st["preconditioned_history"] = [h for h in pre if h == h]
    st["iterations"] = n_it
    st["graph"] = g is not None
    st["mv_count"] += n_it + (1 if bad else 0)
    if bad:
        raise RuntimeError("conjugate gradient breakdown: curvature <= 0 or not finite")
    if bool(S["active"]):
        raise RuntimeError(f"PCG did not reach tol={tol} within {max_iter} iterations")
    st["converged"] = True
    return dsys.normalize(S["x"]), st


class NativeBackend:
    """Local compute in the sm_100a library (SpMV, inner solves)."""

    def __init__(self):
        from . import _lib
        from .system import NativeCsr

        self._lib = _lib
        self._csr = NativeCsr
        self.ctx = _lib.Context.default()

    def matrix(self, a):
        return self._csr(self.ctx, sp.csr_matrix(a))

    def spmv(self, h, x):
        return h.matvec(x.contiguous())

    def spmv_split(self, h, x, nsplit, x_ghost, out=None):
        return h.matvec_split(x.contiguous(), nsplit, x_ghost.contiguous(), y=out)

    def inner(self, kind, a, coords=None):
        from .precond import make_inner

        p = make_inner(kind)
        if coords is not None and hasattr(p, "setup") and kind == "ic0":
            p.setup(a, coords=coords)
        else:
            p.setup(a)
        return p

    def inner_apply(self, h, y):
        return h.apply_inverse(y.contiguous())


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
    of other ranks sharing an element with an owned vertex (heart first,
    then torso, each ascending — the order build_local uses)."""
    el = mesh.elements
    m = mesh.heart_vertex_count
    pe = part[el]
    out = []
    for r in range(nprocs):
        touch = (pe == r).any(axis=1)
        v = np.unique(el[touch])
        g = v[part[v] != r]
        out.append(np.concatenate([g[g < m], g[g >= m]]))
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
    (sm_100a kernels), the coupled solve by distributed_pcg."""

    def __init__(self, wl, part: np.ndarray, rank: int, nprocs: int, dist, device, inner=None):
        import torch

        from . import _lib
        from .ionic import site_masks

        self.wl = wl
        self.comm = Comm(dist, device)
        self.lp = build_local_from_mesh(wl.mesh, wl.params, wl.fibers, wl.dt, part, rank, nprocs,
                                        comm_allreduce=self.comm.allreduce,
                                        assembly=os.environ.get("BD_ASSEMBLY", "device"))
        self.backend = NativeBackend()
        self.dsys = DistributedSystem(self.lp, self.comm, self.backend)
        self.prec = DistributedBlockLU(self.dsys, inner or wl.inner, self.lp.beta)
        lp = self.lp
        pts = wl.mesh.vertices[lp.owned[: lp.m_own]]
        masks = site_masks(pts, wl.protocol) if wl.protocol.sites else None
        self.mask = (torch.as_tensor(masks.view(np.int64)).to(device) if masks is not None
                     else None)
        self.mh = torch.as_tensor(lp.heart_mass, device=device)
        self.ctx = _lib.Context.default()
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
        rhs = torch.empty(lp.n_own + lp.m_own, dtype=torch.float64, device=self.device)
        L.check(L.lib().bd_membrane_rhs_raw(
            self.ctx.handle, lp.n_own, lp.m_own, L.ptr(self.mh), lp.gamma, L.ptr(v), L.ptr(w),
            L.ptr(self.mask), int(active_sites(t, wl.protocol)), float(wl.protocol.amplitude),
            float(wl.params.chi), float(ion.v_rest), float(ion.v_span), float(ion.tau_in),
            float(ion.tau_out), float(wl.params.c_m), L.ptr(rhs), None), self.ctx.handle)
        x, st = distributed_pcg(self.dsys, self.prec, rhs, tol=wl.tol, max_iter=20000,
                                x0=torch.cat([u, v]))
        v_new = x[lp.n_own:].contiguous()
        w_new = torch.empty_like(w)
        L.check(L.lib().bd_membrane_gate(
            self.ctx.handle, lp.m_own, L.ptr(v_new), L.ptr(w), float(wl.dt), float(ion.v_rest),
            float(ion.v_span), float(ion.tau_open), float(ion.tau_close), float(ion.u_gate),
            L.ptr(w_new)), self.ctx.handle)
        return (x[: lp.n_own].contiguous(), v_new, w_new, t + wl.dt), st
