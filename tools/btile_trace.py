"""Dev tool: per-tile timestamps of the blocked-tile triangular solve on cfg2
(grab, inputs ready, published) for the backward pass of one IC(0) apply, and
the critical path split into hop (ready - last dependency published) and
compute (published - ready).  Tiles are lattice bins, deps = the +1 bins."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, '/root/repo')
os.environ.setdefault("BD_TRSV", "btile")
import torch
import paper_1711_08708_b200 as bd
from paper_1711_08708_b200 import configs, _lib
from paper_1711_08708_b200.assembly import assemble_stiffness
from paper_1711_08708_b200.conductivity import TensorField
from paper_1711_08708_b200.precond import regularize_stiffness
cells = tuple(int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "128,128,64").split(","))
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl = configs.cfg2(cells)
S1 = assemble_stiffness(wl.mesh, TensorField(wl.params, 3, "bar1", wl.fibers))
g = regularize_stiffness(S1).grounded()
inner = bd.IncompleteCholesky0(); inner.setup(g, coords=wl.mesh.vertices)
L = _lib.lib()
L.bd_debug_tile_trace.argtypes = [C.c_void_p, C.c_int]
L.bd_debug_btile_rows.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
ntc = C.c_int()
L.bd_debug_btile_rows(inner.handle, 1, None, C.byref(ntc)); nt = ntc.value
first = np.zeros(nt, dtype=np.int32)
L.bd_debug_btile_rows(inner.handle, 1, first.ctypes.data, C.byref(ntc))
V = wl.mesh.vertices
rank = [np.searchsorted(np.unique(V[:, a]), V[first, a]) for a in range(3)]
bins = np.stack([r // 4 for r in rank], 1)
key = {tuple(b): t for t, b in enumerate(bins)}
buf = torch.zeros(nt * 8 + 8, dtype=torch.int64, device='cuda')
y = torch.as_tensor(np.random.default_rng(0).standard_normal(g.shape[0])).cuda()
for _ in range(3):
    inner.apply_inverse(y)
torch.cuda.synchronize()
for rep in range(reps):
    buf.zero_()
    L.bd_debug_tile_trace(C.c_void_p(buf.data_ptr()), 1)
    inner.apply_inverse(y); torch.cuda.synchronize()
    L.bd_debug_tile_trace(None, 0)
    tr = buf[: nt * 8].view(nt, 8).cpu().numpy().astype(np.int64)
    t0 = tr[:, 0].min()
    grab, ready, done = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, (tr[:, 2] - t0) / 1e3
    polled, prep = (tr[:, 4] - t0) / 1e3, (tr[:, 5] - t0) / 1e3
    extd, densed = (tr[:, 6] - t0) / 1e3, (tr[:, 7] - t0) / 1e3
    deps = []
    for t in range(nt):
        b = bins[t]
        d = [key[(b[0] + a, b[1] + c, b[2] + e)] for a in (0, 1) for c in (0, 1) for e in (0, 1)
             if (a, c, e) != (0, 0, 0) and (b[0] + a, b[1] + c, b[2] + e) in key]
        deps.append(d)
    last_dep = np.array([max(done[d]) if d else 0.0 for d in deps])
    hop = ready - np.maximum(last_dep, grab)
    comp = done - ready
    # critical path from the last-finishing tile
    t = int(np.argmax(done)); path = []
    while True:
        path.append(t)
        if not deps[t]:
            break
        t = max(deps[t], key=lambda q: done[q])
    path = path[::-1]
    ph, pc = hop[path], comp[path]
    pre = np.array([max(0.0, grab[q] - (max(done[deps[q]]) if deps[q] else 0)) for q in path])
    print(f"rep {rep}: span {done.max():.1f} us, critical path {len(path)} tiles: "
          f"hop sum {ph.sum():.1f} (median {np.median(ph):.2f}), compute sum {pc.sum():.1f} "
          f"(median {np.median(pc):.2f}), grab-after-ready sum {pre.sum():.1f}")
    print("   all tiles: hop median %.2f p90 %.2f; compute median %.2f p90 %.2f" % (
        np.median(hop), np.percentile(hop, 90), np.median(comp), np.percentile(comp, 90)))
    p_poll = polled[path] - np.maximum(last_dep[path], prep[path])
    p_cp = ready[path] - polled[path]
    p_prep = prep[path] - grab[path]
    print(f"   path: poll-after-max(dep,prep) sum {p_poll.sum():.1f} median {np.median(p_poll):.2f}; "
          f"polled->ready sum {p_cp.sum():.1f} median {np.median(p_cp):.2f}; grab->prep median {np.median(p_prep):.2f}; "
          f"prep after last dep: {(prep[path] > last_dep[path]).sum()} tiles")
    P = np.array(path)
    print("   path medians: ext-sum %.2f, sync %.2f, dense %.2f, tail(sync) %.2f" % (
        np.median(extd[P] - polled[P]), np.median(ready[P] - extd[P]), np.median(densed[P] - ready[P]),
        np.median(done[P] - densed[P])))
    dn = densed - ready
    order = np.argsort(ready)
    print("   dense by start order (first 50 / middle / last 50 tiles): %.2f / %.2f / %.2f" % (
        np.median(dn[order[:50]]), np.median(dn[order[len(order)//2-500:len(order)//2+500]]), np.median(dn[order[-50:]])))
    seg = np.array_split(np.arange(len(path)), 6)
    print("   path poll/cp by segment:", [(round(p_poll[s_].mean(), 2), round(p_cp[s_].mean(), 2)) for s_ in seg])
    print("   path hop/compute by segment:", [(round(ph[s].mean(), 2), round(pc[s].mean(), 2)) for s in seg])
    # --- per-phase statistics over ALL tiles (time sixths of the pass) ---
    if rep == reps - 1:
        edges = np.linspace(0, done.max(), 7)
        for s_ in range(6):
            sel = (done >= edges[s_]) & (done < edges[s_ + 1] + (1e-9 if s_ == 5 else 0))
            if not sel.any():
                continue
            lead = last_dep[sel] - grab[sel]          # > 0: grabbed before its last input was published
            pp = prep[sel] - grab[sel]
            late = (prep[sel] > last_dep[sel]).mean()
            resid = done[sel] - grab[sel]
            h2 = polled[sel] - np.maximum(last_dep[sel], prep[sel])
            print(f"   sixth {s_}: {sel.sum()} tiles; grab->prep med {np.median(pp):.2f} p90 {np.percentile(pp,90):.2f}; "
                  f"lead med {np.median(lead):.2f} p10 {np.percentile(lead,10):.2f}; prep-late frac {late:.2f}; "
                  f"residency med {np.median(resid):.2f}; poll-after-max(dep,prep) med {np.median(h2):.2f} p90 {np.percentile(h2,90):.2f}")
        if os.environ.get("BD_BTILE_KERNEL", "auto") in ("rpipe", "auto"):
            top = densed  # rpipe records "became current" in slot 7
            order_c = np.lexsort((top, tr[:, 3] & 0xffffffff))
            cta = (tr[:, 3] & 0xffffffff)[order_c]
            same = cta[1:] == cta[:-1]
            gap = (top[order_c][1:] - done[order_c][:-1])[same]
            mid = (done > done.max() / 3) & (done < 2 * done.max() / 3)
            print("   rpipe mid-pass: mbar wait med %.2f p90 %.2f; landed->regs med %.2f p90 %.2f" % (
                np.median((extd - top)[mid]), np.percentile((extd - top)[mid], 90),
                np.median((prep - extd)[mid]), np.percentile((prep - extd)[mid], 90)))
            print("   rpipe mid-pass: fetch issue->current med %.2f; current->regs loaded (mbar wait+LDS) med %.2f p90 %.2f; "
                  "regs->polled med %.2f; polled->done med %.2f; current->done med %.2f; done->next current med %.2f" % (
                      np.median((top - grab)[mid]), np.median((prep - top)[mid]), np.percentile((prep - top)[mid], 90),
                      np.median((polled - prep)[mid]), np.median((done - polled)[mid]), np.median((done - top)[mid]),
                      np.median(gap)))
        if os.environ.get("BD_BTILE_KERNEL", "auto") in ("rpipe", "auto"):
            # why do tiles become current late?  prev = the CTA's previous tile
            top = densed
            ctaid = tr[:, 3] & 0xffffffff
            order_c = np.lexsort((top, ctaid))
            prev = np.full(nt, -1)
            same = ctaid[order_c][1:] == ctaid[order_c][:-1]
            prev[order_c[1:][same]] = order_c[:-1][same]
            mid = (done > done.max() / 3) & (done < 2 * done.max() / 3) & (prev >= 0)
            late = top - last_dep           # > 0: became current after its last input was published
            pw = (polled - top)[prev]       # how long the previous tile waited for its inputs
            lm = mid & (late > 0)
            print("   mid-pass: %d tiles, late %.2f; of the late ones: previous tile waited > 1.2 us: %.2f "
                  "(median wait %.2f); late by med %.2f p90 %.2f" % (
                      mid.sum(), lm.sum() / max(mid.sum(), 1), (pw[lm] > 1.2).mean(), np.median(pw[lm]),
                      np.median(late[lm]), np.percentile(late[lm], 90)))
            # level structure: spread of completion times within a tile level
            lvl = bins.sum(1)
            lv_done = np.array([[done[lvl == q].min(), np.median(done[lvl == q]), done[lvl == q].max()]
                                for q in range(lvl.max() + 1)])
            dl = np.diff(lv_done[:, 2])
            print("   level max-done increments: first sixth %.2f, middle %.2f, last sixth %.2f; "
                  "spread (max-min) in the middle %.2f" % (
                      np.median(dl[: len(dl) // 6]), np.median(dl[len(dl) // 3: 2 * len(dl) // 3]),
                      np.median(dl[-len(dl) // 6:]),
                      np.median((lv_done[:, 2] - lv_done[:, 0])[len(dl) // 3: 2 * len(dl) // 3])))
        # in-flight tiles over time
        ts = np.linspace(0, done.max(), 13)[1:-1]
        print("   in flight at t:", [(round(float(x), 0), int(((grab <= x) & (done > x)).sum())) for x in ts])
        print("   waiting (prep done, not ready) at t:", [(round(float(x), 0), int(((prep <= x) & (polled > x)).sum())) for x in ts])
np.save("/root/repo/gpurun_out/btile_trace.npy", tr)
