"""Quick GPU sanity run against the small golden fixtures (dev tool)."""
import sys, time, numpy as np, scipy.sparse as sp
sys.path.insert(0, '/root/repo')
import torch
import paper_1711_08708_b200 as B

def csr(g, k):
    return sp.csr_matrix((g[k+'_data'], g[k+'_indices'], g[k+'_indptr']), shape=tuple(g[k+'_shape']))

for case in ("small_coupled2d", "small_square4", "small_cube2"):
    g = np.load(f'/root/repo/tests/golden/{case}.npz')
    sysm = B.BidomainSystem(csr(g,'S1'), csr(g,'Si'), csr(g,'Se'), g['mass'], g['mh'], float(g['gamma']))
    x = B.BlockVector(g['x_u'], g['x_v'])
    q = sysm.apply(x); qu, qv = q.numpy()
    print(case, "lambda rel err", np.abs(qu-g['lam_u']).max()/np.abs(g['lam_u']).max(), np.abs(qv-g['lam_v']).max()/np.abs(g['lam_v']).max())
    for inner in ("ic0", "jacobi", "exact"):
        t0=time.time()
        pre = B.BlockLUPreconditioner(sysm, inner=inner, monodomain_matrix=csr(g,'Km'))
        if inner == "ic0":
            L = pre.inner_bulk.lower_factor
            print("  ic0 L1 bitwise:", np.array_equal(L.data, g['L1_data']), "LK bitwise:", np.array_equal(pre.inner_schur.lower_factor.data, g['LK_data']))
        z = pre.apply_inverse(B.BlockVector(g['y_u'], g['y_v'])); zu, zv = z.numpy()
        ru = g[f'pinv_{inner}_u']; rv = g[f'pinv_{inner}_v']
        print(f"  {inner} pinv rel err u {np.abs(zu-ru).max()/np.abs(ru).max():.2e} v {np.abs(zv-rv).max()/np.abs(rv).max():.2e}")
        b1 = pre._bulk_inverse(np.ones(sysm.n))
        print(f"  {inner} bulk(1) bitwise:", np.array_equal(b1, g[f'bulk1_{inner}']), "counters", pre.p1_count, pre.pk_count, pre.si_count)
        pre.reset_counters()
        xs, st = B.pcg_solve(sysm, pre, B.BlockVector(g['b_u'], g['b_v']), tol=1e-10, max_iter=2000)
        xu, xv = xs.numpy()
        eu = g[f'pcg_{inner}_u']; ev = g[f'pcg_{inner}_v']
        rel = np.sqrt(((xu-eu)**2).sum()+((xv-ev)**2).sum())/np.sqrt((eu**2).sum()+(ev**2).sum())
        print(f"  {inner} pcg iters gpu {st.iterations} ref {int(g[f'pcg_{inner}_iters'])} counts {st.mv_count,st.p1_count,st.pk_count} ref {g[f'pcg_{inner}_counts']} rel {rel:.2e} dev_ms {st.device_time_ms:.2f} wall {st.wall_time_ms:.2f} ({time.time()-t0:.2f}s)")
        print("   res hist diff", np.abs(np.array(st.residual_history)-g[f'pcg_{inner}_res']).max() if len(st.residual_history)==len(g[f'pcg_{inner}_res']) else "LEN MISMATCH")
print("launches", B._lib.Context.default().launches())
