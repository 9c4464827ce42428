"""GPU: every blocked-tile triangular-solve kernel (BD_BTILE_KERNEL)
gives the oracle's IC(0) application on the same factor, on a lattice-ordered
slab (config 2 shape) and on a heart-first heart-in-torso box (config 4
shape: class-separated tiles, rows with more than 8 external entries), with
and without inbox polling.  Tolerance 1e-12 relative (summation order)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1711_08708_b200 as bd  # noqa: E402
from oracle import bidomain_oracle as orc  # noqa: E402
from paper_1711_08708_b200 import configs  # noqa: E402
from paper_1711_08708_b200.precond import regularize_stiffness  # noqa: E402

KERNELS = ["auto", "rpipe", "reg", "rsmem", "regt", "pipe", "smem"]


@pytest.fixture(scope="module")
def problems():
    out = {}
    for name, wl in (("slab", configs.cfg2((16, 16, 8))), ("torso", configs.cfg4(16))):
        sysm = bd.BidomainSystem.build(wl.mesh, wl.params, wl.dt, fibers=wl.fibers,
                                       with_extra=False)
        g = regularize_stiffness(sysm.stiff_total).grounded()
        ref = orc.make_inner("ic0", g)
        out[name] = (g, wl.mesh.vertices, ref)
    return out


@pytest.mark.parametrize("inbox", ["0", "1"])
@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("name", ["slab", "torso"])
def test_tile_kernel_matches_oracle(problems, name, kernel, inbox, monkeypatch, rng):
    if inbox == "1" and kernel != "reg":
        pytest.skip("inbox polling is a reg-kernel option")
    monkeypatch.setenv("BD_TRSV", "btile")
    monkeypatch.setenv("BD_BTILE_KERNEL", kernel)
    monkeypatch.setenv("BD_BTILE_INBOX", inbox)
    g, xyz, ref = problems[name]
    ic = bd.IncompleteCholesky0()
    ic.setup(g, coords=xyz)
    for _ in range(3):
        y = rng.standard_normal(g.shape[0])
        got, want = ic.apply_inverse(y), ref.apply(y)
        assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


@pytest.mark.parametrize("name", ["slab", "torso"])
def test_ring_kernel_wide_matches_oracle(problems, name, monkeypatch, rng):
    """k_trsv_rpipe with the two-inputs-per-thread instantiation (tiles with more
    than 256 inputs) forced."""
    monkeypatch.setenv("BD_TRSV", "btile")
    monkeypatch.setenv("BD_BTILE_KERNEL", "rpipe")
    monkeypatch.setenv("BD_RPIPE_WIDE", "1")
    g, xyz, ref = problems[name]
    ic = bd.IncompleteCholesky0()
    ic.setup(g, coords=xyz)
    for _ in range(3):
        y = rng.standard_normal(g.shape[0])
        got, want = ic.apply_inverse(y), ref.apply(y)
        assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()


@pytest.mark.parametrize("dense_max,pack,inv_min", [("0", "0", "128"), ("0", "1", "128"),
                                                     ("0", "0", "33"), ("0", "0", "0"),
                                                     ("100000", "0", "128")])
@pytest.mark.parametrize("name", ["slab", "torso"])
def test_exact_inner_paths_match_oracle(problems, name, dense_max, pack, inv_min, monkeypatch, rng):
    """The exact inner as supernodal passes (BD_EXACT_DENSE_MAX=0: split
    external phases, panel inverses; BD_SUPER_PACK=1: several small supernodes
    per warp; BD_SUPER_INV_MIN: whole-block inverses from that size, 0 = none)
    and as the dense explicit inverse all give the oracle's exact solve (1e-10
    relative)."""
    monkeypatch.setenv("BD_EXACT_DENSE_MAX", dense_max)
    monkeypatch.setenv("BD_SUPER_PACK", pack)
    monkeypatch.setenv("BD_SUPER_INV_MIN", inv_min)
    g, _, _ = problems[name]
    ref = orc.make_inner("exact", g)
    ex = bd.ExactFactorization()
    ex.setup(g)
    for _ in range(2):
        y = rng.standard_normal(g.shape[0])
        got, want = ex.apply_inverse(y), ref.apply(y)
        assert np.abs(got - want).max() <= 1e-10 * np.abs(want).max()


@pytest.mark.parametrize("mode", ["dtile", "persist", "syncfree", "tiled", "rows", "cluster"])
@pytest.mark.parametrize("name", ["slab", "torso"])
def test_fallback_schedules_match_oracle(problems, name, mode, monkeypatch, rng):
    """The non-default triangular-solve schedules (BD_TRSV):
    dtile and persist are the live fallbacks when a blocked-tile schedule
    cannot be built, syncfree (any other value) is the level-free v0 kernel
    pair; tiled / rows / cluster are the cooperative and cluster variants.
    Each must give the oracle's IC(0) application (1e-12 relative)."""
    monkeypatch.setenv("BD_TRSV", mode)
    g, xyz, ref = problems[name]
    ic = bd.IncompleteCholesky0()
    ic.setup(g, coords=xyz)
    for _ in range(3):
        y = rng.standard_normal(g.shape[0])
        got, want = ic.apply_inverse(y), ref.apply(y)
        assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
