"""SELL column panels (one GPU): the stored superoperator split into column
ranges whose slice of x stays in L2 (c4), partial row sums carried between
the panel kernels.  Forced on the golden cases with QSWG_SELL_PANELS; every
result must still match the reference (same tolerances as
test_gpu_parity.py), and the assembled matrix must be the same canonical CSR."""
import numpy as np
import pytest

from conftest import CASE_NAMES, Case

pytestmark = pytest.mark.gpu
api = pytest.importorskip("paper_2003_02450_b200.api")

RHO_TOL = 1e-10


@pytest.mark.parametrize("panels", [2, 3, 7])
@pytest.mark.parametrize("name", [c for c in CASE_NAMES if not c.startswith("walkthrough")])
def test_panelled_sell_matches_reference(name, panels, monkeypatch):
    monkeypatch.setenv("QSWG_SELL_PANELS", str(panels))
    c = Case(name)
    l = c.build_gpu(api, format="sell")
    assert l.format == "sell"
    L = l.gather_full()
    assert np.array_equal(L.indptr, c.L.indptr) and np.array_equal(L.indices, c.L.indices)
    assert np.abs(L.data - c.L.data).max(initial=0.0) <= 1e-14
    y = l.spmv(c.z["spmv_x"])
    assert np.abs(y - c.z["spmv_y"]).max() <= 1e-13 * max(1.0, np.abs(c.z["spmv_y"]).max())
    t1, tq, q = c.series
    r = api.series(l, l.state().from_probabilities(c.rho0), t1, tq, int(q), states=True)
    keep = c.z["series_keep"]
    assert np.abs(r.states[keep] - c.z["series_states"]).max() <= RHO_TOL
    assert np.abs(r.populations - c.z["series_pops"]).max() <= RHO_TOL
    if name.startswith("c"):
        assert int(r.info.spmvs) == c.series_spmvs
    for t, want in zip(c.z["step_t"], c.z["step_states"]):
        w, _ = api.step(l, l.state().from_probabilities(c.rho0), float(t))
        assert np.abs(w.gather() - want).max() <= RHO_TOL


def test_panels_off_in_bitwise_mode(monkeypatch):
    """The bitwise reference-order mode keeps one pass (panels reorder the sums)."""
    monkeypatch.setenv("QSWG_SELL_PANELS", "3")
    c = Case("c3_n40")
    l3 = c.build_gpu(api, format="sell", group=1)
    monkeypatch.setenv("QSWG_SELL_PANELS", "1")
    l1 = c.build_gpu(api, format="sell", group=1)
    t1, tq, q = c.series
    a = api.series(l3, l3.state().from_probabilities(c.rho0), t1, tq, int(q), states=True)
    b = api.series(l1, l1.state().from_probabilities(c.rho0), t1, tq, int(q), states=True)
    assert np.array_equal(a.states, b.states)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["c3_n40", "c4_n40", "lqsw_src_snk"])
def test_panelled_sell_sharded(name, world, monkeypatch):
    """Row-partitioned ranks with column panels (halo hulls over every panel)
    match the reference like the single-rank run."""
    from test_gpu_multirank import run_ranks
    monkeypatch.setenv("QSWG_SELL_PANELS", "3")
    c = Case(name)
    t1, tq, q = c.series

    def rank_fn(r, comm):
        l = c.build_gpu(api, comm=comm, format="sell")
        res = api.series(l, l.state().from_probabilities(c.rho0), t1, tq, int(q), states=True)
        return l.row0, res.states, res.populations

    parts = sorted(run_ranks(world, rank_fn), key=lambda p: p[0])
    states = np.concatenate([p[1] for p in parts], axis=1)
    keep = c.z["series_keep"]
    assert np.abs(states[keep] - c.z["series_states"]).max() <= RHO_TOL
    assert np.abs(parts[0][2] - c.z["series_pops"]).max() <= RHO_TOL


@pytest.mark.parametrize("cfg,size,panels", [("c3", 256, 1), ("c3", 200, 3), ("c4", 160, 2)])
def test_fused_natural_order_b_part(cfg, size, panels, monkeypatch):
    """Sigma-sorted SELL on one GPU keeps the B (x) I entries in a second,
    natural-order sliced ELL (coalesced gathers) that a block sums per window
    in shared memory before the sorted slices add theirs (kernels.hpp:
    SellView::b_val).  Same canonical matrix, same products and series as with
    every entry in the sorted arrays (QSWG_SELL_FUSE=0) up to the order of the
    sums, over several windows and with column panels."""
    from paper_2003_02450_b200 import graphs
    w = graphs.config(cfg, size=size)
    monkeypatch.setenv("QSWG_SELL_PANELS", str(panels))
    build = (lambda: api.build_local(w.omega, w.h, w.ops[0], format="sell")) if w.kind == "local" else \
        (lambda: api.build_global(w.omega, w.h, w.ops, format="sell"))
    monkeypatch.setenv("QSWG_SELL_FUSE", "1")
    lf = build()
    monkeypatch.setenv("QSWG_SELL_FUSE", "0")
    l0 = build()
    assert bool(lf.info.sell_fused) and not bool(l0.info.sell_fused)
    assert int(lf.info.sell_panels) == panels
    Lf, L0 = lf.gather_full(), l0.gather_full()
    assert np.array_equal(Lf.indptr, L0.indptr) and np.array_equal(Lf.indices, L0.indices)
    assert np.array_equal(Lf.data, L0.data)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(w.dim) + 1j * rng.standard_normal(w.dim)
    yf, y0 = lf.spmv(x), l0.spmv(x)
    assert np.abs(yf - y0).max() <= 1e-13 * np.abs(y0).max()
    rf = api.series(lf, lf.state().from_probabilities(w.rho0), w.t1, w.tq, 6, states=True)
    r0 = api.series(l0, l0.state().from_probabilities(w.rho0), w.t1, w.tq, 6, states=True)
    assert rf.info.spmvs == r0.info.spmvs
    assert np.abs(rf.states - r0.states).max() <= 1e-13
    assert np.abs(rf.populations.sum(axis=1) - 1).max() <= 1e-12
