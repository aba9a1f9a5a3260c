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
