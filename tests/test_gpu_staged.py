"""Staged Hermitian tiles of the KRON series term (kernels.hpp: KronView::staged).

Opt-in (QSWG_KRON_STAGED=1; measured slower than the global gathers, see
DESIGN.md section 2.2).  On lattice-like operand sets (n a multiple of 32,
every 32-row tile of an operand naming at most five column tiles) the
Hermitian series term copies the tiles its operand rows gather from into
shared memory (cp.async, a tile ahead) and runs the operand-index -> gather
-> FMA chains there.  Entries, order and arithmetic are those of the
global-gather kernel, so a series must agree with it bit for bit: same
states, same populations, same SpMV count.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
api = pytest.importorskip("paper_2003_02450_b200.api")
from paper_2003_02450_b200 import graphs  # noqa: E402


def run(w, steps, monkeypatch, staged):
    monkeypatch.setenv("QSWG_KRON_STAGED", "1" if staged else "0")
    build = (lambda: api.build_local(w.omega, w.h, w.ops[0], format="kron")) if w.kind == "local" else \
        (lambda: api.build_global(w.omega, w.h, w.ops, format="kron"))
    l = build()
    assert bool(l.info.kron_staged) == staged
    r = api.series(l, l.state().from_probabilities(w.rho0), w.t1, w.tq, steps, states=True)
    l._query()  # (info is a snapshot)
    assert bool(l.info.kron_hermitian)
    return r


@pytest.mark.parametrize("cfg,size,steps", [("c2", 8, 12), ("c2", 16, 6), ("c5", 4, 10), ("c5", 8, 4)])
def test_staged_series_is_bit_identical_to_global_gathers(cfg, size, steps, monkeypatch):
    w = graphs.config(cfg, size=size)
    a = run(w, steps, monkeypatch, True)
    b = run(w, steps, monkeypatch, False)
    assert a.info.spmvs == b.info.spmvs
    assert np.array_equal(a.states, b.states)
    assert np.array_equal(a.populations, b.populations)
    assert np.abs(a.populations.sum(axis=1) - 1).max() <= 1e-12


def test_irregular_graph_keeps_global_gathers(monkeypatch):
    monkeypatch.setenv("QSWG_KRON_STAGED", "1")
    w = graphs.config("c4", size=256)  # ER: a tile row names far more than five column tiles
    l = api.build_global(w.omega, w.h, w.ops, format="kron")
    assert not l.info.kron_staged
