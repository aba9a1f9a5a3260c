"""The omega re-mix (WalkSystem::set_omega,
walk.cpp:141-145): set_omega re-derives the operator in place on the device.
It must give exactly what a fresh build at that omega gives (same format,
sparsity, values, norms, Taylor terms and states, bit for bit), keep the
handle's states valid, and match the reference's omega sweep of config 3."""
import numpy as np
import pytest

from conftest import Case

pytestmark = pytest.mark.gpu
api = pytest.importorskip("paper_2003_02450_b200.api")

RHO_TOL = 1e-10


def same_operator(a, b):
    assert a.format == b.format and a.nnz == b.nnz and a.dim == b.dim and a.omega == b.omega
    assert np.array_equal(a.one_norms(), b.one_norms())
    if a.format != "kron":
        A, B = a.gather_full(), b.gather_full()
        assert np.array_equal(A.indptr, B.indptr) and np.array_equal(A.indices, B.indices)
        assert np.array_equal(A.data, B.data)


@pytest.mark.parametrize("fmt", ["kron", "sell", "csr"])
@pytest.mark.parametrize("name", ["c2_n36", "c3_n40", "lqsw_src_snk", "gqsw_multi_rot"])
def test_set_omega_equals_fresh_build(name, fmt):
    c = Case(name)
    t1, tq, q = c.series
    l = c.build_gpu(api, format=fmt)
    v = l.state().from_probabilities(c.rho0)  # created before the re-mix, used after it
    for w in (0.25, 1.0, 0.0, c.omega, 0.7):
        l.set_omega(w)
        c_w = Case(name)
        c_w.omega = w
        f = c_w.build_gpu(api, format=fmt)
        same_operator(l, f)
        r = api.series(l, v, t1, tq, int(q), states=True)
        rf = api.series(f, f.state().from_probabilities(c.rho0), t1, tq, int(q), states=True)
        assert int(r.info.spmvs) == int(rf.info.spmvs), w
        assert np.array_equal(r.states, rf.states), w


def test_set_omega_rejects_out_of_range():
    c = Case("c3_n40")
    l = c.build_gpu(api)
    for bad in (-0.1, 1.5, float("nan")):
        with pytest.raises(ValueError, match="omega must be in"):
            l.set_omega(bad)
    assert l.omega == c.omega


@pytest.mark.parametrize("fmt", ["kron", "sell"])
def test_walk_omega_sweep_matches_reference(fmt):
    """Config 3's omega sweep {0.5, 0.1, 0.9} through one WalkSystem: set_omega
    between runs, the initial state kept on the device, against the reference's
    golden series at each omega."""
    base = Case("c3_n40")
    walk = api.WalkSystem.lqsw(base.omega, base.h, base.ops[0])
    if fmt != "kron":
        walk.liouvillian = base.build_gpu(api, format=fmt)
    walk.initial_state(base.rho0)
    for name in ("c3_n40", "c3_n40_w0.1", "c3_n40_w0.9", "c3_n40"):
        c = Case(name)
        walk.set_omega(c.omega)
        assert walk.liouvillian.omega == c.omega
        np.testing.assert_allclose(walk.liouvillian.one_norms(), c.norms, rtol=1e-13, atol=0)
        t1, tq, q = c.series
        r = walk.series(t1, tq, int(q), states=True)
        keep = c.z["series_keep"]
        assert np.abs(r.states[keep] - c.z["series_states"]).max() <= RHO_TOL, name
        assert np.abs(r.populations - c.z["series_pops"]).max() <= RHO_TOL, name


def test_set_omega_replays_no_stale_graph():
    """A captured series graph of the old omega must not be replayed after the re-mix."""
    c = Case("c2_n36")
    t1, tq, q = c.series
    l = c.build_gpu(api, format="kron")
    v = l.state().from_probabilities(c.rho0)
    for _ in range(3):  # the second identical call captures, the third replays
        api.series(l, v, t1, tq, int(q))
    l.set_omega(0.6)
    c6 = Case("c2_n36")
    c6.omega = 0.6
    f = c6.build_gpu(api, format="kron")
    want = api.series(f, f.state().from_probabilities(c.rho0), t1, tq, int(q)).populations
    for _ in range(3):
        assert np.array_equal(api.series(l, v, t1, tq, int(q)).populations, want)


@pytest.mark.parametrize("world", [2, 3])
def test_set_omega_sharded_keeps_partition(world):
    """Row-partitioned ranks re-mix on their fixed partition; results equal a
    fresh single-rank build at the new omega within the parity tolerance."""
    from test_gpu_multirank import run_ranks
    c = Case("c3_n40")
    t1, tq, q = c.series

    def rank_fn(r, comm):
        l = c.build_gpu(api, comm=comm, format="kron")
        st0 = l.partition()[0].copy()
        v = l.state().from_probabilities(c.rho0)
        l.set_omega(0.9)
        assert np.array_equal(l.partition()[0], st0)
        res = api.series(l, v, t1, tq, int(q), states=True)
        return l.row0, res.states

    out = run_ranks(world, rank_fn)
    full = np.concatenate([s for _, s in sorted(out, key=lambda t: t[0])], axis=1)
    ref = Case("c3_n40_w0.9")
    keep = ref.z["series_keep"]
    assert np.abs(full[keep] - ref.z["series_states"]).max() <= RHO_TOL
