"""Behavioural tests of the device exponential action, mirroring the
reference's own test_expm.cpp / test_walk.cpp / test_liouvillian.cpp cases
(cited per test) with the C oracle or closed forms as the checker."""
import numpy as np
import pytest
import scipy.linalg

from oracle.oracle import rho0_vec

pytestmark = pytest.mark.gpu
api = pytest.importorskip("paper_2003_02450_b200.api")
from paper_2003_02450_b200 import graphs  # noqa: E402
from paper_2003_02450_b200.graphs import Csr  # noqa: E402


def random_digraph(rng, n, density=0.4):
    d = (rng.random((n, n)) < density) * rng.uniform(0.1, 2.0, (n, n))
    np.fill_diagonal(d, 0)
    if not d.any():
        d[n - 1, 0] = 1.0
    r, c = np.nonzero(d)
    return Csr.from_coo(n, n, r, c, d[r, c])


def random_lqsw(rng, n, omega, with_ss=False):
    """test_expm.cpp:18-31"""
    g = random_digraph(rng, n)
    src, snk, total = [], [], n
    if with_ss:
        src, snk, total = [(int(rng.integers(n)), 1.0)], [(int(rng.integers(n)), 1.5)], n + 2
    h = api.generator_matrix(1.0, api.symmetrize(g)).to_csr()
    ml = api.local_lindblad(api.generator_matrix(1.0, g)).to_csr()
    pad = lambda m: Csr(total, total, np.concatenate([m.indptr, np.full(total - n, m.indptr[-1])]),  # noqa: E731
                        m.indices, m.data)
    return api.build_local(omega, pad(h), pad(ml), src, snk), (omega, pad(h), pad(ml), src, snk)


def random_vec(rng, dim):
    return rng.uniform(-1, 1, dim) + 1j * rng.uniform(-1, 1, dim)


def dense_expm_action(L: Csr, v, t):
    return scipy.linalg.expm(t * L.to_dense()) @ v


def test_step_t0_returns_state():  # test_expm.cpp:141-147
    rng = np.random.default_rng(89)
    l, _ = random_lqsw(rng, 4, 0.5)
    x = random_vec(rng, l.dim)
    w, info = api.step(l, l.state().upload(x), 0.0)
    assert info.m_star == 0 and info.spmvs == 0
    assert np.array_equal(w.gather(), x)


def test_coherent_dimer_cos2():  # test_expm.cpp:149-161
    dimer = Csr.from_coo(2, 2, [0, 1], [1, 0], [1.0, 1.0])
    h = api.generator_matrix(1.0, dimer)
    l = api.build_local(0.0, h, api.local_lindblad(h))
    v = l.state().upload(np.array([1, 0, 0, 0], complex))
    for t in (0.1, 0.7, 2.0, 5.0):
        w = api.step(l, v, t)[0].gather()
        assert abs(w[0].real - np.cos(t) ** 2) <= 1e-12
        assert abs(w[3].real - np.sin(t) ** 2) <= 1e-12


def test_omega1_dimer_ctrw():  # test_liouvillian.cpp:93-107: p1 = (1 + e^{-2t})/2
    dimer = Csr.from_coo(2, 2, [0, 1], [1, 0], [1.0, 1.0])
    h = api.generator_matrix(1.0, dimer)
    l = api.build_local(1.0, h, api.local_lindblad(h))
    v = l.state().from_probabilities([1.0, 0.0])
    for t in (0.3, 1.0, 4.0):
        p = api.step(l, v, t)[0].populations()
        assert abs(p[0] - 0.5 * (1 + np.exp(-2 * t))) <= 1e-12


@pytest.mark.parametrize("it", range(6))
def test_step_matches_dense_expm(it):  # test_expm.cpp:163-177
    rng = np.random.default_rng(97 + it)
    l, _ = random_lqsw(rng, 4 + it % 3, 0.25 * (it % 5), with_ss=it % 2 == 0)
    L = l.gather_full()
    x = random_vec(rng, l.dim)
    v = l.state().upload(x)
    for t in (0.1, 1.0, 10.0):
        got = api.step(l, v, t)[0].gather()
        assert np.abs(got - dense_expm_action(L, x, t)).max() <= 1e-10


def test_semigroup():  # test_expm.cpp:179-189
    rng = np.random.default_rng(103)
    for _ in range(4):
        l, _ = random_lqsw(rng, 4, 0.5)
        v = l.state().upload(random_vec(rng, l.dim))
        t1, t2 = 0.4 + 0.2 * rng.integers(4), 0.9 + 0.3 * rng.integers(4)
        once = api.step(l, v, t1 + t2)[0].gather()
        twice = api.step(l, api.step(l, v, t1)[0], t2)[0].gather()
        assert np.abs(once - twice).max() <= 1e-11


def test_directed_dimer_long_times():  # test_expm.cpp:191-207
    g = Csr.from_coo(2, 2, [1], [0], [1.0])
    h = api.generator_matrix(1.0, api.symmetrize(g))
    ml = api.local_lindblad(api.generator_matrix(1.0, g))
    for omega in (0.0, 0.5, 1.0):
        l = api.build_local(omega, h, ml)
        L = l.gather_full()
        x = np.array([1, 0, 0, 0], complex)
        for t in (1.0, 10.0, 100.0):
            got = api.step(l, l.state().upload(x), t)[0].gather()
            assert np.abs(got - dense_expm_action(L, x, t)).max() <= 1e-10


def test_negative_time_reverses():  # test_expm.cpp:226-232
    rng = np.random.default_rng(109)
    l, _ = random_lqsw(rng, 4, 0.3)
    x = random_vec(rng, l.dim)
    fwd = api.step(l, l.state().upload(x), 1.0)[0]
    back = api.step(l, fwd, -1.0)[0].gather()
    assert np.abs(back - x).max() <= 1e-8


def test_overflow_is_reported():  # test_expm.cpp:234-244
    g = Csr.from_coo(2, 2, [1], [0], [1.0])
    h = api.generator_matrix(1.0, api.symmetrize(g))
    ml = api.local_lindblad(api.generator_matrix(1.0, g)).to_csr()
    ml = Csr(ml.rows, ml.cols, ml.indptr, ml.indices, ml.data * 300.0)
    l = api.build_local(1.0, h, ml)
    v = l.state().upload(np.array([1, 0, 0, 0], complex))
    with pytest.raises(api.NumericalError):
        api.step(l, v, -40.0)
    # the handle stays usable after the error
    w, _ = api.step(l, v, 0.1)
    assert np.isfinite(w.gather()).all()


def test_series_endpoints_zero_generator_and_args():  # test_expm.cpp:246-270
    rng = np.random.default_rng(113)
    l, _ = random_lqsw(rng, 5, 0.6)
    x = random_vec(rng, l.dim)
    v = l.state().upload(x)
    r = api.series(l, v, 0.5, 2.5, 1, states=True)
    assert np.abs(r.states[0] - api.step(l, v, 0.5)[0].gather()).max() <= 1e-12
    assert np.abs(r.states[1] - api.step(l, v, 2.5)[0].gather()).max() <= 1e-12
    r0 = api.series(l, v, 0.0, 1.0, 4, states=True)
    assert np.array_equal(r0.states[0], x)
    z3 = Csr.from_coo(3, 3, [], [], [])
    lz = api.build_local(0.5, z3, z3)
    assert lz.nnz == 0
    xz = random_vec(rng, 9)
    rz = api.series(lz, lz.state().upload(xz), 0.0, 10.0, 5, states=True)
    assert rz.info.path == 0
    for s in rz.states:
        assert np.array_equal(s, xz)
    with pytest.raises(ValueError):
        api.series(l, v, 2.0, 1.0, 4)
    with pytest.raises(ValueError):
        api.series(l, v, 0.0, 1.0, 0)


@pytest.mark.parametrize("it", range(4))
def test_series_agrees_with_steps(it):  # test_expm.cpp:272-287
    rng = np.random.default_rng(127 + it)
    l, _ = random_lqsw(rng, 4 + it % 3, 0.25 * (it % 5), with_ss=it % 2 == 0)
    v = l.state().upload(random_vec(rng, l.dim))
    r = api.series(l, v, 0.0, 8.0, 16, states=True)
    for k in range(0, 17, 4):
        direct = api.step(l, v, float(r.times[k]))[0].gather()
        assert np.abs(r.states[k] - direct).max() <= 1e-12


def test_series_sequential_path_matches_oracle(port):
    """q <= span.s: q sequential steps (expm.cpp:234-240)."""
    w = graphs.config("c3", size=30)
    l = api.build_local(w.omega, w.h, w.ops[0])
    h = port.build(w)
    v0 = rho0_vec(w.n, w.rho0)
    so, _, nref = h.series(v0, 0.0, 50.0, 4)
    r = api.series(l, l.state().upload(v0), 0.0, 50.0, 4, states=True)
    assert r.info.path == 1
    assert r.info.spmvs == nref
    assert np.abs(r.states - so).max() <= 1e-10


def test_walkthrough_gqsw_moralises():  # test_walk.cpp:42-51
    g3 = Csr.from_coo(3, 3, [2, 2], [0, 1], [1.0, 1.0])
    w = api.WalkSystem.gqsw(1.0, api.generator_matrix(1.0, api.symmetrize(g3)), [g3])
    w.initial_state([1.0, 0.0, 0.0])
    w.step(100.0)
    p = w.gather_populations()
    np.testing.assert_allclose(p, [0.25, 0.25, 0.5], atol=1e-6)
    rho = w.gather_result()
    assert abs(rho[0, 1] - (-0.25)) <= 1e-6  # test_container.cpp:183-195


def test_walkthrough_lqsw_limits():  # test_walk.cpp:66-94
    g3 = Csr.from_coo(3, 3, [2, 2], [0, 1], [1.0, 1.0])
    gu = api.symmetrize(g3)
    w0 = api.WalkSystem.lqsw(0.0, gu, g3)
    w0.initial_state([1.0, 0.0, 0.0])
    w0.step(100.0)
    np.testing.assert_allclose(w0.gather_populations(), [3.80773217e-07, 9.98766244e-01, 1.23337485e-03],
                               rtol=1e-5)
    w1 = api.WalkSystem.lqsw(1.0, gu, g3)
    w1.initial_state([1.0, 0.0, 0.0])
    w1.step(100.0)
    p = w1.gather_populations()
    assert abs(p[0]) <= 1e-12 and abs(p[1]) <= 1e-12 and abs(p[2] - 1.0) <= 1e-12


def test_regular_graph_coherence_death():  # acceptance_main.cpp:293-308
    g = graphs.cycle_graph(20)
    w = api.WalkSystem.lqsw(0.5, graphs.generator_matrix(1.0, g), graphs.markov_chain_matrix(g))
    w.initial_state(np.eye(20)[0])
    w.step(100.0)
    rho = w.gather_result()
    off = rho - np.diag(np.diag(rho))
    assert np.abs(off).max() <= 1e-8
    # the device coherence norm (run()'s "coherence_norm") tells the same story
    r = w.series(0.0, 100.0, 10, coherence=True)
    assert r.coherence[0] == 0.0 and r.coherence[-1] <= 1e-8
    assert np.all(np.diff(r.coherence[1:]) < 0)  # coherences die out monotonically here
    assert abs(r.coherence[-1] - np.abs(off).max()) <= 1e-12


def test_dense_initial_state_and_set_omega():  # walk.hpp:57-66, walk.cpp:141-145
    g = graphs.cycle_graph(6)
    h, m = graphs.generator_matrix(1.0, g), graphs.markov_chain_matrix(g)
    w = api.WalkSystem.lqsw(0.3, h, m)
    psi = np.ones(6) / np.sqrt(6)
    rho = np.outer(psi, psi.conj()).astype(complex)
    w.initial_state(rho)
    np.testing.assert_allclose(w.gather_result(), rho)
    w.step(2.0)
    a = w.gather_result()
    w.set_omega(0.3)
    w.step(2.0)
    assert np.abs(w.gather_result() - a).max() == 0.0  # rebuild is deterministic
    with pytest.raises(ValueError):
        w.initial_state(np.eye(6))  # trace 6
    with pytest.raises(ValueError):
        w.set_omega(1.5)


def test_validation_errors():  # liouvillian.cpp:133-151, 216-229
    g = graphs.cycle_graph(4)
    h, m = graphs.generator_matrix(1.0, g), graphs.markov_chain_matrix(g)
    with pytest.raises(ValueError):
        api.build_local(1.5, h, m)
    nh = Csr.from_coo(4, 4, [0], [1], [1j])  # not Hermitian
    with pytest.raises(ValueError):
        api.build_local(0.5, nh, m)
    with pytest.raises(IndexError):
        api.build_local(0.5, h, m, sources=[(3, 1.0)])  # target in the augmented block
    with pytest.raises(ValueError):
        api.build_global(0.5, h, [Csr.from_coo(3, 3, [], [], [])])
    l = api.build_local(0.5, h, m)
    other = api.build_local(0.5, h, m)
    with pytest.raises(ValueError):
        api.step(l, other.state(), 1.0)


def test_omega_linearity():  # test_liouvillian.cpp:285-294
    rng = np.random.default_rng(5)
    g = random_digraph(rng, 5)
    h = api.generator_matrix(1.0, api.symmetrize(g))
    ml = api.local_lindblad(api.generator_matrix(1.0, g))
    d = {om: api.build_local(om, h, ml, format="csr").gather_full().to_dense() for om in (0.0, 0.3, 1.0)}
    assert np.abs(d[0.3] - (0.7 * d[0.0] + 0.3 * d[1.0])).max() <= 1e-14


def test_global_equals_local_at_omega0():  # test_liouvillian.cpp:119-127
    g = graphs.cycle_graph(5)
    h = graphs.generator_matrix(1.0, g)
    a = api.build_local(0.0, h, graphs.markov_chain_matrix(g), format="csr").gather_full().to_dense()
    b = api.build_global(0.0, h, [graphs.markov_chain_matrix(g)], format="csr").gather_full().to_dense()
    assert np.array_equal(a, b)


def test_trace_preservation_structure():  # test_liouvillian.cpp:268-283
    rng = np.random.default_rng(3)
    l, _ = random_lqsw(rng, 5, 0.7)
    n = 5
    L = l.gather_full().to_dense()  # assembled on demand in the Kron format
    diag_rows = [i * (n + 1) for i in range(n)]
    colsum = L[diag_rows, :].sum(axis=0)
    assert np.abs(colsum).max() <= 1e-14


@pytest.mark.parametrize("group", [1, 2, 4, 8, 16, 32])
def test_every_row_group_width_agrees(group):
    w = graphs.config("c2", size=6)
    l = api.build_global(w.omega, w.h, w.ops, group=group, format="csr")
    assert l.group == group and l.format == "csr"
    x = random_vec(np.random.default_rng(1), l.dim)
    L = l.gather_full()
    want = L.to_dense() @ x
    assert np.abs(l.spmv(x) - want).max() <= 1e-13 * max(1, np.abs(want).max())


def _walkthrough_nm(omega, **kw):  # test_walk.cpp:33-39
    g3 = Csr.from_coo(3, 3, [2, 2], [0, 1], [1.0, 1.0])
    gu = api.symmetrize(g3)
    dims = api.nm_vsets(gu)
    w = api.WalkSystem.gqsw(omega, api.nm_H(1.0, gu, dims), [api.nm_L(1.0, g3, dims)], api.nm_H_rot(dims),
                            dims, **kw)
    w.initial_state([1.0, 0.0, 0.0])
    return w


@pytest.mark.parametrize("fmt", ["kron", "csr"])
def test_demoralised_walk_reaches_the_child(fmt):  # test_walk.cpp:53-64
    w = _walkthrough_nm(1.0, group=1 if fmt == "csr" else 0)
    w.step(100.0)
    p = w.gather_populations()
    assert len(p) == 3
    assert p[2] >= 1.0 - 1e-10
    assert abs(p[0]) <= 1e-12 and abs(p[1]) <= 1e-12


def test_demoralised_coherent_limit_matches_lqsw():  # test_walk.cpp:66-84
    nm = _walkthrough_nm(0.0)
    nm.step(100.0)
    p_nm = nm.gather_populations()
    np.testing.assert_allclose(p_nm, [3.80773381e-07, 9.98766244e-01, 1.23337485e-03], rtol=1e-5)
    g3 = Csr.from_coo(3, 3, [2, 2], [0, 1], [1.0, 1.0])
    lq = api.WalkSystem.lqsw(0.0, api.symmetrize(g3), g3)
    lq.initial_state([1.0, 0.0, 0.0])
    lq.step(100.0)
    assert np.abs(p_nm - lq.gather_populations()).max() <= 1e-9
    r = _walkthrough_nm(0.5).series(0.0, 10.0, 5)
    assert r.populations.shape == (6, 3)
    np.testing.assert_allclose(r.populations.sum(axis=1), 1.0, atol=1e-12)
