"""Device paths specific to this implementation (no reference counterpart,
checked against the reference-pinned C oracle and against each other):

* the Hermitian tile kernels (KRON, one GPU) — taken when the input is an
  exactly Hermitian matrix — against the general kernels on the same input;
* non-Hermitian inputs, which must take the general path;
* the lazily updated running sums of `series` (term ring, bound-settled stop
  tests, flushes) — the ring size must not change a single bit or term count.
"""
import numpy as np
import pytest

from oracle.oracle import rho0_vec
from conftest import Case

pytestmark = pytest.mark.gpu
api = pytest.importorskip("paper_2003_02450_b200.api")
from paper_2003_02450_b200 import graphs  # noqa: E402


def hermitian(rng, n):
    a = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
    h = a + a.conj().T
    return h.reshape(-1, order="F")  # column-major vec


def as_matrix(v, n):
    return np.asarray(v).reshape(n, n, order="F")


CASES = ["c2_n36", "c3_n40", "c4_n40", "c5_n64", "gqsw_multi_rot", "lqsw_src_snk", "walkthrough_nm_w1"]


@pytest.mark.parametrize("name", CASES)
def test_hermitian_spmv_matches_general(name):
    c = Case(name)
    l = c.build_gpu(api, format="kron")
    rng = np.random.default_rng(5)
    x = hermitian(rng, c.n)
    y_h = l.spmv(x)                  # Hermitian kernels
    l.set_hermitian_mode(False)
    y_g = l.spmv(x)                  # general kernels
    Yh, Yg = as_matrix(y_h, c.n), as_matrix(y_g, c.n)
    iu = np.triu_indices(c.n, 1)
    # upper triangle: the same formula, the same order -> the same bits
    assert np.array_equal(Yh[iu], Yg[iu])
    assert np.array_equal(np.diag(Yh).real, np.diag(Yg).real)
    # the Hermitian result is exactly Hermitian with a real diagonal
    assert np.array_equal(Yh, Yh.conj().T)
    # the general lower triangle agrees to rounding
    scale = np.abs(Yg).max()
    assert np.abs(Yh - Yg).max() <= 1e-14 * scale
    # and both are L x of the reference's superoperator
    ref = c.L.to_dense() @ x
    assert np.abs(y_h - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("name", ["c2_n36", "c4_n40", "gqsw_multi_rot", "lqsw_src_snk"])
def test_hermitian_series_matches_general_and_reference(name):
    c = Case(name)
    t1, tq, q = c.series
    l = c.build_gpu(api, format="kron")
    v = l.state().from_probabilities(c.rho0)
    r_h = api.series(l, v, t1, tq, int(q), states=True)
    l.set_hermitian_mode(False)
    r_g = api.series(l, v, t1, tq, int(q), states=True)
    assert r_h.info.spmvs == r_g.info.spmvs == c.series_spmvs
    assert np.abs(r_h.states - r_g.states).max() <= 1e-13
    keep = c.z["series_keep"]
    assert np.abs(r_h.states[keep] - c.z["series_states"]).max() <= 1e-10
    for s in r_h.states:  # every output of the Hermitian path is exactly Hermitian
        S = as_matrix(s, c.n)
        assert np.array_equal(S, S.conj().T)


@pytest.mark.parametrize("name", ["c2_n36", "lqsw_src_snk"])
def test_non_hermitian_input_takes_general_path(name, port):
    c = Case(name)
    rng = np.random.default_rng(17)
    x = rng.uniform(-1, 1, c.n * c.n) + 1j * rng.uniform(-1, 1, c.n * c.n)  # not Hermitian
    l = c.build_gpu(api, format="kron")
    w, info = api.step(l, l.state().upload(x), 0.7)
    o = c.build_oracle(port)
    ref, ns = o.step(x, 0.7)
    assert info.spmvs == ns
    assert np.abs(w.gather() - ref).max() <= 1e-10 * max(1.0, np.abs(ref).max())
    t1, tq, q = c.series
    res = api.series(l, l.state().upload(x), t1, tq, int(q), states=True)
    states, _, nsp = o.series(x, t1, tq, int(q))
    assert res.info.spmvs == nsp
    assert np.abs(res.states - states).max() <= 1e-10 * max(1.0, np.abs(states).max())


@pytest.mark.parametrize("fmt", ["kron", "auto"])
@pytest.mark.parametrize("name", ["c1_n64", "c2_n36", "gqsw_multi_rot"])
def test_term_ring_size_changes_no_bit(name, fmt, monkeypatch):
    """Running sums are added in term order whatever the ring size, and the
    bound-settled stop tests take the decisions the exact tests take."""
    c = Case(name)
    t1, tq, q = c.series
    out = {}
    for pm in ("1", "2", "7", "64"):
        monkeypatch.setenv("QSWG_PEND_MAX", pm)
        l = c.build_gpu(api, format=fmt)
        r = api.series(l, l.state().from_probabilities(c.rho0), t1, tq, int(q), states=True)
        out[pm] = (r.states, r.info.spmvs)
        del l
    base, nsp = out["1"]
    assert nsp == c.series_spmvs
    for pm, (st, n) in out.items():
        assert n == nsp, pm
        assert np.array_equal(st, base), pm


def test_full_size_c2_series_is_hermitian_and_trace_preserving():
    w = graphs.config("c2")
    l = api.build_global(w.omega, w.h, w.ops)
    r = api.series(l, l.state().from_probabilities(w.rho0), w.t1, w.tq, w.steps, final=True)
    assert r.info.spmvs == 760
    assert np.abs(r.populations.sum(axis=1) - 1).max() <= 1e-12
    F = as_matrix(r.final.gather(), w.n)
    assert np.array_equal(F, F.conj().T)


def test_nccl_communicator_single_rank():
    """libnccl is resolved with dlopen and a one-rank communicator drives the
    same series as no communicator (the N > 1 collectives are covered by
    tests/test_gpu_multirank.py through the in-process communicator)."""
    c = Case("c2_n36")
    t1, tq, q = c.series
    comm = api.Comm.from_unique_id(api.Comm.unique_id(), 0, 1, 0)
    l = c.build_gpu(api, comm=comm)
    r = api.series(l, l.state().from_probabilities(c.rho0), t1, tq, int(q), states=True)
    l0 = c.build_gpu(api)
    r0 = api.series(l0, l0.state().from_probabilities(c.rho0), t1, tq, int(q), states=True)
    assert np.array_equal(r.states, r0.states)
    del l
    del comm


def test_non_hermitian_h_rot_disables_the_hermitian_tiles(port):
    """With a rotating Hamiltonian that is not Hermitian (the reference never
    checks H_rot, liouvillian.cpp:217-229) L does not map Hermitian X to
    Hermitian L(X): the Hermitian tile kernels must stay off, and the result
    must be the reference's full product."""
    c = Case("gqsw_multi_rot")
    rng = np.random.default_rng(3)
    n = c.n
    a = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.2)
    from paper_2003_02450_b200.graphs import Csr
    r_, c_ = np.nonzero(a)
    hrot = Csr.from_coo(n, n, r_, c_, a[r_, c_] + 0.3j * a[r_, c_])  # not Hermitian
    l = api.build_global(c.omega, c.h, c.ops, hrot, format="kron")
    o = port.build_global(c.omega, c.h, c.ops, hrot)
    t1, tq, q = c.series
    v0 = rho0_vec(n, c.rho0)
    r = api.series(l, l.state().upload(v0), t1, tq, int(q), states=True)
    l._query()
    assert not l.info.kron_hermitian
    so, _, _ = o.series(v0, t1, tq, int(q))
    assert np.abs(r.states - so).max() <= 1e-10 * max(1.0, np.abs(so).max())


@pytest.mark.parametrize("kind", ["local", "global"])
def test_slices_of_different_row_length(kind, port):
    """Operand slices that are uniform inside but differ from one another: 32
    vertices on a cycle (degree 2) and 32 on a 4-regular circulant.  The
    shuffled operand rows of the KRON kernels take one row length for the
    whole operand, so such operands must stay on the per-row paths (a round-2
    regression: the Hermitian tiles dropped the longer slices' last entries)."""
    from paper_2003_02450_b200.graphs import Csr
    n, r, c = 64, [], []
    for i in range(32):
        for d in (1, -1):
            r.append(i)
            c.append((i + d) % 32)
        for d in (1, -1, 2, -2):
            r.append(32 + i)
            c.append(32 + (i + d) % 32)
    g = Csr.from_coo(n, n, r, c, [1.0] * len(r))
    h, m = graphs.generator_matrix(1.0, g), graphs.markov_chain_matrix(g)
    p = np.zeros(n)
    p[0] = p[40] = 0.5
    v0 = rho0_vec(n, p)
    o = port.build_local(0.3, h, m, [], []) if kind == "local" else port.build_global(0.3, h, [m], None)
    so, _, ns = o.series(v0, 0.0, 3.0, 4)
    for fmt in ("kron", "sell", "csr"):
        l = api.build_local(0.3, h, m, format=fmt) if kind == "local" else api.build_global(0.3, h, [m], format=fmt)
        res = api.series(l, l.state().upload(v0), 0.0, 3.0, 4, states=True)
        assert res.info.spmvs == ns, fmt
        assert np.abs(res.states - so).max() <= 1e-10, fmt
