"""Device path vs the reference: golden fixtures (from the unmodified
reference library) and the C oracle, through the C ABI on a B200.

Tolerances (north star, BASELINE.json): max |rho_gpu - rho_ref| <= 1e-10
elementwise and |Tr rho - 1| <= 1e-12 at every output time, identical
(m*, s) and identical number of Taylor terms taken.  CSR values: the device
sums duplicate contributions in a fixed order that can differ from the
reference's unstable sort, so values are compared at 1e-14 (absolute, all
entries are O(1)) with an identical sparsity pattern; norms at 1e-13
relative.
"""
import numpy as np
import pytest

from conftest import CASE_NAMES, Case
from oracle.oracle import rho0_vec

pytestmark = pytest.mark.gpu
api = pytest.importorskip("paper_2003_02450_b200.api")
from paper_2003_02450_b200 import graphs  # noqa: E402

# (group, storage format): autotuned fast kernels and the bitwise reference
# order (group=1), each over CSR and SELL-32 storage.
MODES = [(0, "csr"), (0, "sell"), (0, "kron"), (1, "csr"), (1, "sell"), (1, "auto")]
RHO_TOL = 1e-10
TRACE_TOL = 1e-12


def trace_err(states, n):
    s = np.asarray(states).reshape(-1, n, n)
    return np.abs(np.trace(s, axis1=1, axis2=2) - 1.0).max()


@pytest.mark.parametrize("fmt", ["csr", "sell", "kron"])
@pytest.mark.parametrize("name", CASE_NAMES)
def test_csr_and_norms_match_reference(name, fmt):
    c = Case(name)
    l = c.build_gpu(api, format=fmt)
    assert l.format == fmt
    # the default: KRON above dim 65536, the stored superoperator below
    assert c.build_gpu(api).format == ("kron" if c.n * c.n > 65536 else ("sell" if c.build_gpu(api, format="sell").padding <= 1.3 else "csr"))
    assert l.dim == c.dim and l.nnz == c.nnz
    L = l.gather_full()
    assert np.array_equal(L.indptr, c.L.indptr)
    assert np.array_equal(L.indices, c.L.indices)
    assert np.abs(L.data - c.L.data).max(initial=0.0) <= 1e-14
    np.testing.assert_allclose(l.one_norms(), c.norms, rtol=1e-13, atol=0)


@pytest.mark.parametrize("group,fmt", MODES)
@pytest.mark.parametrize("name", CASE_NAMES)
def test_spmv_matches_reference(name, group, fmt):
    c = Case(name)
    l = c.build_gpu(api, group=group, format=fmt)
    y = l.spmv(c.z["spmv_x"])
    scale = max(1.0, np.abs(c.z["spmv_y"]).max())
    assert np.abs(y - c.z["spmv_y"]).max() <= 1e-13 * scale


def counts_must_match(name, group):
    """Identical Taylor terms taken.  The bitwise mode (group=1: CSR-order
    sums, no FMA) reproduces the reference's arithmetic, so its stop tests
    fire at the same terms everywhere.  The fast kernels sum in a different
    order; on the BASELINE workloads (c*) that never moves a stop test, but
    once a walk sits at its steady state the Taylor terms are pure rounding
    noise (~1e-17) and the stop test c1 + c2 <= 2^-53 ||sum|| compares noise
    with noise (walkthrough cases), so only rho is compared there."""
    return group == 1 or name.startswith("c")


@pytest.mark.parametrize("name", ["c1_n64", "c2_n36", "c5_n64"])
def test_bitwise_mode_formats_agree(name):
    """Both storage formats visit a row's entries in CSR order, so the
    bitwise mode gives bit-identical states."""
    c = Case(name)
    t1, tq, q = c.series
    out = []
    for fmt in ("csr", "sell"):
        l = c.build_gpu(api, group=1, format=fmt)
        out.append(api.series(l, l.state().from_probabilities(c.rho0), t1, tq, int(q), states=True).states)
    assert np.array_equal(out[0], out[1])


@pytest.mark.parametrize("group,fmt", MODES)
@pytest.mark.parametrize("name", CASE_NAMES)
def test_series_matches_reference(name, group, fmt):
    c = Case(name)
    l = c.build_gpu(api, group=group, format=fmt)
    v = l.state().from_probabilities(c.rho0)
    t1, tq, q = c.series
    r = api.series(l, v, t1, tq, int(q), states=True)
    if counts_must_match(name, group):
        assert r.info.spmvs == c.series_spmvs
    keep = c.z["series_keep"]
    assert np.abs(r.states[keep] - c.z["series_states"]).max() <= RHO_TOL
    assert np.abs(r.populations - c.z["series_pops"]).max() <= RHO_TOL
    assert trace_err(r.states, c.n) <= TRACE_TOL
    np.testing.assert_allclose(r.times, [t1 + (tq - t1) / q * k for k in range(int(q) + 1)])


@pytest.mark.parametrize("group,fmt", MODES)
@pytest.mark.parametrize("name", CASE_NAMES)
def test_step_matches_reference(name, group, fmt):
    c = Case(name)
    l = c.build_gpu(api, group=group, format=fmt)
    v = l.state().from_probabilities(c.rho0)
    for t, want, nsp in zip(c.z["step_t"], c.z["step_states"], c.z["step_spmvs"]):
        w, info = api.step(l, v, float(t))
        assert (info.m_star, info.s) == api.select_parameters(c.norms, float(t))
        if counts_must_match(name, group):
            assert info.spmvs == nsp
        assert np.abs(w.gather() - want).max() <= RHO_TOL


@pytest.mark.parametrize("name,size", [("c1", 24), ("c2", 5), ("c3", 30), ("c4", 24), ("c5", 3)])
def test_series_matches_oracle_live(port, name, size):
    """Fresh seeded inputs (not in the fixtures), GPU vs the C oracle."""
    w = graphs.config(name, size=size)
    l = api.build_local(w.omega, w.h, w.ops[0]) if w.kind == "local" else api.build_global(w.omega, w.h, w.ops)
    h = port.build(w)
    np.testing.assert_allclose(l.one_norms(), h.norms, rtol=1e-13)
    v0 = rho0_vec(w.n, w.rho0)
    so, po, nref = h.series(v0, w.t1, w.tq, w.steps)
    r = api.series(l, l.state().upload(v0), w.t1, w.tq, w.steps, states=True)
    assert r.info.spmvs == nref
    assert np.abs(r.states - so).max() <= RHO_TOL
    assert trace_err(r.states, w.n) <= TRACE_TOL


@pytest.mark.parametrize("factor", ["0", "1"])
@pytest.mark.parametrize("name", ["c2_n36", "c4_n40", "gqsw_multi_rot", "walkthrough_nm_w1", "walkthrough_gqsw"])
def test_kron_factored_dissipator_matches_reference(name, factor, monkeypatch):
    """G-QSW L'L terms applied as L'(L X) and (X L')L (QSWG_KRON_FACTOR
    forces the choice the build otherwise makes from operand counts)."""
    monkeypatch.setenv("QSWG_KRON_FACTOR", factor)
    c = Case(name)
    l = c.build_gpu(api, format="kron")
    t1, tq, q = c.series
    r = api.series(l, l.state().from_probabilities(c.rho0), t1, tq, int(q), states=True)
    keep = c.z["series_keep"]
    assert np.abs(r.states[keep] - c.z["series_states"]).max() <= RHO_TOL
    assert trace_err(r.states, c.n) <= TRACE_TOL
    if name.startswith("c"):
        assert r.info.spmvs == c.series_spmvs
    y = l.spmv(c.z["spmv_x"])
    assert np.abs(y - c.z["spmv_y"]).max() <= 1e-13 * max(1.0, np.abs(c.z["spmv_y"]).max())
