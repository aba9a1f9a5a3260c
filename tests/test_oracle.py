"""The C restatement (oracle/qsw_oracle.c) against the reference's golden
vectors: this is what pins the oracle before it is trusted as a checker."""
import json
import os

import numpy as np
import pytest

from conftest import CASE_NAMES, GOLDEN, Case, load_csr
from oracle.oracle import rho0_vec


def test_theta_matches_reference(port):
    th = json.load(open(os.path.join(GOLDEN, "taylor.json")))["theta"]
    assert np.array_equal(port.theta(), np.array(th["double"]))


def test_select_parameters_matches_reference(port):
    for c in json.load(open(os.path.join(GOLDEN, "taylor.json")))["select"]:
        assert port.select(c["norms"], c["t"]) == (c["m_star"], c["s"]), c


@pytest.mark.parametrize("k", range(4))
@pytest.mark.parametrize("op", ["generator_matrix", "markov_chain_matrix", "symmetrize", "local_lindblad"])
def test_graph_ops_match_reference(port, k, op):
    z = np.load(os.path.join(GOLDEN, "graph_ops.npz"))
    g, want = load_csr(z, f"g{k}"), load_csr(z, f"g{k}_{op}")
    got = port.graph_op(op, g)
    assert np.array_equal(got.indptr, want.indptr) and np.array_equal(got.indices, want.indices)
    assert np.array_equal(got.data, want.data)


@pytest.mark.parametrize("name", CASE_NAMES)
def test_oracle_case_matches_reference(port, name):
    c = Case(name)
    if c.dim > 2000 and c.kind == "global":
        pytest.skip("exact-norm Gustavson powers too slow for the CPU suite at this size")
    h = c.build_oracle(port)
    L = h.csr()
    assert np.array_equal(L.indptr, c.L.indptr) and np.array_equal(L.indices, c.L.indices)
    assert np.abs(L.data - c.L.data).max(initial=0) <= 1e-14
    np.testing.assert_allclose(h.norms, c.norms, rtol=1e-13, atol=0)
    y = h.spmv(c.z["spmv_x"])
    assert np.abs(y - c.z["spmv_y"]).max() <= 1e-13
    t1, tq, q = c.series
    states, pops, nsp = h.series(rho0_vec(c.n, c.rho0), t1, tq, int(q))
    assert nsp == c.series_spmvs
    assert np.abs(states[c.z["series_keep"]] - c.z["series_states"]).max() <= 1e-12
    assert np.abs(pops - c.z["series_pops"]).max() <= 1e-12
