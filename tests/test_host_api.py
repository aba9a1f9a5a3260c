"""CPU-side checks of libqswg.so: it loads, exports every symbol the C
header declares, its host logic (graph -> operators, canonical CSR, Taylor
parameters) matches the reference's golden vectors, and device entry points
fail loudly without a GPU (no CPU fallback)."""
import json
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, has_gpu, load_csr

api = pytest.importorskip("paper_2003_02450_b200.api")
from paper_2003_02450_b200 import _lib, graphs  # noqa: E402


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "qswg.h")).read()
    return sorted(set(re.findall(r"\b(qswg_[A-Za-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(_lib.lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_version():
    import ctypes as C
    a, b = C.c_int(), C.c_int()
    _lib.check(_lib.lib.qswg_version(C.byref(a), C.byref(b)))
    assert (a.value, b.value) == (0, 1)


@pytest.mark.parametrize("k", range(4))
@pytest.mark.parametrize("op", ["generator_matrix", "markov_chain_matrix", "symmetrize", "local_lindblad"])
def test_graph_ops_bit_identical_to_reference(k, op):
    z = np.load(os.path.join(GOLDEN, "graph_ops.npz"))
    g, want = load_csr(z, f"g{k}"), load_csr(z, f"g{k}_{op}")
    fn = {"generator_matrix": lambda m: api.generator_matrix(1.0, m)}.get(op, getattr(api, op))
    got = fn(g).to_csr()
    assert np.array_equal(got.indptr, want.indptr) and np.array_equal(got.indices, want.indices)
    assert np.array_equal(got.data, want.data)


def test_graph_validation_errors():
    bad = graphs.Csr.from_coo(3, 3, [0, 1], [0, 2], [1.0, 1.0])  # self-loop
    with pytest.raises(ValueError):
        api.markov_chain_matrix(bad)
    neg = graphs.Csr.from_coo(3, 3, [1], [0], [-1.0])
    with pytest.raises(ValueError):
        api.symmetrize(neg)
    with pytest.raises(ValueError):
        api.generator_matrix(0.0, graphs.cycle_graph(4))
    with pytest.raises(IndexError):
        api.augment(graphs.cycle_graph(4), sources=[(7, 1.0)])
    with pytest.raises(ValueError):
        api.augment(graphs.cycle_graph(4), sources=[(1, 1.0), (1, 2.0)])


def test_augment_layout():
    a = api.augment(graphs.cycle_graph(4), sources=[(1, 2.0)], sinks=[(3, 3.0)]).to_dense()
    assert a.shape == (6, 6)
    assert a[1, 4] == 2.0 and a[5, 3] == 3.0  # source arc 4 -> 1, sink arc 3 -> 5


def test_sparse_canonicalisation():
    m = api.SparseMatrix.from_triplets(3, 3, [0, 0, 1, 2, 2], [2, 2, 1, 0, 1], [1, 2, 0, 5, -5]).to_csr()
    assert list(m.indptr) == [0, 1, 1, 3] and list(m.indices) == [2, 0, 1]
    assert list(m.data) == [3, 5, -5]
    with pytest.raises(IndexError):
        api.SparseMatrix.from_triplets(2, 2, [0], [5], [1.0])


def test_theta_and_select_match_reference():
    g = json.load(open(os.path.join(GOLDEN, "taylor.json")))
    assert np.array_equal(api.build_theta_table(2.0 ** -53), np.array(g["theta"]["double"]))
    assert np.array_equal(api.build_theta_table(2.0 ** -24), np.array(g["theta"]["single"]))
    np.testing.assert_allclose(api.build_theta_table(1e-10), g["theta"]["1e-10"], rtol=1e-10)
    for c in g["select"]:
        assert api.select_parameters(c["norms"], c["t"]) == (c["m_star"], c["s"]), c
    with pytest.raises(ValueError):
        api.build_theta_table(1.0)


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_device_entry_points_fail_loudly_without_gpu():
    w = graphs.config("c1", size=8)
    with pytest.raises(_lib.CudaError):
        api.build_local(w.omega, w.h, w.ops[0])


@pytest.mark.parametrize("k", range(4))
def test_nm_operators_bit_identical_to_reference(k):
    """operators.cpp nm_vsets / nm_H / nm_L / nm_H_rot against the reference."""
    z = np.load(os.path.join(GOLDEN, "nm_ops.npz"))
    g = load_csr(z, f"g{k}")
    gamma = 1.0 if k == 0 else 0.7
    gu = api.symmetrize(g)
    dims = api.nm_vsets(gu)
    assert np.array_equal(dims, z[f"g{k}_dims"])
    for name, got in (("nm_H", api.nm_H(gamma, gu, dims)), ("nm_L", api.nm_L(gamma, g, dims)),
                      ("nm_H_rot", api.nm_H_rot(dims)), ("nm_H_rot_py", api.nm_H_rot(dims, pauli_y=True))):
        got, want = got.to_csr(), load_csr(z, f"g{k}_{name}")
        assert np.array_equal(got.indptr, want.indptr) and np.array_equal(got.indices, want.indices), name
        assert np.array_equal(got.data, want.data), name


def test_nm_rho_map_and_measure():
    dims = np.array([1, 1, 2])
    e = api.nm_rho_map([0.5, 0.25, 0.25], dims)
    assert list(e) == [0.5, 0.25, 0.125, 0.125]
    assert list(api.nm_measure(e, dims)) == [0.5, 0.25, 0.25]
    with pytest.raises(ValueError):
        api.nm_rho_map([0.5, 0.5, 0.5], dims)
    with pytest.raises(ValueError):
        api.nm_vsets(graphs.Csr.from_coo(3, 3, [2], [0], [1.0]))  # not symmetric
