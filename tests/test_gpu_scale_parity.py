"""Parity at scale for the c4 and c5 families against the UNMODIFIED reference.

SURVEY.md §8(c): full-size c4 (ER N=4096, ≈3.5e9 nnz) and c5 (24³ torus,
≈1 TB of returned states) do not fit the reference in host RAM, so their
parity runs on the reduced instances §8(c) names, with the reference library
(oracle/_ref/libqswref.so, compiled from /root/reference by oracle/Makefile,
shipped flags) run on the GPU box's host cores inside the test:

* ``c4_n1024`` — the c4 family at N=1024: undirected G(1024, 8/1023), seeded,
  G-QSW with H = Laplacian and L = {markov_chain_matrix}, ω=0.5, ρ0 = 1/16 on
  sites 0–15, 21 outputs on [0, 5] (dim 1,048,576, ≈2.2e8 nnz; the c4-like
  super-step plan d = 2) — build_global, liouvillian.cpp:212-307;
* ``c5_n12`` — the c5 family at 12³: periodic cubic torus, L-QSW, ω=0.3,
  ρ0 = |0⟩⟨0|, 201 outputs on [0, 100] (dim 2,985,984) — build_local,
  liouvillian.cpp:129-210;

both through the super-step series of expm.cpp:242-323.  Every device path
that serves these configs is compared with the one reference run: the
default matrix-free KRON path (factored + Hermitian tiles on c4), the stored
SELL-σ superoperator with column panels forced, and a 2-rank row-partitioned
run (in-process communicator).  Bar: max |ρ_gpu − ρ_ref| ≤ 1e-10 at every
output, populations at every output ≤ 1e-10, |Tr ρ − 1| ≤ 1e-12, the same
(span, d, m*) plan and the same executed SpMV count.
"""
import json
import os
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
api = pytest.importorskip("paper_2003_02450_b200.api")

from oracle.oracle import REF_SO, Oracle, rho0_vec  # noqa: E402
from paper_2003_02450_b200 import graphs  # noqa: E402

RHO_TOL = 1e-10
TRACE_TOL = 1e-12

CASES = {"c4_n1024": ("c4", 1024), "c5_n12": ("c5", 12)}


class RefRun:
    """One reference series of a reduced instance (run once per module)."""

    def __init__(self, name):
        cfg, size = CASES[name]
        self.name = name
        self.w = graphs.config(cfg, size=size)
        o = Oracle("reference", fast=False)  # shipped flags: the golden arithmetic
        cores = os.cpu_count() or 1
        t0 = time.perf_counter()
        h = o.build(self.w, workers=cores)
        self.build_s = time.perf_counter() - t0
        self.norms, self.nnz = h.norms.copy(), h.nnz
        self.v0 = rho0_vec(self.w.n, self.w.rho0)
        t0 = time.perf_counter()
        self.states, self.pops, self.spmvs = h.series(self.v0, self.w.t1, self.w.tq, self.w.steps)
        self.series_s = time.perf_counter() - t0
        del h


@pytest.fixture(scope="module", params=list(CASES))
def ref(request):
    """One reference run per reduced instance; pytest groups the tests by it."""
    if not os.path.exists(REF_SO):
        pytest.fail(f"{REF_SO} missing: build it with __graft_entry__.build() where /root/reference exists")
    return RefRun(request.param)


def build(w, **kw):
    if w.kind == "local":
        return api.build_local(w.omega, w.h, w.ops[0], **kw)
    return api.build_global(w.omega, w.h, w.ops, **kw)


def check(r, states, pops, info, tag):
    w = r.w
    d_rho = np.abs(states - r.states).max(axis=1)
    assert d_rho.max() <= RHO_TOL, f"{tag}: max |d rho| = {d_rho.max():.3e} at output {int(d_rho.argmax())}"
    assert np.abs(pops - r.pops).max() <= RHO_TOL, tag
    tr = np.abs(states[:, np.arange(w.n) * (w.n + 1)].sum(axis=1) - 1.0).max()
    assert tr <= TRACE_TOL, f"{tag}: |Tr rho - 1| = {tr:.2e}"
    assert int(info.spmvs) == int(r.spmvs), f"{tag}: {int(info.spmvs)} SpMVs, reference {int(r.spmvs)}"
    log = os.environ.get("QSWG_PARITY_LOG")  # evidence record (profiles/r02_parity_scale.jsonl)
    if log:
        with open(log, "a") as f:
            f.write(json.dumps({"case": r.name, "path": tag, "dim": int(w.dim), "nnz_ref": int(r.nnz),
                                "outputs": int(w.steps + 1), "spmvs_gpu": int(info.spmvs), "spmvs_ref": int(r.spmvs),
                                "plan": [int(info.path), int(info.span_m_star), int(info.span_s), int(info.d),
                                         int(info.sub_m_star)],
                                "max_abs_drho": float(d_rho.max()), "max_pop_err": float(np.abs(pops - r.pops).max()),
                                "max_trace_err": float(tr), "ref_build_s": r.build_s, "ref_series_s": r.series_s,
                                "ref_threads": os.cpu_count()}) + "\n")


def test_default_path_matches_reference(ref):
    """The format the library picks (KRON above dim 65536; on c4 factored and
    Hermitian) against the reference: norms, plan, every output."""
    r = ref
    name = r.name
    w = r.w
    l = build(w)
    assert l.format == "kron"
    np.testing.assert_allclose(l.one_norms(), r.norms, rtol=1e-13)
    assert l.nnz == r.nnz
    res = api.series(l, l.state().upload(r.v0), w.t1, w.tq, w.steps, states=True)
    assert res.info.path == 2
    if name.startswith("c4"):
        assert int(res.info.d) == 2 and bool(l.info.kron_factored)
    check(r, res.states, res.populations, res.info, f"{name} kron")
    l._query()  # the Hermitian tile path really ran (the input is a density matrix)
    assert bool(l.info.kron_hermitian)


def test_stored_sell_panels_match_reference(ref, monkeypatch):
    """The stored SELL-σ superoperator split into column panels (forced)."""
    monkeypatch.setenv("QSWG_SELL_PANELS", "3")
    r = ref
    name = r.name
    w = r.w
    l = build(w, format="sell")
    assert l.format == "sell" and int(l.info.sell_panels) == 3
    res = api.series(l, l.state().upload(r.v0), w.t1, w.tq, w.steps, states=True)
    check(r, res.states, res.populations, res.info, f"{name} sell/3 panels")


def test_two_rank_sharded_matches_reference(ref):
    """Two row-partitioned ranks (halo exchanges, allreduced stop tests and
    populations) on the default format."""
    from test_gpu_multirank import run_ranks
    r = ref
    name = r.name
    w = r.w

    def rank_fn(rank, comm):
        l = build(w, comm=comm)
        res = api.series(l, l.state().from_probabilities(w.rho0), w.t1, w.tq, w.steps, states=True)
        return l.row0, res.states, res.populations, res.info

    parts = sorted(run_ranks(2, rank_fn), key=lambda p: p[0])
    states = np.concatenate([p[1] for p in parts], axis=1)
    for p in parts:
        assert np.array_equal(p[2], parts[0][2])
    check(r, states, parts[0][2], parts[0][3], f"{name} 2 ranks")
