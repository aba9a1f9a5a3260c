"""The multi-GPU code path (row-sharded superoperator, per-term halo
exchange, allreduce(max) stop tests, allreduce(sum) populations) run as
`world` ranks on ONE GPU through the in-process communicator
(qswg_comm_create_local: host-side rendezvous collectives, no kernel waits on
another rank).  Results must equal the single-rank run and the reference."""
import threading

import numpy as np
import pytest

from conftest import Case

pytestmark = pytest.mark.gpu
api = pytest.importorskip("paper_2003_02450_b200.api")


def run_ranks(world, fn):
    comms = api.Comm.local_group(world)
    out, errs = [None] * world, []

    def body(r):
        try:
            out[r] = fn(r, comms[r])
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("group,fmt", [(0, "auto"), (1, "auto"), (0, "kron")])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["c2_n36", "c5_n64", "c3_n40", "c4_n40", "lqsw_src_snk", "gqsw_multi_rot"])
def test_sharded_series_matches_single_and_reference(name, world, group, fmt):
    c = Case(name)
    t1, tq, q = c.series

    def rank_fn(r, comm):
        l = c.build_gpu(api, comm=comm, group=group, format=fmt)
        v = l.state().from_probabilities(c.rho0)
        res = api.series(l, v, t1, tq, int(q), states=True)
        st, lo, hi = l.partition()
        return l.row0, res.states, res.populations, int(res.info.spmvs), st, l.one_norms()

    parts = run_ranks(world, rank_fn)
    starts = parts[0][4]
    assert starts[0] == 0 and starts[-1] == c.dim and np.all(starts % c.n == 0)
    states = np.concatenate([p[1] for p in sorted(parts, key=lambda p: p[0])], axis=1)
    for p in parts:
        np.testing.assert_allclose(p[5], c.norms, rtol=1e-13)  # distributed norm bound
        assert np.array_equal(p[2], parts[0][2])                # allreduced populations agree
    keep = c.z["series_keep"]
    assert np.abs(states[keep] - c.z["series_states"]).max() <= 1e-10
    assert np.abs(parts[0][2] - c.z["series_pops"]).max() <= 1e-10
    if name.startswith("c") or group == 1:
        assert parts[0][3] == c.series_spmvs
    if group == 1:
        # bitwise mode: per-row arithmetic is independent of the partition, so
        # the sharded run is bit-identical to the single-rank run
        l1 = c.build_gpu(api, group=1)
        single = api.series(l1, l1.state().from_probabilities(c.rho0), t1, tq, int(q), states=True)
        assert np.array_equal(states, single.states)


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_step_and_overflow(world):
    c = Case("c1_n64")

    def rank_fn(r, comm):
        l = c.build_gpu(api, comm=comm)
        v = l.state().from_probabilities(c.rho0)
        w, info = api.step(l, v, float(c.z["step_t"][0]))
        return l.row0, w.gather(), info.spmvs

    parts = sorted(run_ranks(world, rank_fn), key=lambda p: p[0])
    got = np.concatenate([p[1] for p in parts])
    assert np.abs(got - c.z["step_states"][0]).max() <= 1e-10
    assert parts[0][2] == c.z["step_spmvs"][0]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_kron_factored(world, monkeypatch):
    monkeypatch.setenv("QSWG_KRON_FACTOR", "1")
    c = Case("c4_n40")
    t1, tq, q = c.series

    def rank_fn(r, comm):
        l = c.build_gpu(api, comm=comm, format="kron")
        res = api.series(l, l.state().from_probabilities(c.rho0), t1, tq, int(q), states=True)
        return l.row0, res.states, int(res.info.spmvs)

    parts = sorted(run_ranks(world, rank_fn), key=lambda p: p[0])
    states = np.concatenate([p[1] for p in parts], axis=1)
    keep = c.z["series_keep"]
    assert np.abs(states[keep] - c.z["series_states"]).max() <= 1e-10
    assert parts[0][2] == c.series_spmvs


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("fmt", ["kron", "sell"])
def test_sharded_coherence_and_set_omega(world, fmt):
    """Coherence norms (allreduce max over ranks) and populations of a sharded
    series equal the single-rank run's, before and after an omega re-mix."""
    c = Case("lqsw_src_snk")
    t1, tq, q = c.series

    def series_of(l):
        v = l.state().from_probabilities(c.rho0)
        r = api.series(l, v, t1, tq, int(q), coherence=True)
        out = [r.populations.copy(), r.coherence.copy(), v.coherence()]
        l.set_omega(0.35)
        r = api.series(l, v, t1, tq, int(q), coherence=True)
        return out + [r.populations.copy(), r.coherence.copy()]

    single = series_of(c.build_gpu(api, format=fmt))
    parts = run_ranks(world, lambda r, comm: series_of(c.build_gpu(api, comm=comm, format=fmt)))
    for p in parts:
        for got, want in zip(p, single):
            assert np.abs(np.asarray(got) - np.asarray(want)).max() <= 1e-12


@pytest.mark.parametrize("factor", ["1", "0"])
@pytest.mark.parametrize("size", [64, 96])
def test_sharded_kron_er_matches_single(size, factor, monkeypatch):
    """The c4 family (ER G-QSW) at n = 64 / 96 on two row-partitioned ranks —
    the general KRON kernels with padded sliced-ELL operand rows, factored and
    not — against the one-GPU run (Hermitian tiles)."""
    from paper_2003_02450_b200 import graphs
    monkeypatch.setenv("QSWG_KRON_FACTOR", factor)
    w = graphs.config("c4", size=size)

    def build(**kw):
        return api.build_global(w.omega, w.h, w.ops, format="kron", **kw)

    l1 = build()
    r1 = api.series(l1, l1.state().from_probabilities(w.rho0), w.t1, w.tq, w.steps, states=True)

    def rank_fn(r, comm):
        l = build(comm=comm)
        res = api.series(l, l.state().from_probabilities(w.rho0), w.t1, w.tq, w.steps, states=True)
        return l.row0, res.states, int(res.info.spmvs)

    parts = sorted(run_ranks(2, rank_fn), key=lambda p: p[0])
    states = np.concatenate([p[1] for p in parts], axis=1)
    assert np.abs(states - r1.states).max() <= 1e-13
    assert parts[0][2] == int(r1.info.spmvs)
