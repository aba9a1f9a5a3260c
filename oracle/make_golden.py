#!/usr/bin/env python3
"""Generate tests/golden/ from the UNMODIFIED reference library (oracle/_ref).

TEST INFRASTRUCTURE ONLY.  Run here (where /root/reference exists):
    make -C oracle ref && python oracle/make_golden.py
Every fixture is produced by the reference's own code path (shipped flags,
no FMA: oracle/_ref/libqswref.so) through oracle/ref_harness.cpp, so the
fixtures pin both the C restatement (tests/test_oracle.py) and the device
path (tests/test_gpu_parity.py).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, rho0_vec  # noqa: E402
from paper_2003_02450_b200 import graphs  # noqa: E402
from paper_2003_02450_b200.graphs import Csr  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def random_digraph(rng, n, density=0.4):
    """Seeded random weighted digraph (weights in [0.1, 2))."""
    r, c, v = [], [], []
    for i in range(n):
        for j in range(n):
            if i != j and rng.random() < density:
                r.append(i)
                c.append(j)
                v.append(0.1 + 1.9 * rng.random())
    if not r:
        r, c, v = [n - 1], [0], [1.0]
    return Csr.from_coo(n, n, r, c, v)


def csr_arrays(prefix, m: Csr):
    return {f"{prefix}_indptr": m.indptr, f"{prefix}_indices": m.indices, f"{prefix}_data": m.data,
            f"{prefix}_shape": np.array([m.rows, m.cols])}


def padded(m: Csr, n):
    return Csr(n, n, np.concatenate([m.indptr, np.full(n - m.rows, m.indptr[-1])]), m.indices, m.data)


def cases():
    """(name, kind, n, omega, h, ops, sources, sinks, h_rot, rho0 probs, series (t1,tq,q), step ts)."""
    out = []
    for name, size in (("c1", None), ("c2", 6), ("c3", 40), ("c4", 40), ("c5", 4)):
        w = graphs.config(name, size=size)
        out.append(dict(name=f"{name}_n{w.n}", kind=w.kind, n=w.n, omega=w.omega, h=w.h, ops=w.ops,
                        sources=[], sinks=[], h_rot=None, rho0=w.rho0, series=(w.t1, w.tq, w.steps),
                        steps=[w.tq / 3, -0.25]))
    for om in (0.1, 0.9):
        w = graphs.config("c3", omega=om, size=40)
        out.append(dict(name=f"c3_n40_w{om}", kind="local", n=w.n, omega=om, h=w.h, ops=w.ops, sources=[],
                        sinks=[], h_rot=None, rho0=w.rho0, series=(w.t1, w.tq, w.steps), steps=[5.0]))
    rng = np.random.default_rng(2003)
    # L-QSW with a source and a sink on a random digraph (augmented vertices)
    g = random_digraph(rng, 7)
    R = Oracle("reference", fast=False)
    h = padded(R.graph_op("generator_matrix", R.graph_op("symmetrize", g)), 9)
    ml = padded(R.graph_op("local_lindblad", R.graph_op("generator_matrix", g)), 9)
    p = np.zeros(9)
    p[:7] = 1.0 / 7
    out.append(dict(name="lqsw_src_snk", kind="local", n=9, omega=0.6, h=h, ops=[ml], sources=[(2, 1.0)],
                    sinks=[(4, 1.5)], h_rot=None, rho0=p, series=(0.0, 6.0, 12), steps=[2.0]))
    # G-QSW with two complex Lindblads and a rotating Hamiltonian
    n = 6
    gg = random_digraph(rng, n, 0.5)
    h = R.graph_op("generator_matrix", R.graph_op("symmetrize", gg))
    l1 = Csr.from_coo(n, n, *np.nonzero(gg.to_dense()),
                      (rng.normal(size=gg.nnz) + 1j * rng.normal(size=gg.nnz)) * 0.5)
    l2 = Csr.from_coo(n, n, np.arange(n), (np.arange(n) + 1) % n, np.full(n, 0.3 + 0.2j))
    hr = Csr.from_coo(n, n, [0, 1, 2, 1], [1, 0, 1, 2], [1j, -1j, 0.5, 0.5])
    p = np.full(n, 1.0 / n)
    out.append(dict(name="gqsw_multi_rot", kind="global", n=n, omega=0.4, h=h, ops=[l1, l2], sources=[],
                    sinks=[], h_rot=hr, rho0=p, series=(0.5, 4.0, 7), steps=[1.5]))
    # paper walkthrough (test_walk.cpp:18-31): 3-vertex digraph, G-QSW omega=1
    g3 = Csr.from_coo(3, 3, [2, 2], [0, 1], [1.0, 1.0])
    gu = R.graph_op("symmetrize", g3)
    out.append(dict(name="walkthrough_gqsw", kind="global", n=3, omega=1.0, h=R.graph_op("generator_matrix", gu),
                    ops=[g3], sources=[], sinks=[], h_rot=None, rho0=np.array([1.0, 0, 0]),
                    series=(0.0, 100.0, 10), steps=[100.0]))
    vs_h, _ = R.nm_op("nm_H", g3, gu, 1.0)
    vs_l, _ = R.nm_op("nm_L", g3, gu, 1.0)
    vs_r, dims3 = R.nm_op("nm_H_rot", g3, gu)
    p_nm = np.concatenate([np.full(int(d), (1.0 if v == 0 else 0.0) / d) for v, d in enumerate(dims3)])
    for om in (1.0, 0.0):
        out.append(dict(name=f"walkthrough_nm_w{int(om)}", kind="global", n=int(dims3.sum()), omega=om, h=vs_h,
                        ops=[vs_l], sources=[], sinks=[], h_rot=vs_r, rho0=p_nm, series=(0.0, 100.0, 10),
                        steps=[100.0]))
    out.append(dict(name="walkthrough_lqsw_w0", kind="local", n=3, omega=0.0, h=gu, ops=[g3], sources=[],
                    sinks=[], h_rot=None, rho0=np.array([1.0, 0, 0]), series=(0.0, 100.0, 10), steps=[100.0]))
    out.append(dict(name="walkthrough_lqsw_w1", kind="local", n=3, omega=1.0, h=gu, ops=[g3], sources=[],
                    sinks=[], h_rot=None, rho0=np.array([1.0, 0, 0]), series=(0.0, 100.0, 10), steps=[100.0]))
    return out


def build(o: Oracle, c):
    if c["kind"] == "local":
        return o.build_local(c["omega"], c["h"], c["ops"][0], c["sources"], c["sinks"])
    return o.build_global(c["omega"], c["h"], c["ops"], c["h_rot"])


def main():
    os.makedirs(OUT, exist_ok=True)
    R = Oracle("reference", fast=False)
    meta = {"generator": "oracle/make_golden.py", "library": os.path.relpath(R.path, ROOT),
            "flags": "-O3 -DNDEBUG (shipped flags, no FMA)", "cases": {}}

    # theta tables and select_parameters
    th = {"double": R.theta(2.0 ** -53).tolist(), "single": R.theta(2.0 ** -24).tolist(),
          "1e-10": R.theta(1e-10).tolist()}
    rng = np.random.default_rng(7)
    sel = []
    for _ in range(200):
        norms = np.cumprod(rng.uniform(0.5, 30.0, size=9))
        t = float(10 ** rng.uniform(-18, 2.5)) * (1 if rng.random() < 0.8 else -1)
        m, s = R.select(norms, t)
        sel.append({"norms": norms.tolist(), "t": t, "m_star": m, "s": s})
    sel.append({"norms": [0.0] * 9, "t": 5.0, "m_star": 0, "s": 1})
    sel.append({"norms": [1.0] * 9, "t": 0.0, "m_star": 0, "s": 1})
    with open(os.path.join(OUT, "taylor.json"), "w") as f:
        json.dump({"theta": th, "select": sel}, f)

    # graph -> operator helpers
    garr = {}
    for k in range(4):
        g = random_digraph(np.random.default_rng(100 + k), 9, 0.35)
        garr.update(csr_arrays(f"g{k}", g))
        for op in ("generator_matrix", "markov_chain_matrix", "symmetrize", "local_lindblad"):
            garr.update(csr_arrays(f"g{k}_{op}", R.graph_op(op, g)))
    np.savez_compressed(os.path.join(OUT, "graph_ops.npz"), **garr)

    # demoralisation operators (operators.cpp nm_*): walkthrough + random digraphs
    narr = {}
    g3 = Csr.from_coo(3, 3, [2, 2], [0, 1], [1.0, 1.0])
    nm_graphs = [g3] + [random_digraph(np.random.default_rng(300 + k), 6, 0.35) for k in range(3)]
    for k, g in enumerate(nm_graphs):
        gu = R.graph_op("symmetrize", g)
        narr.update(csr_arrays(f"g{k}", g))
        for op in ("nm_H", "nm_L", "nm_H_rot"):
            for py in ((0, 1) if op == "nm_H_rot" else (0,)):
                m, dims = R.nm_op(op, g, gu, gamma=1.0 if k == 0 else 0.7, pauli_y=bool(py))
                narr.update(csr_arrays(f"g{k}_{op}{'_py' if py else ''}", m))
                narr[f"g{k}_dims"] = dims
    np.savez_compressed(os.path.join(OUT, "nm_ops.npz"), **narr)

    for c in cases():
        hd = build(R, c)
        arr = {"norms": hd.norms, "rho0": c["rho0"]}
        arr.update(csr_arrays("h", c["h"]))
        for k, op in enumerate(c["ops"]):
            arr.update(csr_arrays(f"op{k}", op))
        if c["h_rot"] is not None:
            arr.update(csr_arrays("hrot", c["h_rot"]))
        arr.update(csr_arrays("L", hd.csr()))
        v0 = rho0_vec(c["n"], c["rho0"])
        t1, tq, q = c["series"]
        states, pops, nsp = hd.series(v0, t1, tq, q)
        arr["series_pops"] = pops
        keep = sorted({0, q // 2, q}) if hd.dim > 1024 else list(range(q + 1))
        arr["series_keep"] = np.array(keep)
        arr["series_states"] = states[keep]
        step_out, step_spmvs = [], []
        for t in c["steps"]:
            o, ns = hd.step(v0, t)
            step_out.append(o)
            step_spmvs.append(ns)
        arr["step_t"] = np.array(c["steps"])
        arr["step_states"] = np.array(step_out)
        arr["step_spmvs"] = np.array(step_spmvs)
        rngx = np.random.default_rng(11)
        x = rngx.uniform(-1, 1, hd.dim) + 1j * rngx.uniform(-1, 1, hd.dim)
        arr["spmv_x"] = x
        arr["spmv_y"] = hd.spmv(x)
        np.savez_compressed(os.path.join(OUT, f"case_{c['name']}.npz"), **arr)
        meta["cases"][c["name"]] = {
            "kind": c["kind"], "n": c["n"], "omega": c["omega"], "dim": int(hd.dim), "nnz": int(hd.nnz),
            "sources": c["sources"], "sinks": c["sinks"], "has_h_rot": c["h_rot"] is not None,
            "n_ops": len(c["ops"]), "series": [t1, tq, q], "series_spmvs": int(nsp)}
        print(c["name"], hd.dim, hd.nnz, nsp, flush=True)
    with open(os.path.join(OUT, "cases.json"), "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    main()
