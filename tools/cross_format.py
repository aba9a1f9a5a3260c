#!/usr/bin/env python3
"""Full-size property checks where the reference cannot run (c4 needs ~200 GB
of host RAM to assemble, c5 ~1 TB for its returned states; the GPU box has
196 GB): the matrix-free (KRON) and stored (SELL/CSR) device paths are
independent implementations of the same operator, so their series must agree
(populations at every output, the final state), take the same SpMV count, keep
|Tr rho - 1| <= 1e-12, and a single step(tq) must agree with the series' last
state (acceptance_main.cpp:245-281 checks step vs series at 1e-12 on small
graphs).  One JSON line per config."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02450_b200 import api, graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c4,c5")
a = ap.parse_args()


def build(w, **kw):
    return (api.build_local(w.omega, w.h, w.ops[0], **kw) if w.kind == "local"
            else api.build_global(w.omega, w.h, w.ops, **kw))


def trace_err(vec, n):
    return abs(vec[np.arange(n) * (n + 1)].sum() - 1.0)


for name in a.configs.split(","):
    w = graphs.config(name)
    out = {"config": name, "dim": w.dim, "outputs": w.steps + 1}
    runs = {}
    for fmt in ("kron", "stored"):
        l = build(w, format="kron" if fmt == "kron" else "sell")
        if fmt == "stored" and l.padding > 1.3:
            del l
            l = build(w, format="csr")
        v = l.state().from_probabilities(w.rho0)
        r = api.series(l, v, w.t1, w.tq, w.steps, final=True)
        fin = r.final.gather()
        runs[fmt] = (r.populations.copy(), fin, int(r.info.spmvs), l.format)
        out[fmt] = {"format": l.format, "spmvs": int(r.info.spmvs), "series_ms": float(r.info.device_ms),
                    "trace_err_final": float(trace_err(fin, w.n)),
                    "pop_sum_err_max": float(np.abs(r.populations.sum(axis=1) - 1).max())}
        if fmt == "kron":
            s, info = api.step(l, v, w.tq)
            out["step_vs_series_final"] = float(np.abs(s.gather() - fin).max())
            out["step_m_star_s"] = [int(info.m_star), int(info.s)]
            del s
        del r, v, l
    pk, fk, nk, _ = runs["kron"]
    ps, fs, ns, _ = runs["stored"]
    out["max_pop_diff"] = float(np.abs(pk - ps).max())
    out["max_final_state_diff"] = float(np.abs(fk - fs).max())
    out["same_spmvs"] = nk == ns
    out["pass"] = bool(out["max_pop_diff"] <= 1e-10 and out["max_final_state_diff"] <= 1e-10 and nk == ns
                       and out["kron"]["trace_err_final"] <= 1e-12 and out["stored"]["trace_err_final"] <= 1e-12
                       and out["step_vs_series_final"] <= 1e-10)
    print(json.dumps(out), flush=True)
    del runs
