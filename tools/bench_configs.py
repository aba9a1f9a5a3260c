#!/usr/bin/env python3
"""Series time of every BASELINE config on one GPU (default Kron path and the
stored-superoperator path), optionally beside the reference on the host
cores.  One JSON line per config; the round's table lives in DESIGN.md."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02450_b200 import api, graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
ap.add_argument("--reference", default="", help="configs to also time with the reference (e.g. c1,c2,c3)")
ap.add_argument("--repeat", type=int, default=4)  # the 2nd call captures the series graph, later ones replay it
a = ap.parse_args()
ref_set = set(filter(None, a.reference.split(",")))
for name in a.configs.split(","):
    w = graphs.config(name)
    out = {"config": name, "dim": w.dim, "outputs": w.steps + 1}
    for fmt in ("auto", "stored"):
        t0 = time.perf_counter()
        kw = {"format": "auto"} if fmt == "auto" else {"group": 0, "format": "sell"}
        l = (api.build_local(w.omega, w.h, w.ops[0], **kw) if w.kind == "local"
             else api.build_global(w.omega, w.h, w.ops, **kw))
        if fmt == "stored" and l.padding > 1.3:
            del l
            kw["format"] = "csr"
            l = (api.build_local(w.omega, w.h, w.ops[0], **kw) if w.kind == "local"
                 else api.build_global(w.omega, w.h, w.ops, **kw))
        build = time.perf_counter() - t0
        v = l.state().from_probabilities(w.rho0)
        best = None
        for _ in range(a.repeat):
            r = api.series(l, v, w.t1, w.tq, w.steps)
            best = r.info.device_ms if best is None else min(best, r.info.device_ms)
        out[fmt] = {"format": l.format, "nnz": int(l.nnz), "build_s": build, "series_ms": best,
                    "spmvs": int(r.info.spmvs), "kron_factored": bool(l.info.kron_factored),
                    "kron_ell": bool(l.info.kron_ell), "trace_err": float(abs(r.populations[-1].sum() - 1))}
        del l, v
    if name in ref_set:
        from oracle.oracle import Oracle, rho0_vec
        o = Oracle("reference")
        cores = os.cpu_count() or 1
        t0 = time.perf_counter()
        h = o.build(w, workers=cores)
        rb = time.perf_counter() - t0
        t0 = time.perf_counter()
        _, pr, nsp = h.series(rho0_vec(w.n, w.rho0), w.t1, w.tq, w.steps, states=False, pops=True)
        out["reference"] = {"build_s": rb, "series_s": time.perf_counter() - t0, "spmvs": int(nsp), "threads": cores,
                            "library": os.path.relpath(o.path)}
    print(json.dumps(out), flush=True)
