#!/usr/bin/env python3
"""Splits one series term into its parts on every config: the bare SpMV
(Kron prepare included) and the fused term at 1 and d running sums, plus the
series plan (d, terms per super-step).  CUDA events on the library stream."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02450_b200 import api, graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c2,c3,c4,c5")
ap.add_argument("--format", default="auto")
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
for name in a.configs.split(","):
    w = graphs.config(name)
    l = (api.build_local(w.omega, w.h, w.ops[0], format=a.format) if w.kind == "local"
         else api.build_global(w.omega, w.h, w.ops, format=a.format))
    v = l.state().from_probabilities(w.rho0)
    r = api.series(l, v, w.t1, w.tq, w.steps)
    d = max(int(r.info.d), 1)
    out = {"config": name, "format": l.format, "dim": l.dim, "series_ms": r.info.device_ms,
           "spmvs": int(r.info.spmvs), "d": d, "path": int(r.info.path),
           "spmv_ms": l.time_spmv(a.iters), "term1_ms": l.time_series_term(a.iters, 1),
           "termd_ms": l.time_series_term(a.iters, d)}
    out["sum_share"] = 1 - out["spmv_ms"] / out["termd_ms"]
    print(json.dumps(out), flush=True)
    del l, v
