#!/usr/bin/env python3
"""Times the SpMV / fused series-term kernels for every row-group width on a
BASELINE config (CUDA events on the library stream) and prints GB/s."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02450_b200 import api, graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--size", type=int, default=None)
ap.add_argument("--count", type=int, default=6)
ap.add_argument("--groups", default="4,8,16,32")
ap.add_argument("--format", default="auto")
a = ap.parse_args()
w = graphs.config(a.config, size=a.size)
out = []
for g in [int(x) for x in a.groups.split(",")]:
    l = (api.build_local(w.omega, w.h, w.ops[0], group=g, format=a.format) if w.kind == "local"
         else api.build_global(w.omega, w.h, w.ops, group=g, format=a.format))
    nnz, dim = l.info.nnz_local, l.dim
    b_spmv = 20 * nnz + 8 * (dim + 1) + 32 * dim  # algorithmic (CSR) bytes, padding not counted
    b_term = b_spmv + 32 * a.count * dim
    t_spmv = l.time_spmv(20, g)
    t_term = l.time_series_term(20, a.count)
    r = {"config": a.config, "group": g, "format": l.format, "padding": l.padding, "nnz": nnz, "dim": dim, "spmv_ms": t_spmv,
         "spmv_gbs": b_spmv / t_spmv / 1e6, "term_ms": t_term, "term_gbs": b_term / t_term / 1e6,
         "count": a.count}
    out.append(r)
    print(json.dumps(r), flush=True)
    del l
