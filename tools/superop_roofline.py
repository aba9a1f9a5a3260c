#!/usr/bin/env python3
"""SURVEY.md 8(d) metric (i): the stored-superoperator SpMV (series term
kernel) in HBM GB/s and as a fraction of the measured peak, on one GPU, for
the BASELINE configs, in both stored formats (SELL-C-sigma and CSR).
Algorithmic bytes per launch: 20 B/nnz + 8 B/row + x read (16 B/elem) + K_p
written (16 B/elem); SELL padding is not counted as useful bytes."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02450_b200 import api, graphs  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c2,c3,c4")
ap.add_argument("--formats", default="sell,csr")
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
for name in a.configs.split(","):
    w = graphs.config(name)
    build = (lambda fmt: api.build_local(w.omega, w.h, w.ops[0], format=fmt)) if w.kind == "local" else \
        (lambda fmt: api.build_global(w.omega, w.h, w.ops, format=fmt))
    for fmt in a.formats.split(","):
        l = build(fmt)
        parts = l.time_series_parts(a.iters, 1)
        nnz = int(l.info.nnz_local)
        b = 20 * nnz + 8 * (l.rows + 1) + 16 * l.dim + 16 * l.rows
        gbs = b / (parts["term"] * 1e-3) / 1e9
        print(json.dumps({"config": name, "format": l.format, "group": int(l.group), "padding": l.padding,
                          "nnz": nnz, "dim": l.dim, "bytes_per_launch": b, "term_ms": parts["term"],
                          "achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak}), flush=True)
        del l
