#!/usr/bin/env python3
"""Times one product (time_spmv, Kron prepare included) and one series term
(time_series_term with d running sums) per config; no series is run, so
kernel experiments that skip work stay finite."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02450_b200 import api, graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c2,c3,c4")
ap.add_argument("--format", default="auto")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--d", type=int, default=1)
ap.add_argument("--tag", default="")
a = ap.parse_args()
for name in a.configs.split(","):
    w = graphs.config(name)
    l = (api.build_local(w.omega, w.h, w.ops[0], format=a.format) if w.kind == "local"
         else api.build_global(w.omega, w.h, w.ops, format=a.format))
    out = {"tag": a.tag, "config": name, "format": l.format, "spmv_us": 1e3 * l.time_spmv(a.iters),
           "term_us": 1e3 * l.time_series_term(a.iters, a.d)}
    print(json.dumps(out), flush=True)
    del l
