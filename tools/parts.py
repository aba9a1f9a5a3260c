#!/usr/bin/env python3
"""Per-part device times of one series term (prepare / term kernel / flush)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02450_b200 import api, graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c2,c3,c4,c5")
ap.add_argument("--format", default="auto")
ap.add_argument("--d", type=int, default=0, help="outputs (0: the config's series plan)")
ap.add_argument("--tag", default="")
a = ap.parse_args()
D = {"c1": 5, "c2": 6, "c3": 1, "c4": 2, "c5": 2}
for name in a.configs.split(","):
    w = graphs.config(name)
    l = (api.build_local(w.omega, w.h, w.ops[0], format=a.format) if w.kind == "local"
         else api.build_global(w.omega, w.h, w.ops, format=a.format))
    p = l.time_series_parts(20, a.d or D.get(name, 1))
    out = {"tag": a.tag, "config": name, "format": l.format, "spmv_us": 1e3 * l.time_spmv(20)}
    out.update({k + "_us": 1e3 * v for k, v in p.items()})
    print(json.dumps(out), flush=True)
    del l
