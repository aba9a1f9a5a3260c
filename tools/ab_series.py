#!/usr/bin/env python3
"""A/B timing of whole series on one config: runs `reps` series per arm in
alternation (env knobs set per arm in child processes is not possible in one
process, so this times the current process's configuration) and prints the
min / median device ms."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02450_b200 import api, graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--reps", type=int, default=12)
ap.add_argument("--tag", default="")
a = ap.parse_args()
w = graphs.config(a.config)
l = (api.build_local(w.omega, w.h, w.ops[0]) if w.kind == "local" else api.build_global(w.omega, w.h, w.ops))
v = l.state().from_probabilities(w.rho0)
ts = []
for _ in range(a.reps):
    r = api.series(l, v, w.t1, w.tq, w.steps, populations=False)
    ts.append(r.info.device_ms)
ts = sorted(ts[min(3, len(ts) - 1):])  # the first calls run uncaptured / capture the graph
print(json.dumps({"tag": a.tag, "config": a.config, "min_ms": ts[0], "median_ms": ts[len(ts) // 2], "all": ts}))
