#!/usr/bin/env python3
"""Config 3's omega sweep {0.5, 0.1, 0.9}: build once,
then set_omega (device re-mix in place) per omega, beside a fresh build per
omega; one full series at each omega.  Prints one JSON line per format."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02450_b200 import api, graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--formats", default="kron,sell")
ap.add_argument("--config", default="c3")
a = ap.parse_args()
w = graphs.config(a.config)
for fmt in a.formats.split(","):
    t0 = time.perf_counter()
    l = api.build_local(w.omega, w.h, w.ops[0], format=fmt)
    build_s = time.perf_counter() - t0
    v = l.state().from_probabilities(w.rho0)
    rows = []
    for om in (0.5, 0.1, 0.9):
        t0 = time.perf_counter()
        l.set_omega(om)
        remix_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        f = api.build_local(om, w.h, w.ops[0], format=fmt)
        fresh_s = time.perf_counter() - t0
        del f
        r = api.series(l, v, w.t1, w.tq, w.steps)
        rows.append({"omega": om, "set_omega_s": remix_s, "fresh_build_s": fresh_s,
                     "series_ms": float(r.info.device_ms), "spmvs": int(r.info.spmvs)})
    print(json.dumps({"config": a.config, "format": l.format, "build_s": build_s, "sweep": rows}), flush=True)
    del v, l
