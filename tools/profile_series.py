#!/usr/bin/env python3
"""One build + one series of a BASELINE config through the C ABI: the
command profiled under ncu (launch list / --set full capture)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2003_02450_b200 import api, graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--size", type=int, default=None)
ap.add_argument("--series", type=int, default=1)
ap.add_argument("--group", type=int, default=0)
ap.add_argument("--format", default="auto")
a = ap.parse_args()
import time  # noqa: E402

w = graphs.config(a.config, size=a.size)
t0 = time.perf_counter()
if w.kind == "local":
    l = api.build_local(w.omega, w.h, w.ops[0], group=a.group, format=a.format)
else:
    l = api.build_global(w.omega, w.h, w.ops, group=a.group, format=a.format)
build_s = time.perf_counter() - t0
v = l.state().from_probabilities(w.rho0)
for _ in range(a.series):
    r = api.series(l, v, w.t1, w.tq, w.steps)
print(f"{a.config}: dim={l.dim} nnz={l.nnz} format={l.format} pad={l.padding:.3f} group={l.group} spmvs={r.info.spmvs} launches={r.info.launches} "
      f"device_ms={r.info.device_ms:.3f} build_s={build_s:.2f} norms={l.one_norms()[:3]} "
      f"plan=({r.info.path},{r.info.span_m_star},{r.info.span_s},d={r.info.d}) pop0={r.populations[-1][0]:.15f} "
      f"trace_err={abs(r.populations[-1].sum() - 1):.2e}")
