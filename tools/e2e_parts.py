#!/usr/bin/env python3
"""Where the end-to-end (host buffers) c2 series spends its time beside the
device-resident one: upload, the Hermiticity check, series with and without
populations, populations download.  Wall clock per part (synchronised)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2003_02450_b200 import api, graphs  # noqa: E402

w = graphs.config(sys.argv[1] if len(sys.argv) > 1 else "c2")
l = api.build_global(w.omega, w.h, w.ops) if w.kind == "global" else api.build_local(w.omega, w.h, w.ops[0])
vec = torch.zeros(2 * l.rows, dtype=torch.float64, pin_memory=True).numpy().view(np.complex128)
vec[np.arange(w.n) * (w.n + 1)] = w.rho0
pops = torch.zeros((w.steps + 1) * w.n, dtype=torch.float64, pin_memory=True).numpy().reshape(w.steps + 1, w.n)
s = l.state()


def timed(f, reps=5):
    f()
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


out = {
    "upload_ms": timed(lambda: s.upload(vec)),
    "series_nopops_ms": timed(lambda: api.series(l, s, w.t1, w.tq, w.steps, populations=False)),
    "series_pops_ms": timed(lambda: api.series(l, s, w.t1, w.tq, w.steps, pops_out=pops)),
    "upload_series_pops_ms": timed(lambda: (s.upload(vec), api.series(l, s, w.t1, w.tq, w.steps, pops_out=pops))),
}
r = api.series(l, s, w.t1, w.tq, w.steps, populations=False)
out["device_ms_nopops"] = float(r.info.device_ms)
out["launches"] = int(r.info.launches)
print(json.dumps(out))

# per-iteration split of upload + series
tu, ts = [], []
for _ in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.upload(vec)
    t1 = time.perf_counter()
    api.series(l, s, w.t1, w.tq, w.steps, pops_out=pops)
    t2 = time.perf_counter()
    tu.append(t1 - t0)
    ts.append(t2 - t1)
print(json.dumps({"split_upload_ms": [round(x * 1e3, 3) for x in tu], "split_series_ms": [round(x * 1e3, 3) for x in ts]}))
s2 = l.state().upload(vec)
print(json.dumps({"fresh_state_series_ms": timed(lambda: api.series(l, s2, w.t1, w.tq, w.steps, pops_out=pops))}))
del s, s2, l
