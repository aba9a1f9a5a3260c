#!/usr/bin/env python3
"""Full-size parity of the device path against the unmodified reference
library (oracle/_ref, all host threads) on one BASELINE config: norms,
(m*, s), executed SpMVs, rho at every output time (max |d rho|), |Tr rho - 1|.
Writes one JSON line; run on the GPU box (the reference .so travels)."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle, rho0_vec  # noqa: E402
from paper_2003_02450_b200 import api, graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--omega", type=float, default=None)
ap.add_argument("--group", type=int, default=0)
a = ap.parse_args()
w = graphs.config(a.config, omega=a.omega)
cores = os.cpu_count() or 1
R = Oracle("reference", fast=False)  # shipped flags (no FMA): the golden arithmetic
t0 = time.perf_counter()
hr = R.build(w, workers=cores)
t_ref_build = time.perf_counter() - t0
v0 = rho0_vec(w.n, w.rho0)
t0 = time.perf_counter()
s_ref, p_ref, n_ref = hr.series(v0, w.t1, w.tq, w.steps, states=True, pops=True)
t_ref = time.perf_counter() - t0
t0 = time.perf_counter()
l = (api.build_local(w.omega, w.h, w.ops[0], group=a.group) if w.kind == "local"
     else api.build_global(w.omega, w.h, w.ops, group=a.group))
t_gpu_build = time.perf_counter() - t0
v = l.state().upload(v0)
r = api.series(l, v, w.t1, w.tq, w.steps, states=True)
d_rho = np.abs(r.states - s_ref).max(axis=1)
tr = np.abs(r.states.reshape(w.steps + 1, w.n, w.n).trace(axis1=1, axis2=2) - 1)
out = {"config": w.name, "omega": w.omega, "dim": int(l.dim), "nnz_gpu": int(l.nnz), "nnz_ref": int(hr.nnz),
       "format": l.format, "group": int(l.group),
       "norms_rel_err": float(np.abs(l.one_norms() / hr.norms - 1).max()),
       "plan": [int(r.info.path), int(r.info.span_m_star), int(r.info.span_s), int(r.info.d)],
       "spmvs_gpu": int(r.info.spmvs), "spmvs_ref": int(n_ref),
       "max_abs_drho": float(d_rho.max()), "max_abs_drho_per_time": d_rho.tolist(),
       "max_trace_err_gpu": float(tr.max()), "max_pop_err": float(np.abs(r.populations - p_ref).max()),
       "ref_build_s": t_ref_build, "ref_series_s": t_ref, "ref_threads": cores,
       "gpu_build_s": t_gpu_build, "gpu_series_ms": float(r.info.device_ms)}
out["pass"] = bool(out["max_abs_drho"] <= 1e-10 and out["max_trace_err_gpu"] <= 1e-12
                   and out["nnz_gpu"] == out["nnz_ref"])
print(json.dumps(out), flush=True)
