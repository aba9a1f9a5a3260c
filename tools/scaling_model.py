#!/usr/bin/env python3
"""Modelled multi-GPU strong scaling of one series term from measurements on
ONE GPU (only one is available to this build): the N row blocks of the real
multi-GPU build (partition, halo plan, local kernels) are built as N
in-process ranks, each rank's term is timed alone on the GPU (prepare + term
kernel + flush, CUDA events; no rank ever waits on another), and the halo
volume each rank receives per term comes from the real halo plan.

  T_N (no overlap)   = max_r compute_r + max_r halo_r / B + L
  T_N (overlap)      = max_r max(compute_r, halo_r / B) + L
with L the per-term collective latency (one allreduce per term since round 2;
reported for L = 0, 10, 20 us — it cannot be measured on one GPU) plus, for
the round-1 flow, one host synchronisation per term (measured here: a stream
synchronisation after a term's launches), and B = 900 GB/s (NVLink 5 per direction; the exchange of the factored KRON
path also moves W, counted as a second x-sized halo).  Efficiency is against
the measured one-GPU term (Hermitian path).  A model, not a measurement:
DESIGN.md section 5 says so beside the numbers."""
import argparse
import json
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02450_b200 import api, graphs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c2,c4")
ap.add_argument("--worlds", default="2,4,8")
ap.add_argument("--format", default="auto")
ap.add_argument("--bw", type=float, default=900e9)
a = ap.parse_args()
LAT_US = (0.0, 10.0, 20.0)


def sync_latency_ms():
    """Host round trip of one stream synchronisation after a small launch."""
    import time
    import numpy as np
    w = graphs.config("c1", size=8)
    l = api.build_local(w.omega, w.h, w.ops[0])
    v = l.state().from_probabilities(w.rho0)
    out = []
    for _ in range(50):
        t0 = time.perf_counter()
        v.populations()  # one tiny kernel + D2H + synchronisation
        out.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(out))


SYNC_MS = sync_latency_ms()
D = {"c1": 5, "c2": 6, "c3": 1, "c4": 2, "c5": 2}


def build(w, comm=None):
    kw = {"format": a.format, "comm": comm}
    return (api.build_local(w.omega, w.h, w.ops[0], **kw) if w.kind == "local"
            else api.build_global(w.omega, w.h, w.ops, **kw))


for name in a.configs.split(","):
    w = graphs.config(name)
    d = D.get(name, 1)
    l1 = build(w)
    p1 = l1.time_series_parts(10, d)
    t1 = p1["prepare"] + p1["term"] + p1["flush"]
    fmt, factored = l1.format, bool(l1.info.kron_factored)
    del l1
    for world in (int(x) for x in a.worlds.split(",")):
        comms = api.Comm.local_group(world)
        ranks = [None] * world
        errs = []

        def body(r):
            try:
                ranks[r] = build(w, comms[r])
            except Exception as e:  # noqa: BLE001
                errs.append(e)

        ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            raise errs[0]
        comp, halo = [], []
        for r, l in enumerate(ranks):
            p = l.time_series_parts(10, d)
            comp.append(p["prepare"] + p["term"] + p["flush"])
            _, lo, hi = l.partition()
            rows = int((hi[r] - lo[r]).sum())  # elements this rank receives per exchange
            halo.append(16.0 * rows * (2 if (fmt == "kron" and factored) else 1))
        t_comm = [h / a.bw * 1e3 for h in halo]
        no_ov = max(comp) + max(t_comm)
        ov = max(max(c, tc) for c, tc in zip(comp, t_comm))
        eff = {f"L{int(lat)}us": {"overlap": t1 / (world * (ov + lat * 1e-3)),
                                  "no_overlap": t1 / (world * (no_ov + lat * 1e-3)),
                                  "round1_flow_overlap": t1 / (world * (ov + lat * 1e-3 + SYNC_MS))}
               for lat in LAT_US}
        print(json.dumps({"config": name, "format": fmt, "world": world, "one_gpu_term_ms": t1,
                          "one_gpu_format": fmt,
                          "rank_compute_ms": comp, "rank_halo_mb": [h / 1e6 for h in halo],
                          "model_term_ms_no_overlap": no_ov, "model_term_ms_overlap": ov,
                          "host_sync_ms_measured": SYNC_MS, "efficiency": eff}),
              flush=True)
        del ranks, comms
