#!/usr/bin/env python3
"""Benchmark of the expmv hot path (BASELINE.json metric).

A "step" is one full `series` call — the reference's time-series driver
(expm.cpp:214-325) — over the BASELINE workload: by default config 2, G-QSW
on the 32x32 periodic torus (dim 1,048,576, 42,991,616 nnz), 101 output
times on [0, 20], populations extracted on the device at every output.

  value     output steps/s with rho(0) and the superoperator resident in HBM
            (assembly and norms excluded; reported separately)
  e2e       the same through the public C ABI with host buffers: upload of
            vec(rho(0)) from pinned memory + series + download of all
            populations, every step
  roofline  the fused series-term kernel (SpMV + axpys + norms): algorithmic
            bytes per launch / mean launch time (CUDA events, same stream)

Multi-GPU: one process per GPU under torchrun; the superoperator is
row-sharded (strong scaling of one series).  `--impl reference` times the
unmodified reference library (oracle/_ref) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "superop SpMV HBM GB/s (% roofline); expmv steps/sec at 1/2/4/8 B200 vs CPU ref"
UNIT = "output steps/s"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled during the timed
    region through NVML in this process (one sample at entry, one at exit and
    every `period` s in between).  nvidia-smi was used before: its start-up and
    each of its polls stalled this GPU's work for tens of ms (c1, 7 ms region:
    1.4 -> 15-21 ms/step), so the in-process NVML queries replace it."""

    def __init__(self, index, period=0.25, enabled=True):
        self.index = index
        self.enabled = enabled
        self.period = period
        self.rows = []
        self.nvml = None

    def _sample(self):
        n, h = self.nvml, self.h
        try:
            sm = n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM)
            mx = n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM)
            r = n.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            return
        flags = [bool(r & getattr(n, name)) for name in
                 ("nvmlClocksEventReasonHwSlowdown", "nvmlClocksEventReasonHwThermalSlowdown",
                  "nvmlClocksEventReasonSwThermalSlowdown", "nvmlClocksEventReasonSwPowerCap")]
        self.rows.append([str(sm), str(mx), "", "", *["Active" if f else "Not Active" for f in flags]])

    def _loop(self):
        # one sample shortly after the region starts (short regions still get one
        # under load), then one every `period` s: each NVML query can stall the
        # GPU's work for milliseconds (20 series of 29 ms measured 28.8 ms per
        # series with ~2 samples in the region, 30-32 ms with ~6), so few of them
        wait = 0.05
        while not self.stop.wait(wait):
            self._sample()
            wait = self.period

    def prepare(self):
        """NVML start-up, long before the timed region: on a fresh box the first
        nvmlInit of a process disturbed the GPU for the next second or so (the
        first bench run of a box measured 40-45 ms per c2 series in the region
        that followed it, 29 ms in every later run and in the region before it)."""
        if not self.enabled or self.nvml is not None:
            return
        try:
            import pynvml
            pynvml.nvmlInit()
            try:  # the NVML device behind this CUDA ordinal (CUDA_VISIBLE_DEVICES may remap)
                import torch
                pr = torch.cuda.get_device_properties(self.index)
                bus = "%08X:%02X:%02X.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = pynvml
            self._sample()
            self.rows.clear()
        except Exception:
            self.nvml = None
            self.enabled = False

    def __enter__(self):
        if not self.enabled:
            return self
        self.prepare()
        if self.nvml is None:
            return self
        try:
            self._sample()
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._loop, daemon=True)
            self.thread.start()
        except Exception:
            self.nvml = None
        return self

    def __exit__(self, *a):
        if self.nvml is not None:
            self.stop.set()
            self.thread.join(timeout=5)
            self._sample()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[4:8]) if v.strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def l2_for(config, fmt):
    """L2 bytes requested by the SMs per launch of the dominant kernel (ncu)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(f"{config}:{fmt}", {}).get("l2_bytes_per_launch")
    except Exception:
        return None


def traffic_for(config, fmt):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel from the committed ncu --set full capture (profiles/traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        e = t.get(f"{config}:{fmt}")
        return e["dram_bytes_per_launch"] if e else None
    except Exception:
        return None


def workload_desc(w):
    """The workload, identical in both arms (implementation details go to
    `impl_config`)."""
    return {"workload": f"{w.name}: {'L-QSW' if w.kind == 'local' else 'G-QSW'} n={w.n} omega={w.omega} "
                        f"t=[{w.t1},{w.tq}] outputs={w.steps + 1}",
            "dim": w.dim, "outputs": w.steps + 1, "omega": w.omega, "kind": w.kind, "seed": w.seed,
            "l2_policy": "no flush: one step (a whole series) streams far more than the 126 MB L2 "
                         "(term ring, running sums, stored superoperator), so no input survives in L2 "
                         "from one step to the next"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------ reference arm
def run_reference(args, w, rank, world):
    if rank != 0:
        return 0
    from oracle.oracle import Oracle, rho0_vec
    o = Oracle("reference")
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    h = o.build(w, workers=cores)
    build_s = time.perf_counter() - t0
    v0 = rho0_vec(w.n, w.rho0)
    for _ in range(args.warmup):
        h.series(v0, w.t1, w.tq, w.steps, states=False, pops=True)
    times, spmvs = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, _, nsp = h.series(v0, w.t1, w.tq, w.steps, states=False, pops=True)
        times.append(time.perf_counter() - t0)
        spmvs = nsp
    sec = float(np.mean(times))
    value = w.steps / sec
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "complex128",
            "data": "synthetic (seeded, BASELINE.json config)",
            "config": workload_desc(w),
            "impl_config": {"parallelism": f"{cores} host threads (reference WorkerPool)",
                            "build_norms_s": build_s, "spmvs_per_step": spmvs,
                            "library": os.path.relpath(o.path, ROOT)},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "cpu_model": cpu_model(),
                             "sample": f"full {w.name} series ({w.steps + 1} outputs) per step, "
                                       f"n_workers={cores}"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(w):
    """The reference on this box's host cores, one bounded sample (one full
    series of the same workload)."""
    from oracle.oracle import Oracle, rho0_vec
    try:
        o = Oracle("reference")
        kind = "reference"
    except FileNotFoundError:
        o = Oracle("port")
        kind = "port"
    cores = (os.cpu_count() or 1) if kind == "reference" else 1
    h = o.build(w, workers=cores) if kind == "reference" else o.build(w)
    t0 = time.perf_counter()
    _, _, nsp = h.series(rho0_vec(w.n, w.rho0), w.t1, w.tq, w.steps, states=False, pops=True)
    sec = time.perf_counter() - t0
    return {"value": w.steps / sec, "unit": UNIT, "cores": cores, "kind": kind, "cpu_model": cpu_model(),
            "sample": f"one full {w.name} series ({w.steps + 1} outputs, {nsp} SpMVs) in {sec:.2f} s; "
                      f"library {os.path.relpath(o.path, ROOT)}"}


# ----------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="qswg", choices=["qswg", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--size", type=int, default=None, help="shrink the graph (debug only)")
    ap.add_argument("--group", type=int, default=0)
    ap.add_argument("--format", default="auto", choices=["auto", "kron", "sell", "csr"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true", help="debug: no clock sampling (its NVML queries)")
    ap.add_argument("--no-superop", action="store_true", help="skip the stored-superoperator comparison")
    ap.add_argument("--configs", default="c3,c4,c5",
                    help="other BASELINE configs measured on one GPU after the headline ('' to skip)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    from paper_2003_02450_b200 import graphs
    w = graphs.config(args.config, size=args.size)

    if args.impl == "reference":
        return run_reference(args, w, rank, world)

    import torch
    from paper_2003_02450_b200 import api

    torch.cuda.set_device(local_rank)
    clocks = ClockSampler(local_rank, enabled=not args.no_clocks)
    clocks.prepare()
    comm = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        comm = api.Comm.create(rank, world, local_rank)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def build(fmt):
        if w.kind == "local":
            return api.build_local(w.omega, w.h, w.ops[0], device=local_rank, group=args.group, comm=comm,
                                   format=fmt)
        return api.build_global(w.omega, w.h, w.ops, device=local_rank, group=args.group, comm=comm, format=fmt)

    t0 = time.perf_counter()
    l = build(args.format)
    barrier()
    build_s = time.perf_counter() - t0

    stream = torch.cuda.ExternalStream(l.stream(), device=torch.device("cuda", local_rank))
    v = l.state().from_probabilities(w.rho0)

    # ---- end to end through the public API, host buffers ----
    # (measured before the device-resident region: the clock sampler's start
    # and stop around that region perturb the GPU for a while).  Host buffers
    # are page-locked by the library (qswg_host_alloc), so every step's H2D of
    # vec(rho(0)) and D2H of the populations are direct DMA transfers.
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    vec_host = api.pinned_empty(l.rows, np.complex128)
    vec_host[:] = 0
    diag = np.arange(w.n) * (w.n + 1) - l.row0
    own = (diag >= 0) & (diag < l.rows)
    vec_host[diag[own]] = w.rho0[own]
    pops_host = api.pinned_empty((w.steps + 1, w.n), np.float64)
    e2e_state = l.state()
    impl_rows = l.rows
    for _ in range(args.warmup):  # the second identical call captures the series graph: keep it out of the timing
        e2e_state.upload_local(vec_host)
        api.series(l, e2e_state, w.t1, w.tq, w.steps, pops_out=pops_host)
    barrier()
    host_parts = {"upload_ms": [], "series_call_ms": [], "series_device_ms": []}
    ev0.record(stream)
    for _ in range(args.steps):
        h0 = time.perf_counter()
        e2e_state.upload_local(vec_host)                                        # H2D of vec(rho(0))
        h1 = time.perf_counter()
        r_e2e = api.series(l, e2e_state, w.t1, w.tq, w.steps, pops_out=pops_host)  # + D2H populations
        h2 = time.perf_counter()
        host_parts["upload_ms"].append(1e3 * (h1 - h0))
        host_parts["series_call_ms"].append(1e3 * (h2 - h1))
        host_parts["series_device_ms"].append(float(r_e2e.info.device_ms))
    ev1.record(stream)
    barrier()
    e2e_ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_parts = {k: float(np.median(v)) for k, v in host_parts.items()}
    e2e_parts["note"] = ("host wall time per call (median): upload = H2D + the one-time Hermiticity check of the "
                         "uploaded state (one synchronisation); series call = enqueue/graph replay + D2H of the "
                         "populations + one synchronisation; series_device_ms = CUDA events around the series")

    # ---- device-resident timed region ----
    for _ in range(args.warmup):  # (re-)captures this call's series graph
        r = api.series(l, v, w.t1, w.tq, w.steps, populations=False)
    with clocks:
        barrier()
        ev0.record(stream)
        launches = 0
        step_device_ms = []  # CUDA-event time of every series (library stream): shows outlier steps
        for _ in range(args.steps):
            r = api.series(l, v, w.t1, w.tq, w.steps, populations=False)
            launches += r.info.launches
            step_device_ms.append(float(r.info.device_ms))
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    info = r.info
    value = w.steps / (ms_per_step / 1e3)

    # ---- roofline of the dominant kernel (the series term kernel) ----
    d_active = int(info.d) if info.path == 2 else 1
    peak, peak_src = load_peaks()
    n_lind = len(w.ops) if w.kind == "global" else 0
    parts = l.time_series_parts(iters=20, count=d_active)
    term_ms = parts["term"]
    achieved = term_bytes(l, n_lind) / (term_ms * 1e-3) / 1e9
    share = info.spmvs * term_ms / ms_per_step
    kernel_name = {"kron": "kron_series_term_kernel", "sell": "sell_series_term_kernel",
                   "csr": "series_term_kernel"}[l.format]
    parts_line = {"prepare_ms": parts["prepare"], "term_ms": parts["term"], "flush_ms": parts["flush"],
                  "prepare_kernels": ("kron_w_kernel" + ((" (W_k and its row-major copy; V_k = conj Wt_k)" if world == 1
                                                          else " + kron_v_kernel") if l.info.kron_factored else ""))
                  if l.format == "kron" else None,
                  "prepare_gbs": prepare_bytes(l, n_lind) / (parts["prepare"] * 1e-3) / 1e9 if parts["prepare"] > 0 else None,
                  "flush_kernel": "series_flush_kernel (amortised over the term ring)",
                  "count": d_active}
    impl_config = {
        "parallelism": f"row-block x{world}" if world > 1 else "1 GPU", "nnz": int(l.nnz),
        "format": l.format, "kron_factored": bool(l.info.kron_factored), "kron_ell": bool(l.info.kron_ell),
        "build_norms_s": build_s, "one_norms": l.one_norms().tolist(), "group": int(l.group),
        "plan": {"path": int(info.path), "span": [int(info.span_m_star), int(info.span_s)],
                 "d": int(info.d), "n_super": int(info.n_super), "remainder": int(info.remainder),
                 "sub_m_star": int(info.sub_m_star)},
        "spmvs_per_step": int(info.spmvs)}
    roofline = {"bound": "l2" if l.format == "kron" else "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic_for(w.name, l.format), "kernel": kernel_name,
                "format": l.format, "kron_factored": bool(l.info.kron_factored), "kron_ell": bool(l.info.kron_ell),
                "bytes_per_launch": term_bytes(l, n_lind), "ms_per_launch": term_ms,
                "peak_source": peak_src, "share_of_step": share, "parts": parts_line}
    if l.format == "kron":
        l2b = l2_for(w.name, l.format)
        roofline["bound_note"] = (
            "matrix-free (KRON) term: its algorithmic HBM bytes (x read, K_p written, W_k read) are small; "
            "the bound is the SM<-L2 traffic of its ~20 operand-weighted 512-byte segment gathers per element "
            "and the dependent index -> gather -> FMA chains (DESIGN.md section 3); achieved/frac are reported "
            "against HBM as the contract asks.  The stored-superoperator kernel (superop_spmv) is the HBM-bound one.")
        if l2b:
            roofline["l2"] = {"bytes_per_launch": l2b, "achieved_gbs": l2b / (term_ms * 1e-3) / 1e9,
                              "source": "ncu lts__t_sectors_srcunit_tex (profiles/traffic.json)"}

    # ---- the stored-superoperator SpMV (BASELINE's "superop SpMV HBM GB/s") ----
    superop = None
    if l.format == "kron" and world == 1 and not args.no_superop:
        del e2e_state, v
        lk = l
        l = None
        ls = build("sell")
        if ls.padding > 1.3:
            del ls
            ls = build("csr")
        sp = ls.time_series_parts(iters=20, count=d_active)
        s_ms = sp["term"]
        vs = ls.state().from_probabilities(w.rho0)
        api.series(ls, vs, w.t1, w.tq, w.steps, populations=False)  # warm-up
        rs = min((api.series(ls, vs, w.t1, w.tq, w.steps, populations=False) for _ in range(3)),
                 key=lambda r: r.info.device_ms)  # best of 3 (a secondary number; shared boxes are noisy)
        sb = term_bytes(ls, n_lind)
        superop = {"format": ls.format, "kernel": "sell_series_term_kernel" if ls.format == "sell" else
                   "series_term_kernel", "bytes_per_launch": sb, "ms_per_launch": s_ms,
                   "achieved_gbs": sb / (s_ms * 1e-3) / 1e9, "frac": sb / (s_ms * 1e-3) / 1e9 / peak,
                   "flush_ms": sp["flush"],
                   "series_ms": float(rs.info.device_ms), "output_steps_per_s": w.steps / (rs.info.device_ms / 1e3),
                   "bytes_note": "20 B/nnz + 8 B/row + x read + K_p written (SURVEY.md 8(d))"}
        del ls, vs
        l = lk

    # ---- the other BASELINE configs on one GPU (assembly excluded) ----
    configs = None
    if world == 1 and args.configs:
        del l
        l = None
        configs = [config_block(name, peak) for name in args.configs.split(",") if name]

    if rank != 0:
        return 0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "complex128",
        "data": "synthetic (seeded graph of BASELINE.json config; no public dataset exists for this path)",
        "config": workload_desc(w),
        "impl_config": impl_config,
        "roofline": roofline,
        "superop_spmv": superop,
        "configs": configs,
        "e2e": {"value": w.steps / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 16 * int(impl_rows),
                "d2h_bytes_per_step": 8 * (w.steps + 1) * w.n, "ms_per_step": e2e_ms, "h2d_pinned": True,
                "parts": e2e_parts},
        "gpu_launches": int(launches),
        "step_device_ms": {"min": min(step_device_ms), "median": float(np.median(step_device_ms)),
                           "max": max(step_device_ms),
                           "note": "CUDA-event time of each timed series; ms_per_step is their mean plus the host "
                                   "gaps between calls.  On the shared boxes single series intermittently run "
                                   "28.5 -> 40 ms on the device with unchanged clocks (DESIGN.md section 6)"},
        "clocks": clocks.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w)
    print(json.dumps(line), flush=True)
    return 0


def term_bytes(lv, n_lind):
    """Algorithmic HBM bytes of one term-kernel launch: the
    input x read once, K_p written once, plus the stored superoperator
    (20 B/nnz + 8 B/row) or, matrix-free, the W_k (and V_k) work vectors
    read once."""
    vec = 16 * lv.dim + 16 * lv.rows
    if lv.format == "kron":  # W_k and/or its row-major copy, as the kernels read them
        return vec + 16 * n_lind * lv.dim * int(lv.info.kron_term_vectors)
    return vec + 20 * int(lv.info.nnz_local) + 8 * (lv.rows + 1)


def prepare_bytes(lv, n_lind):
    """Kron prepare kernels: x read once per Lindblad term, W_k and/or its
    row-major copy written."""
    if lv.format != "kron":
        return 0
    return n_lind * (1 + int(lv.info.kron_term_vectors)) * 16 * lv.dim


def config_block(name, peak):
    """One BASELINE config on one GPU: the default (matrix-free) series with
    assembly excluded — series time, SpMVs, plan, the dominant kernel's
    algorithmic bytes and fraction — and the stored-superoperator SpMV
    (SELL-C-sigma, column panels where x exceeds L2) with its HBM fraction."""
    from paper_2003_02450_b200 import api, graphs
    w = graphs.config(name)
    n_lind = len(w.ops) if w.kind == "global" else 0

    def build(fmt):
        if w.kind == "local":
            return api.build_local(w.omega, w.h, w.ops[0], format=fmt)
        return api.build_global(w.omega, w.h, w.ops, format=fmt)

    out = {"config": name, "workload": workload_desc(w)["workload"], "dim": int(w.dim)}
    t0 = time.perf_counter()
    l = build("auto")
    out["build_s"] = time.perf_counter() - t0
    out["nnz"] = int(l.nnz)
    out["format"] = l.format
    v = l.state().from_probabilities(w.rho0)
    # warm-up: allocates the workspace (term ring, sums) with a short series of the same plan shape
    api.series(l, v, w.t1, w.t1 + (w.tq - w.t1) / w.steps * 2, 2, populations=False)
    reps = 1 if w.dim > 100_000_000 else 3  # best of 3 (c5: one 12 s series)
    best = None
    for _ in range(reps):
        r = api.series(l, v, w.t1, w.tq, w.steps, populations=False)
        best = r.info.device_ms if best is None else min(best, r.info.device_ms)
    info = r.info
    out.update({"series_ms": float(best), "output_steps_per_s": w.steps / (best / 1e3), "spmvs": int(info.spmvs),
                "plan": [int(info.path), int(info.span_m_star), int(info.span_s), int(info.d), int(info.sub_m_star)],
                "trace_err": float(abs(r.populations[-1].sum() - 1)) if r.populations is not None else None})
    d_active = int(info.d) if info.path == 2 else 1
    parts = l.time_series_parts(iters=10 if w.dim > 100_000_000 else 20, count=d_active)
    tb = term_bytes(l, n_lind)
    out["dominant"] = {"kernel": "kron_series_term_kernel" if l.format == "kron" else "sell_series_term_kernel",
                       "bytes_per_launch": tb, "ms_per_launch": parts["term"],
                       "achieved_gbs": tb / (parts["term"] * 1e-3) / 1e9,
                       "frac": tb / (parts["term"] * 1e-3) / 1e9 / peak,
                       "bound": "l2" if l.format == "kron" else "hbm",
                       "prepare_ms": parts["prepare"], "flush_ms": parts["flush"],
                       "note": ("path 1 (c3): its series runs kron_step_term_kernel, the same tiles plus "
                                "the running-sum epilogue" if info.path == 1 else None)}
    del l, v
    ls = build("sell")
    sp = ls.time_series_parts(iters=5 if w.dim > 10_000_000 else 20, count=d_active)
    sb = term_bytes(ls, n_lind)
    out["superop_spmv"] = {"format": ls.format, "panels": int(ls.info.sell_panels), "padding": float(ls.padding),
                           "bytes_per_launch": sb, "ms_per_launch": sp["term"],
                           "achieved_gbs": sb / (sp["term"] * 1e-3) / 1e9,
                           "frac": sb / (sp["term"] * 1e-3) / 1e9 / peak}
    del ls
    return out


if __name__ == "__main__":
    sys.exit(main())
