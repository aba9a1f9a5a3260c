#!/usr/bin/env python3
"""A/B runs of bench.py under environment variants (kernel experiments):
  python tools/ab_bench.py --config c1 --runs 3 --var coop: --var nocoop:QSWG_COOP=0 -- --steps 40
Prints ms_per_step and e2e ms per run and variant (interleaved)."""
import argparse
import json
import os
import subprocess
import sys

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--runs", type=int, default=2)
ap.add_argument("--var", action="append", default=[], help="name:ENV=V,ENV2=V2")
ap.add_argument("rest", nargs="*")
a = ap.parse_args()
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for run in range(a.runs):
    for v in a.var:
        name, _, envs = v.partition(":")
        env = dict(os.environ)
        for kv in filter(None, envs.split(",")):
            k, _, val = kv.partition("=")
            env[k] = val
        out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", a.config,
                              "--no-cpu-baseline", "--no-superop", *a.rest],
                             env=env, capture_output=True, text=True)
        try:
            d = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
            print(json.dumps({"run": run, "variant": name, "ms_per_step": d["ms_per_step"],
                              "e2e_ms": d["e2e"]["ms_per_step"], "launches": d["gpu_launches"]}), flush=True)
        except Exception:
            print(json.dumps({"run": run, "variant": name, "error": out.stderr[-500:]}), flush=True)
