#!/usr/bin/env python3
"""Small runs of every round-2 kernel path (a quick check; also the command for compute-sanitizer
where one is available): the streamed SELL kernels, the fused
B (x) I windows, the register path, and the staged KRON tiles."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02450_b200 import api, graphs  # noqa: E402


def run(cfg, size, fmt, steps, **env):
    for k, v in env.items():
        os.environ[k] = v
    w = graphs.config(cfg, size=size)
    l = (api.build_local(w.omega, w.h, w.ops[0], format=fmt) if w.kind == "local"
         else api.build_global(w.omega, w.h, w.ops, format=fmt))
    r = api.series(l, l.state().from_probabilities(w.rho0), w.t1, w.tq, steps)
    x = np.ones(w.dim, complex)
    l.spmv(x)
    st, _ = api.step(l, l.state().from_probabilities(w.rho0), 0.5)
    print(cfg, size, fmt, env, "spmvs", r.info.spmvs, "trace", float(r.populations[-1].sum()), flush=True)
    for k in env:
        os.environ.pop(k)


run("c5", 4, "sell", 3)                                   # streamed (short regular rows)
run("c2", 8, "sell", 3)                                   # register path (long regular rows)
run("c3", 96, "sell", 2, QSWG_SELL_FUSE="1")              # fused windows, several windows
run("c4", 96, "sell", 2, QSWG_SELL_PANELS="3", QSWG_SELL_FUSE="1")  # fused windows + column panels
run("c4", 96, "sell", 2, QSWG_SELL_PANELS="2", QSWG_SELL_FUSE="0")  # sorted register path + panels
run("c2", 8, "kron", 3, QSWG_KRON_STAGED="1")             # staged tiles, factored
run("c5", 4, "kron", 3, QSWG_KRON_STAGED="1")             # staged tiles, L-QSW
run("c2", 8, "kron", 3)                                   # default Hermitian tiles
