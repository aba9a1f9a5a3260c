import json, os, sys
sys.path.insert(0, os.getcwd())
from paper_2003_02450_b200 import api, graphs
for name in ["c3", "c4"]:
    w = graphs.config(name)
    for fmt in ["sell", "csr"]:
        l = (api.build_local(w.omega, w.h, w.ops[0], format=fmt) if w.kind == "local" else api.build_global(w.omega, w.h, w.ops, format=fmt))
        p = l.time_series_parts(10, 1)
        nnz = int(l.info.nnz_local)
        b = 20 * nnz + 8 * (l.rows + 1) + 32 * l.dim
        print(json.dumps({"config": name, "format": l.format, "padding": l.padding, "term_ms": p["term"], "gbs": b / (p["term"] * 1e-3) / 1e9}), flush=True)
        del l
