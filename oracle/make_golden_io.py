#!/usr/bin/env python3
"""Generate tests/golden/io/ — the output-path fixtures — from the UNMODIFIED
reference (oracle/_ref/libqswref.so via oracle/ref_io_harness.cpp).

TEST INFRASTRUCTURE ONLY.  Run here (where /root/reference exists):
    make -C oracle ref && python oracle/make_golden_io.py

  mtx/<case>.mtx            Matrix Market inputs (valid and malformed), our own
  mtx_expected.json         the reference parser's verdict per case: the CSR it
                            builds, or its error class code and message
  mtx/<case>.saved.mtx      save_matrix_market of every valid case
  container_ref.qswbox      a container written by the reference
  plot_<quantity>.txt       the reference's emit_plot_data of it
  graphs/*.mtx, runs.json   run() inputs (seeded graphs) and configs
  run_<name>.qswbox         the reference's run() output per config
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.ref_io import RefIo  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "io")
BANNER = "%%MatrixMarket matrix coordinate real general\n"

MTX_CASES = {
    # valid
    "cycle8": BANNER + "8 8 16\n" + "".join(f"{(i + 1) % 8 + 1} {i + 1} 1\n{i + 1} {(i + 1) % 8 + 1} 1\n"
                                            for i in range(8)),
    "path_symmetric_integer": "%%MatrixMarket matrix coordinate integer symmetric\n% a path\n4 4 3\n2 1 1\n3 2 2\n4 3 3\n",
    "comments_blank_upper": "%%MatrixMarket MATRIX Coordinate REAL General\n%\n% comment\n\n   \n5 5 4\n"
                            "% inside\n2 1 0.25\n\n3 1 1.5e-3\n%x\n1 5 7\n4 2 0.125\n",
    "empty_graph": BANNER + "3 3 0\n",
    "trailing_lines": BANNER + "3 3 2\n2 1 1.0\n3 2 2.0\n1 3 9.0\nnot an entry\n",
    "extra_tokens": BANNER + "3 3 2\n2 1 0.5 extra\n1 3 0.75 0\n",
    "weights_17_digits": BANNER + "4 4 4\n2 1 0.10000000000000001\n3 2 0.33333333333333331\n"
                          "4 3 1.2345678901234567e-05\n1 4 123456789.12345679\n",
    # malformed
    "empty_stream": "",
    "bad_banner": "%MatrixMarket matrix coordinate real general\n3 3 0\n",
    "array_format": "%%MatrixMarket matrix array real general\n3 3\n",
    "complex_field": "%%MatrixMarket matrix coordinate complex general\n3 3 0\n",
    "pattern_field": "%%MatrixMarket matrix coordinate pattern general\n3 3 0\n",
    "hermitian": "%%MatrixMarket matrix coordinate real hermitian\n3 3 0\n",
    "size_two_numbers": BANNER + "3 3\n",
    "size_negative": BANNER + "3 3 -1\n",
    "not_square": BANNER + "3 4 1\n2 1 1\n",
    "truncated": BANNER + "3 3 3\n2 1 1\n3 2 1\n",
    "malformed_entry": BANNER + "3 3 1\n1 x 2\n",
    "index_out_of_bounds": BANNER + "3 3 1\n4 1 1.0\n",
    "index_zero": BANNER + "3 3 1\n0 1 1.0\n",
    "self_loop": BANNER + "3 3 1\n2 2 1.0\n",
    "negative_weight": BANNER + "3 3 1\n1 2 -0.5\n",
    "zero_weight": BANNER + "3 3 1\n1 2 0\n",
    "duplicate": BANNER + "3 3 2\n1 2 1\n1 2 2\n",
    "symmetric_duplicate": "%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 1.0\n1 2 1.0\n",
    "only_comments_newline": BANNER + "% nothing\n%\n",
    "only_comments_no_newline": BANNER + "% nothing",
}


def mtx_text(n, arcs):
    """arcs: (i, j, w) = arc j -> i, 0-based."""
    return BANNER + f"{n} {n} {len(arcs)}\n" + "".join(f"{i + 1} {j + 1} {w!r}\n" for i, j, w in arcs)


def graphs():
    rng = np.random.default_rng(20030245)
    out = {"cycle8": mtx_text(8, [(a, b, 1.0) for i in range(8) for a, b in ((i, (i + 1) % 8), ((i + 1) % 8, i))])}
    arcs = []
    for j in range(6):
        for i in range(6):
            if i != j and rng.random() < 0.35:
                arcs.append((i, j, float(np.round(0.1 + rng.random(), 6))))
    out["digraph6"] = mtx_text(6, arcs)
    tor = []
    for y in range(3):
        for x in range(3):
            v = 3 * y + x
            for u in (3 * y + (x + 1) % 3, 3 * ((y + 1) % 3) + x):
                tor += [(u, v, 1.0), (v, u, 1.0)]
    out["torus3x3"] = mtx_text(9, tor)
    out["walkthrough"] = mtx_text(3, [(2, 0, 1.0), (2, 1, 1.0)])  # paper walkthrough: 1 -> 3 <- 2
    er = set()
    while len(er) < 16:
        a, b = rng.integers(0, 10, 2)
        if a != b:
            er.add((int(min(a, b)), int(max(a, b))))
    out["er10"] = mtx_text(10, [(a, b, 1.0) for a, b in sorted(er)] + [(b, a, 1.0) for a, b in sorted(er)])
    return out


def runs():
    g = "tests/golden/io/graphs/"
    return {
        "local_series": dict(graph_path=g + "cycle8.mtx", walk_kind="local", omega=0.5, gamma=1.0, is_series=True,
                             t1=0.0, tq=5.0, steps=10, initial_kind="vertex", initial_vertex=0,
                             out_populations=True, out_full_rho=True, out_coherence_norm=True),
        "local_src_snk": dict(graph_path=g + "digraph6.mtx", walk_kind="local", omega=0.3, gamma=1.0, is_series=True,
                              t1=0.5, tq=4.5, steps=8, initial_kind="mixed", sources=[[0, 0.7]], sinks=[[5, 0.9]],
                              out_populations=True, out_full_rho=False, out_coherence_norm=True),
        "global_step_file": dict(graph_path=g + "torus3x3.mtx", walk_kind="global", omega=0.1, gamma=1.0,
                                 is_series=False, t=2.0, initial_kind="file",
                                 initial_file="tests/golden/io/graphs/torus3x3.prob",
                                 out_populations=True, out_full_rho=True, out_coherence_norm=True),
        "nm_series": dict(graph_path=g + "walkthrough.mtx", walk_kind="nm_global", omega=0.5, gamma=1.0,
                          is_series=True, t1=0.0, tq=4.0, steps=4, initial_kind="vertex", initial_vertex=0,
                          out_populations=True, out_full_rho=True, out_coherence_norm=True),
        "global_series_gamma": dict(graph_path=g + "er10.mtx", walk_kind="global", omega=0.9, gamma=0.5,
                                    is_series=True, t1=0.0, tq=3.0, steps=6, initial_kind="mixed",
                                    out_populations=True, out_full_rho=False, out_coherence_norm=False),
        "local_step_pops_only": dict(graph_path=g + "digraph6.mtx", walk_kind="local", omega=1.0, gamma=2.0,
                                     is_series=False, t=1.5, initial_kind="vertex", initial_vertex=3,
                                     out_populations=True),
    }


def main():
    ref = RefIo()
    os.chdir(ROOT)
    os.makedirs(os.path.join(OUT, "mtx"), exist_ok=True)
    os.makedirs(os.path.join(OUT, "graphs"), exist_ok=True)
    expected = {}
    for name, text in MTX_CASES.items():
        path = os.path.join(OUT, "mtx", name + ".mtx")
        with open(path, "w") as f:
            f.write(text)
        rc, res = ref.parse_mtx(text.encode())
        if rc:
            expected[name] = {"code": rc, "message": res}
        else:
            ip, ix, dv = res
            expected[name] = {"code": 0, "indptr": ip.tolist(), "indices": ix.tolist(),
                              "re": dv.real.tolist(), "im": dv.imag.tolist()}
            ref.save_mtx(text.encode(), os.path.join(OUT, "mtx", name + ".saved.mtx"))
    with open(os.path.join(OUT, "mtx_expected.json"), "w") as f:
        json.dump(expected, f, indent=1)

    arrays = {"times": np.linspace(0.0, 1.0, 5), "populations": np.arange(15.0).reshape(5, 3) / 7.0,
              "scalar": np.array(3.25), "empty": np.zeros((0, 4)), "cube": np.arange(24.0).reshape(2, 3, 4) - 0.5}
    rc, msg = ref.write_container(os.path.join(OUT, "container_ref.qswbox"),
                                  "qsw_version = 0.1.0\nnote = ünïcode ok\n", arrays)
    assert rc == 0, msg
    for q in ("populations", "times", "scalar", "cube"):
        rc, msg = ref.plot_data(os.path.join(OUT, "container_ref.qswbox"), q, os.path.join(OUT, f"plot_{q}.txt"))
        assert rc == 0, msg

    for name, text in graphs().items():
        with open(os.path.join(OUT, "graphs", name + ".mtx"), "w") as f:
            f.write(text)
    with open(os.path.join(OUT, "graphs", "torus3x3.prob"), "w") as f:
        f.write("0.5 0.25\n0.25\n0 0 0 0 0 0\n")
    cfgs = runs()
    with open(os.path.join(OUT, "runs.json"), "w") as f:
        json.dump(cfgs, f, indent=1)
    for name, cfg in cfgs.items():
        rc, msg = ref.run(cfg, os.path.join(OUT, f"run_{name}.qswbox"))
        assert rc == 0, (name, msg)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
