"""The compiled C++ consumer of the C ABI: tests/cpp/facade_test.cpp through
the RAII facade include/qswg/qsw_gpu.hpp (WalkSystem / step / series in the
reference's own language, walk.hpp:39-84, expm.hpp:51-63), linked against
libqswg.so exactly as INTEGRATION.md's glue would be.

* CPU: the program compiles and links, and its host-only checks pass —
  sparse round trip, graph -> operator helpers, and the reference's
  exception types rethrown from the C codes (std::out_of_range,
  std::invalid_argument) before any device is touched.
* GPU: golden cases written to disk, evolved by the C++ program, compared with
  the reference-generated fixtures (populations at every output <= 1e-10,
  identical SpMV counts, step(tq) == the series' last output)."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, Case

CPP = os.path.join(ROOT, "tests", "cpp")
BIN = os.path.join(CPP, "build", "facade_test")


def build():
    subprocess.run(["make", "-s", "-C", CPP], check=True, capture_output=True, text=True)
    assert os.path.exists(BIN)


def test_facade_compiles_and_maps_reference_errors():
    build()
    r = subprocess.run([BIN, "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "0 failure(s)" in r.stderr


def write_matrix(f, name, m):
    rows = np.repeat(np.arange(m.rows), np.diff(m.indptr))
    f.write(f"matrix {name} {m.rows} {m.cols} {len(m.data)}\n")
    for r, c, v in zip(rows, m.indices, m.data):
        f.write(f"{int(r)} {int(c)} {float(v.real)!r} {float(v.imag)!r}\n")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1_n64", "c2_n36", "c5_n64", "gqsw_multi_rot"])
def test_facade_series_matches_reference(name, tmp_path):
    build()
    c = Case(name)
    assert not c.sources and not c.sinks
    t1, tq, q = c.series
    with open(tmp_path / "input.txt", "w") as f:
        f.write(f"kind {c.kind}\nomega {float(c.omega)!r}\nops {c.n_ops}\nrot {int(bool(c.has_h_rot))}\n")
        write_matrix(f, "h", c.h)
        for k, m in enumerate(c.ops):
            write_matrix(f, f"op{k}", m)
        if c.has_h_rot:
            write_matrix(f, "hrot", c.h_rot)
        f.write(f"rho0 {c.n} " + " ".join(repr(float(x)) for x in c.rho0) + "\n")
        f.write(f"times {float(t1)!r} {float(tq)!r} {int(q)}\n")
    r = subprocess.run([BIN, "series", str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = (tmp_path / "output.txt").read_text().split("\n")
    spmvs = int(lines[0].split()[1])
    pops = np.array([[float(x) for x in ln.split()] for ln in lines[1:int(q) + 2]])
    final = np.array([float(x) for x in lines[int(q) + 2].split()[1:]])
    step = np.array([float(x) for x in lines[int(q) + 3].split()[1:]])
    assert np.abs(pops - c.z["series_pops"]).max() <= 1e-10
    assert spmvs == c.series_spmvs
    assert np.array_equal(final, pops[-1])
    assert np.abs(step - pops[-1]).max() <= 1e-10
