"""The data formats either side of the hot path:
Matrix Market graphs, the QSWBOX result container, plot data and run().

Pinned against the unmodified reference through tests/golden/io/ (written by
oracle/make_golden_io.py from oracle/_ref) and, where oracle/_ref is built,
live against it.  The CPU tests exercise libqswg's host code (parser,
container writer/reader); the GPU tests run whole walks through run() on the
device and compare the containers with the reference's run() output.
"""
import json
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, has_gpu

api = pytest.importorskip("paper_2003_02450_b200.api")
from paper_2003_02450_b200 import run as qrun  # noqa: E402

IO = os.path.join(GOLDEN, "io")
EXPECTED = json.load(open(os.path.join(IO, "mtx_expected.json")))
RUNS = json.load(open(os.path.join(IO, "runs.json")))
EXC = {1: api.InvalidArgument, 2: api.OutOfRange, 10: api.FileFormatError, 11: api.IoError}


def mtx(name):
    with open(os.path.join(IO, "mtx", name + ".mtx"), "rb") as f:
        return f.read()


def ref_io():
    from oracle import ref_io
    if not ref_io.available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    return ref_io.RefIo()


# ----------------------------------------------------------- Matrix Market
@pytest.mark.parametrize("name", sorted(EXPECTED))
def test_matrix_market_parse_matches_reference(name):
    exp = EXPECTED[name]
    if exp["code"]:
        with pytest.raises(EXC[exp["code"]]) as ei:
            api.parse_matrix_market(mtx(name))
        assert str(ei.value) == exp["message"]
        return
    c = api.parse_matrix_market(mtx(name)).to_csr()
    assert c.indptr.tolist() == exp["indptr"]
    assert c.indices.tolist() == exp["indices"]
    assert c.data.real.tolist() == exp["re"] and c.data.imag.tolist() == exp["im"]  # bit-identical


@pytest.mark.parametrize("name", sorted(k for k, v in EXPECTED.items() if v["code"] == 0))
def test_matrix_market_save_matches_reference(name, tmp_path):
    out = tmp_path / "g.mtx"
    api.save_matrix_market(api.parse_matrix_market(mtx(name)), out)
    with open(os.path.join(IO, "mtx", name + ".saved.mtx"), "rb") as f:
        assert out.read_bytes() == f.read()
    again = api.load_matrix_market(out).to_csr()  # save -> load is the identity
    first = api.parse_matrix_market(mtx(name)).to_csr()
    assert np.array_equal(again.indptr, first.indptr) and np.array_equal(again.indices, first.indices)
    assert np.array_equal(again.data, first.data)


def test_matrix_market_file_errors(tmp_path):
    missing = tmp_path / "nope.mtx"
    with pytest.raises(api.IoError, match="cannot open graph file"):
        api.load_matrix_market(missing)
    p = tmp_path / "loop.mtx"
    p.write_bytes(mtx("self_loop"))
    with pytest.raises(api.FileFormatError) as ei:  # run.cpp:19-23 wraps invalid_argument
        api.load_matrix_market(p)
    assert str(ei.value) == f"invalid graph file `{p}`: diagonal entry at vertex 2 violates the simple-graph requirement"
    p.write_bytes(mtx("bad_banner"))
    with pytest.raises(api.FileFormatError, match="^missing %%MatrixMarket banner$"):
        api.load_matrix_market(p)


def test_matrix_market_large_roundtrip(tmp_path):
    """A c2-sized graph (32x32 torus) through save -> load."""
    from paper_2003_02450_b200 import graphs
    g = api.SparseMatrix.of(graphs.torus2d(32))
    api.save_matrix_market(g, tmp_path / "t.mtx")
    a, b = g.to_csr(), api.load_matrix_market(tmp_path / "t.mtx").to_csr()
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.data, b.data)


def test_matrix_market_live_reference_fuzz():
    """Random perturbations of valid files: same verdict and message as the reference."""
    ref = ref_io()
    rng = np.random.default_rng(7)
    base = [mtx(k) for k, v in sorted(EXPECTED.items()) if v["code"] == 0]
    for trial in range(300):
        b = bytearray(base[trial % len(base)])
        for _ in range(rng.integers(1, 4)):
            op = rng.integers(0, 3)
            pos = int(rng.integers(0, max(len(b), 1)))
            if op == 0 and b:
                del b[pos]
            elif op == 1:
                b.insert(pos, int(rng.choice(list(b" \n%-0123456789.eE"))))
            elif b:
                b[pos] = int(rng.choice(list(b" \n%-0123456789")))
        text = bytes(b)
        rc, res = ref.parse_mtx(text)
        if rc:
            with pytest.raises(EXC[rc]) as ei:
                api.parse_matrix_market(text)
            assert str(ei.value) == res, text
        else:
            c = api.parse_matrix_market(text).to_csr()
            assert np.array_equal(c.indptr, res[0]) and np.array_equal(c.indices, res[1]), text
            assert np.array_equal(c.data, res[2]), text


# ----------------------------------------------------------- QSWBOX
REF_ARRAYS = {"times": np.linspace(0.0, 1.0, 5), "populations": np.arange(15.0).reshape(5, 3) / 7.0,
              "scalar": np.array(3.25), "empty": np.zeros((0, 4)), "cube": np.arange(24.0).reshape(2, 3, 4) - 0.5}
REF_META = "qsw_version = 0.1.0\nnote = ünïcode ok\n"


def ref_container_bytes():
    with open(os.path.join(IO, "container_ref.qswbox"), "rb") as f:
        return f.read()


def test_container_bytes_identical_to_reference(tmp_path):
    api.ResultContainer(REF_META, REF_ARRAYS).write(tmp_path / "c.qswbox")
    assert (tmp_path / "c.qswbox").read_bytes() == ref_container_bytes()


def test_container_reads_reference_file():
    c = api.ResultContainer.read(os.path.join(IO, "container_ref.qswbox"))
    assert c.metadata == REF_META
    assert sorted(c.arrays) == sorted(REF_ARRAYS)
    for k, v in REF_ARRAYS.items():
        assert c.arrays[k].shape == v.shape and np.array_equal(c.arrays[k], v), k


def corrupt(kind, b):
    if kind == "short":
        return b[:11]
    if kind == "magic":
        return b"QSWBOY" + b[6:]
    if kind == "crc":
        return b[:20] + bytes([b[20] ^ 1]) + b[21:]
    if kind == "truncated":
        return b[:-9]
    raise ValueError(kind)


CORRUPT_MSG = {"short": "container file too short", "magic": "not a qsw container (bad magic bytes)",
               "crc": "container checksum mismatch (truncated or corrupted file)",
               "truncated": "container checksum mismatch (truncated or corrupted file)"}


@pytest.mark.parametrize("kind", sorted(CORRUPT_MSG))
def test_container_rejects_corrupt_files(kind, tmp_path):
    p = tmp_path / "bad.qswbox"
    p.write_bytes(corrupt(kind, ref_container_bytes()))
    with pytest.raises(api.FileFormatError) as ei:
        api.ResultContainer.read(p)
    assert str(ei.value) == CORRUPT_MSG[kind]


def _with_crc(body: bytes) -> bytes:
    import zlib
    return body + zlib.crc32(body).to_bytes(4, "little")  # zlib's CRC-32 is the container's


def test_container_structural_errors(tmp_path):
    body = ref_container_bytes()[:-4]
    p = tmp_path / "x.qswbox"
    p.write_bytes(_with_crc(body[:6] + (2).to_bytes(2, "little") + body[8:]))
    with pytest.raises(api.FileFormatError, match="^unsupported container version 2$"):
        api.ResultContainer.read(p)
    p.write_bytes(_with_crc(body + (50).to_bytes(4, "little") + b"ab"))
    with pytest.raises(api.FileFormatError, match="^truncated container section name$"):
        api.ResultContainer.read(p)
    p.write_bytes(_with_crc(body + (1).to_bytes(4, "little") + b"z" + (99).to_bytes(8, "little")))
    with pytest.raises(api.FileFormatError, match="^truncated container payload$"):
        api.ResultContainer.read(p)
    bad = (1).to_bytes(8, "little") + (3).to_bytes(8, "little") + np.zeros(2).tobytes()
    p.write_bytes(_with_crc(body + (1).to_bytes(4, "little") + b"z" + len(bad).to_bytes(8, "little") + bad))
    with pytest.raises(api.FileFormatError, match="^array section `z` has inconsistent dimensions$"):
        api.ResultContainer.read(p)


def test_container_live_reference_roundtrip(tmp_path):
    """Reference reader -> reference writer on our file gives our bytes back, and
    the reference rejects exactly the corrupt files we reject."""
    ref = ref_io()
    rng = np.random.default_rng(3)
    arrays = {f"a{k}": rng.standard_normal(rng.integers(0, 4, rng.integers(0, 3))) for k in range(6)}
    api.ResultContainer("meta\n" * 3, arrays).write(tmp_path / "ours.qswbox")
    assert ref.rewrite_container(str(tmp_path / "ours.qswbox"), str(tmp_path / "back.qswbox")) == (0, "")
    assert (tmp_path / "back.qswbox").read_bytes() == (tmp_path / "ours.qswbox").read_bytes()
    for kind in CORRUPT_MSG:
        (tmp_path / "bad.qswbox").write_bytes(corrupt(kind, ref_container_bytes()))
        assert ref.rewrite_container(str(tmp_path / "bad.qswbox"), str(tmp_path / "o.qswbox")) == (10, CORRUPT_MSG[kind])


def test_container_write_errors(tmp_path):
    with pytest.raises(api.IoError, match="for writing"):
        api.ResultContainer("", {}).write(tmp_path / "no" / "such" / "dir.qswbox")
    with pytest.raises(api.IoError):
        api.ResultContainer.read(tmp_path / "missing.qswbox")


@pytest.mark.parametrize("q", ["populations", "times", "scalar", "cube"])
def test_plot_data_matches_reference(q, tmp_path):
    c = api.ResultContainer.read(os.path.join(IO, "container_ref.qswbox"))
    c.emit_plot_data(q, tmp_path / "p.txt")
    with open(os.path.join(IO, f"plot_{q}.txt"), "rb") as f:
        assert (tmp_path / "p.txt").read_bytes() == f.read()


def test_plot_data_errors(tmp_path):
    c = api.ResultContainer("", {"x": np.ones(2)})
    with pytest.raises(ValueError, match="no quantity requested"):
        c.emit_plot_data("", tmp_path / "p.txt")
    with pytest.raises(ValueError, match="quantity `y` is not present in the container"):
        c.emit_plot_data("y", tmp_path / "p.txt")


# ----------------------------------------------------------- run()
def config(name, **over):
    cfg = dict(RUNS[name])
    cfg.update(over)
    cfg["sources"] = [tuple(s) for s in cfg.get("sources", [])]
    cfg["sinks"] = [tuple(s) for s in cfg.get("sinks", [])]
    return qrun.RunConfig(**cfg)


def test_run_config_validation(monkeypatch):
    monkeypatch.chdir(ROOT)
    cases = [(dict(graph_path=""), "no graph file given"),
             (dict(graph_path="nope.mtx"), "graph file `nope.mtx` does not exist"),
             (dict(omega=1.5), "omega must lie in [0, 1]"),
             (dict(gamma=0.0), "gamma must be positive"),
             (dict(workers=0), "workers must be at least 1"),
             (dict(tq=0.0), "series requires tq > t1"),
             (dict(steps=0), "series requires steps >= 1"),
             (dict(walk_kind="global", sources=[(0, 1.0)]), "sources/sinks are only supported for local walks"),
             (dict(walk_kind="quantum"), "unknown walk kind `quantum` (expected local, global or nm_global)")]
    for over, msg in cases:
        with pytest.raises(qrun.ConfigError) as ei:
            config("local_series", **over).validate()
        assert str(ei.value) == msg


def test_run_describe_matches_reference_metadata(monkeypatch):
    """The describe() block of every golden run's metadata, line for line."""
    monkeypatch.chdir(ROOT)
    for name in RUNS:
        ref = api.ResultContainer.read(os.path.join(IO, f"run_{name}.qswbox")).metadata
        assert config(name).describe() in ref, name


def _cmp_containers(ours: api.ResultContainer, ref: api.ResultContainer, name):
    assert sorted(ours.arrays) == sorted(ref.arrays), name
    for k, r in ref.arrays.items():
        o = ours.arrays[k]
        assert o.shape == r.shape, (name, k)
        if k == "times":
            assert np.array_equal(o, r), name  # expm.cpp:222-223, bit-identical
        else:
            assert np.abs(o - r).max(initial=0.0) <= 1e-10, (name, k, np.abs(o - r).max())
    ol = [x for x in ours.metadata.splitlines() if not x.startswith("timestamp_unix")]
    rl = [x for x in ref.metadata.splitlines() if not x.startswith("timestamp_unix")]
    assert ol == rl, (name, ol, rl)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(RUNS))
def test_run_matches_reference_container(name, monkeypatch, tmp_path):
    """run() on the device vs the reference's run() (tests/golden/io/run_*.qswbox):
    same arrays and shapes, rho / populations / coherence norms within 1e-10,
    identical times and metadata (bar the timestamp)."""
    monkeypatch.chdir(ROOT)
    out = qrun.run(config(name))
    out.write(tmp_path / "ours.qswbox")
    ours = api.ResultContainer.read(tmp_path / "ours.qswbox")
    _cmp_containers(ours, api.ResultContainer.read(os.path.join(IO, f"run_{name}.qswbox")), name)
    if "populations" in ours.arrays:
        assert np.abs(ours.arrays["populations"].sum(axis=1) - 1.0).max() <= 1e-12


@pytest.mark.gpu
def test_run_live_reference_extra_configs(monkeypatch, tmp_path):
    """Configs beyond the golden set, against the reference's run() live (oracle/_ref)."""
    ref = ref_io()
    monkeypatch.chdir(ROOT)
    extra = {
        "nm_step": dict(RUNS["nm_series"], is_series=False, t=7.5, out_full_rho=False),
        "local_cycle_mixed_gamma": dict(RUNS["local_series"], initial_kind="mixed", gamma=0.25, omega=0.9,
                                        t1=1.0, tq=2.0, steps=3),
        "global_torus_series": dict(RUNS["global_step_file"], is_series=True, t1=0.0, tq=6.0, steps=12),
    }
    for name, cfg in extra.items():
        rc, msg = ref.run(cfg, str(tmp_path / f"{name}.ref.qswbox"))
        assert rc == 0, msg
        c = dict(cfg)
        c["sources"] = [tuple(s) for s in c.get("sources", [])]
        c["sinks"] = [tuple(s) for s in c.get("sinks", [])]
        ours = qrun.run(qrun.RunConfig(**c))
        _cmp_containers(ours, api.ResultContainer.read(tmp_path / f"{name}.ref.qswbox"), name)


@pytest.mark.gpu
def test_series_coherence_matches_states():
    """Device coherence norms = max off-diagonal |rho| of the downloaded states."""
    from paper_2003_02450_b200 import graphs
    for fmt in ("kron", "sell", "csr"):
        w = graphs.config("c2", size=6)
        l = api.build_global(w.omega, w.h, w.ops, format=fmt)
        v = l.state().from_probabilities(w.rho0)
        r = api.series(l, v, 0.0, 3.0, 6, states=True, coherence=True)
        for k in range(7):
            rho = r.states[k].reshape(w.n, w.n)
            off = np.abs(rho[~np.eye(w.n, dtype=bool)]).max()
            assert abs(r.coherence[k] - off) <= 1e-15 * off, (fmt, k)
        assert r.coherence[0] == 0.0  # rho(0) is diagonal
        assert api.series(l, v, 0.0, 3.0, 6).coherence is None
        r2 = api.series(l, v, 0.0, 3.0, 6, coherence=True)  # graph replay on the second identical call
        r3 = api.series(l, v, 0.0, 3.0, 6, coherence=True)
        assert np.array_equal(r2.coherence, r.coherence) and np.array_equal(r3.coherence, r.coherence)
        assert v.coherence() == 0.0


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_run_fails_loudly_without_gpu(monkeypatch):
    monkeypatch.chdir(ROOT)
    with pytest.raises(api.CudaError):
        qrun.run(config("local_series"))
