"""TEST INFRASTRUCTURE ONLY — ctypes front-end to the reference's file formats
and run() (oracle/ref_io_harness.cpp inside oracle/_ref/libqswref.so).

Used by oracle/make_golden_io.py (fixtures under tests/golden/io/) and by
tests/test_io.py for live cross-checks when oracle/_ref is built.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libqswref.so")

_i64 = C.c_int64
_i64p = C.POINTER(C.c_int64)
_dp = C.POINTER(C.c_double)
KINDS = {"local": 0, "global": 1, "nm_global": 2}
INITIAL = {"mixed": 0, "vertex": 1, "file": 2}


def available() -> bool:
    return os.path.exists(REF_LIB)


class RefIo:
    def __init__(self, path: str = REF_LIB):
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_mtx_parse.argtypes = [C.c_char_p, _i64, C.POINTER(C.c_void_p), C.c_char_p, C.c_int]
        L.ref_mtx_save.argtypes = [C.c_void_p, C.c_char_p, C.c_char_p, C.c_int]
        L.ref_container_write.argtypes = [C.c_char_p, C.c_char_p, _i64, _i64, C.POINTER(C.c_char_p), _i64p, _i64p,
                                          _dp, C.c_char_p, C.c_int]
        L.ref_container_rewrite.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int]
        L.ref_plot_data.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_int]
        L.ref_run.argtypes = [C.c_char_p, C.c_int, C.c_double, C.c_double, C.c_int, C.c_double, C.c_double,
                              C.c_double, _i64, C.c_int, _i64, C.c_char_p, _i64, _i64p, _dp, _i64, _i64p, _dp,
                              _i64, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_char_p, C.c_int]
        L.ref_sparse_shape.argtypes = [C.c_void_p, _i64p, _i64p, _i64p]
        L.ref_sparse_export.argtypes = [C.c_void_p, _i64p, _i64p, _dp]
        L.ref_sparse_free.argtypes = [C.c_void_p]

    @staticmethod
    def _err():
        return C.create_string_buffer(1024)

    def parse_mtx(self, text: bytes):
        """-> (0, (indptr, indices, data)) or (code, message)."""
        out, err = C.c_void_p(), self._err()
        rc = self.lib.ref_mtx_parse(text, len(text), C.byref(out), err, 1024)
        if rc:
            return rc, err.value.decode()
        r, c, nnz = _i64(), _i64(), _i64()
        self.lib.ref_sparse_shape(out, C.byref(r), C.byref(c), C.byref(nnz))
        ip = np.zeros(r.value + 1, np.int64)
        ix = np.zeros(max(nnz.value, 1), np.int64)
        dv = np.zeros(2 * max(nnz.value, 1))
        self.lib.ref_sparse_export(out, ip.ctypes.data_as(_i64p), ix.ctypes.data_as(_i64p), dv.ctypes.data_as(_dp))
        self.lib.ref_sparse_free(out)
        return 0, (ip, ix[: nnz.value], dv[: 2 * nnz.value].view(np.complex128))

    def save_mtx(self, text: bytes, path: str):
        """Parse with the reference, then its save_matrix_market into path."""
        out, err = C.c_void_p(), self._err()
        rc = self.lib.ref_mtx_parse(text, len(text), C.byref(out), err, 1024)
        assert rc == 0, err.value
        rc = self.lib.ref_mtx_save(out, path.encode(), err, 1024)
        self.lib.ref_sparse_free(out)
        assert rc == 0, err.value

    def write_container(self, path: str, meta: str, arrays: dict):
        names = list(arrays)
        blocks = [np.array(arrays[k], dtype=np.float64, order="C") for k in names]  # keeps 0-d
        cn = (C.c_char_p * max(len(names), 1))(*[k.encode() for k in names])
        ranks = np.array([b.ndim for b in blocks] or [0], np.int64)
        shapes = np.array([d for b in blocks for d in b.shape] or [0], np.int64)
        data = np.concatenate([b.reshape(-1) for b in blocks] + [np.zeros(1)])
        m = meta.encode()
        err = self._err()
        rc = self.lib.ref_container_write(path.encode(), m, len(m), len(names), cn, ranks.ctypes.data_as(_i64p),
                                          shapes.ctypes.data_as(_i64p), data.ctypes.data_as(_dp), err, 1024)
        return rc, err.value.decode()

    def rewrite_container(self, src: str, dst: str):
        err = self._err()
        rc = self.lib.ref_container_rewrite(src.encode(), dst.encode(), err, 1024)
        return rc, err.value.decode()

    def plot_data(self, src: str, quantity: str, dst: str):
        err = self._err()
        rc = self.lib.ref_plot_data(src.encode(), quantity.encode(), dst.encode(), err, 1024)
        return rc, err.value.decode()

    def run(self, cfg: dict, out_path: str):
        """cfg: the RunConfig fields of paper_2003_02450_b200.run.RunConfig."""
        src = cfg.get("sources", [])
        snk = cfg.get("sinks", [])
        st = np.array([s[0] for s in src] or [0], np.int64)
        sr = np.array([s[1] for s in src] or [0.0])
        kt = np.array([s[0] for s in snk] or [0], np.int64)
        kr = np.array([s[1] for s in snk] or [0.0])
        err = self._err()
        rc = self.lib.ref_run(cfg["graph_path"].encode(), KINDS[cfg.get("walk_kind", "local")], cfg.get("omega", 0.0),
                              cfg.get("gamma", 1.0), int(cfg.get("is_series", False)), cfg.get("t", 0.0),
                              cfg.get("t1", 0.0), cfg.get("tq", 0.0), cfg.get("steps", 0),
                              INITIAL[cfg.get("initial_kind", "mixed")], cfg.get("initial_vertex", 0),
                              cfg.get("initial_file", "").encode(), len(src), st.ctypes.data_as(_i64p),
                              sr.ctypes.data_as(_dp), len(snk), kt.ctypes.data_as(_i64p), kr.ctypes.data_as(_dp),
                              cfg.get("workers", 1), int(cfg.get("out_populations", True)),
                              int(cfg.get("out_full_rho", False)), int(cfg.get("out_coherence_norm", False)),
                              out_path.encode(), err, 1024)
        return rc, err.value.decode()
