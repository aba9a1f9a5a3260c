"""TEST INFRASTRUCTURE ONLY — ctypes front-end to the two CPU checkers.

* ``Oracle("port")``      -> oracle/build/libqsworacle.so, the plain-C
  restatement (oracle/qsw_oracle.c).  Travels to the GPU box (built by
  __graft_entry__.build()).
* ``Oracle("reference")`` -> oracle/_ref/libqswref[_v3].so, the UNMODIFIED
  reference library compiled from /root/reference by oracle/Makefile, behind
  oracle/ref_harness.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
legs may import this module — as the checker, never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "build", "libqsworacle.so")
REF_SO = os.path.join(HERE, "_ref", "libqswref.so")
REF_V3_SO = os.path.join(HERE, "_ref", "libqswref_v3.so")

_i64p = C.POINTER(C.c_int64)
_dp = C.POINTER(C.c_double)


def _p(a, t=_dp):
    return a.ctypes.data_as(t) if a is not None else None


def _cvec(a):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a, a.view(np.float64).ctypes.data_as(_dp)


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def cpu_has_avx2() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            flags = f.read()
        return " avx2" in flags and " fma" in flags and " bmi2" in flags
    except OSError:
        return False


class _Csr(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("nnz", C.c_int64),
                ("rowptr", _i64p), ("col", _i64p), ("val", _dp)]


class Oracle:
    def __init__(self, kind: str = "port", fast: bool = True):
        self.kind = kind
        if kind == "port":
            path = PORT_SO
        elif kind == "reference":
            path = REF_V3_SO if (fast and os.path.exists(REF_V3_SO) and cpu_has_avx2()) else REF_SO
        else:
            raise ValueError(kind)
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (run __graft_entry__.build())")
        self.path = path
        self.lib = C.CDLL(path)
        self._setup()

    # ------------------------------------------------------------------ ABI
    def _setup(self):
        L = self.lib
        if self.kind == "port":
            L.orc_csr_from_arrays.restype = C.POINTER(_Csr)
            L.orc_csr_from_arrays.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, _dp]
            L.orc_csr_free.argtypes = [C.c_void_p]
            for f in ("orc_generator_matrix",):
                getattr(L, f).restype = C.POINTER(_Csr)
                getattr(L, f).argtypes = [C.c_double, C.c_void_p]
            for f in ("orc_markov_chain_matrix", "orc_symmetrize", "orc_local_lindblad"):
                getattr(L, f).restype = C.POINTER(_Csr)
                getattr(L, f).argtypes = [C.c_void_p]
            L.orc_build_local.restype = C.c_int
            L.orc_build_local.argtypes = [C.c_double, C.c_void_p, C.c_void_p, C.c_int64, _i64p, _dp,
                                          C.c_int64, _i64p, _dp, C.POINTER(C.c_void_p)]
            L.orc_build_global.restype = C.c_int
            L.orc_build_global.argtypes = [C.c_double, C.c_void_p, C.c_int64, C.POINTER(C.c_void_p),
                                           C.c_void_p, C.POINTER(C.c_void_p)]
            L.orc_free.argtypes = [C.c_void_p]
            L.orc_matrix.restype = C.POINTER(_Csr)
            L.orc_matrix.argtypes = [C.c_void_p]
            L.orc_norms.argtypes = [C.c_void_p, _dp]
            L.orc_theta.argtypes = [_dp]
            L.orc_select.argtypes = [_dp, C.c_double, _i64p, _i64p]
            L.orc_spmv.argtypes = [C.c_void_p, _dp, _dp]
            L.orc_step.restype = C.c_int
            L.orc_step.argtypes = [C.c_void_p, _dp, C.c_double, _dp]
            L.orc_series.restype = C.c_int
            L.orc_series.argtypes = [C.c_void_p, _dp, C.c_double, C.c_double, C.c_int64, _dp, _dp]
            L.orc_spmv_counter.restype = C.c_uint64
        else:
            L.ref_sparse_new.restype = C.c_void_p
            L.ref_sparse_new.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, _dp]
            L.ref_sparse_free.argtypes = [C.c_void_p]
            L.ref_sparse_shape.argtypes = [C.c_void_p, _i64p, _i64p, _i64p]
            L.ref_sparse_export.argtypes = [C.c_void_p, _i64p, _i64p, _dp]
            L.ref_graph_op.restype = C.c_void_p
            L.ref_graph_op.argtypes = [C.c_int, C.c_double, C.c_void_p, C.c_char_p, C.c_int]
            L.ref_nm_op.restype = C.c_void_p
            L.ref_nm_op.argtypes = [C.c_int, C.c_double, C.c_void_p, C.c_void_p, C.c_int, _i64p, C.c_char_p, C.c_int]
            L.ref_build_local.restype = C.c_void_p
            L.ref_build_local.argtypes = [C.c_double, C.c_void_p, C.c_void_p, C.c_int64, _i64p, _dp,
                                          C.c_int64, _i64p, _dp, C.c_int64, C.POINTER(C.c_int),
                                          C.c_char_p, C.c_int]
            L.ref_build_global.restype = C.c_void_p
            L.ref_build_global.argtypes = [C.c_double, C.c_void_p, C.c_int64, C.POINTER(C.c_void_p),
                                           C.c_void_p, C.c_int64, C.POINTER(C.c_int), C.c_char_p, C.c_int]
            L.ref_free.argtypes = [C.c_void_p]
            L.ref_info.argtypes = [C.c_void_p, _i64p, _i64p, _dp]
            L.ref_csr.argtypes = [C.c_void_p, _i64p, _i64p, _dp]
            L.ref_spmv.argtypes = [C.c_void_p, _dp, _dp]
            L.ref_step.restype = C.c_int
            L.ref_step.argtypes = [C.c_void_p, _dp, C.c_double, _dp, C.c_char_p, C.c_int]
            L.ref_series.restype = C.c_int
            L.ref_series.argtypes = [C.c_void_p, _dp, C.c_double, C.c_double, C.c_int64, _dp, _dp,
                                     C.c_char_p, C.c_int]
            L.ref_theta.restype = C.c_int
            L.ref_theta.argtypes = [C.c_double, _dp]
            L.ref_select.argtypes = [_dp, C.c_double, C.c_double, _i64p, _i64p]
            L.ref_spmv_counter.restype = C.c_uint64

    # ------------------------------------------------------------- sparse
    def _sparse_in(self, m):
        ip = np.ascontiguousarray(m.indptr, dtype=np.int64)
        ix = np.ascontiguousarray(m.indices, dtype=np.int64)
        dv = np.ascontiguousarray(m.data, dtype=np.complex128).view(np.float64)
        keep = (ip, ix, dv)
        if self.kind == "port":
            h = self.lib.orc_csr_from_arrays(m.rows, m.cols, _p(ip, _i64p), _p(ix, _i64p), _p(dv))
            return C.cast(h, C.c_void_p), keep
        return C.c_void_p(self.lib.ref_sparse_new(m.rows, m.cols, _p(ip, _i64p), _p(ix, _i64p), _p(dv))), keep

    def _sparse_free(self, h):
        (self.lib.orc_csr_free if self.kind == "port" else self.lib.ref_sparse_free)(h)

    def _sparse_out(self, h):
        from paper_2003_02450_b200.graphs import Csr
        if self.kind == "port":
            s = C.cast(h, C.POINTER(_Csr)).contents
            ip = np.ctypeslib.as_array(s.rowptr, shape=(s.rows + 1,)).copy()
            ix = np.ctypeslib.as_array(s.col, shape=(max(s.nnz, 1),))[: s.nnz].copy()
            dv = np.ctypeslib.as_array(s.val, shape=(max(2 * s.nnz, 1),))[: 2 * s.nnz].copy()
            return Csr(s.rows, s.cols, ip, ix, dv.view(np.complex128))
        r, c, z = C.c_int64(), C.c_int64(), C.c_int64()
        self.lib.ref_sparse_shape(h, C.byref(r), C.byref(c), C.byref(z))
        ip = np.zeros(r.value + 1, np.int64)
        ix = np.zeros(max(z.value, 1), np.int64)
        dv = np.zeros(max(2 * z.value, 2), np.float64)
        self.lib.ref_sparse_export(h, _p(ip, _i64p), _p(ix, _i64p), _p(dv))
        return Csr(r.value, c.value, ip, ix[: z.value], dv[: 2 * z.value].view(np.complex128))

    def graph_op(self, what: str, m, gamma: float = 1.0):
        """what in {generator_matrix, markov_chain_matrix, symmetrize, local_lindblad}."""
        h, keep = self._sparse_in(m)
        try:
            if self.kind == "port":
                fn = getattr(self.lib, "orc_" + what)
                out = fn(gamma, h) if what == "generator_matrix" else fn(h)
                if not out:
                    raise OracleError(1, what)
                res = self._sparse_out(out)
                self.lib.orc_csr_free(out)
                return res
            code = {"generator_matrix": 0, "markov_chain_matrix": 1, "symmetrize": 2,
                    "local_lindblad": 3}[what]
            err = C.create_string_buffer(512)
            out = self.lib.ref_graph_op(code, gamma, h, err, 512)
            if not out:
                raise OracleError(1, err.value.decode())
            res = self._sparse_out(C.c_void_p(out))
            self.lib.ref_sparse_free(C.c_void_p(out))
            return res
        finally:
            self._sparse_free(h)

    def nm_op(self, what: str, g, gu, gamma: float = 1.0, pauli_y: bool = False):
        """Reference demoralisation operators: what in {nm_H, nm_L, nm_H_rot};
        returns (matrix, vsets dims).  Reference library only."""
        assert self.kind == "reference"
        gh, k1 = self._sparse_in(g)
        uh, k2 = self._sparse_in(gu)
        dims = np.zeros(g.rows, np.int64)
        err = C.create_string_buffer(512)
        code = {"nm_H": 0, "nm_L": 1, "nm_H_rot": 2}[what]
        try:
            out = self.lib.ref_nm_op(code, gamma, gh, uh, int(pauli_y), _p(dims, _i64p), err, 512)
            if not out:
                raise OracleError(1, err.value.decode())
            res = self._sparse_out(C.c_void_p(out))
            self.lib.ref_sparse_free(C.c_void_p(out))
            return res, dims
        finally:
            self._sparse_free(gh)
            self._sparse_free(uh)

    # -------------------------------------------------------- liouvillian
    def build_local(self, omega, h, m_l, sources=(), sinks=(), workers=1):
        hh, k1 = self._sparse_in(h)
        mh, k2 = self._sparse_in(m_l)
        st = np.array([s[0] for s in sources], np.int64)
        sr = np.array([s[1] for s in sources], np.float64)
        kt = np.array([s[0] for s in sinks], np.int64)
        kr = np.array([s[1] for s in sinks], np.float64)
        try:
            if self.kind == "port":
                out = C.c_void_p()
                rc = self.lib.orc_build_local(omega, hh, mh, len(st), _p(st, _i64p), _p(sr), len(kt),
                                              _p(kt, _i64p), _p(kr), C.byref(out))
                if rc:
                    raise OracleError(rc)
                return _Handle(self, out, h.rows)
            code = C.c_int()
            err = C.create_string_buffer(512)
            out = self.lib.ref_build_local(omega, hh, mh, len(st), _p(st, _i64p), _p(sr), len(kt),
                                           _p(kt, _i64p), _p(kr), workers, C.byref(code), err, 512)
            if not out:
                raise OracleError(code.value, err.value.decode())
            return _Handle(self, C.c_void_p(out), h.rows)
        finally:
            self._sparse_free(hh)
            self._sparse_free(mh)

    def build_global(self, omega, h, lindblads, h_rot=None, workers=1):
        hh, k1 = self._sparse_in(h)
        ls = [self._sparse_in(x) for x in lindblads]
        arr = (C.c_void_p * max(len(ls), 1))(*[x[0] for x in ls])
        hr = self._sparse_in(h_rot) if h_rot is not None else (None, None)
        try:
            if self.kind == "port":
                out = C.c_void_p()
                rc = self.lib.orc_build_global(omega, hh, len(ls), arr, hr[0], C.byref(out))
                if rc:
                    raise OracleError(rc)
                return _Handle(self, out, h.rows)
            code = C.c_int()
            err = C.create_string_buffer(512)
            out = self.lib.ref_build_global(omega, hh, len(ls), arr, hr[0], workers, C.byref(code), err, 512)
            if not out:
                raise OracleError(code.value, err.value.decode())
            return _Handle(self, C.c_void_p(out), h.rows)
        finally:
            self._sparse_free(hh)
            for x in ls:
                self._sparse_free(x[0])
            if hr[0] is not None:
                self._sparse_free(hr[0])

    def build(self, w, workers=1):
        if w.kind == "local":
            return self.build_local(w.omega, w.h, w.ops[0], workers=workers)
        return self.build_global(w.omega, w.h, w.ops, workers=workers)

    # ------------------------------------------------------------- Taylor
    def theta(self, tol=2.0 ** -53):
        out = np.zeros(55)
        if self.kind == "port":
            self.lib.orc_theta(_p(out))
        else:
            self.lib.ref_theta(tol, _p(out))
        return out

    def select(self, norms, t, tol=2.0 ** -53):
        nm = np.ascontiguousarray(norms, dtype=np.float64)
        m, s = C.c_int64(), C.c_int64()
        if self.kind == "port":
            self.lib.orc_select(_p(nm), t, C.byref(m), C.byref(s))
        else:
            self.lib.ref_select(_p(nm), t, tol, C.byref(m), C.byref(s))
        return m.value, s.value

    def counter(self):
        return int(self.lib.orc_spmv_counter() if self.kind == "port" else self.lib.ref_spmv_counter())


def rho0_vec(n, probabilities):
    v = np.zeros(n * n, dtype=np.complex128)
    v[np.arange(n) * (n + 1)] = probabilities
    return v


class _Handle:
    def __init__(self, o: Oracle, h, n):
        self.o, self.h, self.n = o, h, n
        self.dim, self.nnz, self.norms = self._info()

    def __del__(self):
        try:
            (self.o.lib.orc_free if self.o.kind == "port" else self.o.lib.ref_free)(self.h)
        except Exception:
            pass

    def _info(self):
        norms = np.zeros(9)
        if self.o.kind == "port":
            s = self.o.lib.orc_matrix(self.h).contents
            self.o.lib.orc_norms(self.h, _p(norms))
            return s.rows, s.nnz, norms
        d, z = C.c_int64(), C.c_int64()
        self.o.lib.ref_info(self.h, C.byref(d), C.byref(z), _p(norms))
        return d.value, z.value, norms

    def csr(self):
        from paper_2003_02450_b200.graphs import Csr
        if self.o.kind == "port":
            return self.o._sparse_out(C.cast(self.o.lib.orc_matrix(self.h), C.c_void_p))
        ip = np.zeros(self.dim + 1, np.int64)
        ix = np.zeros(max(self.nnz, 1), np.int64)
        dv = np.zeros(max(2 * self.nnz, 2))
        self.o.lib.ref_csr(self.h, _p(ip, _i64p), _p(ix, _i64p), _p(dv))
        return Csr(self.dim, self.dim, ip, ix[: self.nnz], dv[: 2 * self.nnz].view(np.complex128))

    def spmv(self, x):
        x, xp = _cvec(x)
        y = np.zeros(self.dim, np.complex128)
        (self.o.lib.orc_spmv if self.o.kind == "port" else self.o.lib.ref_spmv)(
            self.h, xp, y.view(np.float64).ctypes.data_as(_dp))
        return y

    def step(self, v, t):
        v, vp = _cvec(v)
        out = np.zeros(self.dim, np.complex128)
        c0 = self.o.counter()
        if self.o.kind == "port":
            rc = self.o.lib.orc_step(self.h, vp, t, out.view(np.float64).ctypes.data_as(_dp))
            msg = ""
        else:
            err = C.create_string_buffer(512)
            rc = self.o.lib.ref_step(self.h, vp, t, out.view(np.float64).ctypes.data_as(_dp), err, 512)
            msg = err.value.decode()
        if rc:
            raise OracleError(rc, msg)
        return out, self.o.counter() - c0

    def series(self, v, t1, tq, steps, states=True, pops=True):
        v, vp = _cvec(v)
        so = np.zeros((steps + 1, self.dim), np.complex128) if states else None
        po = np.zeros((steps + 1, self.n)) if pops else None
        sp = so.view(np.float64).ctypes.data_as(_dp) if states else None
        pp = _p(po) if pops else None
        c0 = self.o.counter()
        if self.o.kind == "port":
            rc = self.o.lib.orc_series(self.h, vp, t1, tq, steps, sp, pp)
            msg = ""
        else:
            err = C.create_string_buffer(512)
            rc = self.o.lib.ref_series(self.h, vp, t1, tq, steps, sp, pp, err, 512)
            msg = err.value.decode()
        if rc:
            raise OracleError(rc, msg)
        return so, po, self.o.counter() - c0
