"""Python mirror of the reference library surface for the expmv hot path.

Every name follows proj/core/include/qsw/* (cited per item) and calls the
C ABI of libqswg.so (include/qswg.h); nothing here computes on the CPU
beyond argument marshalling.  Error behaviour matches the reference's
exceptions: ValueError (std::invalid_argument), IndexError
(std::out_of_range), NumericalError, LogicError (std::logic_error).
"""
from __future__ import annotations

import ctypes as C
import dataclasses

import numpy as np

from . import _lib
from ._lib import (CudaError, FileFormatError, InvalidArgument, IoError, LogicError,  # noqa: F401
                   NumericalError, OutOfRange, QswgError, check, lib)
from .graphs import Csr

DOUBLE_TOL = 2.0 ** -53  # expm.hpp:18
SINGLE_TOL = 2.0 ** -24  # expm.hpp:19


def _dp(a):
    return a.ctypes.data_as(_lib.dp)


def _i64p(a):
    return a.ctypes.data_as(_lib.i64p)


def _cplx(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    if n is not None and a.size != n:
        raise ValueError(f"expected {n} complex values, got {a.size}")
    return a


class _Pinned:
    """Owner of one qswg_host_alloc block (freed with the last array view)."""

    def __init__(self, nbytes):
        self.ptr = C.c_void_p()
        check(lib.qswg_host_alloc(int(nbytes), C.byref(self.ptr)))
        self.nbytes = int(nbytes)

    def __del__(self):
        if getattr(self, "ptr", None) is not None and self.ptr.value:
            lib.qswg_host_free(self.ptr)
            self.ptr = None


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """A numpy array in page-locked host memory (qswg_host_alloc): uploads from
    it and population reads into it are direct DMA transfers.  The block is
    freed when the last view of the array goes away."""
    dt = np.dtype(dtype)
    shape = tuple(int(d) for d in (shape if isinstance(shape, (tuple, list)) else (shape,)))
    owner = _Pinned(max(int(np.prod(shape)) * dt.itemsize, 1))
    owner.__array_interface__ = {"shape": shape, "typestr": dt.str, "data": (owner.ptr.value, False),
                                 "version": 3}
    return np.asarray(owner)  # .base is the owner


# --------------------------------------------------------------- sparse
class SparseMatrix:
    """Host canonical CSR (sparse.hpp:29-84) owned by the C library."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.qswg_sparse_destroy(h)
            self._h = None

    @staticmethod
    def from_triplets(rows, cols, r, c, v) -> "SparseMatrix":
        r = np.ascontiguousarray(r, dtype=np.int64)
        c = np.ascontiguousarray(c, dtype=np.int64)
        v = _cplx(v)
        out = C.c_void_p()
        check(lib.qswg_sparse_from_triplets(rows, cols, len(r), _i64p(r), _i64p(c),
                                            _dp(v.view(np.float64)), C.byref(out)))
        return SparseMatrix(out)

    @staticmethod
    def from_csr(m: Csr) -> "SparseMatrix":
        ip = np.ascontiguousarray(m.indptr, dtype=np.int64)
        ix = np.ascontiguousarray(m.indices, dtype=np.int64)
        dv = _cplx(m.data)
        out = C.c_void_p()
        check(lib.qswg_sparse_from_csr(m.rows, m.cols, _i64p(ip), _i64p(ix),
                                       _dp(dv.view(np.float64)) if dv.size else None, C.byref(out)))
        return SparseMatrix(out)

    @staticmethod
    def of(x) -> "SparseMatrix":
        if isinstance(x, SparseMatrix):
            return x
        if isinstance(x, Csr):
            return SparseMatrix.from_csr(x)
        if hasattr(x, "tocsr"):  # scipy.sparse
            s = x.tocsr()
            return SparseMatrix.from_csr(Csr(s.shape[0], s.shape[1], s.indptr.astype(np.int64),
                                             s.indices.astype(np.int64), s.data.astype(np.complex128)))
        d = np.asarray(x, dtype=np.complex128)
        r, c = np.nonzero(d)
        return SparseMatrix.from_triplets(d.shape[0], d.shape[1], r, c, d[r, c])

    @property
    def shape(self):
        r, c, z = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.qswg_sparse_shape(self._h, C.byref(r), C.byref(c), C.byref(z)))
        return r.value, c.value

    @property
    def nnz(self) -> int:
        z = C.c_int64()
        check(lib.qswg_sparse_shape(self._h, None, None, C.byref(z)))
        return z.value

    def to_csr(self) -> Csr:
        rows, cols = self.shape
        z = self.nnz
        ip = np.zeros(rows + 1, np.int64)
        ix = np.zeros(max(z, 1), np.int64)
        dv = np.zeros(max(z, 1), np.complex128)
        check(lib.qswg_sparse_export(self._h, _i64p(ip), _i64p(ix), _dp(dv.view(np.float64))))
        return Csr(rows, cols, ip, ix[:z], dv[:z])

    def to_dense(self) -> np.ndarray:
        return self.to_csr().to_dense()


def _unary(fn, *args):
    keep = [a for a in args if isinstance(a, SparseMatrix)]  # handles must outlive the call
    out = C.c_void_p()
    check(fn(*[a._h if isinstance(a, SparseMatrix) else a for a in args], C.byref(out)))
    del keep
    return SparseMatrix(out)


def symmetrize(adjacency) -> SparseMatrix:  # graph.hpp:75
    return _unary(lib.qswg_symmetrize, SparseMatrix.of(adjacency))


def generator_matrix(gamma: float, adjacency) -> SparseMatrix:  # graph.hpp:84-85
    return _unary(lib.qswg_generator_matrix, C.c_double(gamma), SparseMatrix.of(adjacency))


def markov_chain_matrix(adjacency) -> SparseMatrix:  # graph.hpp:88
    return _unary(lib.qswg_markov_chain_matrix, SparseMatrix.of(adjacency))


def local_lindblad(m) -> SparseMatrix:  # operators.hpp:53-54
    return _unary(lib.qswg_local_lindblad, SparseMatrix.of(m))


def global_lindblad(adjacency) -> SparseMatrix:  # operators.hpp:56-57
    return SparseMatrix.of(adjacency)


def _arcs(sources, sinks):
    src = (_lib.SourceArc * max(len(sources), 1))(*[_lib.SourceArc(int(t), float(r)) for t, r in sources])
    snk = (_lib.SinkArc * max(len(sinks), 1))(*[_lib.SinkArc(int(o), float(r)) for o, r in sinks])
    return src, snk


def augment(adjacency, sources=(), sinks=()) -> SparseMatrix:  # graph.hpp:93-95
    src, snk = _arcs(sources, sinks)
    return _unary(lib.qswg_augment, SparseMatrix.of(adjacency), src, len(sources), snk, len(sinks))


# ------------------------------------------------- demoralisation (NM-G-QSW)
def nm_vsets(gu) -> np.ndarray:
    """Subspace dimension per vertex of the symmetric graph gu (operators.hpp:59-60)."""
    m = SparseMatrix.of(gu)
    dims = np.zeros(m.shape[0], np.int64)
    check(lib.qswg_nm_vsets(m._h, _i64p(dims)))
    return dims


def nm_H(gamma, gu, dims) -> SparseMatrix:  # operators.hpp:66-68
    d = np.ascontiguousarray(dims, np.int64)
    return _unary(lib.qswg_nm_H, C.c_double(gamma), SparseMatrix.of(gu), _i64p(d), len(d))


def nm_L(gamma, g, dims) -> SparseMatrix:  # operators.hpp:70-75
    d = np.ascontiguousarray(dims, np.int64)
    return _unary(lib.qswg_nm_L, C.c_double(gamma), SparseMatrix.of(g), _i64p(d), len(d))


def nm_H_rot(dims, pauli_y: bool = False) -> SparseMatrix:  # operators.hpp:77-79
    d = np.ascontiguousarray(dims, np.int64)
    return _unary(lib.qswg_nm_H_rot, _i64p(d), len(d), int(pauli_y))


def nm_rho_map(p, dims) -> np.ndarray:  # operators.hpp:80-81
    d = np.ascontiguousarray(dims, np.int64)
    p = np.ascontiguousarray(p, np.float64)
    out = np.zeros(int(d.sum()))
    check(lib.qswg_nm_rho_map(_dp(p), _i64p(d), len(d), _dp(out)))
    return out


def nm_measure(diag, dims) -> np.ndarray:  # operators.hpp:82-83
    d = np.ascontiguousarray(dims, np.int64)
    diag = np.ascontiguousarray(diag, np.float64)
    out = np.zeros(len(d))
    check(lib.qswg_nm_measure(_dp(diag), _i64p(d), len(d), _dp(out)))
    return out


# ----------------------------------------------------------- Liouvillian
class Liouvillian:
    """Device superoperator (DistributedLiouvillian, liouvillian.hpp:21-63)."""

    def __init__(self, handle):
        self._h = handle
        self._query()

    def _query(self):
        info = _lib.LiouvillianInfo()
        check(lib.qswg_liouvillian_query(self._h, C.byref(info)))
        self.info = info

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.qswg_liouvillian_destroy(h)
            self._h = None

    n = property(lambda self: self.info.n)
    dim = property(lambda self: self.info.dim)
    nnz = property(lambda self: self.info.nnz)
    omega = property(lambda self: self.info.omega)
    group = property(lambda self: self.info.group)
    row0 = property(lambda self: self.info.row0)
    rows = property(lambda self: self.info.rows)
    format = property(lambda self: {1: "csr", 2: "sell", 3: "kron"}[self.info.format])
    padding = property(lambda self: self.info.padding)

    def one_norms(self) -> np.ndarray:
        return np.array(list(self.info.one_norms))

    def gather_full(self) -> Csr:
        """Local row block (the full matrix on one GPU), liouvillian.hpp:34."""
        z = self.info.nnz_local
        ip = np.zeros(self.rows + 1, np.int64)
        ix = np.zeros(max(z, 1), np.int64)
        dv = np.zeros(max(z, 1), np.complex128)
        check(lib.qswg_liouvillian_download(self._h, _i64p(ip), _i64p(ix), _dp(dv.view(np.float64))))
        return Csr(self.rows, self.dim, ip, ix[:z], dv[:z])

    def spmv(self, x) -> np.ndarray:
        """y = L x (liouvillian.hpp:93)."""
        x = _cplx(x, self.dim)
        y = np.zeros(self.rows, np.complex128)
        check(lib.qswg_spmv(self._h, _dp(x.view(np.float64)), _dp(y.view(np.float64))))
        return y

    def time_spmv(self, iters: int = 20, group: int = 0) -> float:
        ms = C.c_double()
        check(lib.qswg_time_spmv(self._h, iters, group, C.byref(ms)))
        return ms.value

    def partition(self):
        """(starts[world+1], halo_lo[world, world], halo_hi[world, world])."""
        w = self.info.world
        st = np.zeros(w + 1, np.int64)
        lo, hi = np.zeros((w, w), np.int64), np.zeros((w, w), np.int64)
        check(lib.qswg_liouvillian_partition(self._h, _i64p(st), _i64p(lo), _i64p(hi)))
        return st, lo, hi

    def time_series_term(self, iters: int = 20, count: int = 1) -> float:
        ms = C.c_double()
        check(lib.qswg_time_series_term(self._h, iters, count, C.byref(ms)))
        return ms.value

    def set_omega(self, omega: float) -> None:
        """Re-mix for a new omega in place on the device (qswg_liouvillian_set_omega);
        states of this operator stay valid."""
        check(lib.qswg_liouvillian_set_omega(self._h, float(omega)))
        self._query()

    def set_hermitian_mode(self, on: bool) -> None:
        """KRON on one GPU: allow (default) or forbid the Hermitian tile kernels."""
        check(lib.qswg_liouvillian_set_hermitian_mode(self._h, 1 if on else 0))

    def time_series_parts(self, iters: int = 20, count: int = 1) -> dict:
        """Mean device ms of one series term split into prepare / term kernel / flush."""
        ms = (C.c_double * 4)()
        check(lib.qswg_time_series_parts(self._h, iters, count, ms))
        return {"prepare": ms[0], "term": ms[1], "flush": ms[2], "total": ms[3]}

    def stream(self) -> int:
        """cudaStream_t of this handle (for CUDA events recorded by callers)."""
        s = C.c_void_p()
        check(lib.qswg_liouvillian_stream(self._h, C.byref(s)))
        return s.value or 0

    def state(self) -> "StateVector":
        return StateVector(self)


FORMATS = {"auto": 0, "csr": 1, "sell": 2, "kron": 3}


def _config(device, group, comm, format="auto"):
    return _lib.DeviceConfig(device, group, FORMATS[format], comm._h if comm is not None else None)


def build_local(omega, h, m_l, sources=(), sinks=(), device: int = 0, group: int = 0, comm=None,
                format: str = "auto") -> Liouvillian:
    """build_local (liouvillian.hpp:65-71)."""
    src, snk = _arcs(sources, sinks)
    cfg = _config(device, group, comm, format)
    out = C.c_void_p()
    hs, ms = SparseMatrix.of(h), SparseMatrix.of(m_l)
    check(lib.qswg_build_local(float(omega), hs._h, ms._h, src, len(sources), snk, len(sinks),
                               C.byref(cfg), C.byref(out)))
    return Liouvillian(out)


def build_global(omega, h, lindblads, h_rot=None, device: int = 0, group: int = 0, comm=None,
                 format: str = "auto") -> Liouvillian:
    """build_global (liouvillian.hpp:73-85)."""
    cfg = _config(device, group, comm, format)
    hs = SparseMatrix.of(h)
    ls = [SparseMatrix.of(x) for x in lindblads]
    arr = (C.c_void_p * max(len(ls), 1))(*[x._h.value for x in ls])
    hr = SparseMatrix.of(h_rot) if h_rot is not None else None
    out = C.c_void_p()
    check(lib.qswg_build_global(float(omega), hs._h, arr, len(ls), hr._h if hr else None,
                                C.byref(cfg), C.byref(out)))
    return Liouvillian(out)


# ------------------------------------------------------------------ state
class StateVector:
    """Device vec(rho), column-major (state.hpp:13-27)."""

    def __init__(self, l: Liouvillian):
        self.l = l
        h = C.c_void_p()
        check(lib.qswg_state_create(l._h, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.qswg_state_destroy(h)
            self._h = None

    def upload(self, vec) -> "StateVector":
        v = _cplx(vec, self.l.dim)
        check(lib.qswg_state_upload(self._h, _dp(v.view(np.float64))))
        return self

    def upload_local(self, vec_local) -> "StateVector":
        """Upload only this rank's rows (vec_local has `rows` entries)."""
        v = _cplx(vec_local, self.l.rows)
        # qswg_state_upload reads vec + row0; pass a pointer shifted back by row0
        base = v.ctypes.data - 16 * self.l.row0
        check(lib.qswg_state_upload(self._h, C.cast(C.c_void_p(base), _lib.dp)))
        return self

    def from_probabilities(self, p) -> "StateVector":
        p = np.ascontiguousarray(p, dtype=np.float64)
        check(lib.qswg_state_from_probabilities(self._h, _dp(p), len(p)))
        return self

    def gather(self) -> np.ndarray:
        out = np.zeros(self.l.rows, np.complex128)
        check(lib.qswg_state_download(self._h, _dp(out.view(np.float64))))
        return out

    def populations(self) -> np.ndarray:
        out = np.zeros(self.l.n)
        check(lib.qswg_state_populations(self._h, _dp(out)))
        return out

    def coherence(self) -> float:
        """max_{i != j} |rho(i, j)| on the device (DensityMatrix::max_coherence, walk.cpp:32-40)."""
        out = C.c_double()
        check(lib.qswg_state_coherence(self._h, C.byref(out)))
        return out.value


# ----------------------------------------------------------------- Taylor
def build_theta_table(tolerance: float = DOUBLE_TOL) -> np.ndarray:
    out = np.zeros(55)
    check(lib.qswg_theta_table(tolerance, _dp(out)))
    return out


def select_parameters(one_norms, t: float, tolerance: float = DOUBLE_TOL):
    n = np.ascontiguousarray(one_norms, dtype=np.float64)
    m, s = C.c_int64(), C.c_int64()
    check(lib.qswg_select_parameters(_dp(n), t, tolerance, C.byref(m), C.byref(s)))
    return m.value, s.value


def step(l: Liouvillian, v: StateVector, t: float, tolerance: float = DOUBLE_TOL):
    """w = exp(tL) v (expm.hpp:47-51). Returns (StateVector, StepInfo)."""
    out = StateVector(l)
    info = _lib.StepInfo()
    check(lib.qswg_step(l._h, v._h, t, tolerance, out._h, C.byref(info)))
    return out, info


@dataclasses.dataclass
class SeriesResult:
    """expm.hpp:53-58 plus the device populations and plan."""
    times: np.ndarray
    populations: np.ndarray | None
    states: np.ndarray | None
    final: StateVector | None
    info: object
    coherence: np.ndarray | None = None


def series(l: Liouvillian, v: StateVector, t1: float, tq: float, steps: int, tolerance: float = DOUBLE_TOL,
           populations: bool = True, states: bool = False, final: bool = False, pops_out=None,
           coherence: bool = False) -> SeriesResult:
    """States at t1 + k (tq - t1)/steps, k = 0..steps (expm.hpp:60-63).
    `pops_out` may be a preallocated (e.g. pinned) float64 [(steps+1), n] array;
    `coherence` adds max_{i != j} |rho_k(i, j)| per output, computed on the device."""
    if pops_out is not None:
        assert pops_out.dtype == np.float64 and pops_out.size == (steps + 1) * l.n and pops_out.flags.c_contiguous
        pops = pops_out
    else:
        pops = np.zeros((steps + 1, l.n)) if populations else None
    st = np.zeros((steps + 1, l.rows), np.complex128) if states else None
    fin = StateVector(l) if final else None
    coh = np.zeros(steps + 1) if coherence and steps >= 1 else None
    info = _lib.SeriesInfo()
    check(lib.qswg_series_observe(l._h, v._h, t1, tq, steps, tolerance,
                                  _dp(pops) if pops is not None else None,
                                  _dp(coh) if coh is not None else None,
                                  _dp(st.view(np.float64)) if st is not None else None,
                                  fin._h if fin is not None else None, C.byref(info)))
    h = (tq - t1) / steps if steps >= 1 else 0.0
    times = np.array([t1 + h * float(k) for k in range(steps + 1)])  # expm.cpp:222-223
    return SeriesResult(times, pops, st, fin, info, coh)


# ------------------------------------------------------------ file formats
def parse_matrix_market(text) -> SparseMatrix:
    """WeightedDigraph::load_matrix_market on an in-memory stream (graph.cpp:54-136):
    the adjacency matrix, entry (i, j) = arc j -> i.  FileFormatError for a
    malformed stream, ValueError for a self-loop or a non-positive weight."""
    b = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    check(lib.qswg_matrix_market_parse(b, len(b), C.byref(h)))
    return SparseMatrix(h)


def load_matrix_market(path) -> SparseMatrix:
    """The graph-file loader of run() (run.cpp:14-25): IoError when the file
    cannot be opened, FileFormatError (naming the file) for anything else."""
    h = C.c_void_p()
    check(lib.qswg_matrix_market_load(str(path).encode(), C.byref(h)))
    return SparseMatrix(h)


def save_matrix_market(adjacency, path) -> None:
    """WeightedDigraph::save_matrix_market (graph.cpp:138-150)."""
    check(lib.qswg_matrix_market_save(SparseMatrix.of(adjacency)._h, str(path).encode()))


class ResultContainer:
    """qsw::ResultContainer (container.hpp:19-46): `metadata` text plus named
    float64 arrays; `write`/`read` use the QSWBOX v1 bytes of the reference."""

    def __init__(self, metadata: str = "", arrays=None):
        self.metadata = metadata
        self.arrays = dict(arrays or {})

    def _handle(self):
        h = C.c_void_p()
        check(lib.qswg_container_create(C.byref(h)))
        try:
            m = self.metadata.encode() if isinstance(self.metadata, str) else bytes(self.metadata)
            check(lib.qswg_container_set_metadata(h, m, len(m)))
            for name, a in self.arrays.items():
                a = np.array(a, dtype=np.float64, order="C")  # keeps 0-d arrays 0-d
                shape = np.asarray(a.shape, np.int64)
                check(lib.qswg_container_put_array(h, str(name).encode(), a.ndim, _i64p(shape), _dp(a)))
        except Exception:
            lib.qswg_container_destroy(h)
            raise
        return h

    @staticmethod
    def _from_handle(h) -> "ResultContainer":
        n = C.c_int64()
        check(lib.qswg_container_get_metadata(h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(max(n.value, 1))
        check(lib.qswg_container_get_metadata(h, buf, n.value, C.byref(n)))
        out = ResultContainer(buf.raw[: n.value].decode(errors="replace"))
        check(lib.qswg_container_array_count(h, C.byref(n)))
        for k in range(n.value):
            nl, rank = C.c_int64(), C.c_int64()
            check(lib.qswg_container_array_info(h, k, None, 0, C.byref(nl), C.byref(rank), None, 0))
            name = C.create_string_buffer(max(nl.value, 1))
            shape = np.zeros(max(rank.value, 1), np.int64)
            check(lib.qswg_container_array_info(h, k, name, nl.value, C.byref(nl), C.byref(rank),
                                                _i64p(shape), rank.value))
            shp = tuple(int(d) for d in shape[: rank.value])
            data = np.zeros(int(np.prod(shp)) if shp else 1)
            check(lib.qswg_container_array_data(h, k, _dp(data)) if data.size else 0)
            out.arrays[name.raw[: nl.value].decode(errors="replace")] = data.reshape(shp)
        return out

    def write(self, path) -> None:
        """write_container (container.hpp:48)."""
        h = self._handle()
        try:
            check(lib.qswg_container_write(h, str(path).encode()))
        finally:
            lib.qswg_container_destroy(h)

    @staticmethod
    def read(path) -> "ResultContainer":
        """read_container (container.hpp:49): FileFormatError on bad magic,
        version, checksum or section layout."""
        h = C.c_void_p()
        check(lib.qswg_container_read(str(path).encode(), C.byref(h)))
        try:
            return ResultContainer._from_handle(h)
        finally:
            lib.qswg_container_destroy(h)

    def emit_plot_data(self, quantity: str, path) -> None:
        """emit_plot_data (container.hpp:51-56): one text row per time."""
        h = self._handle()
        try:
            check(lib.qswg_container_plot_data(h, quantity.encode(), str(path).encode()))
        finally:
            lib.qswg_container_destroy(h)


# -------------------------------------------------------------- multi-GPU
def plan_rows(n: int, colptr, world: int) -> np.ndarray:
    """Row partition on rho-column boundaries balanced by nnz (host planner)."""
    cp = np.ascontiguousarray(colptr, dtype=np.int64)
    out = np.zeros(world + 1, np.int64)
    check(lib.qswg_plan_rows(n, _i64p(cp), world, _i64p(out)))
    return out


def plan_halo(cols, starts, rank: int):
    """Per-peer hull [lo, hi) of the columns a rank's block references."""
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    st = np.ascontiguousarray(starts, dtype=np.int64)
    world = len(st) - 1
    lo, hi = np.zeros(world, np.int64), np.zeros(world, np.int64)
    check(lib.qswg_plan_halo(_i64p(cols) if cols.size else None, cols.size, _i64p(st), world, rank,
                             _i64p(lo), _i64p(hi)))
    return lo, hi

class Comm:
    """NCCL communicator for one rank (qswg_comm_*); one process per GPU."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.qswg_comm_destroy(h)
            self._h = None

    @staticmethod
    def unique_id() -> bytes:
        n = lib.qswg_comm_unique_id_size()
        buf = (C.c_uint8 * n)()
        check(lib.qswg_comm_get_unique_id(buf))
        return bytes(buf)

    @staticmethod
    def from_unique_id(uid: bytes, rank: int, world: int, device: int) -> "Comm":
        buf = (C.c_uint8 * len(uid)).from_buffer_copy(uid)
        h = C.c_void_p()
        check(lib.qswg_comm_create(buf, rank, world, device, C.byref(h)))
        return Comm(h)

    @staticmethod
    def local_group(world: int) -> list:
        """`world` linked in-process communicators (one per host thread)."""
        arr = (C.c_void_p * world)()
        check(lib.qswg_comm_create_local(world, arr))
        return [Comm(C.c_void_p(arr[r])) for r in range(world)]

    @staticmethod
    def create(rank: int, world: int, device: int) -> "Comm":
        """Rendezvous through an initialised torch.distributed process group."""
        import torch.distributed as dist
        obj = [Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return Comm.from_unique_id(obj[0], rank, world, device)


# ------------------------------------------------------------------- walk
class WalkSystem:
    """walk.hpp:28-101 for the L-QSW / G-QSW paths (one GPU or one rank)."""

    def __init__(self):
        self._initial = None
        self._result = None

    @staticmethod
    def lqsw(omega, h, m_l, sources=(), sinks=(), device=0, group=0, comm=None) -> "WalkSystem":
        w = WalkSystem()
        w.kind, w._omega = "local", float(omega)
        w._h, w._ops, w._src, w._snk = SparseMatrix.of(h), [SparseMatrix.of(m_l)], list(sources), list(sinks)
        w._h_rot = None
        w._dev = (device, group, comm)
        w._rebuild()
        return w

    @staticmethod
    def gqsw(omega, h, lindblads, h_rot=None, vsets=None, device=0, group=0, comm=None) -> "WalkSystem":
        """Pass both h_rot and vsets (subspace dims) for the non-moralising
        walk, neither for the plain one (walk.hpp:43-48)."""
        if (h_rot is None) != (vsets is None):
            raise ValueError("non-moralising walks need both the rotating Hamiltonian and the vertex subspaces")
        w = WalkSystem()
        w.kind, w._omega = "global", float(omega)
        w._h, w._ops, w._src, w._snk = SparseMatrix.of(h), [SparseMatrix.of(x) for x in lindblads], [], []
        w._h_rot = SparseMatrix.of(h_rot) if h_rot is not None else None
        w._vsets = None if vsets is None else np.asarray(vsets, np.int64)
        if w._vsets is not None and int(w._vsets.sum()) != w._h.shape[0]:
            raise ValueError("vertex subspaces do not match the operator dimension")
        w._dev = (device, group, comm)
        w._rebuild()
        return w

    def _rebuild(self):
        d, g, c = self._dev
        if self.kind == "local":
            self.liouvillian = build_local(self._omega, self._h, self._ops[0], self._src, self._snk, d, g, c)
        else:
            self.liouvillian = build_global(self._omega, self._h, self._ops, self._h_rot, d, g, c)

    omega = property(lambda self: self._omega)
    dimension = property(lambda self: self.liouvillian.n)
    _vsets = None

    def measured_vertex_count(self) -> int:  # walk.hpp:55
        return len(self._vsets) if self._vsets is not None else self.liouvillian.n

    def initial_state(self, rho):
        """Probabilities (walk.cpp:101-126) or a dense Hermitian unit-trace rho (128-139)."""
        rho = np.asarray(rho)
        n = self.liouvillian.n
        s = StateVector(self.liouvillian)
        if rho.ndim == 1:
            p = rho.astype(np.float64)
            if self._vsets is not None and len(p) == len(self._vsets):
                p = nm_rho_map(p, self._vsets)  # walk.cpp:103-105
            if self.kind == "local" and len(p) < n and len(p) == n - len(self._src) - len(self._snk):
                p = np.concatenate([p, np.zeros(n - len(p))])
            s.from_probabilities(p)
        else:
            if rho.shape != (n, n):
                raise ValueError("density matrix dimension does not match the walk")
            if abs(np.trace(rho) - 1.0) > 1e-12:
                raise ValueError("density matrix must have unit trace")
            if np.abs(rho - rho.conj().T).max() > 1e-12:
                raise ValueError("density matrix must be Hermitian")
            s.upload(np.asarray(rho, np.complex128).T.reshape(-1))  # column-major vec
        self._initial, self._result = s, None

    def set_omega(self, omega):
        if not (0.0 <= omega <= 1.0):
            raise ValueError("omega must be in [0, 1]")
        self._omega = float(omega)
        self.liouvillian.set_omega(omega)  # walk.cpp:141-145; the states stay on the device

    def step(self, t, tolerance=DOUBLE_TOL):
        if self._initial is None:
            raise LogicError("no initial state: call initial_state first")
        self._result, info = step(self.liouvillian, self._initial, t, tolerance)
        return info

    def series(self, t1, tq, steps, tolerance=DOUBLE_TOL, states=False, coherence=False):
        if self._initial is None:
            raise LogicError("no initial state: call initial_state first")
        r = series(self.liouvillian, self._initial, t1, tq, steps, tolerance, True, states, True,
                   coherence=coherence)
        self._result = r.final
        if self._vsets is not None:
            r.populations = np.stack([nm_measure(p, self._vsets) for p in r.populations])
        return r

    def _current(self):
        if self._result is not None:
            return self._result
        if self._initial is not None:
            return self._initial
        raise LogicError("no state available: call initial_state first")

    def gather_result(self) -> np.ndarray:
        n = self.liouvillian.n
        return self._current().gather().reshape(n, n).T  # unvec (state.cpp:37-44)

    def gather_populations(self) -> np.ndarray:
        return self.populations_of(self._current())

    def populations_of(self, state: StateVector) -> np.ndarray:
        """Vertex populations; NM walks are folded back onto the original
        vertices (walk.cpp:177-186)."""
        p = state.populations()
        return nm_measure(p, self._vsets) if self._vsets is not None else p
