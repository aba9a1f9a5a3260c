"""ctypes binding of libqswg.so (include/qswg.h).

The shared library is built in-tree by __graft_entry__.build() (make -C
paper_2003_02450_b200/csrc).  Importing this module without it raises
immediately: there is no CPU fallback for the product path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QSWG_LIB_PATH") or os.path.join(HERE, "libqswg.so")  # override: kernel experiments

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(qswg has no CPU fallback)")

lib = C.CDLL(LIB_PATH)

i64 = C.c_int64
i64p = C.POINTER(C.c_int64)
dp = C.POINTER(C.c_double)
vp = C.c_void_p

OK, EINVAL, ERANGE, ENUMERICAL, ESTATE, ECUDA, ENCCL, ENOMEM, EINTERNAL = 0, 1, 2, 3, 4, 5, 6, 7, 9
EFORMAT, EIO = 10, 11


class QswgError(RuntimeError):
    code = EINTERNAL


class NumericalError(QswgError, ArithmeticError):
    """qsw::NumericalError (expm.hpp:13-17)."""
    code = ENUMERICAL


class CudaError(QswgError):
    code = ECUDA


class InvalidArgument(QswgError, ValueError):
    code = EINVAL


class OutOfRange(QswgError, IndexError):
    code = ERANGE


class LogicError(QswgError):
    code = ESTATE


class FileFormatError(QswgError):
    """qsw::FileFormatError (graph.hpp:11-15)."""
    code = EFORMAT


class IoError(QswgError, OSError):
    """qsw::IoError (container.hpp:13-17)."""
    code = EIO


_EXC = {EINVAL: InvalidArgument, ERANGE: OutOfRange, ENUMERICAL: NumericalError,
        ESTATE: LogicError, ECUDA: CudaError, ENCCL: CudaError, ENOMEM: MemoryError,
        EFORMAT: FileFormatError, EIO: IoError}


def check(rc: int):
    if rc != OK:
        msg = lib.qswg_last_error().decode(errors="replace")
        exc = _EXC.get(rc, QswgError)
        raise exc(msg)


class SourceArc(C.Structure):
    _fields_ = [("target", i64), ("rate", C.c_double)]


class SinkArc(C.Structure):
    _fields_ = [("origin", i64), ("rate", C.c_double)]


class DeviceConfig(C.Structure):
    _fields_ = [("device", C.c_int), ("group", C.c_int), ("format", C.c_int), ("comm", vp)]


class LiouvillianInfo(C.Structure):
    _fields_ = [("n", i64), ("dim", i64), ("nnz", i64), ("nnz_local", i64), ("row0", i64), ("rows", i64),
                ("omega", C.c_double), ("one_norms", C.c_double * 9),
                ("group", C.c_int), ("device", C.c_int), ("rank", C.c_int), ("world", C.c_int),
                ("format", C.c_int), ("padding", C.c_double), ("kron_factored", C.c_int), ("kron_ell", C.c_int),
                ("kron_term_vectors", C.c_int), ("sell_panels", C.c_int), ("kron_hermitian", C.c_int),
                ("kron_staged", C.c_int), ("sell_fused", C.c_int)]


class StepInfo(C.Structure):
    _fields_ = [("m_star", i64), ("s", i64), ("spmvs", i64), ("launches", i64)]


class SeriesInfo(C.Structure):
    _fields_ = [("path", C.c_int), ("span_m_star", i64), ("span_s", i64), ("d", i64), ("n_super", i64),
                ("remainder", i64), ("sub_m_star", i64), ("spmvs", i64), ("launches", i64),
                ("device_ms", C.c_double), ("host_waits", i64)]


# Every symbol include/qswg.h declares, with its ctypes signature.
SIGNATURES = {
    "qswg_last_error": (C.c_char_p, []),
    "qswg_version": (C.c_int, [C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "qswg_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "qswg_host_alloc": (C.c_int, [i64, C.POINTER(vp)]),
    "qswg_host_free": (None, [vp]),
    "qswg_sparse_from_triplets": (C.c_int, [i64, i64, i64, i64p, i64p, dp, C.POINTER(vp)]),
    "qswg_sparse_from_csr": (C.c_int, [i64, i64, i64p, i64p, dp, C.POINTER(vp)]),
    "qswg_sparse_shape": (C.c_int, [vp, i64p, i64p, i64p]),
    "qswg_sparse_export": (C.c_int, [vp, i64p, i64p, dp]),
    "qswg_sparse_destroy": (None, [vp]),
    "qswg_symmetrize": (C.c_int, [vp, C.POINTER(vp)]),
    "qswg_generator_matrix": (C.c_int, [C.c_double, vp, C.POINTER(vp)]),
    "qswg_markov_chain_matrix": (C.c_int, [vp, C.POINTER(vp)]),
    "qswg_local_lindblad": (C.c_int, [vp, C.POINTER(vp)]),
    "qswg_augment": (C.c_int, [vp, C.POINTER(SourceArc), i64, C.POINTER(SinkArc), i64, C.POINTER(vp)]),
    "qswg_nm_vsets": (C.c_int, [vp, i64p]),
    "qswg_nm_H": (C.c_int, [C.c_double, vp, i64p, i64, C.POINTER(vp)]),
    "qswg_nm_L": (C.c_int, [C.c_double, vp, i64p, i64, C.POINTER(vp)]),
    "qswg_nm_H_rot": (C.c_int, [i64p, i64, C.c_int, C.POINTER(vp)]),
    "qswg_nm_rho_map": (C.c_int, [dp, i64p, i64, dp]),
    "qswg_nm_measure": (C.c_int, [dp, i64p, i64, dp]),
    "qswg_build_local": (C.c_int, [C.c_double, vp, vp, C.POINTER(SourceArc), i64, C.POINTER(SinkArc), i64,
                                   C.POINTER(DeviceConfig), C.POINTER(vp)]),
    "qswg_build_global": (C.c_int, [C.c_double, vp, C.POINTER(vp), i64, vp, C.POINTER(DeviceConfig),
                                    C.POINTER(vp)]),
    "qswg_liouvillian_query": (C.c_int, [vp, C.POINTER(LiouvillianInfo)]),
    "qswg_liouvillian_download": (C.c_int, [vp, i64p, i64p, dp]),
    "qswg_liouvillian_destroy": (None, [vp]),
    "qswg_spmv": (C.c_int, [vp, dp, dp]),
    "qswg_time_spmv": (C.c_int, [vp, C.c_int, C.c_int, dp]),
    "qswg_time_series_term": (C.c_int, [vp, C.c_int, C.c_int, dp]),
    "qswg_time_series_parts": (C.c_int, [vp, C.c_int, C.c_int, dp]),
    "qswg_liouvillian_set_hermitian_mode": (C.c_int, [vp, C.c_int]),
    "qswg_liouvillian_stream": (C.c_int, [vp, C.POINTER(vp)]),
    "qswg_state_create": (C.c_int, [vp, C.POINTER(vp)]),
    "qswg_state_upload": (C.c_int, [vp, dp]),
    "qswg_state_from_probabilities": (C.c_int, [vp, dp, i64]),
    "qswg_state_download": (C.c_int, [vp, dp]),
    "qswg_state_populations": (C.c_int, [vp, dp]),
    "qswg_state_destroy": (None, [vp]),
    "qswg_theta_table": (C.c_int, [C.c_double, dp]),
    "qswg_select_parameters": (C.c_int, [dp, C.c_double, C.c_double, i64p, i64p]),
    "qswg_step": (C.c_int, [vp, vp, C.c_double, C.c_double, vp, C.POINTER(StepInfo)]),
    "qswg_series": (C.c_int, [vp, vp, C.c_double, C.c_double, i64, C.c_double, dp, dp, vp,
                              C.POINTER(SeriesInfo)]),
    "qswg_series_observe": (C.c_int, [vp, vp, C.c_double, C.c_double, i64, C.c_double, dp, dp, dp, vp,
                                      C.POINTER(SeriesInfo)]),
    "qswg_state_coherence": (C.c_int, [vp, dp]),
    "qswg_liouvillian_set_omega": (C.c_int, [vp, C.c_double]),
    "qswg_matrix_market_parse": (C.c_int, [C.c_char_p, i64, C.POINTER(vp)]),
    "qswg_matrix_market_load": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "qswg_matrix_market_save": (C.c_int, [vp, C.c_char_p]),
    "qswg_container_create": (C.c_int, [C.POINTER(vp)]),
    "qswg_container_destroy": (None, [vp]),
    "qswg_container_set_metadata": (C.c_int, [vp, C.c_char_p, i64]),
    "qswg_container_get_metadata": (C.c_int, [vp, C.c_char_p, i64, i64p]),
    "qswg_container_put_array": (C.c_int, [vp, C.c_char_p, i64, i64p, dp]),
    "qswg_container_array_count": (C.c_int, [vp, i64p]),
    "qswg_container_array_info": (C.c_int, [vp, i64, C.c_char_p, i64, i64p, i64p, i64p, i64]),
    "qswg_container_array_data": (C.c_int, [vp, i64, dp]),
    "qswg_container_write": (C.c_int, [vp, C.c_char_p]),
    "qswg_container_read": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "qswg_container_plot_data": (C.c_int, [vp, C.c_char_p, C.c_char_p]),
    "qswg_plan_rows": (C.c_int, [i64, i64p, C.c_int, i64p]),
    "qswg_plan_halo": (C.c_int, [i64p, i64, i64p, C.c_int, C.c_int, i64p, i64p]),
    "qswg_liouvillian_partition": (C.c_int, [vp, i64p, i64p, i64p]),
    "qswg_comm_unique_id_size": (C.c_int, []),
    "qswg_comm_get_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "qswg_comm_create": (C.c_int, [C.POINTER(C.c_uint8), C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    "qswg_comm_destroy": (None, [vp]),
    "qswg_comm_create_local": (C.c_int, [C.c_int, C.POINTER(vp)]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args
