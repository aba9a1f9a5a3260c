"""One declarative walk run -> ResultContainer, on the device.

The B200 counterpart of qsw::run (proj/core/src/run.cpp:88-171) for the
callers either side of the hot path: Matrix Market
graph in (libqswg's parser, graph.cpp:54-136), operators as run.cpp:40-68
builds them, the series / step on the GPU, and a QSWBOX container out whose
arrays and metadata keys are the reference's.  Populations and coherence
norms are computed on the device at every output time, so a series never
brings its states back to the host (the reference gathers every full state,
run.cpp:114-133); only `full_rho` downloads the final state.

The JSON/CLI front end (config.cpp, tools/qsw) is out of scope: a RunConfig
is built directly, with the fields, validation and `describe()` text of
config.hpp:31-64 / config.cpp:111-155.
"""
from __future__ import annotations

import dataclasses
import os
import re
import time

import numpy as np

from . import api

VERSION_STRING = "0.1.0"  # version.hpp:9: the metadata names the reference version it mirrors


class ConfigError(RuntimeError):
    """qsw::ConfigError (config.hpp:13-17)."""


_KINDS = ("local", "global", "nm_global")
_NUMBER = re.compile(r"[+-]?(\d+\.?\d*|\.\d+)([eE][+-]?\d+)?")


def _g(x: float) -> str:
    """std::ostream << double with default flags (%g, precision 6)."""
    return "%g" % x


@dataclasses.dataclass
class RunConfig:
    """config.hpp:31-64 (time: `t` for a single point, or t1/tq/steps)."""
    graph_path: str = ""
    walk_kind: str = "local"
    omega: float = 0.0
    gamma: float = 1.0
    is_series: bool = False
    t: float = 0.0
    t1: float = 0.0
    tq: float = 0.0
    steps: int = 0
    initial_kind: str = "mixed"  # mixed | vertex | file
    initial_vertex: int = 0
    initial_file: str = ""
    sources: list = dataclasses.field(default_factory=list)  # [(target, rate)]
    sinks: list = dataclasses.field(default_factory=list)    # [(origin, rate)]
    workers: int = 1
    out_populations: bool = True
    out_full_rho: bool = False
    out_coherence_norm: bool = False

    def validate(self) -> None:
        """config.cpp:111-127."""
        if not self.graph_path:
            raise ConfigError("no graph file given")
        if not os.path.exists(self.graph_path):
            raise ConfigError(f"graph file `{self.graph_path}` does not exist")
        if self.walk_kind not in _KINDS:
            raise ConfigError(f"unknown walk kind `{self.walk_kind}` (expected local, global or nm_global)")
        if not (0.0 <= self.omega <= 1.0):
            raise ConfigError("omega must lie in [0, 1]")
        if not (self.gamma > 0.0):
            raise ConfigError("gamma must be positive")
        if self.workers < 1:
            raise ConfigError("workers must be at least 1")
        if self.is_series:
            if not (self.tq > self.t1):
                raise ConfigError("series requires tq > t1")
            if self.steps < 1:
                raise ConfigError("series requires steps >= 1")
        if self.walk_kind != "local" and (self.sources or self.sinks):
            raise ConfigError("sources/sinks are only supported for local walks")

    def describe(self) -> str:
        """One `key = value` line per field (config.cpp:129-155)."""
        out = [f"walk = {self.walk_kind}", f"graph = {self.graph_path}", f"omega = {_g(self.omega)}",
               f"gamma = {_g(self.gamma)}"]
        if self.is_series:
            out.append(f"time = series t1 = {_g(self.t1)} tq = {_g(self.tq)} steps = {self.steps}")
        else:
            out.append(f"time = single t = {_g(self.t)}")
        if self.initial_kind == "mixed":
            out.append("initial_state = mixed")
        elif self.initial_kind == "vertex":
            out.append(f"initial_state = vertex {self.initial_vertex}")
        else:
            out.append(f"initial_state = file {self.initial_file}")
        out += [f"source = {t} rate {_g(r)}" for t, r in self.sources]
        out += [f"sink = {o} rate {_g(r)}" for o, r in self.sinks]
        out.append(f"workers = {self.workers}")
        return "".join(line + "\n" for line in out)


def _resized(m: api.SparseMatrix, n: int) -> api.SparseMatrix:
    """SparseMatrix::resized: the same entries in an n x n matrix."""
    c = m.to_csr()
    ip = np.concatenate([c.indptr, np.full(n - c.rows, c.indptr[-1], np.int64)])
    return api.SparseMatrix.from_csr(api.Csr(n, n, ip, c.indices, c.data))


def make_walk(config: RunConfig, g: api.SparseMatrix, device=0, group=0, comm=None) -> api.WalkSystem:
    """Operators exactly as run.cpp:40-68 builds them."""
    gu = api.symmetrize(g)
    if config.walk_kind == "local":
        h = api.generator_matrix(config.gamma, gu)
        m_l = api.local_lindblad(api.generator_matrix(config.gamma, g))
        total = g.shape[0] + len(config.sources) + len(config.sinks)
        return api.WalkSystem.lqsw(config.omega, _resized(h, total), _resized(m_l, total),
                                   config.sources, config.sinks, device=device, group=group, comm=comm)
    if config.walk_kind == "global":
        return api.WalkSystem.gqsw(config.omega, api.generator_matrix(config.gamma, gu),
                                   [api.global_lindblad(g)], device=device, group=group, comm=comm)
    dims = api.nm_vsets(gu)
    return api.WalkSystem.gqsw(config.omega, api.nm_H(config.gamma, gu, dims), [api.nm_L(config.gamma, g, dims)],
                               api.nm_H_rot(dims), dims, device=device, group=group, comm=comm)


def load_probability_file(path) -> np.ndarray:
    """run.cpp:27-35: whitespace-separated doubles."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise api.IoError(f"cannot open initial state file `{path}`") from None
    p = []
    for tok in text.split():
        m = _NUMBER.match(tok)  # what `in >> x` accepts: no inf/nan words
        if m is None:
            break  # `in >> x` stops at the first token that is not a number
        if re.match(r"[eE][+-]?(?![0-9])", tok[m.end():]):
            break  # an exponent without digits ("1e", "1e+"): libstdc++ fails the whole extraction
        p.append(float(m.group(0)))
        if m.end() != len(tok):
            break  # a number followed by junk: the stream fails on the junk
    if not p:
        raise api.FileFormatError(f"initial state file `{path}` is empty")
    return np.asarray(p)


def make_initial(config: RunConfig, n_base: int) -> np.ndarray:
    """run.cpp:70-86."""
    if config.initial_kind == "mixed":
        return np.full(n_base, 1.0 / n_base)
    if config.initial_kind == "vertex":
        if config.initial_vertex >= n_base:
            raise ConfigError("initial vertex out of range")
        p = np.zeros(n_base)
        p[config.initial_vertex] = 1.0
        return p
    return load_probability_file(config.initial_file)


def run(config: RunConfig, device: int = 0, group: int = 0, comm=None) -> api.ResultContainer:
    """qsw::run (run.cpp:88-171) with the evolution on the GPU."""
    config.validate()
    g = api.load_matrix_market(config.graph_path)
    walk = make_walk(config, g, device, group, comm)
    walk.initial_state(make_initial(config, g.shape[0]))
    out = api.ResultContainer()

    if config.is_series:
        r = walk.series(config.t1, config.tq, config.steps, coherence=config.out_coherence_norm)
        times, t_final = r.times, config.tq
        pops, coh = r.populations, r.coherence
    else:
        walk.step(config.t)
        times, t_final = np.array([config.t]), config.t
        pops = walk.gather_populations()[None, :] if config.out_populations else None
        coh = np.array([walk._current().coherence()]) if config.out_coherence_norm else None
    out.arrays["times"] = np.asarray(times, np.float64)
    if config.out_populations:
        out.arrays["populations"] = np.asarray(pops, np.float64).reshape(len(times), walk.measured_vertex_count())
    if config.out_coherence_norm:
        out.arrays["coherence_norm"] = np.asarray(coh, np.float64)
    if config.out_full_rho:
        rho = walk.gather_result()
        out.arrays["rho_re"] = np.ascontiguousarray(rho.real)
        out.arrays["rho_im"] = np.ascontiguousarray(rho.imag)

    # run.cpp:151-169: parameter diagnostics for the final-time exponential
    norms = walk.liouvillian.one_norms()
    m_star, s = api.select_parameters(norms, t_final)
    out.metadata = (f"qsw_version = {VERSION_STRING}\n"
                    f"timestamp_unix = {int(time.time())}\n"
                    + config.describe()
                    + f"liouvillian_dim = {walk.liouvillian.dim}\n"
                    f"liouvillian_one_norm = {_g(norms[0])}\n"
                    f"taylor_m_star = {m_star}\n"
                    f"taylor_s = {s}\n")
    return out
