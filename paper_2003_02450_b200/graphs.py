"""Seeded synthetic workloads for the BASELINE.json configs.

Pure data: each workload is a graph plus the operators the reference's
library API would be called with (WalkSystem::lqsw / gqsw, walk.hpp:39-48),
built with the reference's own definitions:

* generator_matrix(gamma, G): M_ij = -gamma*G_ij, M_jj = gamma*OutDeg(j)
  (graph.cpp:193-211) -- for an undirected graph, gamma * Laplacian;
* markov_chain_matrix(G): C_ij = 1/OutDeg(j) wherever an arc j->i exists
  (graph.cpp:217-228);
* symmetrize(G): w_ij = w_ji = max of the two (graph.cpp:152-173).

Index convention (graph.hpp:32-41): column j holds the out-arcs of vertex j.
There is no public dataset for this path; every graph is generated from a
fixed seed with numpy's PCG64, so the oracle and the device see identical
inputs on any host.
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass
class Csr:
    """Canonical complex128 CSR: sorted columns, summed duplicates, no zeros."""

    rows: int
    cols: int
    indptr: np.ndarray  # int64 [rows+1]
    indices: np.ndarray  # int64 [nnz]
    data: np.ndarray  # complex128 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    @staticmethod
    def from_coo(rows, cols, r, c, v) -> "Csr":
        r = np.asarray(r, dtype=np.int64)
        c = np.asarray(c, dtype=np.int64)
        v = np.asarray(v, dtype=np.complex128)
        order = np.lexsort((c, r))
        r, c, v = r[order], c[order], v[order]
        if len(r):
            key = r * cols + c
            first = np.ones(len(key), dtype=bool)
            first[1:] = key[1:] != key[:-1]
            grp = np.cumsum(first) - 1
            vs = np.zeros(int(first.sum()), dtype=np.complex128)
            np.add.at(vs, grp, v)
            r, c, v = r[first], c[first], vs
            keep = v != 0
            r, c, v = r[keep], c[keep], v[keep]
        indptr = np.zeros(rows + 1, dtype=np.int64)
        np.add.at(indptr, r + 1, 1)
        return Csr(rows, cols, np.cumsum(indptr), c, v)

    def row_of(self) -> np.ndarray:
        return np.repeat(np.arange(self.rows, dtype=np.int64), np.diff(self.indptr))

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.rows, self.cols), dtype=np.complex128)
        d[self.row_of(), self.indices] = self.data
        return d

    def transpose(self) -> "Csr":
        return Csr.from_coo(self.cols, self.rows, self.indices, self.row_of(), self.data)


# --- reference operator definitions (numpy restatements, see module doc) ---

def generator_matrix(gamma: float, adj: Csr) -> Csr:
    cs = np.zeros(adj.cols)
    np.add.at(cs, adj.indices, adj.data.real)
    r = adj.row_of()
    diag = np.nonzero(cs != 0.0)[0]
    rr = np.concatenate([r, diag])
    cc = np.concatenate([adj.indices, diag])
    vv = np.concatenate([-gamma * adj.data.real, gamma * cs[diag]]).astype(np.complex128)
    return Csr.from_coo(adj.rows, adj.cols, rr, cc, vv)


def markov_chain_matrix(adj: Csr) -> Csr:
    deg = np.zeros(adj.cols)
    np.add.at(deg, adj.indices, adj.data.real)
    return Csr.from_coo(adj.rows, adj.cols, adj.row_of(), adj.indices,
                        1.0 / deg[adj.indices])


def symmetrize(adj: Csr) -> Csr:
    t = adj.transpose()
    r = np.concatenate([adj.row_of(), t.row_of()])
    c = np.concatenate([adj.indices, t.indices])
    v = np.concatenate([adj.data.real, t.data.real])
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    key = r * adj.cols + c
    first = np.ones(len(key), dtype=bool)
    first[1:] = key[1:] != key[:-1]
    grp = np.cumsum(first) - 1
    vm = np.full(int(first.sum()), -np.inf)
    np.maximum.at(vm, grp, v)
    return Csr.from_coo(adj.rows, adj.cols, r[first], c[first], vm)


# --- graphs ---------------------------------------------------------------

def _undirected(n, edges) -> Csr:
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    e = e[e[:, 0] != e[:, 1]]
    r = np.concatenate([e[:, 0], e[:, 1]])
    c = np.concatenate([e[:, 1], e[:, 0]])
    key = np.unique(r * n + c)
    return Csr.from_coo(n, n, key // n, key % n, np.ones(len(key)))


def cycle_graph(n: int) -> Csr:
    i = np.arange(n)
    return _undirected(n, np.stack([i, (i + 1) % n], axis=1))


def torus2d(side: int) -> Csr:
    """Periodic square lattice, vertex id y*side + x."""
    y, x = np.divmod(np.arange(side * side), side)
    right = y * side + (x + 1) % side
    down = ((y + 1) % side) * side + x
    v = np.arange(side * side)
    return _undirected(side * side, np.concatenate([np.stack([v, right], 1), np.stack([v, down], 1)]))


def torus3d(side: int) -> Csr:
    """Periodic cubic lattice, vertex id (z*side + y)*side + x."""
    v = np.arange(side ** 3)
    z, rem = np.divmod(v, side * side)
    y, x = np.divmod(rem, side)
    idx = lambda zz, yy, xx: (zz * side + yy) * side + xx  # noqa: E731
    nb = [idx(z, y, (x + 1) % side), idx(z, (y + 1) % side, x), idx((z + 1) % side, y, x)]
    return _undirected(side ** 3, np.concatenate([np.stack([v, b], 1) for b in nb]))


def er_graph(n: int, p: float, seed: int) -> Csr:
    """Undirected G(n, p), unit weights."""
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, k=1)
    keep = rng.random(len(iu)) < p
    return _undirected(n, np.stack([iu[keep], ju[keep]], 1))


def er_digraph_weighted(n: int, p: float, seed: int) -> Csr:
    """Directed G(n, p) over ordered pairs i != j, weights 1 - U[0,1) in (0, 1];
    a vertex with no out-arc gets one random out-arc (BASELINE config 3)."""
    rng = np.random.default_rng(seed)
    src, dst = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    src, dst = src.ravel(), dst.ravel()
    off = src != dst
    src, dst = src[off], dst[off]
    keep = rng.random(len(src)) < p
    src, dst = src[keep], dst[keep]
    w = 1.0 - rng.random(len(src))
    outdeg = np.bincount(src, minlength=n)
    lonely = np.nonzero(outdeg == 0)[0]
    extra_dst = rng.integers(0, n - 1, size=len(lonely))
    extra_dst = extra_dst + (extra_dst >= lonely)  # skip the self-loop
    src = np.concatenate([src, lonely])
    dst = np.concatenate([dst, extra_dst])
    w = np.concatenate([w, 1.0 - rng.random(len(lonely))])
    # arc j -> i is entry (row i, col j)
    return Csr.from_coo(n, n, dst, src, w)


def column_normalised(adj: Csr) -> Csr:
    """M_ij = w_ij / OutDeg_j (BASELINE config 3's weighted Markov matrix)."""
    deg = np.zeros(adj.cols)
    np.add.at(deg, adj.indices, adj.data.real)
    return Csr.from_coo(adj.rows, adj.cols, adj.row_of(), adj.indices,
                        adj.data.real / deg[adj.indices])


# --- workloads --------------------------------------------------------------

@dataclasses.dataclass
class Workload:
    name: str
    kind: str  # "local" (L-QSW) or "global" (G-QSW)
    n: int
    omega: float
    h: Csr
    ops: list  # [m_l] for local, Lindblad list for global
    rho0: np.ndarray  # vertex probabilities (diagonal rho(0))
    t1: float
    tq: float
    steps: int
    seed: int | None = None

    @property
    def dim(self) -> int:
        return self.n * self.n


def _point(n, i):
    p = np.zeros(n)
    p[i] = 1.0
    return p


def config(name: str, omega: float | None = None, size: int | None = None) -> Workload:
    """BASELINE.json configs c1..c5; `size` shrinks the graph for parity cases
    (cycle length, torus side, ER vertex count) keeping every other setting."""
    if name == "c1":
        n = size or 64
        g = cycle_graph(n)
        return Workload("c1", "local", n, 0.5 if omega is None else omega,
                        generator_matrix(1.0, g), [markov_chain_matrix(g)],
                        _point(n, 0), 0.0, 10.0, 20)
    if name == "c2":
        side = size or 32
        g = torus2d(side)
        n = side * side
        centre = (side // 2) * side + side // 2
        return Workload("c2", "global", n, 0.1 if omega is None else omega,
                        generator_matrix(1.0, g), [markov_chain_matrix(g)],
                        _point(n, centre), 0.0, 20.0, 100)
    if name == "c3":
        n = size or 2048
        seed = 12345
        g = er_digraph_weighted(n, 0.005 if size is None else min(1.0, 10.0 / n), seed)
        return Workload("c3", "local", n, 0.5 if omega is None else omega,
                        generator_matrix(1.0, symmetrize(g)), [column_normalised(g)],
                        _point(n, 0), 0.0, 50.0, 50, seed)
    if name == "c4":
        n = size or 4096
        seed = 4096
        g = er_graph(n, 8.0 / (n - 1), seed)
        p = np.zeros(n)
        p[:16] = 1.0 / 16
        return Workload("c4", "global", n, 0.5 if omega is None else omega,
                        generator_matrix(1.0, g), [markov_chain_matrix(g)],
                        p, 0.0, 5.0, 20, seed)
    if name == "c5":
        side = size or 24
        g = torus3d(side)
        n = side ** 3
        return Workload("c5", "local", n, 0.3 if omega is None else omega,
                        generator_matrix(1.0, g), [markov_chain_matrix(g)],
                        _point(n, 0), 0.0, 100.0, 200)
    raise ValueError(f"unknown config {name!r}")
