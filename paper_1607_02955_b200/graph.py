"""Graph container and matrix views (reference pkg/src/cfcent/graph.py).

Only the parts on the solve path are provided: the immutable CSR
:class:`Graph` (graph.py:30-147), ``laplacian`` (:253-258),
``incidence_and_weights`` (:261-276) and ``largest_connected_component``
(:217-250).  Edge-list parsing and the noise experiment are out of scope
(SURVEY.md §2 rows 4, 8, 9).

Besides the reference views, :func:`edge_index_view` produces the device
upload format of the JL right-hand sides: per adjacency entry the canonical
(u<v, sorted) edge id, plus sqrt(w) per edge.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

from .errors import DomainError

__all__ = ["Graph", "check_connected", "largest_connected_component", "laplacian", "incidence_and_weights",
           "edge_index_view"]


def _row_ids(indptr: np.ndarray) -> np.ndarray:
    return np.repeat(np.arange(indptr.size - 1, dtype=np.int64), np.diff(indptr))


@dataclass(frozen=True)
class Graph:
    """Undirected weighted graph, sorted CSR adjacency, each edge stored at
    both endpoints with equal weight (graph.py:30-55)."""

    indptr: np.ndarray
    indices: np.ndarray
    weights: np.ndarray
    node_labels: np.ndarray = field(default=None)  # type: ignore[assignment]

    def __post_init__(self):
        if self.node_labels is None:
            object.__setattr__(self, "node_labels", np.arange(self.n, dtype=np.int64))
        for a in (self.indptr, self.indices, self.weights, self.node_labels):
            a.setflags(write=False)

    @property
    def n(self) -> int:
        return self.indptr.size - 1

    @property
    def m(self) -> int:
        return self.indices.size // 2

    def degrees(self) -> np.ndarray:
        return np.bincount(_row_ids(self.indptr), weights=self.weights, minlength=self.n)

    def neighbors(self, u: int):
        lo, hi = self.indptr[u], self.indptr[u + 1]
        return self.indices[lo:hi], self.weights[lo:hi]

    def has_edge(self, u: int, v: int) -> bool:
        nb, _ = self.neighbors(u)
        k = np.searchsorted(nb, v)
        return bool(k < nb.size and nb[k] == v)

    def edge_array(self):
        """(u, v, w) with u < v sorted by (u, v) (graph.py:78-86)."""
        src = _row_ids(self.indptr)
        up = src < self.indices
        return src[up], self.indices[up], self.weights[up]

    def adjacency_matrix(self) -> sp.csr_matrix:
        return sp.csr_matrix((self.weights, (_row_ids(self.indptr), self.indices)),
                             shape=(self.n, self.n))

    def is_connected(self) -> bool:
        if self.n <= 1:
            return True
        return connected_components(self.adjacency_matrix(), directed=False)[0] == 1

    @staticmethod
    def from_edges(u: Sequence[int], v: Sequence[int], w: Sequence[float] | None = None,
                   n: int | None = None, node_labels: np.ndarray | None = None) -> "Graph":
        """Drop self-loops, symmetrise, merge duplicates by summing weights
        (graph.py:100-147)."""
        u = np.asarray(u, dtype=np.int64)
        v = np.asarray(v, dtype=np.int64)
        w = np.ones(u.size) if w is None else np.asarray(w, dtype=np.float64)
        if u.size != v.size or u.size != w.size:
            raise DomainError("endpoint and weight arrays must have equal length")
        if u.size and (np.any(w <= 0) or not np.all(np.isfinite(w))):
            raise DomainError("edge weights must be finite and strictly positive")
        keep = u != v
        if not keep.all():
            u, v, w = u[keep], v[keep], w[keep]
        if n is None:
            n = int(max(u.max(initial=-1), v.max(initial=-1)) + 1)
        if u.size and (min(u.min(), v.min()) < 0 or max(u.max(), v.max()) >= n):
            raise DomainError("node ids out of range")
        # symmetrise, sort neighbours, merge duplicates (graph.py:133-146):
        # native counting sort (csrc/cf_setup.cpp) when no edge repeats
        from . import _native as N

        u = np.ascontiguousarray(u, dtype=np.int64)
        v = np.ascontiguousarray(v, dtype=np.int64)
        w = np.ascontiguousarray(w, dtype=np.float64)
        indptr = np.empty(n + 1, dtype=np.int64)
        dst = np.empty(2 * u.size, dtype=np.int64)
        wt = np.empty(2 * u.size, dtype=np.float64)
        nnz = np.zeros(1, dtype=np.int64)
        if _device_ingest(u.size):
            # large edge lists: stable radix sort of the adjacency entries on
            # the GPU (csrc/cf_graph.cu), the same arrays as the host route
            st = np.zeros(1, dtype=np.int32)
            N.check(N.lib().cf_csr_from_edges_dev(_ingest_device(), n, u.size, N.ptr(u, N.i64p),
                                                  N.ptr(v, N.i64p), N.ptr(w, N.f64p),
                                                  N.ptr(indptr, N.i64p), N.ptr(dst, N.i64p),
                                                  N.ptr(wt, N.f64p), N.ptr(st, N.i32p)))
            if st[0] == 2:
                raise DomainError("node ids out of range")
            nnz[0] = 2 * u.size if st[0] == 0 else -1
        else:
            N.check(N.lib().cf_build_csr(n, u.size, N.ptr(u, N.i64p), N.ptr(v, N.i64p),
                                         N.ptr(w, N.f64p), N.ptr(indptr, N.i64p),
                                         N.ptr(dst, N.i64p), N.ptr(wt, N.f64p),
                                         N.ptr(nnz, N.i64p)))
        if nnz[0] == 2 * u.size:
            dst, wt = dst[:nnz[0]], wt[:nnz[0]]
        else:
            # duplicates were merged: redo with numpy's own reduction so the
            # summed weights match the reference bit-for-bit on this machine
            src = np.concatenate([u, v])
            dst = np.concatenate([v, u])
            wt = np.concatenate([w, w])
            order = np.lexsort((dst, src))
            src, dst, wt = src[order], dst[order], wt[order]
            first = np.empty(src.size, dtype=bool)
            first[0] = True
            np.logical_or(src[1:] != src[:-1], dst[1:] != dst[:-1], out=first[1:])
            starts = np.flatnonzero(first)
            wt = np.add.reduceat(wt, starts)
            src, dst = src[starts], dst[starts]
            indptr = np.zeros(n + 1, dtype=np.int64)
            np.cumsum(np.bincount(src, minlength=n), out=indptr[1:])
        return Graph(indptr=indptr, indices=dst, weights=wt, node_labels=node_labels)


# Edge lists of at least this many edges are sorted / labelled on the GPU when
# one is visible; smaller ones, and any process without
# a device, take the native host route -- both produce identical arrays
# (tests/test_gpu_solver.py::test_device_ingestion_matches_host).
DEVICE_INGEST_MIN_EDGES = 1 << 20


def _device_ingest(m: int) -> bool:
    import os

    if os.environ.get("CF_DEVICE_INGEST", "1") == "0" or m < DEVICE_INGEST_MIN_EDGES:
        return False
    from . import _native as N

    return N.device_available()


def _ingest_device() -> int:
    import os

    return int(os.environ.get("LOCAL_RANK", "0"))


def largest_connected_component(g: Graph):
    """LCC, ties to the component holding the smallest label
    (graph.py:217-250).  Returns (subgraph, {old: new})."""
    if g.n == 0:
        raise DomainError("cannot extract a component of an empty graph")
    eu = ev = ew = None
    if _device_ingest(g.m):
        # component roots (smallest node id per component) from the GPU's
        # hook / pointer-jumping rounds; roots in ascending order number the
        # components exactly as scipy does (first occurrence)
        from . import _native as N

        eu, ev, ew = g.edge_array()
        eu = np.ascontiguousarray(eu, dtype=np.int64)
        ev = np.ascontiguousarray(ev, dtype=np.int64)
        root = np.empty(g.n, dtype=np.int64)
        rounds = np.zeros(1, dtype=np.int32)
        N.check(N.lib().cf_components_dev(_ingest_device(), g.n, eu.size, N.ptr(eu, N.i64p),
                                          N.ptr(ev, N.i64p), N.ptr(root, N.i64p),
                                          N.ptr(rounds, N.i32p)))
        is_root = root == np.arange(g.n)
        ncomp = int(is_root.sum())
        comp = (np.cumsum(is_root) - 1)[root]
    else:
        ncomp, comp = connected_components(g.adjacency_matrix(), directed=False)
    if ncomp == 1:
        return g, {i: i for i in range(g.n)}
    sizes = np.bincount(comp, minlength=ncomp)
    cands = np.flatnonzero(sizes == sizes.max())
    if cands.size == 1:
        pick = cands[0]
    else:
        pick = cands[int(np.argmin([g.node_labels[comp == c].min() for c in cands]))]
    keep = np.flatnonzero(comp == pick)
    remap = np.full(g.n, -1, dtype=np.int64)
    remap[keep] = np.arange(keep.size)
    if eu is None:
        eu, ev, ew = g.edge_array()
    sel = remap[eu] >= 0
    sub = Graph.from_edges(remap[eu[sel]], remap[ev[sel]], ew[sel], n=keep.size,
                           node_labels=g.node_labels[keep].copy())
    return sub, {int(a): int(b) for a, b in zip(keep, remap[keep])}


def check_connected(g: Graph) -> None:
    """DomainError unless ``g`` is connected (graph.py:338-348); one
    connected-components pass over the CSR adjacency."""
    if g.n == 0:
        raise DomainError("empty graph")
    if g.n == 1:
        return
    ncomp, _ = connected_components(g.adjacency_matrix(), directed=False)
    if ncomp != 1:
        raise DomainError("graph is not connected; extract the LCC first")


def laplacian(g: Graph) -> sp.csr_matrix:
    """L = D - A (graph.py:253-258)."""
    a = g.adjacency_matrix()
    deg = np.asarray(a.sum(axis=1)).ravel()
    return (sp.diags(deg, format="csr") - a).tocsr()


def incidence_and_weights(g: Graph):
    """B (m x n; +1 at the smaller id) and w, canonical edge order
    (graph.py:261-276)."""
    eu, ev, ew = g.edge_array()
    m = eu.size
    cols = np.empty(2 * m, dtype=np.int64)
    cols[0::2] = eu
    cols[1::2] = ev
    b = sp.csr_matrix((np.tile(np.array([1.0, -1.0]), m),
                       (np.repeat(np.arange(m, dtype=np.int64), 2), cols)), shape=(m, g.n))
    return b, ew.copy()


def edge_index_view(g: Graph):
    """Device upload view for the JL right-hand sides: for each adjacency
    entry (i, nbr) the canonical id of edge {i, nbr} (its row in
    ``incidence_and_weights``), and sqrt(w) per canonical edge.

    Since canonical ids ascend with (min, max) endpoints, node i's entries in
    sorted-neighbour order visit its edges in ascending id order -- the order
    in which the reference's CSR product (resistance.py:192) accumulates them.
    """
    src = _row_ids(g.indptr)
    up = src < g.indices
    m = int(up.sum())
    eid_up = np.arange(m, dtype=np.int64)
    # id of the mirrored entry (nbr, i) for i > nbr: position of (nbr, i) in canonical order
    eid = np.empty(g.indices.size, dtype=np.int64)
    eid[up] = eid_up
    lo = ~up
    # canonical key of the lower-triangle entries: (indices, src)
    key_up = src[up] * g.n + g.indices[up]
    key_lo = g.indices[lo] * g.n + src[lo]
    eid[lo] = np.searchsorted(key_up, key_lo)
    _, _, ew = g.edge_array()
    return eid, np.sqrt(ew)
