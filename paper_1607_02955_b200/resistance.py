"""Effective resistances, exact and sketched (reference
pkg/src/cfcent/resistance.py), on the device solve path.

* ``build_sketch`` generates the seeded projection Q on the GPU (numpy PCG64
  stream reproduced bit-for-bit, csrc/cf_estimators.cu), forms and centres the
  right-hand sides, solves them as one block and returns ``z`` (k x n).
* ``node_solution`` builds the ``e_x - 1/n`` supplies on the device.
* :func:`sketch_closeness_sums` is the fused path used by
  ``cf_closeness_projection``: Z never leaves the GPU; only the per-row sums
  and the query columns are read back.
"""

from __future__ import annotations

import math
import weakref
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native as N
from .errors import DomainError
from .graph import Graph, edge_index_view, incidence_and_weights  # noqa: F401
from .solver import MultigridHierarchy, SolverConfig, _params, solve

__all__ = ["SupplySpec", "ResistanceSketch", "effective_resistance", "resistances_from_node",
           "node_solution", "build_sketch", "sketch_distance", "sketch_distance_sums",
           "sketch_dimension"]

SKETCH_ROW_BLOCK = 256  # reference constant (resistance.py:34); the device chunks by 256 too


@dataclass(frozen=True)
class SupplySpec:
    """Unit current injection: +1 at ``source``, -1 at ``sink``
    (resistance.py:37-54)."""

    source: int
    sink: int

    def __post_init__(self):
        if self.source == self.sink:
            raise DomainError("source and sink must differ")

    def vector(self, n: int) -> np.ndarray:
        if not (0 <= self.source < n and 0 <= self.sink < n):
            raise DomainError("supply nodes out of range")
        b = np.zeros(n)
        b[self.source] = 1.0
        b[self.sink] = -1.0
        return b


def effective_resistance(hierarchy: MultigridHierarchy, u: int, v: int,
                         config: SolverConfig | None = None) -> float:
    """Potential difference under a unit u-v supply; exactly 0 for u == v
    without solving (resistance.py:57-74)."""
    n = hierarchy.n
    if not (0 <= u < n and 0 <= v < n):
        raise DomainError("node ids out of range")
    if u == v:
        return 0.0
    pot = solve(hierarchy, SupplySpec(u, v).vector(n), config)
    return float(pot.values[u] - pot.values[v])


def _node_solve(hierarchy: MultigridHierarchy, nodes: np.ndarray, config: SolverConfig,
                full: bool):
    """Device solve of L z_x = e_x - 1/n for each x in ``nodes`` (sorted).
    Returns (sub|None, z_rows|None, residuals): sub[a, b] = z_{nodes[a]}[nodes[b]]
    (only when the full solutions are not requested)."""
    n = hierarchy.n
    cnt = nodes.size
    sub = None if full else np.empty((cnt, cnt))
    z = np.empty((cnt, n)) if full else None
    res = np.zeros(cnt)
    if cnt == 0:
        return sub, z, res
    dev = hierarchy.device()
    st = N.CfSolveStats()
    nd = np.ascontiguousarray(dev.inv0[np.asarray(nodes, dtype=np.int64)], dtype=np.int64)
    N.check(N.lib().cf_node_solutions(dev.handle, N.ptr(nd, N.i64p), cnt,
                                      N.C.byref(_params(config, n)), N.ptr(sub, N.f64p),
                                      N.ptr(z, N.f64p), N.ptr(res, N.f64p), N.C.byref(st)), st)
    hierarchy.stats.record(res, int(st.fallback_solves), int(st.vcycles),
                           int(st.krylov_solves))
    return sub, z, res


def node_solution(hierarchy: MultigridHierarchy, nodes: Sequence[int],
                  config: SolverConfig | None = None, cache: dict[int, np.ndarray] | None = None,
                  threads: int = 1) -> dict[int, np.ndarray]:
    """Mean-centred solutions of ``L z_x = e_x - (1/n) 1`` (resistance.py:77-99);
    only nodes missing from ``cache`` are solved."""
    config = config or hierarchy.config
    cache = cache if cache is not None else {}
    missing = np.asarray(sorted({int(x) for x in nodes} - cache.keys()), dtype=np.int64)
    if missing.size:
        if missing.min() < 0 or missing.max() >= hierarchy.n:
            raise DomainError("node ids out of range")
        _, z, _ = _node_solve(hierarchy, missing, config, full=True)
        for i, x in enumerate(missing):
            cache[int(x)] = z[i]
    return cache


def resistances_from_node(hierarchy: MultigridHierarchy, v: int, targets: Sequence[int],
                          config: SolverConfig | None = None,
                          cache: dict[int, np.ndarray] | None = None,
                          threads: int = 1) -> np.ndarray:
    """R(v, t) = z_v[v] - z_v[t] - z_t[v] + z_t[t] from cached node solutions
    (resistance.py:102-130)."""
    n = hierarchy.n
    targets = np.asarray(targets, dtype=np.int64)
    if not (0 <= v < n) or (targets.size and (targets.min() < 0 or targets.max() >= n)):
        raise DomainError("node ids out of range")
    cache = node_solution(hierarchy, np.r_[targets, v], config, cache=cache, threads=threads)
    z_v = cache[int(v)]
    at_v = np.fromiter((cache[int(w)][v] for w in targets), np.float64, targets.size)
    at_w = np.fromiter((cache[int(w)][w] for w in targets), np.float64, targets.size)
    out = (z_v[v] - z_v[targets]) - at_v + at_w
    out[targets == v] = 0.0
    return out


def pair_resistance_table(hierarchy: MultigridHierarchy, nodes: np.ndarray,
                          config: SolverConfig | None = None):
    """Device route for the sampling estimator: solve every node of ``nodes``
    (sorted, unique) once and return the |nodes|^2 submatrix of solutions
    (no full solution vectors leave the GPU)."""
    config = config or hierarchy.config
    sub, _, res = _node_solve(hierarchy, np.asarray(nodes, dtype=np.int64), config, full=False)
    return sub, res


@dataclass(frozen=True)
class ResistanceSketch:
    """Random projection whose column distances approximate resistances
    (resistance.py:133-153)."""

    z: np.ndarray
    k: int
    epsilon: float
    seed: int
    max_residual: float = 0.0

    def __post_init__(self):
        self.z.setflags(write=False)

    @property
    def n(self) -> int:
        return self.z.shape[1]


def sketch_dimension(n: int, epsilon: float) -> int:
    """``max(1, ceil(ln n / epsilon^2))`` (resistance.py:156-158)."""
    return max(1, math.ceil(math.log(n) / epsilon ** 2))


class _DeviceGraph:
    """Adjacency + canonical edge ids + sqrt(w) on the device (one per
    (graph, hierarchy) pair)."""

    def __init__(self, g: Graph, hierarchy: MultigridHierarchy):
        eid, sqw = edge_index_view(g)
        self._h = hierarchy.device()
        # adjacency rows in device order (row i' = node perm0[i']), entries of
        # each row kept in ascending canonical edge order
        perm0 = self._h.perm0
        deg = np.diff(g.indptr)[perm0]
        ap = np.zeros(g.n + 1, dtype=np.int64)
        np.cumsum(deg, out=ap[1:])
        src = np.repeat(g.indptr[:-1][perm0] - ap[:-1], deg) + np.arange(ap[-1])
        nb = np.ascontiguousarray(g.indices[src], dtype=np.int32)
        ei = np.ascontiguousarray(eid[src], dtype=np.int32)
        sw = np.ascontiguousarray(sqw, dtype=np.float64)
        h = N.C.c_void_p()
        N.check(N.lib().cf_graph_create(self._h.handle, g.n, sw.size, N.ptr(ap, N.i64p),
                                        N.ptr(nb, N.i32p), N.ptr(ei, N.i32p), N.ptr(sw, N.f64p),
                                        N.C.byref(h)))
        self.handle = h

    def __del__(self):
        try:
            if self.handle is not None and self.handle.value:
                N.lib().cf_graph_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def _device_graph(g: Graph, hierarchy: MultigridHierarchy) -> _DeviceGraph:
    per = hierarchy._graphs
    key = id(g)
    ent = per.get(key)
    if ent is None or ent[0]() is not g:
        # entries of graphs that have died are dropped here, so their device
        # copies (adjacency, edge ids, sqrt(w), sign bits) do not outlive them
        for dead in [k for k, (ref, _) in per.items() if ref() is None]:
            per.pop(dead, None)
        ent = (weakref.ref(g), _DeviceGraph(g, hierarchy))
        per[key] = ent
    return ent[1]


def _pcg_words(seed: int):
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m64 = (1 << 64) - 1
    return (s >> 64) & m64, s & m64, (inc >> 64) & m64, inc & m64


def _sketch_device(g: Graph, hierarchy: MultigridHierarchy, epsilon: float, seed: int,
                   config: SolverConfig, query: np.ndarray | None, want_z: bool,
                   rows: tuple[int, int] | None = None, want_parts: bool = False):
    """Device JL sketch of rows [r0, r1) (all k rows by default).  Returns
    (k, z rows|None, per-query sums over those rows, residuals[, row parts])."""
    if not 0 < epsilon <= 1:
        raise DomainError(f"epsilon must be in (0, 1], got {epsilon}")
    n = g.n
    if hierarchy.n != n:
        raise DomainError("hierarchy does not match graph")
    k = sketch_dimension(n, epsilon)
    r0, r1 = (0, k) if rows is None else rows
    dg = _device_graph(g, hierarchy)
    q = np.zeros(0, dtype=np.int64) if query is None else np.asarray(query, np.int64)
    q = np.ascontiguousarray(hierarchy.device().inv0[q], dtype=np.int64)
    sums = np.zeros(max(q.size, 1))
    parts = np.empty((r1 - r0, 2 + q.size)) if want_parts else None
    z = np.empty((r1 - r0, n)) if want_z else None
    res = np.zeros(r1 - r0)
    st = N.CfSolveStats()
    sh, sl, ih, il = _pcg_words(seed)
    N.check(N.lib().cf_jl_sketch(dg.handle, sh, sl, ih, il, k, r0, r1 - r0, 1.0 / math.sqrt(k),
                                 N.ptr(q, N.i64p), q.size, N.C.byref(_params(config, n)),
                                 N.ptr(sums, N.f64p), N.ptr(parts, N.f64p), N.ptr(z, N.f64p),
                                 N.ptr(res, N.f64p), N.C.byref(st)), st)
    hierarchy.stats.record(res, int(st.fallback_solves), int(st.vcycles),
                           int(st.krylov_solves))
    if want_parts:
        return k, z, sums[:q.size], res, parts
    return k, z, sums[:q.size], res


def build_sketch(g: Graph, hierarchy: MultigridHierarchy, epsilon: float, seed: int,
                 config: SolverConfig | None = None, threads: int = 1) -> ResistanceSketch:
    """Project the resistance embedding onto k = ceil(ln n / eps^2) random
    +-1/sqrt(k) directions (resistance.py:161-204); deterministic per seed and
    Q identical to the reference's."""
    config = config or hierarchy.config
    k, z, _, res = _sketch_device(g, hierarchy, epsilon, seed, config, None, True)
    return ResistanceSketch(z=z, k=k, epsilon=epsilon, seed=seed,
                            max_residual=float(res.max()) if res.size else 0.0)


def jl_rhs_rows(g: Graph, hierarchy: MultigridHierarchy, k: int, seed: int, row0: int = 0,
                rows: int | None = None) -> np.ndarray:
    """Uncentred seeded right-hand sides rows [row0, row0+rows) of
    Q W^1/2 B as formed on the device (for parity tests against
    resistance.py:184-192)."""
    rows = k if rows is None else rows
    dg = _device_graph(g, hierarchy)
    out = np.empty((rows, g.n))
    sh, sl, ih, il = _pcg_words(seed)
    N.check(N.lib().cf_jl_rhs_rows(dg.handle, sh, sl, ih, il, k, row0, rows, N.ptr(out, N.f64p)))
    return out


def sketch_closeness_sums(g: Graph, hierarchy: MultigridHierarchy, epsilon: float, seed: int,
                          query: Sequence[int], config: SolverConfig | None = None,
                          rows: tuple[int, int] | None = None, row_parts: bool = False):
    """Fused device JL path: returns (k, sums_v for query, residuals).  With
    ``rows`` only that range of sketch rows is solved and the sums are its
    share.  With ``row_parts`` a fourth value is returned: the per-row parts
    [T_j, C_j, Z[q, j]...] ((r1 - r0) x (2 + |query|)) that ``combine_row_parts``
    sums in row order -- bitwise the same total for any split of the rows over
    ranks (multi-GPU sharding)."""
    config = config or hierarchy.config
    out = _sketch_device(g, hierarchy, epsilon, seed, config,
                         np.asarray(query, dtype=np.int64), False, rows, row_parts)
    return out[0], out[2], out[3], *out[4:]


def combine_row_parts(parts: np.ndarray, n: int) -> np.ndarray:
    """sum_w ||z_v - z_w||^2 for the query nodes from per-row parts stacked in
    ascending sketch-row order (cf_jl_combine; resistance.py:218-237)."""
    parts = np.ascontiguousarray(parts, dtype=np.float64)
    if parts.ndim != 2 or parts.shape[1] < 2:
        raise DomainError("row parts must be (rows, 2 + |query|)")
    nq = parts.shape[1] - 2
    out = np.zeros(max(nq, 1))
    N.check(N.lib().cf_jl_combine(N.ptr(parts, N.f64p), parts.shape[0], nq, int(n),
                                  N.ptr(out, N.f64p)))
    return out[:nq]


def sketch_distance(sketch: ResistanceSketch, u: int, v: int) -> float:
    """Squared distance between sketch columns (resistance.py:207-215)."""
    n = sketch.n
    if not (0 <= u < n and 0 <= v < n):
        raise DomainError("node ids out of range")
    if u == v:
        return 0.0
    d = sketch.z[:, u] - sketch.z[:, v]
    return float(d @ d)


def sketch_distance_sums(sketch: ResistanceSketch, nodes: Sequence[int] | None = None) -> np.ndarray:
    """sum_w ||z_v - z_w||^2 in closed form (resistance.py:218-237)."""
    z = sketch.z
    col_sq = np.einsum("ij,ij->j", z, z)
    n = sketch.n
    idx = np.arange(n) if nodes is None else np.asarray(nodes, dtype=np.int64)
    if idx.size and (idx.min() < 0 or idx.max() >= n):
        raise DomainError("node ids out of range")
    return col_sq.sum() + n * col_sq[idx] - 2.0 * (z[:, idx].T @ z.sum(axis=1))
