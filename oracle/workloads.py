"""Benchmark workloads C1..C5 built with the oracle's own numpy graph layer.

TEST / BENCH INFRASTRUCTURE ONLY (see ``oracle/__init__.py``): the CPU
reference arm of ``bench.py`` builds its input here so that it runs no
product code (no ``libcfcent_b200.so``).  The recipes are the frozen ones of
SURVEY.md §8(d), identical draw for draw to
``paper_1607_02955_b200/configs.py`` (the product arm), and the graphs are
equal to the product's (``tests/test_oracle_golden.py`` checks C1/C2 and a
small R-MAT/RGG here; the C4 LCC size is pinned in ``test_gpu_solver``).

Each workload is a dict: ``graph`` (indptr, indices, weights), ``tau``,
``jl_k``, ``jl_seed``, ``query``, ``sampling`` (pivots, seed, query) or None.
"""

from __future__ import annotations

import math

import numpy as np

from . import lamg_oracle as O


def rgg_graph(n, seed, mean_degree=10.0):
    """Random geometric graph in the unit square, w = 1/(dist + 1e-3), LCC."""
    from scipy.spatial import cKDTree

    pts = np.random.default_rng(seed).random((n, 2))
    r = math.sqrt(mean_degree / (math.pi * n))
    pairs = cKDTree(pts).query_pairs(r, output_type="ndarray")
    d = np.linalg.norm(pts[pairs[:, 0]] - pts[pairs[:, 1]], axis=1)
    g = O.graph_from_edges(pairs[:, 0], pairs[:, 1], 1.0 / (d + 1e-3), n=n)
    return O.largest_component(g)[0]


def rmat_edges(scale, edge_factor, seed, weighted, abcd=(0.57, 0.19, 0.19, 0.05)):
    """R-MAT edge list: one rng.random(M) draw per bit level picks the
    quadrant; self-loops dropped; duplicates removed (u < v) before the
    weights are drawn (w = 2 - 1.5 U[0,1), i.e. in (0.5, 2])."""
    rng = np.random.default_rng(seed)
    n = 1 << scale
    M = edge_factor * n
    a, b, c, _ = abcd
    u = np.zeros(M, dtype=np.int64)
    v = np.zeros(M, dtype=np.int64)
    for bit in range(scale):
        r = rng.random(M)
        u |= (r >= a + b).astype(np.int64) << bit
        v |= (((r >= a) & (r < a + b)) | (r >= a + b + c)).astype(np.int64) << bit
    keep = u != v
    lo = np.minimum(u[keep], v[keep])
    hi = np.maximum(u[keep], v[keep])
    # sorted unique keys (in-place sort + neighbour compare: the same result as
    # np.unique, without its hash pass -- 19 s of the 31 s scale-20 generation)
    key = lo * n + hi
    key.sort()
    if key.size:
        key = key[np.r_[True, key[1:] != key[:-1]]]
    lo, hi = key // n, key % n
    w = (2.0 - rng.random(lo.size) * 1.5) if weighted else np.ones(lo.size)
    return n, lo, hi, w


def rmat_graph(scale, edge_factor, seed, weighted):
    n, lo, hi, w = rmat_edges(scale, edge_factor, seed, weighted)
    return O.largest_component(O.graph_from_edges(lo, hi, w, n=n))[0]


def _max_degree_node(g):
    return int(np.argmax(np.diff(g[0])))


def make(name):
    name = name.lower()
    if name == "c1":
        g = O.grid_graph(64)
        return dict(graph=g, tau=1e-8, jl_k=64, jl_seed=0, query=np.array([0]),
                    sampling=(64, 0, [0]))
    if name == "c2":
        g = O.barabasi_albert(100000, 4, 1)
        n = g[0].size - 1
        q = np.sort(np.random.default_rng(2).choice(n, 100, replace=False))
        return dict(graph=g, tau=1e-6, jl_k=128, jl_seed=0, query=q, sampling=None)
    if name == "c3":
        g = rgg_graph(1_000_000, 3)
        u = _max_degree_node(g)
        return dict(graph=g, tau=1e-6, jl_k=128, jl_seed=0, query=np.array([u]),
                    sampling=(256, 3, [u]))
    if name == "c4":
        g = rmat_graph(20, 16, 4, True)
        n = g[0].size - 1
        q = np.sort(np.random.default_rng(4).choice(n, 1000, replace=False))
        return dict(graph=g, tau=1e-6, jl_k=256, jl_seed=0, query=q, sampling=None)
    if name == "c5":
        g = rmat_graph(22, 12, 5, False)
        n = g[0].size - 1
        u = _max_degree_node(g)
        k = math.ceil(4 * math.log(n) / 0.09)
        return dict(graph=g, tau=1e-6, jl_k=k, jl_seed=0, query=np.array([u]),
                    sampling=(1024, 5, [u]))
    raise ValueError(f"unknown config {name}")


def hierarchy_from_levels(levels, cfg):
    """Oracle hierarchy dict (lamg_oracle.build_hierarchy's format) from a
    host hierarchy's ``levels`` (objects with the reference ``Level`` fields,
    solver.py:97-120), so the oracle's restatement of the reference solve loop
    (solver.py:526-751) can be timed or checked on a hierarchy the reference's
    own setup cannot produce in bounded time (the R-MAT configurations)."""
    import scipy.sparse as sp

    out = []
    for lv in levels:
        kind = getattr(lv.kind, "value", lv.kind)
        A = sp.csr_matrix(lv.matrix)
        if kind == "elimination":
            out.append({"kind": "elim", "A": A, "f": np.asarray(lv.f_nodes),
                        "c": np.asarray(lv.c_nodes), "d_f": np.asarray(lv.f_degree),
                        "w_cf": sp.csr_matrix(lv.w_cf), "w_fc": sp.csr_matrix(lv.w_cf).T.tocsr()})
        elif kind == "aggregation":
            agg = np.asarray(lv.aggregates)
            n = A.shape[0]
            out.append({"kind": "agg", "A": A, "agg": agg,
                        "P": sp.csr_matrix((np.ones(n), (np.arange(n), agg)),
                                           shape=(n, int(agg.max()) + 1)),
                        "lower": sp.tril(A, 0, format="csr"),
                        "upper": sp.triu(A, 0, format="csr")})
        else:
            out.append({"kind": "coarse", "A": A, "factor": O._coarsest_factor(A)})
    return {"levels": out, "cfg": cfg, "stats": {"solves": 0, "max_residual": 0.0,
                                                  "fallback_solves": 0}}
