"""Benchmark / parity configurations C1..C5 (BASELINE.json ``configs``;
frozen recipes from SURVEY.md §8(d)).  Seeded synthetic inputs stand in for
the paper's SNAP/DIMACS graphs (not available offline).

C1 and C2 use the reference's own generators (same draws).  The RGG (C3) and
R-MAT (C4, C5) generators are not in the reference; their recipes are fixed
here: RGG points ``default_rng(3).random((n, 2))``, radius sqrt(10/(pi n)),
weights 1/(dist+1e-3), LCC; R-MAT with one ``rng.random(M)`` draw per bit
level choosing the quadrant, self-loops dropped, duplicates removed (u<v)
before weights, LCC.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .graph import Graph, largest_connected_component
from .generators import barabasi_albert_graph, grid_graph


@dataclass
class BenchConfig:
    name: str
    description: str
    tau: float
    jl_k: int
    query: np.ndarray
    graph: Graph
    jl_seed: int = 0
    sampling_pivots: int = 0
    sampling_seed: int = 0
    sampling_query: list = field(default_factory=list)

    @property
    def epsilon(self) -> float:
        # eps = sqrt(ln n / (k - 0.5)) makes ceil(ln n / eps^2) == k exactly
        return math.sqrt(math.log(self.graph.n) / (self.jl_k - 0.5))


def rgg_graph(n: int, seed: int, mean_degree: float = 10.0) -> Graph:
    from scipy.spatial import cKDTree

    pts = np.random.default_rng(seed).random((n, 2))
    r = math.sqrt(mean_degree / (math.pi * n))
    pairs = cKDTree(pts).query_pairs(r, output_type="ndarray")
    d = np.linalg.norm(pts[pairs[:, 0]] - pts[pairs[:, 1]], axis=1)
    g = Graph.from_edges(pairs[:, 0], pairs[:, 1], 1.0 / (d + 1e-3), n=n)
    return largest_connected_component(g)[0]


def rmat_graph(scale: int, edge_factor: int, seed: int, weighted: bool,
               abcd=(0.57, 0.19, 0.19, 0.05)) -> Graph:
    rng = np.random.default_rng(seed)
    n = 1 << scale
    M = edge_factor * n
    a, b, c, _ = abcd
    u = np.zeros(M, dtype=np.int64)
    v = np.zeros(M, dtype=np.int64)
    for bit in range(scale):
        r = rng.random(M)
        # quadrant: a -> (0,0), b -> (0,1), c -> (1,0), d -> (1,1)
        ubit = r >= a + b
        vbit = ((r >= a) & (r < a + b)) | (r >= a + b + c)
        u |= ubit.astype(np.int64) << bit
        v |= vbit.astype(np.int64) << bit
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
    g = Graph.from_edges(lo, hi, w, n=n)
    return largest_connected_component(g)[0]


def make(name: str) -> BenchConfig:
    name = name.lower()
    if name == "c1":
        g = grid_graph(64)
        return BenchConfig("c1", "grid 64x64 unit weights; JL k=64 seed 0, query {0}; "
                           "sampling 64 pivots seed 0 for u=0; tau 1e-8", 1e-8, 64,
                           np.array([0]), g, 0, 64, 0, [0])
    if name == "c2":
        g = barabasi_albert_graph(100000, 4, 1)
        q = np.sort(np.random.default_rng(2).choice(g.n, 100, replace=False))
        return BenchConfig("c2", "Barabasi-Albert n=1e5 m0=4 seed 1 unit weights; JL k=128 "
                           "(Q seed 0) for 100 nodes drawn with seed 2; tau 1e-6", 1e-6, 128, q, g)
    if name == "c3":
        g = rgg_graph(1_000_000, 3)
        deg = np.diff(g.indptr)
        u = int(np.argmax(deg))
        return BenchConfig("c3", "RGG n=1e6 (seed 3) mean degree 10, LCC, w=1/(d+1e-3); JL k=128 "
                           "and sampling 256 pivots (seed 3) for the max-degree node; tau 1e-6",
                           1e-6, 128, np.array([u]), g, 0, 256, 3, [u])
    if name == "c4":
        g = rmat_graph(20, 16, 4, weighted=True)
        q = np.sort(np.random.default_rng(4).choice(g.n, 1000, replace=False))
        return BenchConfig("c4", "R-MAT scale 20 ef 16 (.57,.19,.19,.05) seed 4, dedup, LCC, "
                           "w in (0.5,2]; JL k=256 for 1000 nodes; tau 1e-6", 1e-6, 256, q, g)
    if name == "c5":
        g = rmat_graph(22, 12, 5, weighted=False)
        deg = np.diff(g.indptr)
        u = int(np.argmax(deg))
        k = math.ceil(4 * math.log(g.n) / 0.09)
        return BenchConfig("c5", "R-MAT scale 22 ef 12 seed 5, LCC, unit weights; JL k=ceil(4 ln n/"
                           "0.3^2) and sampling 1024 pivots (seed 5) for the max-degree node; "
                           "tau 1e-6", 1e-6, k, np.array([u]), g, 0, 1024, 5, [u])
    raise ValueError(f"unknown config {name}")
