"""GPU parity tests of the solve path (through the C-ABI) against the CPU
oracle, the reference's golden vectors and the reference's known answers
(pkg/tests/test_solver.py cases restated)."""

import numpy as np
import pytest

import paper_1607_02955_b200 as P
from conftest import dense_pinv_resistance, golden, random_connected_graph_edges
from oracle import lamg_oracle as O
from paper_1607_02955_b200 import generators as G

pytestmark = pytest.mark.gpu


def dense_solve(lap, b):
    x = np.zeros(lap.shape[0])
    x[1:] = np.linalg.solve(lap[1:, 1:], b[1:])
    return x - x.mean()


def test_p2_unit_supply():
    h = P.setup(P.laplacian(G.path_graph(2)))
    p = P.solve(h, np.array([1.0, -1.0]))
    assert p.values == pytest.approx([0.5, -0.5], abs=1e-12)


def test_zero_rhs_exact_zeros():
    h = P.setup(P.laplacian(G.path_graph(5)))
    p = P.solve(h, np.zeros(5))
    assert np.all(p.values == 0.0) and p.achieved_residual == 0.0


def test_grid_residual_contract(rng):
    g = G.grid_graph(64)
    h = P.setup(P.laplacian(g))
    b = rng.standard_normal(g.n)
    b -= b.mean()
    p = P.solve(h, b)
    lap = P.laplacian(g)
    assert np.linalg.norm(b - lap @ p.values) / np.linalg.norm(b) <= 1e-5
    assert abs(p.values.mean()) < 1e-12


def test_unbalanced_rejected():
    h = P.setup(P.laplacian(G.path_graph(4)))
    with pytest.raises(P.DomainError):
        P.solve(h, np.array([1.0, 0.0, 0.0, 0.0]))


@pytest.mark.parametrize("t", range(6))
def test_golden_small_graphs(t):
    """Same hierarchy as the reference; solutions of the reference's supplies
    agree with the reference's own solutions and the dense oracle."""
    d = golden("small_graphs.npz")
    g = P.Graph.from_edges(d[f"g{t}_eu"], d[f"g{t}_ev"], d[f"g{t}_ew"], n=int(d[f"g{t}_n"]))
    cfg = P.SolverConfig(tau=1e-10, max_direct_size=int(d[f"g{t}_mds"]))
    h = P.setup(P.laplacian(g), cfg)
    assert h.level_sizes == d[f"g{t}_sizes"].tolist()
    pots = P.solve_many(h, d[f"g{t}_b"])
    x = np.stack([p.values for p in pots])
    ref = d[f"g{t}_x"]
    lap = P.laplacian(g).toarray()
    exact = np.stack([dense_solve(lap, b) for b in d[f"g{t}_b"]])
    scale = np.abs(exact).max()
    assert np.abs(x - ref).max() <= 1e-7 * scale
    assert np.abs(x - exact).max() <= 1e-7 * scale
    assert max(p.achieved_residual for p in pots) <= 1e-10


def test_matches_dense_oracle_random(rng):
    for _ in range(8):
        n = int(rng.integers(3, 40))
        u, v, w = random_connected_graph_edges(n, rng, weighted=True)
        g = P.Graph.from_edges(u, v, w, n=n)
        h = P.setup(P.laplacian(g), P.SolverConfig(tau=1e-10, max_direct_size=2))
        b = rng.standard_normal(n)
        b -= b.mean()
        p = P.solve(h, b)
        exp = dense_solve(P.laplacian(g).toarray(), b)
        assert p.values == pytest.approx(exp, abs=1e-7 * max(1, np.abs(exp).max()))


def test_determinism_columns_negation_batch(rng):
    g = G.grid_graph(16)
    h = P.setup(P.laplacian(g))
    b = rng.standard_normal(g.n)
    b -= b.mean()
    r = P.solve_many(h, [b, b, -b])
    assert np.array_equal(r[0].values, r[1].values)
    assert np.array_equal(r[0].values, -r[2].values)
    others = rng.standard_normal((70, g.n))
    others -= others.mean(axis=1, keepdims=True)
    alone = P.solve_many(h, [b])[0]
    grouped = P.solve_many(h, np.vstack([others, b[None, :]]))[-1]
    # per-column independence on the device: bitwise, stronger than the
    # reference's 1e-12 (pkg/tests/test_solver.py:273-285)
    assert np.array_equal(alone.values, grouped.values)
    t1 = P.solve_many(h, others, threads=1)
    t4 = P.solve_many(h, others, threads=4)
    assert all(np.array_equal(a.values, c.values) for a, c in zip(t1, t4))


def test_many_rhs_random_graph(rng):
    u, v, w = random_connected_graph_edges(1000, rng)
    g = P.Graph.from_edges(u, v, w, n=1000)
    h = P.setup(P.laplacian(g))
    lap = P.laplacian(g)
    s = rng.standard_normal((300, g.n))
    s -= s.mean(axis=1, keepdims=True)
    for pot, b in zip(P.solve_many(h, s), s):
        assert np.linalg.norm(b - lap @ pot.values) / np.linalg.norm(b) <= 1e-5


def test_fallback_rescues_starved_multigrid(rng):
    g = G.grid_graph(20)
    cfg = P.SolverConfig(max_cycles=1, smoothing_steps=(1, 1), max_direct_size=2)
    h = P.setup(P.laplacian(g), cfg)
    b = rng.standard_normal(g.n)
    b -= b.mean()
    p = P.solve(h, b, cfg)
    assert np.linalg.norm(b - P.laplacian(g) @ p.values) / np.linalg.norm(b) <= 1e-5
    assert h.stats.fallback_solves >= 1


def test_unreachable_tolerance_raises(rng):
    cfg = P.SolverConfig(tau=1e-300, max_cycles=8)
    h = P.setup(P.laplacian(G.path_graph(30)), cfg)
    b = rng.standard_normal(30)
    b -= b.mean()
    with pytest.raises(P.ConvergenceError) as err:
        P.solve(h, b, cfg)
    assert 0 < err.value.best_residual < 1e-10


def test_block_widths_agree(rng):
    """Every device block width computes each column identically."""
    g = G.grid_graph(12)
    h = P.setup(P.laplacian(g))
    s = rng.standard_normal((200, g.n))
    s -= s.mean(axis=1, keepdims=True)
    full = np.stack([p.values for p in P.solve_many(h, s)])
    for cnt in (1, 5, 9, 17, 33, 65, 129, 161, 192):  # widths 1..128, 160, 192
        part = np.stack([p.values for p in P.solve_many(h, s[:cnt])])
        assert np.array_equal(part, full[:cnt]), cnt


def test_vs_oracle_bigger(rng):
    """BA 20k: device solutions vs the oracle's reference-algorithm solutions."""
    g = G.barabasi_albert_graph(20000, 4, 7)
    og = O.barabasi_albert(20000, 4, 7)
    cfg = P.SolverConfig(tau=1e-10)
    h = P.setup(P.laplacian(g), cfg)
    oh = O.build_hierarchy(O.laplacian(og), O.OracleConfig(tau=1e-10))
    assert h.level_sizes == [l["A"].shape[0] for l in oh["levels"]]
    b = rng.standard_normal((40, g.n))
    b -= b.mean(axis=1, keepdims=True)
    x = np.stack([p.values for p in P.solve_many(h, b)])
    ref, _ = O.solve_rows(oh, b)
    assert np.abs(x - ref).max() <= 1e-8 * np.abs(ref).max()


@pytest.mark.slow
def test_config3_properties():
    """C3 (RGG 1e6): hierarchy equals the reference's recorded shape
    (SURVEY.md A.2), every solve meets tau, JL sums additive over row ranges."""
    import math
    from paper_1607_02955_b200 import configs
    from paper_1607_02955_b200.resistance import sketch_closeness_sums
    bc = configs.make("c3")
    assert (bc.graph.n, bc.graph.m) == (999896, 4995274)
    cfg = P.SolverConfig(tau=bc.tau)
    h = P.setup(P.laplacian(bc.graph), cfg)
    assert h.level_sizes == [999896, 194376, 144154, 35917, 25678, 6364, 4862, 1165, 894, 209, 154]
    eps = math.sqrt(math.log(bc.graph.n) / (bc.jl_k - 0.5))
    k, full, res = sketch_closeness_sums(bc.graph, h, eps, 0, bc.query, cfg)
    assert k == 128 and res.max() <= bc.tau
    # strong multi-GPU split (distributed.py): row parts of two ranges stacked
    # in row order and combined give the single run's sums BITWISE
    from paper_1607_02955_b200.resistance import combine_row_parts
    _, a, _, pa = sketch_closeness_sums(bc.graph, h, eps, 0, bc.query, cfg, rows=(0, 50),
                                        row_parts=True)
    _, b, _, pb = sketch_closeness_sums(bc.graph, h, eps, 0, bc.query, cfg, rows=(50, 128),
                                        row_parts=True)
    assert np.allclose(a + b, full, rtol=1e-10)
    assert combine_row_parts(np.concatenate([pa, pb]), bc.graph.n).tobytes() == full.tobytes()
    lap = P.laplacian(bc.graph)
    rng = np.random.default_rng(3)
    s = rng.standard_normal((3, bc.graph.n))
    s -= s.mean(axis=1, keepdims=True)
    for pot, b_ in zip(P.solve_many(h, s, cfg), s):
        assert np.linalg.norm(b_ - lap @ pot.values) / np.linalg.norm(b_) <= bc.tau


@pytest.mark.slow
def test_config4_properties():
    """C4 (R-MAT scale 20): generator reproduces the survey's LCC, the stall
    breaker keeps the hierarchy shallow, solves meet tau."""
    from paper_1607_02955_b200 import configs
    bc = configs.make("c4")
    assert (bc.graph.n, bc.graph.m) == (646140, 15700710)
    cfg = P.SolverConfig(tau=bc.tau)
    h = P.setup(P.laplacian(bc.graph), cfg)
    assert len(h.levels) < 80
    lap = P.laplacian(bc.graph)
    rng = np.random.default_rng(4)
    s = rng.standard_normal((9, bc.graph.n))
    s -= s.mean(axis=1, keepdims=True)
    for pot, b_ in zip(P.solve_many(h, s, cfg), s):
        assert np.linalg.norm(b_ - lap @ pot.values) / np.linalg.norm(b_) <= bc.tau
    assert h.stats.fallback_solves == 0


def test_split_aggregates(rng, monkeypatch):
    """Aggregates larger than the restriction piece (8 members; hub levels of
    power-law graphs use cap 64) are restricted in pieces combined in a fixed
    order: solutions match the dense oracle and stay bitwise independent of the
    block width."""
    from paper_1607_02955_b200 import solver as S
    monkeypatch.setattr(S, "MAX_AGGREGATE_SIZE", 64)
    g = G.barabasi_albert_graph(6000, 2, 7)
    lap = P.laplacian(g)
    h = P.setup(lap, P.SolverConfig(tau=1e-10))
    big = [int(np.bincount(lv.aggregates).max()) for lv in h.levels
           if lv.aggregates is not None]
    assert max(big) > 8, big
    b = rng.standard_normal((9, g.n))
    b -= b.mean(axis=1, keepdims=True)
    x = np.stack([p.values for p in P.solve_many(h, b)])
    dense = lap.toarray()
    for r in range(3):
        ref = dense_solve(dense, b[r])
        assert np.abs(x[r] - ref).max() <= 1e-7 * np.abs(ref).max()
    one = P.solve(h, b[4]).values
    assert np.array_equal(one, x[4])


def test_tolerance_not_baked_into_solve_graph(rng):
    """The solve loop runs as a captured CUDA graph; its stop rule must follow
    each call's tau (regression: a graph captured for one tau was replayed for
    another)."""
    g = G.grid_graph(32)
    h = P.setup(P.laplacian(g))
    b = rng.standard_normal(g.n)
    b -= b.mean()
    tight = P.solve(h, b, P.SolverConfig(tau=1e-12))
    loose = P.solve(h, b, P.SolverConfig(tau=1e-3))
    tight2 = P.solve(h, b, P.SolverConfig(tau=1e-12))
    assert tight.achieved_residual <= 1e-12 and tight2.achieved_residual <= 1e-12
    assert 1e-9 < loose.achieved_residual <= 1e-3
    assert np.array_equal(tight.values, tight2.values)


def test_pinned_multiblock_overlap_matches(rng):
    """More right-hand sides than one device block with page-locked host
    buffers take the overlapped copy-in / solve / copy-out pipeline; results
    are bitwise those of the pageable path and of single solves."""
    import torch
    g = G.barabasi_albert_graph(5000, 3, 3)
    h = P.setup(P.laplacian(g), P.SolverConfig(tau=1e-8))
    k = 300  # 128 + 128 + 44 columns
    b = rng.standard_normal((k, g.n))
    b -= b.mean(axis=1, keepdims=True)
    ref = np.stack([p.values for p in P.solve_many(h, b)])
    b_pin = torch.empty(b.shape, dtype=torch.float64, pin_memory=True).numpy()
    b_pin[:] = b
    out = torch.empty(b.shape, dtype=torch.float64, pin_memory=True).numpy()
    pots = P.solve_many(h, b_pin, out=out)
    assert np.array_equal(out, ref)
    assert all(p.achieved_residual <= 1e-8 for p in pots)
    assert np.array_equal(P.solve(h, b[257]).values, ref[257])


def test_krylov_handoff_grid(rng):
    """Slowly converging columns (a grid: ~0.6 residual reduction per V-cycle)
    are handed to FCG after the third cycle: solutions match the dense oracle,
    stay bitwise independent of the batch, and need far fewer V-cycles than
    the stationary iteration (37 per column on C1 at 1e-8)."""
    g = G.grid_graph(48)
    lap = P.laplacian(g)
    h = P.setup(lap, P.SolverConfig(tau=1e-10))
    b = rng.standard_normal((20, g.n))
    b -= b.mean(axis=1, keepdims=True)
    v0 = h.stats.vcycles
    x = np.stack([p.values for p in P.solve_many(h, b)])
    per_col = (h.stats.vcycles - v0) / b.shape[0]
    assert per_col < 35, per_col
    dense = lap.toarray()
    for r in range(3):
        ref = dense_solve(dense, b[r])
        assert np.abs(x[r] - ref).max() <= 1e-7 * np.abs(ref).max()
    assert np.array_equal(P.solve(h, b[7]).values, x[7])
    assert np.array_equal(np.stack([p.values for p in P.solve_many(h, -b[:5])]), -x[:5])


def test_pinned_pipeline_error_drains_copies(rng):
    """an unbalanced column in the SECOND block of the overlapped
    pinned multi-block path raises DomainError only after the copy stream has
    drained (no DMA into the caller's buffers after the raise); the next call
    on the same hierarchy works."""
    import torch
    g = G.grid_graph(40)
    h = P.setup(P.laplacian(g), P.SolverConfig(tau=1e-8))
    b = rng.standard_normal((200, g.n))
    b -= b.mean(axis=1, keepdims=True)
    rows = torch.empty(b.shape, dtype=torch.float64, pin_memory=True).numpy()
    out = torch.empty(b.shape, dtype=torch.float64, pin_memory=True).numpy()
    rows[...] = b
    rows[150, 3] += 1.0  # block 2 (columns 128..199)
    out[...] = 7.0
    with pytest.raises(P.DomainError):
        P.solve_many(h, rows, out=out)
    snap = out.copy()
    torch.cuda.synchronize()
    import time
    time.sleep(0.05)
    assert np.array_equal(out, snap)  # nothing still being written
    rows[150, 3] -= 1.0
    got = P.solve_many(h, rows, out=out)
    assert max(p.achieved_residual for p in got) <= 1e-8


def test_device_ingestion_matches_host(monkeypatch):
    """Graph.from_edges and largest_connected_component
    on the GPU (csrc/cf_graph.cu: stable radix sort of the adjacency entries,
    min-id hooking + pointer jumping) produce exactly the host route's arrays
    (graph.py:100-147, 217-250): random sparse graph with many components,
    weighted; duplicate edges are detected and summed on the host route."""
    from paper_1607_02955_b200 import graph as GR

    r = np.random.default_rng(11)
    n, m = 300_000, 420_000  # mean degree 2.8: a giant component plus many small ones
    u = r.integers(0, n, m)
    v = r.integers(0, n, m)
    keep = u != v
    u, v = u[keep], v[keep]
    key = np.unique(np.minimum(u, v) * n + np.maximum(u, v))
    u, v = key // n, key % n
    w = r.random(u.size) + 0.5

    def build(dev):
        monkeypatch.setattr(GR, "DEVICE_INGEST_MIN_EDGES", 1 if dev else 1 << 62)
        g = P.Graph.from_edges(u, v, w, n=n)
        sub, remap = P.largest_connected_component(g)
        return g, sub, remap

    gh, sh, rh = build(False)
    gd, sd, rd = build(True)
    for a, b in ((gh, gd), (sh, sd)):
        assert np.array_equal(a.indptr, b.indptr)
        assert np.array_equal(a.indices, b.indices)
        assert np.array_equal(a.weights, b.weights)
        assert np.array_equal(a.node_labels, b.node_labels)
    assert rh == rd and sh.n < n and sh.is_connected()
    # duplicates (and both orientations) go through the host sum, same result
    u2, v2, w2 = np.r_[u, v[:1000]], np.r_[v, u[:1000]], np.r_[w, w[:1000] * 0.25]
    monkeypatch.setattr(GR, "DEVICE_INGEST_MIN_EDGES", 1)
    a = P.Graph.from_edges(u2, v2, w2, n=n)
    monkeypatch.setattr(GR, "DEVICE_INGEST_MIN_EDGES", 1 << 62)
    b = P.Graph.from_edges(u2, v2, w2, n=n)
    assert np.array_equal(a.indices, b.indices) and np.array_equal(a.weights, b.weights)
    # equal-size components: the tie goes to the smallest label on both routes
    monkeypatch.setattr(GR, "DEVICE_INGEST_MIN_EDGES", 1)
    t = P.Graph.from_edges([0, 1, 3, 4, 6], [1, 2, 4, 5, 7], n=8)
    sub, remap = P.largest_connected_component(t)
    assert sorted(remap) == [0, 1, 2]
    with pytest.raises(P.DomainError):
        P.Graph.from_edges([0, 9], [1, 2], n=4)


def test_device_coarse_operators_match_host(rng):
    """the Galerkin product and the Schur complement
    (+ Laplacian rebuild) computed on the GPU (csrc/cf_setup_dev.cu: triples,
    stable radix sort, runs summed in order) against the host route
    (solver.py:251-261, 383-386, 167-187 via scipy): identical sparsity
    pattern, values to rounding (the summation order differs), exact zero row
    sums structure (diagonal = minus the off-diagonal sum)."""
    from paper_1607_02955_b200 import solver as S

    n = 6000  # sparse connected graph: a path plus 2n random edges (mean degree ~6)
    ru, rv = rng.integers(0, n, 2 * n), rng.integers(0, n, 2 * n)
    keep = ru != rv
    u = np.r_[np.arange(n - 1), ru[keep]]
    v = np.r_[np.arange(1, n), rv[keep]]
    g = P.Graph.from_edges(u, v, rng.random(u.size) + 0.5, n=n)
    A = S._validate_laplacian(P.laplacian(g))
    # Galerkin: random aggregation with aggregates of 1..6 nodes
    agg = np.sort(rng.integers(0, 2000, 6000))
    agg = np.unique(agg, return_inverse=True)[1]
    nc = int(agg.max()) + 1
    host = S._galerkin(A, agg, nc)
    dev = S._coarse_operator_dev(A, agg, nc)
    for a, b in ((host, dev),):
        assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
        assert np.allclose(a.data, b.data, rtol=1e-13, atol=0)
    assert np.abs(np.asarray(dev.sum(axis=1))).max() <= 1e-12 * np.abs(dev.data).max()
    # Schur complement of a greedy independent low-degree set
    f = S._elim_select(A, 6)
    assert f.size > 100
    host, rec = S._eliminate_set(A, f)
    cmap = np.full(A.shape[0], -1, dtype=np.int64)
    cmap[rec.c_nodes] = np.arange(rec.c_nodes.size)
    dev = S._coarse_operator_dev(A, cmap, rec.c_nodes.size, f)
    assert np.array_equal(host.indptr, dev.indptr) and np.array_equal(host.indices, dev.indices)
    assert np.allclose(host.data, dev.data, rtol=1e-12, atol=0)
    # a hierarchy built with the device operators solves to the same answers
    saved = S.DEVICE_SETUP_MIN_NNZ, S.DEVICE_SETUP_MIN_N0, S.HUB_DEGREE_RATIO
    try:
        S.DEVICE_SETUP_MIN_NNZ, S.DEVICE_SETUP_MIN_N0, S.HUB_DEGREE_RATIO = 1, 1, 0.0
        h_dev = P.setup(P.laplacian(g), P.SolverConfig(tau=1e-10))
        assert S._device_setup_on and len(h_dev.levels) >= 2
    finally:
        S.DEVICE_SETUP_MIN_NNZ, S.DEVICE_SETUP_MIN_N0, S.HUB_DEGREE_RATIO = saved
        S._device_setup_on = False
    b = rng.standard_normal((4, g.n))
    b -= b.mean(axis=1, keepdims=True)
    x = np.stack([p.values for p in P.solve_many(h_dev, b)])
    L = P.laplacian(g)
    assert max(np.linalg.norm(L @ x[i] - b[i]) / np.linalg.norm(b[i]) for i in range(4)) <= 1e-10


def test_device_validation_matches_host(rng, monkeypatch):
    """_validate_laplacian's checks (solver.py:190-211) on the GPU for large
    inputs: same verdicts and the same rebuilt matrix as the host route."""
    import scipy.sparse as sp
    from paper_1607_02955_b200 import solver as S

    u, v, w = random_connected_graph_edges(800, rng, weighted=True)
    L = P.laplacian(P.Graph.from_edges(u, v, w, n=800))
    host = S._validate_laplacian(L)
    monkeypatch.setattr(S, "DEVICE_SETUP_MIN_NNZ", 1)
    dev = S._validate_laplacian(L)
    assert np.array_equal(host.indptr, dev.indptr) and np.array_equal(host.indices, dev.indices)
    assert np.array_equal(host.data, dev.data)
    bad = L.tolil(copy=True)
    bad[3, 7] = bad[3, 7] - 0.5
    with pytest.raises(P.DomainError, match="symmetric"):
        S._validate_laplacian(bad.tocsr())
    bad = L.tolil(copy=True)
    bad[5, 5] = bad[5, 5] + 1.0
    with pytest.raises(P.DomainError, match="row sums"):
        S._validate_laplacian(bad.tocsr())
    bad = L.tolil(copy=True)
    j = L[9].indices[L[9].indices != 9][0]
    bad[9, j] = 0.25
    bad[j, 9] = 0.25
    bad[9, 9] = bad[9, 9] - 0.25 + L[9, j]
    bad[j, j] = bad[j, j] - 0.25 + L[j, 9]
    with pytest.raises(P.DomainError, match="positive off-diagonal"):
        S._validate_laplacian(bad.tocsr())
    two = sp.block_diag([L, L], format="csr")
    with pytest.raises(P.DomainError, match="not connected"):
        S._validate_laplacian(two)


def test_segment_launch_forms_agree_bitwise():
    """Hub rows: the sweep segments computed by a k_seg launch of their own
    (with column windows and the bounded first sweep's leading-segment lists)
    give bit for bit the solution of the in-kernel segment form."""
    import hashlib
    import os
    import subprocess
    import sys

    code = r'''
import hashlib, numpy as np
import paper_1607_02955_b200 as P
rng = np.random.default_rng(3)
n = 4000
hubs = np.arange(12)
u = [np.arange(n - 1)]; v = [np.arange(1, n)]
for hb in hubs:  # hubs of 700-3000 neighbours
    nb = rng.choice(np.arange(12, n), size=700 + 200 * int(hb), replace=False)
    u.append(np.full(nb.size, hb)); v.append(nb)
u = np.concatenate(u); v = np.concatenate(v)
keep = u != v
g = P.Graph.from_edges(u[keep], v[keep], rng.random(int(keep.sum())) + 0.5, n=n)
h = P.setup(P.laplacian(g), P.SolverConfig(tau=1e-9), stall_breaker=False)
b = rng.standard_normal((40, n)); b -= b.mean(axis=1, keepdims=True)
x = np.stack([p.values for p in P.solve_many(h, b)])
assert max(p for p in [h.stats.max_residual]) <= 1e-9
print("HASH", hashlib.sha256(x.tobytes()).hexdigest())
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for name, pre in (("own_launch", "1"), ("in_kernel", "1000000000")):
        env = dict(os.environ, PYTHONPATH=root, CF_PRE_SEG_MIN=pre, CF_WIN_ROWS="256",
                   CF_WIN_DEG="128")
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out[name] = [ln for ln in r.stdout.splitlines() if ln.startswith("HASH")][0]
    assert out["own_launch"] == out["in_kernel"]
