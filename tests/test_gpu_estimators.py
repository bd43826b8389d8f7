"""GPU parity tests of the estimator path: bit-exact seeded JL right-hand
sides, closeness values vs the reference's golden values, the oracle and the
exact pseudo-inverse (SURVEY.md §8(c) parity protocol)."""

import math

import numpy as np
import pytest

import paper_1607_02955_b200 as P
from conftest import dense_pinv_resistance, golden, random_connected_graph_edges
from oracle import lamg_oracle as O
from paper_1607_02955_b200 import generators as G
from paper_1607_02955_b200.resistance import jl_rhs_rows

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [0, 1, 17])
def test_jl_rhs_bit_exact_vs_oracle(seed, rng):
    # odd edge count so rows start at odd half-word offsets too
    u, v, w = random_connected_graph_edges(300, np.random.default_rng(seed), weighted=True)
    g = P.Graph.from_edges(u, v, w, n=300)
    og = O.graph_from_edges(u, v, w, n=300)
    h = P.setup(P.laplacian(g))
    for k in (1, 7, 64, 300):
        ref, _ = O.jl_rhs(og, k, seed)
        got = jl_rhs_rows(g, h, k, seed)
        assert np.array_equal(got, ref), (k, np.abs(got - ref).max())
    ref, _ = O.jl_rhs(og, 300, seed)
    got = jl_rhs_rows(g, h, 300, seed, row0=37, rows=100)
    assert np.array_equal(got, ref[37:137])


def test_config1_rhs_golden():
    d = golden("config1.npz")
    g = G.grid_graph(64)
    h = P.setup(P.laplacian(g))
    got = jl_rhs_rows(g, h, 64, 0, rows=4)
    assert np.array_equal(got, d["y_rows_0_3"])


def test_config1_closeness_parity():
    """C1: JL (k=64, seed 0) and sampling (64 pivots, seed 0) vs the reference
    at tau 1e-8 (rel 1e-6) and both vs the exact pseudo-inverse."""
    d = golden("config1.npz")
    g = G.grid_graph(64)
    eps = float(d["eps"])
    q = d["query"]
    for tau, tag in ((1e-8, "1em08"), (1e-10, "1em10")):
        cfg = P.SolverConfig(tau=tau)
        h = P.setup(P.laplacian(g), cfg)
        jl = P.cf_closeness_projection(g, h, q, eps, 0, cfg)
        assert jl.params["k"] == 64
        assert np.allclose(jl.vector(q), d[f"jl_{tag}"], rtol=1e-6 if tau == 1e-8 else 1e-8)
        sm = P.cf_closeness_sampling(g, h, [0], 64, 0, cfg)
        assert np.allclose(sm.vector([0]), d[f"samp_{tag}"], rtol=1e-6 if tau == 1e-8 else 1e-8)
        assert h.stats.max_residual <= tau
    exact_jl = O.jl_exact_pinv(O.grid_graph(64), 64, 0, q)
    cfg = P.SolverConfig(tau=1e-8)
    h = P.setup(P.laplacian(g), cfg)
    jl = P.cf_closeness_projection(g, h, q, eps, 0, cfg)
    assert np.allclose(jl.vector(q), exact_jl, rtol=1e-6)


def test_sketch_and_sums_match_oracle(rng):
    u, v, w = random_connected_graph_edges(120, rng, weighted=True)
    g = P.Graph.from_edges(u, v, w, n=120)
    og = O.graph_from_edges(u, v, w, n=120)
    cfg = P.SolverConfig(tau=1e-11)
    h = P.setup(P.laplacian(g), cfg)
    sk = P.build_sketch(g, h, 0.3, 5, cfg)
    assert sk.k == O.sketch_rows(120, 0.3)
    _, rhs = O.jl_rhs(og, sk.k, 5)
    pinv = np.linalg.pinv(O.laplacian(og).toarray())
    z_exact = rhs @ pinv
    assert np.abs(sk.z - z_exact).max() <= 1e-8 * np.abs(z_exact).max()
    assert np.abs(sk.z.mean(axis=1)).max() < 1e-10
    sums = P.sketch_distance_sums(sk, [3, 50])
    fused = P.cf_closeness_projection(g, h, [3, 50], 0.3, 5, cfg).vector([3, 50])
    assert np.allclose((120 - 1) / sums, fused, rtol=1e-10)


def test_resistance_kats():
    d = golden("kats.npz")
    h = P.setup(P.laplacian(G.path_graph(3)))
    assert P.effective_resistance(h, 0, 2) == pytest.approx(2.0, rel=1e-6)
    assert P.effective_resistance(h, 1, 1) == 0.0
    h = P.setup(P.laplacian(G.complete_graph(3)))
    assert P.effective_resistance(h, 0, 1) == pytest.approx(float(d["k3_r01"]), rel=1e-6)
    g = P.Graph.from_edges([0, 1, 2], [1, 2, 3], [2.0, 4.0, 0.5])
    h = P.setup(P.laplacian(g))
    assert P.effective_resistance(h, 0, 3) == pytest.approx(2.75, rel=1e-6)
    g = P.Graph.from_edges([0, 0], [1, 1], [1.5, 0.5])
    h = P.setup(P.laplacian(g))
    assert P.effective_resistance(h, 0, 1) == pytest.approx(0.5, rel=1e-8)
    g = G.complete_graph(3)
    h = P.setup(P.laplacian(g))
    assert np.allclose(P.cf_closeness_exact(g, h, [0, 1, 2]).vector([0, 1, 2]), 1.5, rtol=1e-6)


def test_sampling_and_exact_vs_pinv(rng):
    u, v, w = random_connected_graph_edges(40, rng, weighted=True)
    g = P.Graph.from_edges(u, v, w, n=40)
    cfg = P.SolverConfig(tau=1e-10, max_direct_size=16)
    h = P.setup(P.laplacian(g), cfg)
    r = dense_pinv_resistance(P.laplacian(g).toarray())
    exact = (40 - 1) / r.sum(axis=1)
    got = P.cf_closeness_exact(g, h, range(40), cfg).vector(range(40))
    assert np.allclose(got, exact, rtol=1e-7)
    samp = P.cf_closeness_sampling(g, h, range(40), k=40, seed=5, config=cfg).vector(range(40))
    assert np.allclose(samp, exact, rtol=1e-7)
    piv = P.pivot_set(40, 9, 3)
    s = P.cf_closeness_sampling(g, h, [0, 7], k=9, seed=3, config=cfg).vector([0, 7])
    for v_, sv in zip([0, 7], s):
        assert sv == pytest.approx((9 / 40) * 39 / r[v_, piv].sum(), rel=1e-7)


def test_k1_own_pivot_undefined():
    g = G.path_graph(3)
    h = P.setup(P.laplacian(g))
    piv = int(P.pivot_set(3, 1, 0)[0])
    with pytest.raises(P.UndefinedScoreError):
        P.cf_closeness_sampling(g, h, [piv], k=1, seed=0)


@pytest.mark.slow
def test_config2_closeness_parity():
    """C2 (BA 1e5, JL k=128, 100 queries): vs the reference at tau_parity=1e-10
    (both sides) within 1e-8, and at the config tau 1e-6 within 1e-6."""
    d = golden("config2.npz")
    g = G.barabasi_albert_graph(100000, 4, 1)
    assert g.m == int(d["m"])
    eps = float(d["eps"])
    q = d["query"]
    for tau, tag, tol in ((1e-10, "1em10", 1e-8), (1e-6, "1em06", 1e-6)):
        cfg = P.SolverConfig(tau=tau)
        h = P.setup(P.laplacian(g), cfg)
        assert h.level_sizes == d["sizes"].tolist()
        jl = P.cf_closeness_projection(g, h, q, eps, 0, cfg)
        rel = np.abs(jl.vector(q) / d[f"jl_{tag}"] - 1).max()
        assert rel <= tol, (tau, rel)
        assert h.stats.max_residual <= tau


def test_jl_rhs_bit_exact_with_hub_nodes():
    """Nodes above the hub threshold take the CTA-per-hub path; still
    bit-identical to the reference's ascending-edge sums."""
    rng = np.random.default_rng(8)
    n = 6000
    u = np.r_[np.zeros(n - 1, dtype=np.int64), np.ones(2500, dtype=np.int64),
              rng.integers(0, n, 3000)]
    v = np.r_[np.arange(1, n), rng.integers(2, n, 2500), rng.integers(0, n, 3000)]
    w = rng.uniform(0.5, 2.0, u.size)
    g = P.Graph.from_edges(u, v, w, n=n)
    og = O.graph_from_edges(u, v, w, n=n)
    assert np.diff(g.indptr).max() > 2048
    h = P.setup(P.laplacian(g))
    for k in (8, 64, 200):
        ref, _ = O.jl_rhs(og, k, 5)
        assert np.array_equal(jl_rhs_rows(g, h, k, 5), ref)


@pytest.mark.slow
def test_config3_closeness_parity():
    """C3 (RGG 1e6, max-degree node): JL k=128 (Q seed 0) and sampling with 256
    pivots (seed 3) vs the reference's own values (tests/golden/config3.npz,
    make_golden.py c3 / c3tau10).

    SURVEY.md 8(c) parity protocol: closeness at tau_parity 1e-10 on both
    sides, held to the north star's 1e-6 relative (measured: JL 6.4e-8,
    sampling 2.2e-11).  A residual tolerance does not pin closeness to its own
    size on a geometric graph (the Laplacian's condition number amplifies it;
    SURVEY A.3: 2.2e-5 between two valid reference settings on the grid), so at
    each tolerance the accuracy bar is: our value is no further from the
    tightly converged value (ours at 1e-12) than max(1e-8, 2x) the reference's
    value at the same tolerance is."""
    import os
    from conftest import GOLDEN
    from paper_1607_02955_b200 import configs
    if not os.path.exists(os.path.join(GOLDEN, "config3.npz")):
        pytest.skip("config3.npz not generated")
    d = golden("config3.npz")
    bc = configs.make("c3")
    g = bc.graph
    assert (g.n, g.m, int(bc.query[0])) == (int(d["n"]), int(d["m"]), int(d["u"]))
    u = [int(d["u"])]
    h = P.setup(P.laplacian(g), P.SolverConfig(tau=1e-12))
    assert h.level_sizes == d["sizes"].tolist()
    ours = {}
    for tau in (1e-12, 1e-10, 1e-6):  # stats accumulate: strict tolerances first
        cfg = P.SolverConfig(tau=tau)
        jl = P.cf_closeness_projection(g, h, u, float(d["eps"]), 0, cfg).vector(u)[0]
        sm = P.cf_closeness_sampling(g, h, u, 256, 3, cfg).vector(u)[0]
        assert h.stats.max_residual <= tau
        ours[tau] = {"jl": jl, "samp": sm}
    for est in ("jl", "samp"):
        conv = ours[1e-12][est]
        for tau, tag in ((1e-10, "1em10"), (1e-6, "1em06")):
            if f"{est}_{tag}" not in d.files:
                continue
            ref = float(d[f"{est}_{tag}"][0])
            err_ref = abs(ref / conv - 1)
            err_ours = abs(ours[tau][est] / conv - 1)
            print(est, tau, "ours vs ref", abs(ours[tau][est] / ref - 1), "err ref", err_ref,
                  "err ours", err_ours)
            assert err_ours <= max(1e-8, 2 * err_ref), (est, tau, err_ours, err_ref)
            if tau == 1e-10:
                assert abs(ours[tau][est] / ref - 1) <= 1e-6, (est, tau)


def _rmat_row_range_parity(name, cfg_name, eps_of):
    """Shared body of the C4 / C5 parity tests: JL partial closeness sums over
    sketch rows [0, jl_rows) -- S_v is additive over sketch rows
    (resistance.py:218-237), so a row range pins the whole estimate -- against
    the golden values, at tau_parity 1e-10 (north-star bar 1e-6 relative) and
    at the configuration's tau 1e-6 (our error against the tightly converged
    value at most max(1e-8, 2x) the golden side's at the same tolerance)."""
    import os
    from conftest import GOLDEN
    from paper_1607_02955_b200 import configs
    from paper_1607_02955_b200.resistance import sketch_closeness_sums
    if not os.path.exists(os.path.join(GOLDEN, name)):
        pytest.skip(f"{name} not generated")
    d = golden(name)
    if "jl_psum_1em10" not in d.files:
        pytest.skip(f"{name} holds no JL values yet")
    bc = configs.make(cfg_name)
    g = bc.graph
    assert (g.n, g.m, bc.jl_k) == (int(d["n"]), int(d["m"]), int(d["k"]))
    q = np.asarray(d["query"], dtype=np.int64)
    assert np.array_equal(np.asarray(bc.query, dtype=np.int64), q)
    rows = int(d["jl_rows"])
    h = P.setup(P.laplacian(g), P.SolverConfig(tau=1e-12))
    eps = eps_of(bc)
    ours = {}
    for tau in (1e-12, 1e-10, 1e-6):
        cfg = P.SolverConfig(tau=tau)
        k, sums, res = sketch_closeness_sums(g, h, eps, bc.jl_seed, q, cfg, rows=(0, rows))
        assert k == bc.jl_k and res.max() <= tau
        ours[tau] = sums
    conv = ours[1e-12]
    ref10 = np.asarray(d["jl_psum_1em10"])
    rel10 = np.abs(ours[1e-10] / ref10 - 1).max()
    print(cfg_name, "tau 1e-10: ours vs golden", rel10)
    assert rel10 <= 1e-6
    if "jl_psum_1em06" in d.files:
        err_ref = np.abs(np.asarray(d["jl_psum_1em06"]) / conv - 1).max()
        err_ours = np.abs(ours[1e-6] / conv - 1).max()
        print(cfg_name, "tau 1e-6: err ours", err_ours, "err golden", err_ref)
        assert err_ours <= max(1e-8, 2 * err_ref)
    return d, bc, g, h


@pytest.mark.slow
def test_config4_closeness_parity():
    """C4 (R-MAT scale 20, weighted, 1000 query nodes, k = 256): partial JL sums
    over the first sketch rows vs the REFERENCE PACKAGE's own values
    (tests/golden/config4.npz: reference setup 3,576 levels / 1,432 s, then its
    solve_many on the centred rows; tests/golden/make_golden.py c4).  This is
    the graph where this build's hierarchy differs from the reference's (stall
    breaker, hub aggregates), so the check is on closeness, not on levels."""
    _rmat_row_range_parity("config4.npz", "c4", lambda bc: bc.epsilon)


@pytest.mark.slow
def test_config5_closeness_parity():
    """C5 (R-MAT scale 22, max-degree node, k = 650): partial JL sums and the
    sampling estimator's amortised resistances R(u, t) for the first pivots vs
    the CPU oracle's restatement of the reference solve loop on an exported
    copy of this build's host hierarchy (tests/golden/make_golden_c5.py; the
    reference's own setup cannot finish at this scale -- see that script).  At
    tau_parity the solutions are the pseudo-inverse solutions to ~1e-10, so the
    values do not depend on the hierarchy that preconditioned them."""
    d, bc, g, h = _rmat_row_range_parity("config5.npz", "c5", lambda bc: bc.epsilon)
    if "samp_r_1em10" in d.files:
        from paper_1607_02955_b200.resistance import resistances_from_node
        u = int(d["query"][0])
        piv = np.asarray(d["samp_pivots"], dtype=np.int64)
        cfg = P.SolverConfig(tau=1e-10)
        rr = resistances_from_node(h, u, piv, cfg, cache={})
        rel = np.abs(rr / np.asarray(d["samp_r_1em10"]) - 1).max()
        print("c5 sampling R(u, t) vs golden", rel)
        assert rel <= 1e-6


def test_exact_closeness_device_reduction_vs_pinv_and_host_route():
    """cf_closeness_exact reduces the n node solutions on the device
    (cf_exact_sums); it equals the dense pseudo-inverse value and the host
    four-term route of resistances_from_node (resistance.py:102-130) summed
    over every target, at n ~ 1,600 (several 128-column chunks + a tail)."""
    g = G.barabasi_albert_graph(1600, 3, 11)
    cfg = P.SolverConfig(tau=1e-10)
    h = P.setup(P.laplacian(g), cfg)
    q = [0, 5, 801, 1599]
    got = P.cf_closeness_exact(g, h, q, cfg).vector(q)
    r = dense_pinv_resistance(P.laplacian(g).toarray())
    exact = (g.n - 1) / r[q].sum(axis=1)
    assert np.allclose(got, exact, rtol=1e-8)
    cache = {}
    host = [(g.n - 1) / P.resistances_from_node(h, v, np.arange(g.n), cfg, cache=cache).sum()
            for v in q]
    assert np.allclose(got, host, rtol=1e-9)
    assert h.stats.max_residual <= 1e-10


@pytest.mark.slow
def test_exact_closeness_vs_reference_10k():
    """n = 10^4 BA graph: device exact closeness vs the reference's own
    cf_closeness_exact (tests/golden/exact10k.npz, tau 1e-8)."""
    d = golden("exact10k.npz")
    g = G.barabasi_albert_graph(10000, 3, 9)
    cfg = P.SolverConfig(tau=1e-8)
    h = P.setup(P.laplacian(g), cfg)
    assert h.level_sizes == d["sizes"].tolist()
    q = d["query"].tolist()
    got = P.cf_closeness_exact(g, h, q, cfg).vector(q)
    assert np.allclose(got, d["exact"], rtol=1e-6), np.abs(got / d["exact"] - 1).max()


def test_jl_multi_chunk_pipeline_bitwise():
    """A sketch of several device chunks (the next chunk's right-hand sides
    are built on a second stream while the current chunk solves, and a
    129..192-row remainder runs as one wide chunk) gives bit for bit the
    per-row parts of the same rows solved in separate single-chunk calls."""
    from paper_1607_02955_b200.resistance import combine_row_parts, sketch_closeness_sums

    g = G.grid_graph(40)
    cfg = P.SolverConfig(tau=1e-8)
    h = P.setup(P.laplacian(g), cfg)
    q = np.array([0, 777, 1599])
    eps = math.sqrt(math.log(g.n) / (430 - 0.5))
    k, sums, res, parts = sketch_closeness_sums(g, h, eps, 5, q, cfg, row_parts=True)
    assert k == 430 and res.max() <= 1e-8  # chunks of 128, 128, 174 (wide)
    pieces = []
    for lo, hi in ((0, 128), (128, 256), (256, 384), (384, 430)):
        pieces.append(sketch_closeness_sums(g, h, eps, 5, q, cfg, rows=(lo, hi), row_parts=True)[3])
    assert np.array_equal(parts, np.vstack(pieces))
    assert np.array_equal(sums, combine_row_parts(np.vstack(pieces), g.n))
