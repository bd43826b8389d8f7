"""Pin the CPU oracle (oracle/lamg_oracle.py) against golden vectors produced
by the reference package itself (tests/golden/make_golden.py)."""

import math

import numpy as np
import pytest

from conftest import golden
from oracle import lamg_oracle as O


def _graph_from_fixture(d, t):
    return O.graph_from_edges(d[f"g{t}_eu"], d[f"g{t}_ev"], d[f"g{t}_ew"], n=int(d[f"g{t}_n"]))


KIND = {"elim": 0, "agg": 1, "coarse": 2}


@pytest.mark.parametrize("t", range(6))
def test_small_graph_hierarchy_and_solutions(t):
    d = golden("small_graphs.npz")
    g = _graph_from_fixture(d, t)
    cfg = O.OracleConfig(tau=1e-10, max_direct_size=int(d[f"g{t}_mds"]))
    h = O.build_hierarchy(O.laplacian(g), cfg)
    kinds = [KIND[l["kind"]] for l in h["levels"]]
    sizes = [l["A"].shape[0] for l in h["levels"]]
    nnz = [l["A"].nnz for l in h["levels"]]
    assert kinds == d[f"g{t}_kinds"].tolist()
    assert sizes == d[f"g{t}_sizes"].tolist()
    assert nnz == d[f"g{t}_nnz"].tolist()
    agg = next((l["agg"] for l in h["levels"] if l["kind"] == "agg"), np.zeros(0))
    assert np.array_equal(agg, d[f"g{t}_agg0"])
    x, res = O.solve_rows(h, d[f"g{t}_b"], cfg)
    # same operations in the same order: agreement at roundoff level
    scale = np.abs(d[f"g{t}_x"]).max()
    assert np.abs(x - d[f"g{t}_x"]).max() <= 1e-12 * scale
    assert np.all(res <= 1e-10)


def test_kats():
    d = golden("kats.npz")
    h = O.build_hierarchy(O.laplacian(O.path_graph(2)))
    x, _ = O.solve_rows(h, np.array([1.0, -1.0]))
    assert np.allclose(x[0], d["p2_solve"], atol=1e-15)
    assert np.allclose(d["p2_solve"], [0.5, -0.5], atol=1e-12)
    assert d["p3_r02"] == pytest.approx(2.0, rel=1e-6)
    assert d["k3_r01"] == pytest.approx(2.0 / 3.0, rel=1e-6)
    assert d["wpath_r03"] == pytest.approx(0.5 + 0.25 + 2.0, rel=1e-6)
    assert d["par_r01"] == pytest.approx(0.5, rel=1e-8)
    assert np.allclose(d["k3_exact"], 1.5, rtol=1e-6)
    for seed in (0, 5, 11):
        bits = np.random.default_rng(seed).integers(0, 2, size=(3, 777))
        assert np.array_equal(bits, d[f"bits_seed{seed}"])
    assert np.array_equal(O.pivots(4096, 64, 0), d["piv_4096_64_0"])
    assert np.array_equal(O.pivots(1000, 30, 3), d["piv_1000_30_3"])
    assert d["sketch_dims"].tolist() == [
        O.sketch_rows(2, 0.5), O.sketch_rows(500, 0.2),
        O.sketch_rows(4096, math.sqrt(math.log(4096) / 63.5)), O.sketch_rows(2234040, 0.15)]
    assert d["sketch_dims"].tolist()[2] == 64 and d["sketch_dims"].tolist()[3] == 650
    # star: elimination removes every leaf
    h = O.build_hierarchy(O.laplacian(O.graph_from_edges(np.zeros(99, int), np.arange(1, 100))),
                          O.OracleConfig(max_direct_size=10))
    assert np.array_equal(h["levels"][0]["f"], d["star_f"])


def test_config1_hierarchy_rhs_and_scores():
    d = golden("config1.npz")
    g = O.grid_graph(64)
    eps = float(d["eps"])
    k = O.sketch_rows(4096, eps)
    assert k == 64
    raw, _ = O.jl_rhs(g, k, 0)
    assert np.array_equal(raw[:4], d["y_rows_0_3"])  # bit-exact seeded RHS
    assert np.array_equal(np.abs(raw).sum(axis=1), d["y_sum_abs"])
    cfg = O.OracleConfig(tau=1e-8)
    h = O.build_hierarchy(O.laplacian(g), cfg)
    assert [l["A"].shape[0] for l in h["levels"]] == d["sizes"].tolist()
    q = d["query"]
    s, _, _ = O.closeness_projection(g, h, q, eps, 0, cfg)
    assert np.allclose(s, d["jl_1em08"], rtol=1e-12)
    samp = O.closeness_sampling(g, h, [0], 64, 0, cfg)
    assert np.allclose(samp, d["samp_1em08"], rtol=1e-12)
    # the reference itself vs the exact pseudo-inverse with the same Q
    exact_jl = O.jl_exact_pinv(g, k, 0, q)
    assert np.allclose(d["jl_1em10"], exact_jl, rtol=1e-8)
    assert np.allclose(d["jl_1em08"], exact_jl, rtol=1e-6)


def test_workload_graphs_match_product_generators():
    """bench.py's CPU reference arm builds its input with oracle/workloads.py
    (no product code); the product arm with paper_1607_02955_b200/configs.py.
    Same recipe, same draws -> the same graph (small R-MAT / RGG / C1 / C2)."""
    from oracle import workloads as OW
    from paper_1607_02955_b200 import configs
    for og, pg in ((OW.rmat_graph(12, 8, 4, True), configs.rmat_graph(12, 8, 4, weighted=True)),
                   (OW.rmat_graph(11, 12, 5, False), configs.rmat_graph(11, 12, 5, weighted=False)),
                   (OW.rgg_graph(5000, 3), configs.rgg_graph(5000, 3)),
                   (OW.make("c1")["graph"], configs.make("c1").graph)):
        assert np.array_equal(og[0], pg.indptr)
        assert np.array_equal(og[1], pg.indices)
        assert np.array_equal(og[2], pg.weights)
    wl, bc = OW.make("c2"), configs.make("c2")
    assert np.array_equal(wl["graph"][1], bc.graph.indices)
    assert np.array_equal(wl["query"], bc.query)


def test_rmat_goldens_are_wired():
    """C4 / C5 fixtures (tests/golden/make_golden.py c4, make_golden_c5.py): the
    values the -m gpu parity tests compare against are present, converged to
    their tolerances and mutually consistent (the tau 1e-6 sums within 1e-6 of
    the tau 1e-10 ones -- the reference's own accuracy at the config tau)."""
    for name, rows, nq in (("config4.npz", 4, 1000), ("config5.npz", 8, 1)):
        d = golden(name)
        assert int(d["jl_rows"]) == rows and d["query"].size == nq
        for tag, tau in (("1em06", 1e-6), ("1em10", 1e-10)):
            assert d[f"jl_psum_{tag}"].shape == (nq,)
            assert d[f"jl_res_{tag}"].shape == (rows,) and d[f"jl_res_{tag}"].max() <= tau
        rel = np.abs(d["jl_psum_1em06"] / d["jl_psum_1em10"] - 1).max()
        assert rel <= 1e-6, rel
    d4, d5 = golden("config4.npz"), golden("config5.npz")
    # C4 comes from the reference package itself (its stalled 3,576-level hierarchy)
    assert (int(d4["n"]), int(d4["m"]), int(d4["k"])) == (646140, 15700710, 256)
    assert d4["sizes"].size == 3576 and float(d4["t_setup"]) > 1000
    # C5 from the oracle solve loop on this build's hierarchy (reference setup cannot finish)
    assert (int(d5["n"]), int(d5["m"]), int(d5["k"])) == (2234040, 48492111, 650)
    assert "oracle" in str(d5["source"]) and d5["samp_r_1em10"].shape == d5["samp_pivots"].shape
    assert np.all(d5["samp_r_1em10"] > 0)
