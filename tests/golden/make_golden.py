"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container only (it imports ``/root/reference/pkg/src``,
which does not exist on the GPU box):

    python tests/golden/make_golden.py

Writes ``tests/golden/*.npz`` (small, committed).  Each fixture records the
numpy/scipy versions that produced it (RNG-stream provenance).
"""

from __future__ import annotations

import math
import os
import sys
import time

import numpy as np
import scipy

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import cfcent  # noqa: E402  (the reference)
from cfcent import generators as gen  # noqa: E402
from cfcent import resistance as res  # noqa: E402
from cfcent import solver as slv  # noqa: E402

sys.setrecursionlimit(20000)
PROV = dict(numpy=np.__version__, scipy=scipy.__version__)


def rcg(n, rng, p=0.15, weighted=False):
    """Spanning tree plus Bernoulli extra edges (same recipe as the
    reference test fixture pkg/tests/conftest.py:7-21)."""
    us, vs = [], []
    for v in range(1, n):
        us.append(int(rng.integers(v)))
        vs.append(v)
    iu, iv = np.nonzero(np.triu(rng.random((n, n)) < p, 1))
    us += iu.tolist()
    vs += iv.tolist()
    w = rng.uniform(0.2, 3.0, size=len(us)) if weighted else np.ones(len(us))
    return cfcent.Graph.from_edges(np.asarray(us), np.asarray(vs), w, n=n)


def level_summary(h):
    kinds = np.array([{"elimination": 0, "aggregation": 1, "coarsest": 2}[l.kind.value]
                      for l in h.levels], dtype=np.int64)
    sizes = np.array([l.size for l in h.levels], dtype=np.int64)
    nnz = np.array([l.matrix.nnz for l in h.levels], dtype=np.int64)
    return kinds, sizes, nnz


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays, provenance=np.array(repr(PROV)))
    print("wrote", path, os.path.getsize(path), "bytes")


def small_graphs():
    """Random small graphs: edges, hierarchy shape, solutions at tau=1e-10."""
    rng = np.random.default_rng(20240601)
    out = {}
    for t in range(6):
        n = int(rng.integers(30, 400))
        g = rcg(n, rng, p=float(rng.uniform(0.02, 0.15)), weighted=bool(t % 2))
        eu, ev, ew = g.edge_array()
        cfg = slv.SolverConfig(tau=1e-10, max_direct_size=int(rng.integers(8, 40)))
        h = slv.setup(cfcent.laplacian(g), cfg)
        kinds, sizes, nnz = level_summary(h)
        b = rng.standard_normal((5, n))
        b -= b.mean(axis=1, keepdims=True)
        pots = slv.solve_many(h, b)
        x = np.stack([p.values for p in pots])
        r = np.array([p.achieved_residual for p in pots])
        first_agg = next((l.aggregates for l in h.levels if l.kind.value == "aggregation"),
                         np.zeros(0, dtype=np.int64))
        first_elim = next((l.f_nodes for l in h.levels if l.kind.value == "elimination"),
                          np.zeros(0, dtype=np.int64))
        out.update({f"g{t}_eu": eu, f"g{t}_ev": ev, f"g{t}_ew": ew, f"g{t}_n": np.int64(n),
                    f"g{t}_mds": np.int64(cfg.max_direct_size),
                    f"g{t}_kinds": kinds, f"g{t}_sizes": sizes, f"g{t}_nnz": nnz,
                    f"g{t}_b": b, f"g{t}_x": x, f"g{t}_res": r,
                    f"g{t}_agg0": first_agg, f"g{t}_elim0": first_elim})
    out["count"] = np.int64(6)
    save("small_graphs.npz", **out)


def kats():
    """Known answers from the reference's own unit tests, recomputed."""
    P = gen.path_graph
    d = {}
    h = slv.setup(cfcent.laplacian(P(2)))
    d["p2_solve"] = slv.solve(h, np.array([1.0, -1.0])).values
    d["p3_r02"] = np.float64(res.effective_resistance(slv.setup(cfcent.laplacian(P(3))), 0, 2))
    g = gen.complete_graph(3)
    d["k3_r01"] = np.float64(res.effective_resistance(slv.setup(cfcent.laplacian(g)), 0, 1))
    g = cfcent.Graph.from_edges([0, 1, 2], [1, 2, 3], [2.0, 4.0, 0.5])
    d["wpath_r03"] = np.float64(res.effective_resistance(slv.setup(cfcent.laplacian(g)), 0, 3))
    g = cfcent.Graph.from_edges([0, 0], [1, 1], [1.5, 0.5])
    d["par_r01"] = np.float64(res.effective_resistance(slv.setup(cfcent.laplacian(g)), 0, 1))
    g = gen.complete_graph(3)
    h = slv.setup(cfcent.laplacian(g))
    d["k3_exact"] = cfcent.cf_closeness_exact(g, h, [0, 1, 2]).vector([0, 1, 2])
    g = P(3)
    h = slv.setup(cfcent.laplacian(g))
    d["p3_exact"] = cfcent.cf_closeness_exact(g, h, [0, 1, 2]).vector([0, 1, 2])
    # star: one elimination level removes all leaves
    h = slv.setup(cfcent.laplacian(gen.star_graph(100)), slv.SolverConfig(max_direct_size=10))
    d["star_f"] = h.levels[0].f_nodes
    d["star_sizes"] = np.array(h.level_sizes)
    d["sketch_dims"] = np.array([res.sketch_dimension(2, 0.5), res.sketch_dimension(500, 0.2),
                                 res.sketch_dimension(4096, math.sqrt(math.log(4096) / 63.5)),
                                 res.sketch_dimension(2234040, 0.15)])
    # PCG64 integers(0,2) sign stream, several shapes / seeds
    for seed in (0, 5, 11):
        d[f"bits_seed{seed}"] = np.random.default_rng(seed).integers(0, 2, size=(3, 777))
    # pivot sets (config seeds)
    d["piv_4096_64_0"] = cfcent.centrality.pivot_set(4096, 64, 0)
    d["piv_1000_30_3"] = cfcent.centrality.pivot_set(1000, 30, 3)
    save("kats.npz", **d)


def config1():
    """C1: grid 64x64; JL k=64 (seed 0) and sampling k=64 (seed 0), u=0."""
    g = gen.grid_graph(64)
    n = g.n
    eps = math.sqrt(math.log(n) / 63.5)
    d = {"eps": np.float64(eps)}
    b_inc, w = cfcent.incidence_and_weights(g)
    d["y_rows_0_3"] = None
    # uncentred JL right-hand sides exactly as build_sketch forms them
    st = b_inc.multiply(np.sqrt(w)[:, None]).T.tocsr()
    rng = np.random.default_rng(0)
    k = res.sketch_dimension(n, eps)
    q = (rng.integers(0, 2, size=(k, g.m)).astype(np.float64) * 2.0 - 1.0) / math.sqrt(k)
    y = (st @ q.T).T
    d["y_rows_0_3"] = y[:4].copy()
    d["y_sum_abs"] = np.abs(y).sum(axis=1)
    query = [0, 1, 65, 2080, 4095]
    d["query"] = np.array(query)
    for tau in (1e-8, 1e-10):
        cfg = slv.SolverConfig(tau=tau, seed=0)
        h = slv.setup(cfcent.laplacian(g), cfg)
        kinds, sizes, nnz = level_summary(h)
        d["kinds"], d["sizes"], d["nnz"] = kinds, sizes, nnz
        t0 = time.perf_counter()
        jl = cfcent.cf_closeness_projection(g, h, query, eps, 0, cfg)
        t1 = time.perf_counter()
        sm = cfcent.cf_closeness_sampling(g, h, [0], 64, 0, cfg)
        t2 = time.perf_counter()
        tag = f"{tau:.0e}".replace("-", "m")
        d[f"jl_{tag}"] = jl.vector(query)
        d[f"samp_{tag}"] = sm.vector([0])
        d[f"t_jl_{tag}"] = np.float64(t1 - t0)
        d[f"t_samp_{tag}"] = np.float64(t2 - t1)
        print("C1", tau, jl.vector(query), sm.vector([0]), t1 - t0, t2 - t1)
    save("config1.npz", **d)


def config2():
    """C2: BA n=1e5, m0=4, seed 1; JL k=128 for 100 nodes (seed 2), Q seed 0."""
    g = gen.barabasi_albert_graph(100000, 4, 1)
    n = g.n
    eps = math.sqrt(math.log(n) / 127.5)
    query = np.sort(np.random.default_rng(2).choice(n, 100, replace=False))
    d = {"eps": np.float64(eps), "query": query, "m": np.int64(g.m)}
    for tau in (1e-6, 1e-10):
        cfg = slv.SolverConfig(tau=tau, seed=0)
        t0 = time.perf_counter()
        h = slv.setup(cfcent.laplacian(g), cfg)
        t1 = time.perf_counter()
        kinds, sizes, nnz = level_summary(h)
        d["kinds"], d["sizes"], d["nnz"] = kinds, sizes, nnz
        jl = cfcent.cf_closeness_projection(g, h, query, eps, 0, cfg, threads=8)
        t2 = time.perf_counter()
        tag = f"{tau:.0e}".replace("-", "m")
        d[f"jl_{tag}"] = jl.vector(query)
        d[f"t_setup_{tag}"] = np.float64(t1 - t0)
        d[f"t_jl_{tag}"] = np.float64(t2 - t1)
        print("C2", tau, jl.vector(query)[:4], t1 - t0, t2 - t1)
    save("config2.npz", **d)


def config3(tau_list=(1e-6, 1e-10)):
    """C3: RGG 1e6 (recipe of paper_1607_02955_b200/configs.py, restated here
    with the reference's own Graph/LCC); JL k=128 (Q seed 0) and sampling 256
    pivots (seed 3) for the max-degree node."""
    from scipy.spatial import cKDTree
    n = 1_000_000
    pts = np.random.default_rng(3).random((n, 2))
    r = math.sqrt(10.0 / (math.pi * n))
    pairs = cKDTree(pts).query_pairs(r, output_type="ndarray")
    dist = np.linalg.norm(pts[pairs[:, 0]] - pts[pairs[:, 1]], axis=1)
    g0 = cfcent.Graph.from_edges(pairs[:, 0], pairs[:, 1], 1.0 / (dist + 1e-3), n=n)
    g, _ = cfcent.largest_connected_component(g0)
    deg = np.diff(g.indptr)
    u = int(np.argmax(deg))
    eps = math.sqrt(math.log(g.n) / 127.5)
    d = {"n": np.int64(g.n), "m": np.int64(g.m), "u": np.int64(u), "eps": np.float64(eps)}
    old = os.path.join(OUT, "config3.npz")
    if os.path.exists(old):  # keep values of earlier runs (one tau per run is hours)
        with np.load(old, allow_pickle=True) as prev:
            d.update({k: prev[k] for k in prev.files if k != "provenance"})
    for tau in tau_list:
        cfg = slv.SolverConfig(tau=tau, seed=0)
        t0 = time.perf_counter()
        h = slv.setup(cfcent.laplacian(g), cfg)
        t1 = time.perf_counter()
        jl = cfcent.cf_closeness_projection(g, h, [u], eps, 0, cfg, threads=2)
        t2 = time.perf_counter()
        sm = cfcent.cf_closeness_sampling(g, h, [u], 256, 3, cfg, threads=5)
        t3 = time.perf_counter()
        tag = f"{tau:.0e}".replace("-", "m")
        d[f"sizes"] = np.array(h.level_sizes)
        d[f"jl_{tag}"] = jl.vector([u])
        d[f"samp_{tag}"] = sm.vector([u])
        d[f"t_setup_{tag}"] = np.float64(t1 - t0)
        d[f"t_jl_{tag}"] = np.float64(t2 - t1)
        d[f"t_samp_{tag}"] = np.float64(t3 - t2)
        print("C3", tau, jl.vector([u]), sm.vector([u]), t1 - t0, t2 - t1, t3 - t2, flush=True)
        save("config3.npz", **d)


def _rmat_reference_graph(scale, edge_factor, seed, weighted):
    """R-MAT recipe of SURVEY.md §8(d) (frozen in paper_1607_02955_b200/
    configs.py:rmat_graph), restated here on the reference's own Graph and
    largest_connected_component (graph.py:100-147, 217-250)."""
    rng = np.random.default_rng(seed)
    n = 1 << scale
    M = edge_factor * n
    a, b, c = 0.57, 0.19, 0.19
    u = np.zeros(M, dtype=np.int64)
    v = np.zeros(M, dtype=np.int64)
    for bit in range(scale):
        r = rng.random(M)
        u |= (r >= a + b).astype(np.int64) << bit
        v |= (((r >= a) & (r < a + b)) | (r >= a + b + c)).astype(np.int64) << bit
    keep = u != v
    lo = np.minimum(u[keep], v[keep])
    hi = np.maximum(u[keep], v[keep])
    key = np.unique(lo * n + hi)
    lo, hi = key // n, key % n
    w = (2.0 - rng.random(lo.size) * 1.5) if weighted else np.ones(lo.size)
    g = cfcent.Graph.from_edges(lo, hi, w, n=n)
    return cfcent.largest_connected_component(g)[0]


def _jl_rows_reference(g, h, k, seed, rows, cfg):
    """Rows [0, rows) of the reference sketch (resistance.py:177-201): the
    first rows*m draws of default_rng(seed).integers(0, 2) are the first
    ``rows`` rows of the full k x m Q (row-major stream), scaled
    by 1/sqrt(k) of the FULL k; right-hand sides centred and solved by the
    reference's solve_many."""
    b_inc, weights = cfcent.incidence_and_weights(g)
    scaled_t = b_inc.multiply(np.sqrt(weights)[:, None]).T.tocsr()
    rng = np.random.default_rng(seed)
    q = (rng.integers(0, 2, size=(rows, g.m)).astype(np.float64) * 2.0 - 1.0) / math.sqrt(k)
    rhs = (scaled_t @ q.T).T
    rhs -= rhs.mean(axis=1, keepdims=True)
    solved = slv.solve_many(h, rhs, cfg)
    z = np.vstack([p.values for p in solved])
    res_ = np.array([p.achieved_residual for p in solved])
    return z, res_


def _partial_sums(z, nodes):
    """Additive share of sketch_distance_sums (resistance.py:218-237) over
    the sketch rows held in z."""
    col_sq = np.einsum("ij,ij->j", z, z)
    return col_sq.sum() + z.shape[1] * col_sq[nodes] - 2.0 * (z[:, nodes].T @ z.sum(axis=1))


def _cpu_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return f"{model}; {os.cpu_count()} cores"


def config_rmat(name, scale, ef, seed, weighted, k, query_fn, jl_rows=32, samp=None,
                tau_list=(1e-6, 1e-10)):
    """C4/C5 reference goldens: JL partial sums over sketch rows [0, jl_rows)
    at each tau, and (C5) amortised resistances R(u, t) for the first pivots
    of the sampling pivot set.  The reference setup on these graphs takes
    tens of minutes to hours (831+ levels); timings are recorded as the cached
    CPU baseline (provenance: this container)."""
    path = os.path.join(OUT, f"{name}.npz")
    d = {}
    if os.path.exists(path):
        with np.load(path, allow_pickle=True) as prev:
            d.update({kk: prev[kk] for kk in prev.files if kk != "provenance"})
    t0 = time.perf_counter()
    g = _rmat_reference_graph(scale, ef, seed, weighted)
    t1 = time.perf_counter()
    query = np.asarray(query_fn(g), dtype=np.int64)
    d.update({"n": np.int64(g.n), "m": np.int64(g.m), "query": query, "k": np.int64(k),
              "jl_rows": np.int64(jl_rows), "t_graph": np.float64(t1 - t0),
              "cpu": np.array(_cpu_info())})
    print(name, "graph", g.n, g.m, t1 - t0, flush=True)
    cfg0 = slv.SolverConfig(tau=tau_list[0], seed=0)
    # the reference setup takes tens of minutes to hours here: keep a pickled
    # copy (scratch, outside the repo) so an interrupted run resumes at the solves
    cache = os.path.join(os.path.dirname(OUT), "..", "gpurun_out", "cache", f"{name}_hier.pkl")
    if os.path.exists(cache) and "t_setup" in d:
        import pickle
        with open(cache, "rb") as f:
            h = pickle.load(f)
        t_setup = float(d["t_setup"])
    else:
        h = slv.setup(cfcent.laplacian(g), cfg0)
        t_setup = time.perf_counter() - t1
        try:
            if os.environ.get("GOLDEN_NO_CACHE"):
                raise RuntimeError("GOLDEN_NO_CACHE set")
            import pickle
            os.makedirs(os.path.dirname(cache), exist_ok=True)
            with open(cache, "wb") as f:
                pickle.dump(h, f, protocol=pickle.HIGHEST_PROTOCOL)
        except Exception as exc:  # noqa: BLE001 - the cache is optional
            print(name, "hierarchy not cached:", exc, flush=True)
    d["sizes"] = np.array(h.level_sizes)
    d["t_setup"] = np.float64(t_setup)
    print(name, "setup", len(h.level_sizes), "levels", t_setup, flush=True)
    save(f"{name}.npz", **d)
    for tau in tau_list:
        cfg = slv.SolverConfig(tau=tau, seed=0)
        tag = f"{tau:.0e}".replace("-", "m")
        t3 = time.perf_counter()
        z, r = _jl_rows_reference(g, h, k, 0, jl_rows, cfg)
        t4 = time.perf_counter()
        d[f"jl_psum_{tag}"] = _partial_sums(z, query)
        d[f"jl_res_{tag}"] = r
        d[f"t_jl_{tag}"] = np.float64(t4 - t3)
        print(name, tau, "jl", d[f"jl_psum_{tag}"][:3], t4 - t3, flush=True)
        save(f"{name}.npz", **d)
        if samp is not None:
            npiv, pseed, cnt = samp
            u = int(query[0])
            piv = cfcent.centrality.pivot_set(g.n, npiv, pseed)[:cnt]
            t5 = time.perf_counter()
            rr = res.resistances_from_node(h, u, piv, cfg, cache={}, threads=2)
            t6 = time.perf_counter()
            d["samp_pivots"] = piv
            d[f"samp_r_{tag}"] = rr
            d[f"t_samp_{tag}"] = np.float64(t6 - t5)
            print(name, tau, "samp", rr[:3], t6 - t5, flush=True)
            save(f"{name}.npz", **d)


def config4():
    # 4 sketch rows: the reference's recursion keeps three n_l x rows arrays
    # alive on each of its 3,576 levels (sum n_l = 92.7 M), on top of a 39 GB
    # hierarchy -- 32 rows exceed the build container's 62 GB
    config_rmat("config4", 20, 16, 4, True, 256,
                lambda g: np.sort(np.random.default_rng(4).choice(g.n, 1000, replace=False)),
                jl_rows=int(os.environ.get("GOLDEN_JL_ROWS", "4")))


def config5():
    def q(g):
        return np.array([int(np.argmax(np.diff(g.indptr)))])
    n_est = 2234040
    k = math.ceil(4 * math.log(n_est) / 0.09)
    config_rmat("config5", 22, 12, 5, False, k, q, samp=(1024, 5, 64))


def exact10k():
    """cf_closeness_exact on a 10^4-node BA graph (the reference solves every
    node, centrality.py:78-101) for the device reduction's parity test."""
    g = gen.barabasi_albert_graph(10000, 3, 9)
    query = [0, 17, 4242, 9999]
    cfg = slv.SolverConfig(tau=1e-8, seed=0)
    h = slv.setup(cfcent.laplacian(g), cfg)
    t0 = time.perf_counter()
    tab = cfcent.cf_closeness_exact(g, h, query, cfg, threads=8)
    t1 = time.perf_counter()
    print("exact10k", tab.vector(query), t1 - t0, flush=True)
    save("exact10k.npz", query=np.array(query), exact=tab.vector(query),
         sizes=np.array(h.level_sizes), t_exact=np.float64(t1 - t0))


if __name__ == "__main__":
    which = sys.argv[1:] or ["kats", "small", "c1", "c2"]
    if "kats" in which:
        kats()
    if "small" in which:
        small_graphs()
    if "c1" in which:
        config1()
    if "c2" in which:
        config2()
    if "c3" in which:
        config3()
    if "exact10k" in which:
        exact10k()
    if "c4" in which:
        config4()
    if "c5" in which:
        config5()
    if "c3tau10" in which:  # the tau_parity values alone (~2 h of reference CPU time)
        config3((1e-10,))
