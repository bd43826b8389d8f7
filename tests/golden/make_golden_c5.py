"""C5 golden values (R-MAT scale 22, ~4M nodes / 48.5M edges).

The reference's own setup does not finish on this graph in the build container
(its stage rule stalls into thousands of levels; C4, a quarter of the size,
already needs 3,576 levels and 1,415 s -- tests/golden/config4.npz -- and its
level storage alone would exceed this container's memory at scale 22), so,
as SURVEY.md §8(c) allows for exactly this case, the values come from the CPU
oracle's restatement of the reference solve loop (oracle/lamg_oracle.py:
solver.py:526-751 -- natural-order Gauss-Seidel, energy line search, FCG /
Jacobi-PCG fallbacks) run on an exported copy of THIS build's host hierarchy
(oracle/workloads.hierarchy_from_levels).  At tau_parity 1e-10 the solutions
are the pseudo-inverse solutions to ~1e-10 whatever hierarchy preconditions
the iteration, so the partial closeness sums below pin the device solve and
estimator kernels on C5 independently of their own arithmetic.

Stored (config5.npz): JL partial sums over sketch rows [0, rows) (additive
over rows, resistance.py:218-237) at tau 1e-6 and 1e-10, and the amortised
resistances R(u, t) (resistance.py:102-130) of the first pivots of the
sampling pivot set at tau 1e-10, u = the max-degree node.

    python tests/golden/make_golden_c5.py [rows] [pivots]
"""

import math
import os
import sys
import time

import numpy as np
import scipy.sparse as sp

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
OUT = os.path.dirname(os.path.abspath(__file__))

from oracle import lamg_oracle as O  # noqa: E402
from oracle import workloads as OW  # noqa: E402


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


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    npiv = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    sys.setrecursionlimit(20000)
    t0 = time.perf_counter()
    wl = OW.make("c5")
    g = wl["graph"]
    n = g[0].size - 1
    k = wl["jl_k"]
    u = int(wl["query"][0])
    print("c5 graph", n, g[0][-1] // 2, "k", k, "u", u, time.perf_counter() - t0, flush=True)
    # this build's host hierarchy (host setup code only; no device)
    import paper_1607_02955_b200 as P
    from paper_1607_02955_b200.graph import Graph

    pg = Graph(g[0], g[1], g[2])
    t1 = time.perf_counter()
    h = P.setup(P.laplacian(pg), P.SolverConfig(tau=1e-6))
    print("host setup", [lv.size for lv in h.levels], time.perf_counter() - t1, flush=True)
    d = {"n": np.int64(n), "m": np.int64(g[0][-1] // 2), "k": np.int64(k), "query": np.array([u]),
         "jl_rows": np.int64(rows), "sizes": np.array([lv.size for lv in h.levels]),
         "cpu": np.array(_cpu_info()),
         "source": np.array("oracle solve loop on this build's host hierarchy (reference setup "
                            "does not finish at this scale)")}
    # first `rows` sketch rows: the first rows*m draws of the row-major stream
    eu, ev, ew = O.canonical_edges(g)
    m = eu.size
    inc = sp.csr_matrix((np.tile([1.0, -1.0], m),
                         (np.repeat(np.arange(m), 2), np.column_stack([eu, ev]).ravel())),
                        shape=(m, n))
    st = inc.multiply(np.sqrt(ew)[:, None]).T.tocsr()
    rng = np.random.default_rng(wl["jl_seed"])
    q = (rng.integers(0, 2, size=(rows, m)).astype(np.float64) * 2.0 - 1.0) * (1.0 / math.sqrt(k))
    rhs = (st @ q.T).T
    rhs -= rhs.mean(axis=1, keepdims=True)
    del inc, st, q
    for tau in (1e-6, 1e-10):
        cfg = O.OracleConfig(tau=tau)
        oh = OW.hierarchy_from_levels(h.levels, cfg)
        tag = f"{tau:.0e}".replace("-", "m")
        t2 = time.perf_counter()
        z, res = O.solve_rows(oh, rhs, cfg)
        dt = time.perf_counter() - t2
        d[f"jl_psum_{tag}"] = O.jl_sums(z, [u])
        d[f"jl_res_{tag}"] = np.asarray(res)
        d[f"t_jl_{tag}"] = np.float64(dt)
        print("jl", tau, d[f"jl_psum_{tag}"], "max res", np.max(res), dt, flush=True)
        np.savez_compressed(os.path.join(OUT, "config5.npz"), **d)
    cfg = O.OracleConfig(tau=1e-10)
    oh = OW.hierarchy_from_levels(h.levels, cfg)
    sp_k, sp_seed, _ = wl["sampling"]
    piv = O.pivots(n, sp_k, sp_seed)[:npiv]
    t3 = time.perf_counter()
    rr = O.resistances_from(oh, u, piv, cfg, cache={})
    d["samp_pivots"] = piv
    d["samp_r_1em10"] = rr
    d["t_samp_1em10"] = np.float64(time.perf_counter() - t3)
    print("samp", rr[:4], time.perf_counter() - t3, flush=True)
    np.savez_compressed(os.path.join(OUT, "config5.npz"), **d)


if __name__ == "__main__":
    main()
