"""Closeness of a config's first query node at several tolerances (our solver).

    python tools/tau_sweep.py --config c3 --taus 1e-6,1e-8,1e-10
"""
import argparse
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1607_02955_b200 as P  # noqa: E402
from paper_1607_02955_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--taus", default="1e-6,1e-8,1e-10")
args = ap.parse_args()
bc = configs.make(args.config)
g = bc.graph
q = [int(bc.query[0])]
eps = math.sqrt(math.log(g.n) / (bc.jl_k - 0.5))
for tau in (float(t) for t in args.taus.split(",")):
    cfg = P.SolverConfig(tau=tau)
    h = P.setup(P.laplacian(g), cfg)
    t = time.perf_counter()
    jl = P.cf_closeness_projection(g, h, q, eps, bc.jl_seed, cfg).vector(q)[0]
    t1 = time.perf_counter()
    line = f"tau={tau:.0e} jl={jl!r} ({t1 - t:.2f}s)"
    if bc.sampling_pivots:
        sm = P.cf_closeness_sampling(g, h, q, bc.sampling_pivots, bc.sampling_seed, cfg).vector(q)[0]
        line += f" sampling={sm!r} ({time.perf_counter() - t1:.2f}s)"
    print(line, f"maxres={h.stats.max_residual:.2e}", flush=True)
