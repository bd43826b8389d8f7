"""Smoother-schedule sweep on one configuration: JL estimate time and V-cycles
per right-hand side for several (pre, post) sweep counts.

    python tools/smooth_sweep.py --config c4 --steps 1,2 2,1 1,1 2,2
"""
import argparse
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1607_02955_b200 as P  # noqa: E402
from paper_1607_02955_b200 import configs  # noqa: E402
from paper_1607_02955_b200.resistance import sketch_closeness_sums  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--steps", nargs="+", default=["1,2", "1,1", "2,1", "2,2"])
args = ap.parse_args()
bc = configs.make(args.config)
h = P.setup(P.laplacian(bc.graph), P.SolverConfig(tau=bc.tau))
eps = math.sqrt(math.log(bc.graph.n) / (bc.jl_k - 0.5))
for st in args.steps:
    nu = tuple(int(x) for x in st.split(","))
    cfg = P.SolverConfig(tau=bc.tau, smoothing_steps=nu)
    for rep in range(3):
        v0 = h.stats.vcycles
        t = time.perf_counter()
        k, sums, res = sketch_closeness_sums(bc.graph, h, eps, bc.jl_seed, bc.query, cfg)
        dt = time.perf_counter() - t
    print(f"{args.config} nu={nu} {dt * 1e3:.1f} ms  vcycles/rhs={(h.stats.vcycles - v0) / k:.2f} "
          f"score={(bc.graph.n - 1) / sums[0]:.10g} maxres={res.max():.2e}", flush=True)
