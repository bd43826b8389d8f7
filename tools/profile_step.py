"""Run one JL estimate step of a configuration (for ncu / compute-sanitizer).

    python tools/profile_step.py --config c3 --steps 1
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
ap.add_argument("--config", default="c2")
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--profile", action="store_true",
                help="eager launches, each inside an NVTX range cf:<kind>@L<level> (ncu --nvtx)")
args = ap.parse_args()
bc = configs.make(args.config)
cfg = P.SolverConfig(tau=bc.tau)
h = P.setup(P.laplacian(bc.graph), cfg)
if args.profile:
    h.profile(True)
eps = math.sqrt(math.log(bc.graph.n) / (bc.jl_k - 0.5))
for _ in range(args.steps):
    t = time.perf_counter()
    k, sums, res = sketch_closeness_sums(bc.graph, h, eps, bc.jl_seed, bc.query, cfg)
    print(f"step {time.perf_counter() - t:.3f}s k={k} score={(bc.graph.n - 1) / sums[0]:.12g} "
          f"maxres={res.max():.3e}", flush=True)
