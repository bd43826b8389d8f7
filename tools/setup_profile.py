"""cProfile of graph generation, host/device setup and the device upload of a
configuration (where the seconds before the first solve go).

    python tools/setup_profile.py --config c5
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1607_02955_b200 as P  # noqa: E402
from paper_1607_02955_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--top", type=int, default=22)
args = ap.parse_args()
for name, fn in (("generate", lambda: configs.make(args.config)),
                 ("setup", lambda: P.setup(P.laplacian(bc.graph), P.SolverConfig(tau=bc.tau))),
                 ("upload", lambda: h.device())):
    pr = cProfile.Profile()
    t = time.perf_counter()
    pr.enable()
    out = fn()
    pr.disable()
    print(f"== {name}: {time.perf_counter() - t:.1f} s", flush=True)
    pstats.Stats(pr).sort_stats("cumulative").print_stats(args.top)
    if name == "generate":
        bc = out
    elif name == "setup":
        h = out
