"""Structure of the hub levels of a configuration's hierarchy: how the
nonzeros split between heavy and light rows/columns (what an L2-resident hot
set or column windows could save).  Host only.

    python tools/hub_stats.py --config c4
"""
import argparse
import os
import pickle
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1607_02955_b200 as P  # noqa: E402
from paper_1607_02955_b200 import configs  # noqa: E402
from paper_1607_02955_b200.solver import device_levels  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--cache", default="gpurun_out/cache")
args = ap.parse_args()
path = os.path.join(args.cache, f"levels_{args.config}.pkl")
if os.path.exists(path):
    with open(path, "rb") as f:
        mats = pickle.load(f)
else:
    t = time.perf_counter()
    bc = configs.make(args.config)
    h = P.setup(P.laplacian(bc.graph), P.SolverConfig(tau=bc.tau))
    print(f"gen+setup {time.perf_counter() - t:.1f}s")
    mats = [(l.kind.value, l.matrix) for l in device_levels(h.levels)]
    os.makedirs(args.cache, exist_ok=True)
    with open(path, "wb") as f:
        pickle.dump(mats, f)
for j, (kind, a) in enumerate(mats):
    a = a.tocsr()
    n = a.shape[0]
    deg = np.diff(a.indptr) - 1
    nnz = int(deg.sum())
    print(f"L{j} {kind[:5]} n={n} offnnz={nnz} mean={deg.mean():.1f} max={deg.max()}")
    if n < 5000:
        continue
    rows = np.repeat(np.arange(n), np.diff(a.indptr))
    cols = a.indices
    off = rows != cols
    rows, cols = rows[off], cols[off]
    for thr in (64, 256, 1024, 4096):
        hv = deg >= thr
        hr, hc = hv[rows], hv[cols]
        print(f"   thr {thr:5d}: heavy rows {hv.sum():7d} nnz HH {np.mean(hr & hc):.3f} "
              f"HL {np.mean(hr & ~hc):.3f} LH {np.mean(~hr & hc):.3f} LL {np.mean(~hr & ~hc):.3f}")
    order = np.argsort(-deg, kind="stable")
    for top in (1024, 4096, 16384):
        if top < n:
            intop = np.zeros(n, dtype=bool)
            intop[order[:top]] = True
            blk = int(np.sum(intop[rows] & intop[cols]))
            print(f"   top {top:6d} x {top:6d} block: {blk} nnz = {blk / nnz:.3f} of the level, "
                  f"{blk / (top * top):.3f} full")
    cum = np.cumsum(deg[order]) / nnz
    for top in (4096, 16384, 32768, 65536, 131072):
        if top < n:
            print(f"   top {top:6d} nodes hold {cum[top - 1]:.3f} of the endpoints")
