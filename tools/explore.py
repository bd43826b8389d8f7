"""One-hierarchy exploration on a configuration (setup once, then several
measurements): block-width cost of cf_solve_block_dev, and JL-estimate time /
V-cycles per right-hand side for smoother schedules.

    python tools/explore.py --config c5 --widths 16,32,64,128,256 --nu 1,2 1,1 2,1
"""
import argparse
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1607_02955_b200 as P  # noqa: E402
from paper_1607_02955_b200 import _native as N  # noqa: E402
from paper_1607_02955_b200 import configs  # noqa: E402
from paper_1607_02955_b200.resistance import sketch_closeness_sums  # noqa: E402
from paper_1607_02955_b200.solver import _params, device_levels  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--widths", default="")
ap.add_argument("--nu", nargs="*", default=[])
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
t = time.perf_counter()
bc = configs.make(args.config)
tg = time.perf_counter() - t
cfg = P.SolverConfig(tau=bc.tau)
t = time.perf_counter()
h = P.setup(P.laplacian(bc.graph), cfg)
ts = time.perf_counter() - t
t = time.perf_counter()
dev = h.device()
tu = time.perf_counter() - t
print(f"{args.config}: n={bc.graph.n} gen {tg:.1f}s setup {ts:.1f}s upload {tu:.1f}s", flush=True)
for j, l in enumerate(device_levels(h.levels)):
    od = np.diff(l.matrix.indptr) - 1
    print(f"  L{j} {l.kind.value[:5]} n={l.size} nnz={l.matrix.nnz} maxdeg={od.max()} "
          f"mean={od.mean():.1f}", flush=True)
n = bc.graph.n
gen = torch.Generator(device="cuda").manual_seed(0)
for k in (int(x) for x in args.widths.split(",") if x):
    b = torch.randn((n, k), dtype=torch.float64, device="cuda", generator=gen)
    b -= b.mean(dim=0, keepdim=True)
    x = torch.empty_like(b)
    res = np.zeros(k)
    times = []
    for r in range(args.reps + 1):
        st = N.CfSolveStats()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        N.check(N.lib().cf_solve_block_dev(dev.handle, C.c_void_p(b.data_ptr()),
                                           C.c_void_p(x.data_ptr()), k,
                                           C.byref(_params(cfg, n)), N.ptr(res, N.f64p),
                                           C.byref(st),
                                           C.c_void_p(torch.cuda.current_stream().cuda_stream)),
                st)
        torch.cuda.synchronize()
        if r:
            times.append((time.perf_counter() - t0) * 1e3)
    ms = min(times)
    print(f"width k={k:4d} ms={ms:9.2f} vcycles/col={st.vcycles / k:6.2f} ms/col={ms / k:8.3f} "
          f"maxres={res.max():.2e}", flush=True)
    del b, x
eps = bc.epsilon
for stp in args.nu:
    nu = tuple(int(v) for v in stp.split(","))
    c2 = P.SolverConfig(tau=bc.tau, smoothing_steps=nu)
    for rep in range(args.reps):
        v0 = h.stats.vcycles
        torch.cuda.synchronize()
        t = time.perf_counter()
        k, sums, res = sketch_closeness_sums(bc.graph, h, eps, bc.jl_seed, bc.query, c2)
        dt = time.perf_counter() - t
    print(f"nu={nu} {dt * 1e3:.1f} ms vcycles/rhs={(h.stats.vcycles - v0) / k:.2f} "
          f"score={(n - 1) / sums[0]:.10g} maxres={res.max():.2e}", flush=True)
