"""Cost of one device block solve per block width (chunk-planner calibration).

    python tools/kc_cost.py --config c3 --widths 1,8,16,32,64,128,256

Solves k random balanced right-hand sides already resident on the device
(cf_solve_block_dev) and prints milliseconds, V-cycles and ms per column.
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
from paper_1607_02955_b200.solver import _params  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--widths", default="1,8,16,32,64,128,256")
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
bc = configs.make(args.config)
cfg = P.SolverConfig(tau=bc.tau)
t = time.perf_counter()
h = P.setup(P.laplacian(bc.graph), cfg)
dev = h.device()
print(f"{args.config}: n={bc.graph.n} setup {time.perf_counter() - t:.1f}s levels {h.level_sizes[:12]}",
      flush=True)
n = bc.graph.n
gen = torch.Generator(device="cuda").manual_seed(0)
for k in (int(x) for x in args.widths.split(",")):
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
    print(f"k={k:4d} ms={ms:9.2f} vcycles/col={st.vcycles / k:6.2f} ms/col={ms / k:8.3f} "
          f"maxres={res.max():.2e}", flush=True)
