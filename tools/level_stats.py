"""Print per-level statistics of the host and device hierarchies of a config."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1607_02955_b200 as P
from paper_1607_02955_b200 import configs
from paper_1607_02955_b200.solver import device_levels
bc = configs.make(sys.argv[1])
t = time.time()
h = P.setup(P.laplacian(bc.graph), P.SolverConfig(tau=bc.tau))
print(f"setup {time.time() - t:.1f}s levels {len(h.levels)}")
for j, l in enumerate(device_levels(h.levels)):
    A = l.matrix
    deg = np.diff(A.indptr) - 1
    print(f"{j:3d} {l.kind.value[:5]:5s} n={l.size:9d} nnz={A.nnz:11d} avgdeg={deg.mean():8.1f} "
          f"maxdeg={deg.max():8d} nnz_in_rows>64={deg[deg > 64].sum() / max(1, deg.sum()):.2f}")
