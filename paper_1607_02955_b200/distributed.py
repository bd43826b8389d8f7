"""Multi-GPU split of one JL estimate.

Every sketch row is an independent solve on a read-only hierarchy
(``SPEC.md:195-196``; the reference parallelises the same independence over
64-column blocks, ``solver.py:791-807``).  The K rows of ONE estimate are
split into contiguous ranges, one per rank (one process per GPU, hierarchy
replicated), so the workload is the same at every GPU count (strong split).
The closeness denominator

    S_v = sum_j ( T_j + n Z_vj^2 - 2 Z_vj C_j ),  T_j = sum_i Z_ij^2,  C_j = sum_i Z_ij

is assembled from per-row parts [T_j, C_j, Z_vj ...]: each rank produces its
rows' parts on the device (``cf_jl_sketch``), one all-gather (NCCL over
NVLink on the GPU box, gloo in the CPU tests) stacks them in row order, and
``cf_jl_combine`` sums them in ascending row order -- the same bits for
every number of ranks.  There is no exchange inside the solve.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

from .resistance import combine_row_parts, sketch_closeness_sums


def row_range(k: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous share of ``k`` sketch rows owned by ``rank``."""
    return (k * rank) // world, (k * (rank + 1)) // world


def gather_row_parts(local: np.ndarray, k: int, device: str = "cpu") -> np.ndarray:
    """All-gather every rank's row parts (``row_range`` shares of ``k`` rows,
    each (rows x W)) over the default process group and stack them in rank
    (= row) order.  Shares differ by at most one row; they are padded to the
    largest share for the collective and trimmed after."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    local = np.ascontiguousarray(local, dtype=np.float64)
    width = local.shape[1]
    cap = max(b - a for a, b in (row_range(k, world, r) for r in range(world)))
    buf = torch.zeros((cap, width), dtype=torch.float64, device=device)
    if local.shape[0]:
        buf[: local.shape[0]] = torch.from_numpy(local).to(device)
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    pieces = []
    for r, t in enumerate(outs):
        a, b = row_range(k, world, r)
        pieces.append(t[: b - a].cpu().numpy())
    return np.concatenate(pieces, axis=0)


def sharded_sketch_sums(g, hierarchy, epsilon: float, seed: int, query: Sequence[int],
                        config=None, device: str = "cpu"):
    """One JL estimate split over the ranks of the default process group.
    Returns (k, S_v for ``query``, this rank's residuals, its row range)."""
    import torch.distributed as dist

    from .resistance import sketch_dimension

    world, rank = dist.get_world_size(), dist.get_rank()
    k = sketch_dimension(g.n, epsilon)
    r0, r1 = row_range(k, world, rank)
    _, _, res, parts = sketch_closeness_sums(g, hierarchy, epsilon, seed, query, config,
                                             rows=(r0, r1), row_parts=True)
    allp = gather_row_parts(parts, k, device)
    return k, combine_row_parts(allp, g.n), res, (r0, r1)


def sharded_closeness(n: int, sums: np.ndarray) -> np.ndarray:
    """(n - 1) / S_v (centrality.py:154-160)."""
    return (n - 1) / np.asarray(sums)
