"""Multi-GPU decomposition of the JL estimator.

Every sketch row is an independent solve on a read-only hierarchy, so the k
rows are split into contiguous ranges, one per rank (one process per GPU,
hierarchy replicated).  The closeness denominator is additive over rows:

    S_v = sum_j ( T_j + n Z_vj^2 - 2 Z_vj C_j ),  T_j = sum_i Z_ij^2,  C_j = sum_i Z_ij

so each rank reports its rows' share and one all-reduce of |q| doubles
(NCCL over NVLink on the GPU box, gloo in the CPU tests) combines them.
There is no exchange inside the solve.
"""

from __future__ import annotations

import math
from typing import Sequence

import numpy as np


def row_range(k: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous share of ``k`` sketch rows owned by ``rank``."""
    return (k * rank) // world, (k * (rank + 1)) // world


def partial_sums(z_rows: np.ndarray, query: Sequence[int]) -> np.ndarray:
    """Share of S_v from the given sketch rows (rows x n), host restatement of
    the device reduction in csrc/cf_estimators.cu (``cf_jl_sketch``)."""
    z = np.asarray(z_rows, dtype=np.float64)
    n = z.shape[1]
    q = np.asarray(query, dtype=np.int64)
    t = np.einsum("ji,ji->j", z, z)
    c = z.sum(axis=1)
    zq = z[:, q]
    return t.sum() + n * np.einsum("jq,jq->q", zq, zq) - 2.0 * (zq.T @ c)


def allreduce_sums(local: np.ndarray, device: str = "cpu") -> np.ndarray:
    """Sum the per-rank shares over the default process group."""
    import torch
    import torch.distributed as dist

    t = torch.as_tensor(np.ascontiguousarray(local), dtype=torch.float64, device=device)
    dist.all_reduce(t)
    return t.cpu().numpy()


def sharded_closeness(n: int, sums: np.ndarray) -> np.ndarray:
    """(n - 1) / S_v (centrality.py:154-160)."""
    return (n - 1) / np.asarray(sums)


def weak_scaling_epsilon(n: int, k_per_rank: int, world: int) -> float:
    """epsilon giving exactly k_per_rank * world sketch rows (ceil rule of
    resistance.py:156-158)."""
    return math.sqrt(math.log(n) / (k_per_rank * world - 0.5))
