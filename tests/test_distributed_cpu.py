"""Multi-rank split of one JL estimate on CPU (gloo, world sizes 2 and 3):
each rank owns a row range of the sketch and contributes its per-row parts;
``gather_row_parts`` + ``combine_row_parts`` -- the functions the GPU bench
uses (``distributed.sharded_sketch_sums``) -- reproduce the single-process
sums BITWISE, and match the oracle's closed form (resistance.py:218-237)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1607_02955_b200.distributed import gather_row_parts, row_range, sharded_closeness
from paper_1607_02955_b200.resistance import combine_row_parts


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _z_exact(k, seed):
    from oracle import lamg_oracle as O
    g = O.grid_graph(12)
    _, rhs = O.jl_rhs(g, k, seed)
    pinv = np.linalg.pinv(O.laplacian(g).toarray())
    return g, rhs @ pinv


def _row_parts(z, query):
    """Per-row parts [T_j, C_j, Z[q, j]...] as cf_jl_sketch returns them."""
    q = np.asarray(query, dtype=np.int64)
    return np.column_stack([np.einsum("ji,ji->j", z, z), z.sum(axis=1), z[:, q]])


def _worker(rank, world, port, k, seed, query, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, z = _z_exact(k, seed)
        r0, r1 = row_range(k, world, rank)
        parts = _row_parts(z[r0:r1], query)
        allp = gather_row_parts(parts, k)
        out[rank] = combine_row_parts(allp, z.shape[1]).tobytes()
    finally:
        dist.destroy_process_group()


def test_row_range_partition():
    for k in (1, 7, 64, 650):
        for world in (1, 2, 3, 8):
            rr = [row_range(k, world, r) for r in range(world)]
            assert rr[0][0] == 0 and rr[-1][1] == k
            assert all(a[1] == b[0] for a, b in zip(rr, rr[1:]))


def test_combine_matches_oracle_and_is_split_invariant():
    from oracle import lamg_oracle as O
    k, seed, query = 37, 3, [0, 5, 77, 143]
    g, z = _z_exact(k, seed)
    parts = _row_parts(z, query)
    full = combine_row_parts(parts, z.shape[1])
    assert np.allclose(full, O.jl_sums(z, query), rtol=1e-12)
    # any split of the rows, parts stacked back in row order: same bits
    for world in (2, 3, 5, 8):
        stacked = np.concatenate([parts[a:b] for a, b in
                                  (row_range(k, world, r) for r in range(world))])
        assert combine_row_parts(stacked, z.shape[1]).tobytes() == full.tobytes()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_split_sums_bitwise_equal_single_process(world):
    k, seed, query = 24, 3, [0, 5, 77]
    g, z = _z_exact(k, seed)
    ref = combine_row_parts(_row_parts(z, query), z.shape[1])
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, k, seed, query, out), nprocs=world, join=True)
    for rank in range(world):
        assert out[rank] == ref.tobytes()
    n = g[0].size - 1
    got = np.frombuffer(out[0], dtype=np.float64)
    assert np.array_equal(sharded_closeness(n, got), (n - 1) / ref)
