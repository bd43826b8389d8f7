"""World-size-2 gloo test of the multi-GPU decomposition on CPU: each rank
owns a row range of the sketch, computes its share of the closeness sums and
one all-reduce combines them; the result equals the single-process sums."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1607_02955_b200.distributed import (allreduce_sums, partial_sums, row_range,
                                                sharded_closeness, weak_scaling_epsilon)


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


def _worker(rank, world, port, k, seed, query, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, z = _z_exact(k, seed)
        r0, r1 = row_range(k, world, rank)
        total = allreduce_sums(partial_sums(z[r0:r1], query))
        out[rank] = total.tolist()
    finally:
        dist.destroy_process_group()


def test_row_range_partition():
    for k in (1, 7, 64, 650):
        for world in (1, 2, 3, 8):
            rr = [row_range(k, world, r) for r in range(world)]
            assert rr[0][0] == 0 and rr[-1][1] == k
            assert all(a[1] == b[0] for a, b in zip(rr, rr[1:]))


def test_weak_scaling_epsilon_gives_k():
    from paper_1607_02955_b200.resistance import sketch_dimension
    for n in (4096, 100000, 2234040):
        for world in (1, 2, 4, 8):
            assert sketch_dimension(n, weak_scaling_epsilon(n, 128, world)) == 128 * world


def test_gloo_world2_sums_match_single_process():
    k, seed, query = 24, 3, [0, 5, 77]
    g, z = _z_exact(k, seed)
    ref = partial_sums(z, query)
    from oracle import lamg_oracle as O
    assert np.allclose(ref, O.jl_sums(z, query), rtol=1e-12)
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, k, seed, query, out), nprocs=2, join=True)
    for rank in range(2):
        assert np.allclose(out[rank], ref, rtol=1e-12)
    n = g[0].size - 1
    assert np.allclose(sharded_closeness(n, out[0]), (n - 1) / ref, rtol=1e-12)
