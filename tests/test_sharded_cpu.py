"""World-size > 1 coverage of the column-sharded path on CPU (torch.distributed, gloo).

The device engine needs a GPU, so these tests run the sharded protocol's numpy
restatement (oracle/sharded.py) across two gloo ranks and check that it reproduces the
single-process greedy QRCP exactly: the same pivots (global positions and tie rule), the
same R rows, the same pass-2 decisions from the reduced TSQR triangles, and the carry
blocks reassembled in the order csrc/sweep.cu uses. The native shard planner
(ttg_shard_range, host-only) is checked against the restatement.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port
from oracle import sharded as sh


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _allgather_dist(x):
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return np.stack([o.numpy() for o in out])


def _allgather_one(x):
    return np.asarray(x, dtype=np.float64)[None, :]


def _matrix(kind, k, n, seed):
    rng = np.random.default_rng(seed)
    if kind == "lowrank":
        return rng.standard_normal((k, 5)) @ rng.standard_normal((5, n)) + 1e-6 * rng.standard_normal((k, n))
    if kind == "ties":  # repeated columns: exact ties resolve to the lowest global position
        base = rng.standard_normal((k, n // 4))
        return np.hstack([base, base, base[:, ::-1], base])
    i = np.arange(1, k + 1)[:, None] + np.arange(1, n + 1)[None, :]
    return 1.0 / (i - 1.0)  # Hilbert-type, rapidly decaying


def _worker(rank, world, port_, kind, k, n, s, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W = _matrix(kind, k, n, 7)
        nl = n // world
        off = rank * nl
        piv, R, Q = sh.sharded_pass1(W[:, off:off + nl], off, n, s, _allgather_dist)
        piv1, R1, Q1 = sh.sharded_pass1(W, 0, n, s, _allgather_one)
        np.testing.assert_array_equal(piv, piv1)
        np.testing.assert_allclose(R, R1[:, off:off + nl], rtol=0, atol=1e-12 * np.abs(R1).max())
        np.testing.assert_allclose(Q, Q1, rtol=0, atol=1e-12)
        # the reference algorithm itself (plain-C restatement, pinned to the reference)
        if port.available():
            _, Rref, perm = port.qr_col_pivot(W)
            # pivots agree wherever they are decided above rounding (Hilbert-type decay
            # reaches the noise floor within the s steps)
            dref = np.abs(np.diag(Rref)[:s])
            sig = int(np.sum(dref > 1e-8 * dref[0]))
            np.testing.assert_array_equal(piv1[:sig], perm[:sig])
            np.testing.assert_allclose(np.abs(np.diag(R1[:, piv1]))[:sig], dref[:sig], rtol=1e-8,
                                       atol=1e-14 * dref[0])
        # pass 2 from the reduced triangles: same pivots and |R| as QRCP of the full B
        RB = sh.sharded_rb(R, _allgather_dist)
        RB1 = sh.sharded_rb(R1, _allgather_one)
        if port.available():
            _, r2, p2 = port.qr_col_pivot(RB)
            _, r21, p21 = port.qr_col_pivot(RB1)
            np.testing.assert_array_equal(p2, p21)
            np.testing.assert_allclose(np.abs(np.diag(r2)), np.abs(np.diag(r21)), rtol=1e-9,
                                       atol=1e-13 * abs(r21[0, 0]))
        # carries reassembled like decompose_sharded does
        sel = np.arange(min(3, s))
        urv = sh.gather_carry_urv(np.ascontiguousarray(R[sel, :].T), _allgather_dist)
        np.testing.assert_allclose(urv, R1[sel, :].T, rtol=0, atol=1e-12 * np.abs(R1).max())
        ulv = sh.gather_carry_ulv(np.ascontiguousarray(R[sel, :]), _allgather_dist)
        np.testing.assert_allclose(ulv, R1[sel, :], rtol=0, atol=1e-12 * np.abs(R1).max())
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,k,n,s", [("lowrank", 12, 64, 8), ("ties", 10, 48, 10), ("hilbert", 16, 40, 12)])
def test_gloo_world2_sharded_first_cut(kind, k, n, s):
    mp.spawn(_worker, args=(2, _free_port(), kind, k, n, s, None), nprocs=2, join=True)


@pytest.mark.parametrize("dims", [[20, 20, 20, 20], [6, 12, 9], [16, 24], [4, 8, 2, 6]])
@pytest.mark.parametrize("method", ["ulv", "urv"])
@pytest.mark.parametrize("G", [1, 2, 4])
def test_shard_range_native_matches_restatement(dims, method, G):
    from paper_2501_07904_b200 import api
    first = dims[0] if method == "ulv" else dims[-1]
    if (int(np.prod(dims)) // first) % G:
        with pytest.raises(Exception, match="not divisible"):
            api.shard_range(dims, method, G, 0)
        return
    blocks = [api.shard_range(dims, method, G, g) for g in range(G)]
    assert blocks == [sh.shard_range(dims, method, G, g) for g in range(G)]
    # the blocks tile the sharded index range
    assert blocks[0][0] == 0 and blocks[-1][1] == int(np.prod(dims)) // first
    assert all(blocks[g][1] == blocks[g + 1][0] for g in range(G - 1))


def test_shard_block_tiles_the_tensor():
    from paper_2501_07904_b200 import api
    dims = [6, 12, 9]
    a = np.arange(np.prod(dims), dtype=np.float64)
    for method in ("ulv", "urv"):
        G = 3
        parts = [api.shard_block(a, dims, method, G, g) for g in range(G)]
        assert sum(p.size for p in parts) == a.size
        if method == "ulv":
            np.testing.assert_array_equal(np.concatenate(parts), a)
        else:
            m = a.size // dims[-1]
            c = a.reshape((m, dims[-1]), order="F")
            back = np.vstack([p.reshape((m // G, dims[-1]), order="F") for p in parts])
            np.testing.assert_array_equal(back, c)


def _worker_kshard(rank, world, port_):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(3)
        k, N, s = 96, 12, 6
        W = rng.standard_normal((k, 6)) @ rng.standard_normal((6, N)) + 1e-3 * rng.standard_normal((k, N))
        kl = k // world
        piv, R, Q = sh.kshard_gram_pass1(W[rank * kl:(rank + 1) * kl], s, _allgather_dist)
        piv1, R1, Q1 = sh.kshard_gram_pass1(W, s, _allgather_one)
        np.testing.assert_array_equal(piv, piv1)
        np.testing.assert_allclose(R, R1, rtol=0, atol=1e-12 * np.abs(R1).max())
        np.testing.assert_allclose(Q, Q1[rank * kl:(rank + 1) * kl], rtol=0, atol=1e-10)
        # the Householder QRCP of the whole matrix picks the same pivots and |R|
        if port.available():
            _, Rref, perm = port.qr_col_pivot(W)
            np.testing.assert_array_equal(piv1, perm[:s])
            np.testing.assert_allclose(np.abs(np.diag(R1[:, piv1])), np.abs(np.diag(Rref)[:s]), rtol=1e-9)
        # and the local Q rows stack into orthonormal columns
        Qall = _allgather_dist(np.ascontiguousarray(Q.reshape(-1, order="F"))).reshape(world, -1)
        Qs = np.vstack([q.reshape(kl, s, order="F") for q in Qall])
        np.testing.assert_allclose(Qs.T @ Qs, np.eye(s), atol=1e-10)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_gloo_world2_k_sharded_gram_pass1():
    mp.spawn(_worker_kshard, args=(2, _free_port()), nprocs=2, join=True)
