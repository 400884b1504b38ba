"""Column-sharded sweeps vs the reference oracle and the single-GPU engine.

One GPU is available to the tests, so G ranks run as a loopback group: G host threads of
this process, each driving its own stream and its own shard, exchanging pivot records,
TSQR triangles and the carry through host-side barriers around device copies (no kernel
waits on another). The NCCL communicator is covered at world size 1.

Contract: the sharded result equals the reference's like the single-GPU result does
(identical ranks, |RSE - RSE_ref| <= 1e-10, kept |T_ii| within 1e-10 |T_00|), every rank
returns the same train bit for bit, and it matches the single-GPU train to rounding.
"""
import threading

import numpy as np
import pytest

from tests.fixtures import cfg1, planted_plus_noise, shifted_hilbert
from tests.replay import replay

pytestmark = pytest.mark.gpu

TOL_RSE = 1e-10
TOL_DIAG = 1e-10


def _run_group(dev, a, dims, method, G, **kw):
    comms = dev.loopback_group(G)
    out, errs = [None] * G, [None] * G

    def work(g):
        try:
            blk = dev.shard_block(a, dims, method, G, g)
            sweep = "l2r" if method == "ulv" else "r2l"
            out[g] = dev.decompose_sharded(blk, dims, comms[g], method, sweep, **kw)
        except Exception as e:  # surfaced below
            errs[g] = e

    th = [threading.Thread(target=work, args=(g,)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in errs:
        if e is not None:
            raise e
    return out


def _check(dev, ref, a, dims, method, G, ranks=None, eps=None):
    sweep = "l2r" if method == "ulv" else "r2l"
    res = _run_group(dev, a, dims, method, G, ranks=ranks, eps=eps)
    reps = [r.report() for r in res]
    # every rank holds the same train, bit for bit
    for r in res[1:]:
        for k in range(len(dims)):
            np.testing.assert_array_equal(r.core(k), res[0].core(k))
    assert all(rp.ranks_chosen == reps[0].ranks_chosen for rp in reps)
    rep = reps[0]
    rr = ref.decompose(a, dims, method, sweep, ranks=ranks, eps=eps or 0.0)
    assert rep.ranks_chosen == rr.ranks_chosen
    gpu_rse = res[0].rse(a)
    ref_rse = ref.rse(rr, a, dims)
    assert abs(gpu_rse - ref_rse) <= TOL_RSE, (gpu_rse, ref_rse)
    cuts = replay(ref, a, dims, method, ranks=ranks, eps=eps)
    for c, (g, r) in enumerate(zip(rep.cuts, cuts)):
        assert g["rank"] == r["rank"]
        assert np.max(np.abs(g["diag"] - r["diag"])) <= TOL_DIAG * r["diag"][0], (c, g["diag"], r["diag"])
    # and the single-GPU engine
    one = dev.decompose_device(a, dims, method, sweep, ranks=ranks, eps=eps)
    assert one.report().ranks_chosen == rep.ranks_chosen
    assert abs(one.rse(a) - gpu_rse) <= 1e-12
    return rep


@pytest.mark.parametrize("G", [1, 2, 4])
@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_cfg1_fixed_rank_sharded(dev, ref, method, G):
    a, dims, ranks = cfg1(ref)
    rep = _check(dev, ref, a, dims, method, G, ranks=ranks)
    assert rep.ranks_chosen == ranks


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_cfg1_tolerance_sharded(dev, ref, method, G):
    a, dims, _ = cfg1(ref)
    _check(dev, ref, a, dims, method, G, eps=1e-6)


@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_hilbert_tolerance_sharded(dev, ref, method):
    dims = [10] * 4
    _check(dev, ref, shifted_hilbert(dims), dims, method, 2, eps=1e-6)


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_planted_uneven_modes_sharded(dev, ref, method, G):
    dims, ranks = [6, 12, 9], [1, 4, 5, 1]
    a = planted_plus_noise(ref, dims, ranks, 11, 1e-5)
    _check(dev, ref, a, dims, method, G, ranks=ranks)


@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_order_two_sharded(dev, ref, method):
    dims, ranks = [16, 24], [1, 6, 1]
    a = planted_plus_noise(ref, dims, ranks, 5, 1e-6)
    _check(dev, ref, a, dims, method, 4, ranks=ranks)


def test_sharded_zero_tensor(dev):
    dims = [4, 6, 8]
    res = _run_group(dev, np.zeros(int(np.prod(dims))), dims, "urv", 2, ranks=[1, 3, 3, 1])
    rep = res[0].report()
    assert rep.ranks_chosen == [1, 1, 1, 1]
    assert any("zero" in w for w in rep.warnings)


def test_sharded_rejects_indivisible(dev, ref):
    from paper_2501_07904_b200._native import ArgumentError
    with pytest.raises(ArgumentError, match="not divisible"):
        dev.shard_range([5, 7, 3], "urv", 2, 0)


def test_nccl_world_of_one(dev, ref):
    a, dims, ranks = cfg1(ref)
    comm = dev.nccl_comm(dev.nccl_unique_id(), 1, 0)
    res = dev.decompose_sharded(a, dims, comm, "urv", "r2l", ranks=ranks)
    one = dev.decompose_device(a, dims, "urv", "r2l", ranks=ranks)
    assert res.report().ranks_chosen == one.report().ranks_chosen
    assert abs(res.rse(a) - one.rse(a)) <= 1e-13


@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_planted_rank48_gram_sharded(dev, ref, method):
    # the Gram matrices of the ranks' R1 blocks are all-gathered and summed in rank order
    dims, ranks = [64, 64, 64], [1, 48, 48, 1]
    a = planted_plus_noise(ref, dims, ranks, 21, 1e-6)
    _check(dev, ref, a, dims, method, 4, ranks=ranks)


@pytest.mark.parametrize("G", [2, 4])
def test_k_sharded_second_cut(dev, ref, G):
    # URV: the second cut's W' = c'^T is tall and its rows are the ranks' carry blocks, so
    # it runs k-sharded (rank-summed Gram matrix) without gathering the carry
    dims, ranks = [16, 64, 64], [1, 8, 8, 1]
    a = planted_plus_noise(ref, dims, ranks, 33, 1e-6)
    _check(dev, ref, a, dims, "urv", G, ranks=ranks)


@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_long_pass2_beyond_160_steps_sharded(dev, ref, method):
    """A fixed rank above 160 on the sharded first cut: pass 2 no longer fits the TSQR / Gram
    routes, so the ranks' blocks of B = R1^T are all-gathered and factored in place (before:
    an InvariantError). 176 x 48 x 48, first-cut rank 170."""
    dims, ranks = [176, 48, 48], [1, 170, 30, 1]
    a = planted_plus_noise(ref, dims, [1, 24, 12, 1], 31, 1e-3)
    rk = [1, 170, 30, 1] if method == "ulv" else [1, 30, 40, 1]
    if method == "urv":  # URV shards the last mode: its first cut has W = 48 x 36,864 (p = 48)
        dims, rk = [48, 48, 176], [1, 30, 170, 1]
        a = planted_plus_noise(ref, dims, [1, 12, 24, 1], 31, 1e-3)
    _check(dev, ref, a, dims, method, 2, ranks=rk)
