"""The real engine across separate processes: two ranks (two processes) run the column-sharded
TT-URV / TT-ULV with a communicator whose exchanges go over torch.distributed's
gloo backend (ttg_comm_callback_create). One GPU is visible to the tests, so both processes
use it; the exchange happens on the host between kernel launches (no kernel waits on another).
Checked: both ranks hold the same train, and it matches the single-process result."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, method, out_path):
    import pickle
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2501_07904_b200 import api, inputs
    dims, ranks = [20] * 4, [1, 5, 5, 5, 1]
    a = inputs.planted(dims, ranks, 1, 1e-8)

    def allgather(payload: bytes) -> bytes:
        t = torch.frombuffer(bytearray(payload), dtype=torch.uint8)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return b"".join(p.numpy().tobytes() for p in parts)

    comm = api.callback_comm(allgather, world, rank)
    blk = api.shard_block(a, dims, method, world, rank)
    res = api.decompose_sharded(blk, dims, comm, method, "l2r" if method == "ulv" else "r2l", ranks=ranks)
    cores = [res.core(k) for k in range(4)]
    rep = res.report()
    with open(f"{out_path}.{rank}", "wb") as f:
        pickle.dump({"cores": cores, "ranks": rep.ranks_chosen, "rse": res.rse(a)}, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("method", ["urv", "ulv"])
def test_two_process_sharded_sweep_over_gloo(dev, tmp_path, method):
    import pickle
    import torch.multiprocessing as mp
    from paper_2501_07904_b200 import inputs
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(2, port, method, out), nprocs=2, join=True)
    r0 = pickle.load(open(f"{out}.0", "rb"))
    r1 = pickle.load(open(f"{out}.1", "rb"))
    for c0, c1 in zip(r0["cores"], r1["cores"]):
        np.testing.assert_array_equal(c0, c1)
    dims, ranks = [20] * 4, [1, 5, 5, 5, 1]
    a = inputs.planted(dims, ranks, 1, 1e-8)
    one = dev.decompose_device(a, dims, method, "l2r" if method == "ulv" else "r2l", ranks=ranks)
    assert r0["ranks"] == one.report().ranks_chosen == ranks
    assert abs(r0["rse"] - one.rse(a)) <= 1e-12
