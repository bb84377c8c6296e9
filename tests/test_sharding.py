"""Multi-GPU partitioning logic on CPU: world_size 2 over gloo.

The GPU box used by this run has one B200, so the N>1 path's host logic --
which streams each rank owns and how the NCCL all-gather of per-head outputs
is reassembled -- is covered here with the gloo backend.
"""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_19769_b200.sharding import ShardPlan, gather_outputs


def test_head_plan_partitions_streams():
    for N in (1, 2, 4, 8):
        seen = []
        for r in range(N):
            p = ShardPlan(r, N, layers=32, kv_heads=8, requests=1, mode="heads")
            ids = p.local_streams()
            assert len(ids) == p.n_local == 256 // N
            seen += ids
        assert sorted(seen) == list(range(256))


def test_request_plan_partitions_streams():
    for N in (1, 2, 4, 8):
        seen = []
        for r in range(N):
            seen += ShardPlan(r, N, 32, 8, 16, "requests").local_streams()
        assert sorted(seen) == list(range(16 * 256))


def test_plan_rejects_uneven_split():
    with pytest.raises(ValueError):
        ShardPlan(0, 3, 32, 8, 1, "heads").local_streams()


def _worker(rank, world, port, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        R = 2 if mode == "requests" else 1
        plan = ShardPlan(rank, world, layers=4, kv_heads=8, requests=R, mode=mode)
        ids = torch.tensor(plan.local_streams(), dtype=torch.float32)
        G, d = 4, 3
        # output value encodes (global stream, head, channel)
        local = ids.view(-1, 1, 1) * 100 + torch.arange(G).view(1, G, 1) * 10 + \
            torch.arange(d).view(1, 1, d)
        full = gather_outputs(local, plan)
        S = 4 * 8 * R
        expect = torch.arange(S, dtype=torch.float32).view(-1, 1, 1) * 100 + \
            torch.arange(G).view(1, G, 1) * 10 + torch.arange(d).view(1, 1, d)
        q.put((rank, bool(torch.equal(full, expect))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["heads", "requests"])
def test_gather_outputs_world2_gloo(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + (0 if mode == "heads" else 1)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert [p.exitcode for p in procs] == [0, 0]
    res = [q.get(timeout=10) for _ in procs]
    assert all(ok for _, ok in res), res
