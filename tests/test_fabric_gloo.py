"""Multi-process (world_size 2, gloo on CPU) tests of the N>1 host path.

The NCCL group the engine uses on B200s is exercised here over gloo: the
engine's own split tables (SP seq->head and head->seq all-to-alls with uneven
token shards and empty shards, TP all-reduce, uneven logits all-gather) must
give exactly what the in-process LoopbackGroup (the reference's simulated-P
model, fabric.py:117-191) gives on the same inputs.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_11830_b200.fabric import LoopbackGroup, NcclGroup
from paper_2507_11830_b200.flops import shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _payload(rank, rows, width, peers, seed):
    g = torch.Generator().manual_seed(seed * 100 + rank)
    return torch.randn(peers * rows, width, generator=g)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grp = NcclGroup(device="cpu")
        out = {}
        for total in (7, 1, 16):  # uneven shards and an empty shard (M=1, P=2)
            rows = shard_rows(total, world)
            W = 12
            send = {rank: _payload(rank, rows[rank], W, world, total)}
            recv = {rank: torch.empty(total, W)}
            grp.all_to_all(send, recv, {r: [rows[r]] * world for r in range(world)},
                           {s: list(rows) for s in range(world)}, row_bytes=W * 4)
            # head -> seq back exchange of the received rows
            back = {rank: torch.empty(world * rows[rank], W)}
            grp.all_to_all(recv, back, {r: list(rows) for r in range(world)},
                           {s: [rows[s]] * world for s in range(world)}, row_bytes=W * 4)
            out[f"a2a{total}"] = recv[rank]
            out[f"back{total}"] = back[rank]
        part = {rank: torch.full((3, 4), float(rank + 1))}
        out["allreduce"] = grp.all_reduce_sum(part)[rank].clone()
        cnt = [2, 0]
        out["gather"] = grp.all_gather_rows({rank: torch.full((2, 3), float(rank))}, cnt)
        # the TP logits gather: equal [R, V/P] blocks -> [P, R, V/P]
        out["blocks"] = grp.all_gather_blocks(torch.full((3, 4), float(rank + 10)))
        out["ledger"] = [(r.kind, r.bytes) for r in grp.records if r.device == 0]
        q.put((rank, {k: (v.tolist() if isinstance(v, torch.Tensor) else v) for k, v in out.items()}))
    finally:
        dist.destroy_process_group()


def test_nccl_group_over_gloo_matches_loopback():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # the same exchanges through the in-process loopback group
    lb = LoopbackGroup(world, device="cpu")
    lb._add = lambda a, b, out: out.copy_(a + b)
    for total in (7, 1, 16):
        rows = shard_rows(total, world)
        W = 12
        send = {r: _payload(r, rows[r], W, world, total) for r in range(world)}
        recv = {r: torch.empty(total, W) for r in range(world)}
        lb.all_to_all(send, recv, {r: [rows[r]] * world for r in range(world)},
                      {s: list(rows) for s in range(world)}, row_bytes=W * 4)
        back = {r: torch.empty(world * rows[r], W) for r in range(world)}
        lb.all_to_all(recv, back, {r: list(rows) for r in range(world)},
                      {s: [rows[s]] * world for s in range(world)}, row_bytes=W * 4)
        for r in range(world):
            assert torch.equal(torch.tensor(res[r][f"a2a{total}"]).view(-1, W), recv[r])
            assert torch.equal(torch.tensor(res[r][f"back{total}"]).view(-1, W), back[r])
            # the back exchange is the inverse of the forward one
            assert torch.equal(back[r], send[r])
    for r in range(world):
        assert res[r]["allreduce"] == [[3.0] * 4] * 3
        assert res[r]["gather"] == [[0.0] * 3] * 2
        assert res[r]["blocks"] == [[[10.0] * 4] * 3, [[11.0] * 4] * 3]
    # byte ledger identical to the reference ring formulas, from every rank's view
    lb.all_reduce_sum({0: torch.ones(3, 4), 1: torch.ones(3, 4)})
    lb.all_gather_rows({0: torch.zeros(2, 3), 1: torch.zeros(2, 3)}, [2, 0])
    lb.charge("all_gather", [(world - 1) / world * world * 3 * 4 * 4] * world)  # Engine._head_tp
    want = [(r.kind, r.bytes) for r in lb.records if r.device == 0]
    assert [tuple(x) for x in res[0]["ledger"]] == want
    assert [tuple(x) for x in res[1]["ledger"]] == want
