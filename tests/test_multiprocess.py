"""World-size-2 gloo tests of the multi-GPU host logic (CPU only): J-balanced mode sharding,
pencil partition, and the theta pencil transpose as an all_to_all that round-trips exactly."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_04827_b200 import shard


def test_partitions_cover_exactly():
    for p, world in [(8, 2), (64, 4), (256, 8), (512, 8)]:
        parts = shard.mode_partition(p, world)
        flat = sorted(s for part in parts for s in part)
        assert flat == list(range(p // 2 + 1))
        sizes = [len(x) for x in parts]
        assert max(sizes) - min(sizes) <= 2
        pen = shard.pencil_partition(p, p // 2, world)
        assert pen[0][0] == 0 and pen[-1][1] == p * (p // 2)
        assert all(a[1] == b[0] for a, b in zip(pen, pen[1:]))
    # 302, 226, 132 MB egress at 256^3 for G = 2, 4, 8
    for g, mb in [(2, 302), (4, 226), (8, 132)]:
        assert abs(shard.alltoall_bytes_per_rank(256, 256, 256, g) / 1e6 - mb) < 2


def _exchange(send, recv, rank):
    """Pairwise all-to-all (what the NCCL path issues as grouped ncclSend/ncclRecv)."""
    ops = []
    for r in range(len(send)):
        if r == rank:
            recv[r].copy_(send[r])
            continue
        ops.append(dist.P2POp(dist.isend, send[r], r))
        ops.append(dist.P2POp(dist.irecv, recv[r], r))
    for w in dist.batch_isend_irecv(ops):
        w.wait()


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p, n, mh = 8, 6, 4
    nslots = p // 2 + 1
    parts = shard.mode_partition(p, world)
    pens = shard.pencil_partition(n, mh, world)
    # global field: value(slot, plane, pencil) = deterministic
    full = torch.arange(nslots * 2 * n * mh, dtype=torch.float64).reshape(nslots, 2, n * mh)
    mine = full[parts[rank]]  # mode-sharded: my slots, all pencils
    # forward transpose: send to rank r my slots restricted to r's pencils
    send = [mine[:, :, a:b].contiguous() for (a, b) in pens]
    recv = [torch.empty(len(parts[r]), 2, pens[rank][1] - pens[rank][0], dtype=torch.float64) for r in range(world)]
    _exchange(send, recv, rank)
    # pencil-sharded: all slots for my pencils
    got = torch.empty(nslots, 2, pens[rank][1] - pens[rank][0], dtype=torch.float64)
    for r in range(world):
        got[parts[r]] = recv[r]
    ok1 = torch.equal(got, full[:, :, pens[rank][0]:pens[rank][1]])
    # backward transpose restores the mode sharding
    send2 = [got[parts[r]].contiguous() for r in range(world)]
    recv2 = [torch.empty(len(parts[rank]), 2, b - a, dtype=torch.float64) for (a, b) in pens]
    _exchange(send2, recv2, rank)
    back = torch.cat(recv2, dim=2)
    ok2 = torch.equal(back, mine)
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # bench.py: max-over-ranks timing
    q.put((rank, bool(ok1), bool(ok2), float(t.item())))
    dist.destroy_process_group()


def test_theta_transpose_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, ok1, ok2, tmax in res:
        assert ok1 and ok2 and tmax == float(world)
