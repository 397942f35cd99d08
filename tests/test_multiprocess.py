"""World-size-2 gloo tests of the mode-sharded host logic (CPU only, csrc/shard.cu model).

* the Python partition equals the library's (host-only ccf_shard_partition);
* a numpy model of one sharded step: per-mode stages on the owned slots, the theta stage on the
  owned rows of all slots with every (slot, row) read from and written to the OWNER's full-extent
  exchange buffer (peer loads / stores at the same offset, modelled by gathering the ranks'
  buffers), two rank barriers; the gathered result equals the unsharded step exactly;
* gather_by_slot / gather_omega reassemble reference-layout fields from owned slices;
* max-over-ranks timing reduction (bench.py)."""
import os

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_04827_b200 import shard


def test_partition_matches_library(P):
    for m, p, world in [(16, 16, 2), (16, 16, 3), (64, 64, 4), (256, 256, 8), (512, 512, 8), (16, 256, 8)]:
        sb, rb = P.shard_partition(m, p, world)
        part = shard.partition(m, p, world)
        assert [x["slot_lo"] for x in part] + [part[-1]["slot_hi"]] == sb
        assert [x["row_lo"] for x in part] + [part[-1]["row_hi"]] == rb
        sizes = [b - a for a, b in zip(sb, sb[1:])]
        assert sb[0] == 0 and sb[-1] == p // 2 + 1 and max(sizes) - min(sizes) <= 1 and min(sizes) >= 1
        assert rb[0] == 0 and rb[-1] == m // 2 and min(b - a for a, b in zip(rb, rb[1:])) >= 1
    # 302, 226, 132 MB of exchange per rank and step at 256^3 for G = 2, 4, 8
    for g, mb in [(2, 302), (4, 226), (8, 132)]:
        assert abs(shard.exchange_bytes_per_rank(256, 256, 256, g) / 1e6 - mb) < 2


def test_slot_ownership_covers_reference_slices():
    p = 16
    parts = shard.partition(16, p, 3)
    masks = [shard.owned_slices(p, x["slot_lo"], x["slot_hi"]) for x in parts]
    assert np.array_equal(np.sum(masks, axis=0), np.ones(p, int))  # every slice owned exactly once
    assert shard.slot_of_slice(0, p) == p // 2 and shard.slot_of_slice(p // 2 + 3, p) == 3
    assert shard.slot_of_slice(p // 2 - 3, p) == 3  # w and -w in the same slot (Hermitian pair)
    rng = np.random.default_rng(0)
    full = rng.standard_normal((p, 4, 6))
    pieces = []
    for x in parts:
        junk = rng.standard_normal(full.shape)  # non-owned slices are meaningless on a rank
        sel = shard.owned_slices(p, x["slot_lo"], x["slot_hi"])
        junk[sel] = full[sel]
        pieces.append((x["slot_lo"], x["slot_hi"], junk))
    assert np.array_equal(shard.gather_by_slot(pieces, p), full)


# ---- model of one sharded step (same index arithmetic as the kernels)
S, NPL, MH, NZ = 9, 2, 6, 5  # slots, planes, rows, z positions
MIX = np.random.default_rng(7).standard_normal((3, S, 6 * S))  # theta stage: couples all slots of a point


def _per_mode_in(x, s):   # stands in for the composite synthesis GEMMs (slot-local)
    return np.sin(x * (1 + s)) + s


def _per_mode_out(y, s):  # stands in for the analysis / curl / decompose GEMMs (slot-local)
    return y * (2.0 + s) - 1.0


def _theta(vals):  # vals: [6][S] at one point -> [3][S]; stands in for FFT x cross x FFT
    return (MIX.reshape(3 * S, 6 * S) @ np.ascontiguousarray(vals).reshape(6 * S)).reshape(3, S)


def _reference_step(x):  # x: [6, S, NPL, MH, NZ]
    v = np.stack([_per_mode_in(x[:, s], s) for s in range(S)], axis=1)
    a = np.empty((3, S, NPL, MH, NZ))
    for pl in range(NPL):
        for j in range(MH):
            for k in range(NZ):
                a[:, :, pl, j, k] = _theta(v[:, :, pl, j, k])
    return np.stack([_per_mode_out(a[:, s], s) for s in range(S)], axis=1)


def _sharded_step(x, rank, world):
    sb = shard.slot_bounds(S, world)
    rb = shard.row_bounds(MH, world)
    xbuf = np.full((9, S, NPL, MH, NZ), np.nan)  # full-extent exchange buffer, owned slots valid
    for s in range(sb[rank], sb[rank + 1]):
        xbuf[:6, s] = _per_mode_in(x[:, s], s)
    # barrier 1, then peer loads: the buffers of all ranks as mapped here
    bufs = [torch.empty(xbuf.shape, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(bufs, torch.from_numpy(xbuf))
    peers = [b.numpy() for b in bufs]
    owner = [max(r for r in range(world) if sb[r] <= s) for s in range(S)]
    stores = np.full((3, S, NPL, MH, NZ), np.nan)  # what this rank stores into the owners' buffers
    for pl in range(NPL):
        for j in range(rb[rank], rb[rank + 1]):
            for k in range(NZ):
                vals = np.stack([peers[owner[s]][:6, s, pl, j, k] for s in range(S)], axis=1)
                stores[:, :, pl, j, k] = _theta(vals)
    # peer stores land in the owner's buffer at the same offset; barrier 2
    allst = [torch.empty(stores.shape, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(allst, torch.from_numpy(stores))
    for r in range(world):
        rows = slice(rb[r], rb[r + 1])
        for s in range(sb[rank], sb[rank + 1]):
            xbuf[6:, s, :, rows] = allst[r].numpy()[:, s, :, rows]
    out = np.full((3, S, NPL, MH, NZ), np.nan)
    for s in range(sb[rank], sb[rank + 1]):
        out[:, s] = _per_mode_out(xbuf[6:, s], s)
    return out, sb


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = np.random.default_rng(3).standard_normal((6, S, NPL, MH, NZ))
    out, sb = _sharded_step(x, rank, world)
    ref = _reference_step(x)
    mine = slice(sb[rank], sb[rank + 1])
    ok = bool(np.array_equal(out[:, mine], ref[:, mine]))
    # gather of owned slots (what shard.gather_omega does with reference-layout tensors)
    full = torch.from_numpy(np.where(np.isnan(out), 0.0, out))
    dist.all_reduce(full)
    ok_gather = bool(np.array_equal(full.numpy(), ref))
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # bench.py: max-over-ranks timing
    q.put((rank, ok, ok_gather, float(t.item())))
    dist.destroy_process_group()


def test_sharded_step_model_gloo_world2():
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
    for rank, ok, okg, tmax in res:
        assert ok and okg and tmax == float(world), res
