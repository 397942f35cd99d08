"""Host side of the mode-sharded NS step (device side in csrc/shard.cu).

Partition (identical to ccf::Ctx::shard_init, checked against the library's host-only
``ccf_shard_partition``): rank r of ``world`` owns the contiguous half-spectrum slots
[sb[r], sb[r+1]) (slot s carries w = s, slot p/2 the Nyquist slice) in every per-mode stage, and
the radial value rows [rb[r], rb[r+1]) of all slots in the theta stage, with
sb[r] = r (p/2+1) // world, rb[r] = r (m/2) // world. Fast diagonalization makes every slot cost the
same, so equal contiguous ranges are balanced (129 slots over 8 ranks: 16 or 17 each).

Exchange: the theta kernel of a rank reads each slot's values of its rows straight from the
owner's exchange buffer and stores the cross product's spectrum back there (CUDA IPC peer memory
over NVLink). ``connect`` swaps the exchange-buffer IPC handles over torch.distributed; ``gather_omega``
reassembles a reference-layout field from the ranks' owned slices.

The reference (proj/src/ptns.cpp) is single-process; nothing here replaces a reference function.
"""
from __future__ import annotations


def slot_bounds(nslots: int, world: int):
    return [(r * nslots) // world for r in range(world + 1)]


def row_bounds(mh: int, world: int):
    return [(r * mh) // world for r in range(world + 1)]


def partition(m: int, p: int, world: int):
    """Per rank: dict(slot_lo, slot_hi, row_lo, row_hi)."""
    sb = slot_bounds(p // 2 + 1, world)
    rb = row_bounds(m // 2, world)
    return [dict(slot_lo=sb[r], slot_hi=sb[r + 1], row_lo=rb[r], row_hi=rb[r + 1]) for r in range(world)]


def slot_of_slice(l: int, p: int) -> int:
    """Half-spectrum slot holding reference slice l (w = l - p/2; slice 0 = Nyquist -> slot p/2)."""
    return p // 2 if l == 0 else abs(l - p // 2)


def owned_slices(p: int, slot_lo: int, slot_hi: int):
    """Boolean mask over the reference slices l = 0..p-1 owned by a rank with slots [slot_lo, slot_hi)."""
    import numpy as np
    return np.array([slot_lo <= slot_of_slice(l, p) < slot_hi for l in range(p)])


def mask_owned(a, p: int, slot_lo: int, slot_hi: int):
    """Zero the slices of a reference-layout (p, n, m) tensor this rank does not own (in place)."""
    a[~owned_slices(p, slot_lo, slot_hi)] = 0
    return a


def gather_by_slot(parts, p: int):
    """Combine per-rank reference-layout tensors [(slot_lo, slot_hi, array)] by slot ownership."""
    import numpy as np
    out = np.zeros_like(parts[0][2])
    for lo, hi, a in parts:
        sel = owned_slices(p, lo, hi)
        out[sel] = a[sel]
    return out


def exchange_bytes_per_rank(m: int, n: int, p: int, world: int, fields: int = 9) -> float:
    """NVLink bytes per rank and step of the theta exchange: the rank's rows (1/G) of
    the slots it does not own ((G-1)/G) of 6 input and 3 output fields, fields x 8N x (G-1)/G^2."""
    N = m * n * p
    return fields * 8.0 * N * (world - 1) / (world * world)


def connect(ctx, group=None):
    """Multi-process: exchange the ranks' exchange-buffer IPC handles over torch.distributed and
    map the peers (device-side rank barriers afterwards). ctx must be sharded (Context.shard)."""
    import torch.distributed as dist
    handles = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, ctx.ipc_handle(), group=group)
    ctx.open_ipc(handles)


def gather_omega(ctx, lam, gam, group=None):
    """All-reduce a stepper's omega() output (own slices valid) into the full field on every rank."""
    import torch
    import torch.distributed as dist
    info = ctx.shard_info()
    out = []
    for a in (lam, gam):
        mask_owned(a, ctx.p, info["slot_lo"], info["slot_hi"])
        t = torch.from_numpy(a.view("float64").copy())
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.all_reduce(t, group=group)
        out.append(t.cpu().numpy().view("complex128").reshape(a.shape))
    return tuple(out)
