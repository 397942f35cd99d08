"""GPU tests of the mode-sharded NS step (csrc/shard.cu) on ONE B200.

Ranks are emulated without any device-side waiting between them (B200_PROFILING.md: kernels of
different ranks that wait on one another must not share a GPU):
  * linked contexts in one process (ccf_shard_link_local), each stepped by its own host thread,
    host barriers between the stages: exercises the partition, the owned-slot GEMM batches and the
    theta kernel's peer addressing (other ranks' exchange buffers are plain device pointers);
  * two processes on the same GPU connected through CUDA IPC handles swapped over gloo
    (ccf_shard_ipc_handle / ccf_shard_open_ipc, the multi-GPU code path), with the rank barrier
    replaced by stream synchronisation + a gloo barrier (ccf_shard_set_host_barrier).
The gathered sharded result must equal the unsharded stepper's (same kernels, same per-tile
arithmetic: bit-identical in practice; gate 1e-13 relative) and the CPU oracle's (1e-10)."""
import os
import threading

import numpy as np
import pytest

from paper_2206_04827_b200 import shard
from tests.inputs import hermitian_coeffs, rel_err

pytestmark = pytest.mark.gpu


def _initial(m, n, p, decay=0.7, seed=3):
    return hermitian_coeffs(m, n, p, decay, seed), hermitian_coeffs(m, n, p, decay, seed + 100)


def run_linked(P, m, n, p, world, lam, gam, steps, reynolds=100.0, h=1e-3, disable_nonlinear=False):
    ctxs = [P.Context(m, n, p, device=0).shard(r, world) for r in range(world)]
    P.Context.link_local(ctxs)
    sts = [P.NSStepper(c, lam, gam, reynolds=reynolds, h=h, disable_nonlinear=disable_nonlinear) for c in ctxs]
    errs = []

    def work(i):
        try:
            sts[i].step(steps)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    parts_l, parts_g = [], []
    for c, st in zip(ctxs, sts):
        info = c.shard_info()
        lo, hi = info["slot_lo"], info["slot_hi"]
        wl, wg = st.omega()
        parts_l.append((lo, hi, wl))
        parts_g.append((lo, hi, wg))
    out = shard.gather_by_slot(parts_l, p), shard.gather_by_slot(parts_g, p)
    infos = [c.shard_info() for c in ctxs]
    for st in sts:
        st.close()
    for c in ctxs:
        c.close()
    return out, infos


def run_single(P, m, n, p, lam, gam, steps, reynolds=100.0, h=1e-3, disable_nonlinear=False):
    ctx = P.Context(m, n, p, device=0)
    st = P.NSStepper(ctx, lam, gam, reynolds=reynolds, h=h, disable_nonlinear=disable_nonlinear)
    st.step(steps)
    out = st.omega()
    st.close()
    ctx.close()
    return out


@pytest.mark.parametrize("size,world", [((16, 16, 16), 2), ((16, 16, 16), 3), ((16, 12, 16), 4),
                                        ((16, 16, 256), 2), ((16, 16, 256), 8), ((32, 32, 32), 4),
                                        ((16, 14, 512), 4)],
                         ids=lambda x: "x".join(map(str, x)) if isinstance(x, tuple) else f"g{x}")
def test_sharded_ns_equals_unsharded(P, size, world):
    m, n, p = size
    lam, gam = _initial(m, n, p)
    steps = 7  # BDF ramp (4 orders) + steady state
    (sl, sg), infos = run_linked(P, m, n, p, world, lam, gam, steps)
    rl, rg = run_single(P, m, n, p, lam, gam, steps)
    err = max(rel_err(sl, rl), rel_err(sg, rg))
    print(f"{size} world {world}: sharded vs unsharded rel err {err:.2e}")
    assert err <= 1e-13
    # the partition the library used is the documented one
    ref = shard.partition(m, p, world)
    for i, info in enumerate(infos):
        assert {k: info[k] for k in ref[i]} == ref[i]


def test_sharded_ns_matches_oracle(P, O):
    m, n, p = 16, 16, 16
    lam, gam = _initial(m, n, p)
    (sl, sg), _ = run_linked(P, m, n, p, 3, lam, gam, 5)
    ons = O.NSStepper(lam, gam, 100.0, 1e-3)
    ons.step(5)
    rl, rg = ons.omega()
    assert max(rel_err(sl, rl), rel_err(sg, rg)) < 1e-10


def test_sharded_heat_equals_unsharded(P):
    m, n, p = 16, 16, 16
    lam, gam = _initial(m, n, p, 0.85, 2)
    (sl, sg), _ = run_linked(P, m, n, p, 2, lam, gam, 6, disable_nonlinear=True)
    rl, rg = run_single(P, m, n, p, lam, gam, 6, disable_nonlinear=True)
    assert max(rel_err(sl, rl), rel_err(sg, rg)) <= 1e-13


def test_sharded_ns_64_world4(P):
    m = n = p = 64
    lam, gam = _initial(m, n, p, 0.7, 3)
    (sl, sg), _ = run_linked(P, m, n, p, 4, lam * 1e-3, gam * 1e-3, 6)
    rl, rg = run_single(P, m, n, p, lam * 1e-3, gam * 1e-3, 6)
    assert max(rel_err(sl, rl), rel_err(sg, rg)) <= 1e-13


def test_sharded_context_refuses_other_entry_points(P):
    ctx = P.Context(16, 16, 16, device=0).shard(1, 2)
    with pytest.raises(P.ConfigError):
        ctx.solve_poisson_3d(hermitian_coeffs(16, 16, 16, 0.8, 1))
    with pytest.raises(P.ConfigError):
        ctx.shard(0, 2)  # already sharded
    ctx.close()


def _ipc_worker(rank, world, port, m, n, p, steps, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        import paper_2206_04827_b200 as P
        dist.init_process_group("gloo", rank=rank, world_size=world)
        lam, gam = _initial(m, n, p)
        ctx = P.Context(m, n, p, device=0).shard(rank, world)
        shard.connect(ctx)                      # CUDA IPC handles over gloo (the multi-GPU path)
        ctx.set_host_barrier(dist.barrier)      # one GPU: no device-side waiting between ranks
        st = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3)
        st.step(steps)
        wl, wg = st.omega()
        gl, gg = shard.gather_omega(ctx, wl, wg)
        st.close()
        dist.barrier()
        ctx.close()
        err = None
        if rank == 0:
            rl, rg = run_single(P, m, n, p, lam, gam, steps)
            err = max(rel_err(gl, rl), rel_err(gg, rg))
        q.put((rank, err, None))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, None, repr(e)))


@pytest.mark.parametrize("size", [(16, 16, 16), (16, 16, 256)], ids=lambda s: "x".join(map(str, s)))
def test_sharded_ipc_two_processes(size):
    import torch.multiprocessing as mp
    m, n, p = size
    world, steps = 2, 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, m, n, p, steps, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, err, exc in res:
        assert exc is None, exc
        if rank == 0:
            print(f"IPC world 2 {size}: gathered vs unsharded rel err {err:.2e}")
            assert err <= 1e-13
