"""NSStepper::seed and ns_run incl. the substeps bootstrap (ptns.cpp:195-203, 269-324) on the device against
the CPU oracle on the same seeded inputs (1e-10 relative max-norm), through the C-ABI (ccf_ns_seed)."""
import numpy as np
import pytest

from tests.inputs import hermitian_coeffs, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _init(m, n, p, scale=1e-3):
    # small amplitude: with O(0.1) data the reference's scheme (explicit nonlinear term, quirk Q1) blows up within
    # the ~100 fine steps of the substeps bootstrap, on the CPU oracle and the GPU alike
    return hermitian_coeffs(m, n, p, 0.7, 21) * scale, hermitian_coeffs(m, n, p, 0.7, 22) * scale


def _err(a, b):
    return max(rel_err(a[0], b[0]), rel_err(a[1], b[1]))


@pytest.mark.parametrize("size", [(16, 16, 16), (24, 20, 16)], ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("order", [2, 4])
def test_ns_run_substeps_matches_oracle(P, O, size, order):
    m, n, p = size
    lam, gam = _init(m, n, p)
    steps = order + 5  # seeded steps, then graph-replayed steady state
    ctx = P.Context(m, n, p)
    got = P.ns_run(ctx, lam, gam, steps, reynolds=100.0, h=2e-3, order=order, bootstrap="substeps")
    ref = O.ns_run(lam, gam, steps, 100.0, 2e-3, order=order, bootstrap="substeps")
    assert _err(got["final_omega"], ref[:2]) < TOL
    assert abs(got["final_time"] - ref[2]) < 1e-15
    ramp = O.ns_run(lam, gam, steps, 100.0, 2e-3, order=order)
    assert _err(ref[:2], ramp[:2]) > 1e-7  # the bootstrap changes the trajectory
    ctx.close()


def test_ns_run_ramp_snapshots(P, O):
    m = n = p = 16
    lam, gam = _init(m, n, p)
    ctx = P.Context(m, n, p)
    got = P.ns_run(ctx, lam, gam, 6, reynolds=100.0, h=1e-3, output_every=3)
    assert len(got["snapshots"]) == 2 and np.allclose(got["snapshot_times"], [3e-3, 6e-3], atol=1e-15)
    ons = O.NSStepper(lam, gam, 100.0, 1e-3)
    for snap in got["snapshots"]:
        ons.step(3)
        assert _err(snap, ons.omega()) < TOL
    assert _err(got["final_omega"], ons.omega()) < TOL
    ctx.close()


@pytest.mark.parametrize("eigen", ["1", "0"])
def test_seed_continues_a_run(P, O, eigen, monkeypatch):
    # a stepper seeded with a run's history (host tensors) continues that run; both state representations
    monkeypatch.setenv("CCF_NS_EIGEN", eigen)
    m = n = p = 16
    lam, gam = _init(m, n, p)
    ctx = P.Context(m, n, p)
    run = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3)
    oh = [(lam, gam)]
    for _ in range(3):
        run.step()
        oh.insert(0, run.omega())
    nh = [ctx.nonlinear_term(*ctx.velocity_from_vorticity(*w), *w) for w in oh[1:]]
    seeded = P.NSStepper(ctx, *oh[0], reynolds=100.0, h=1e-3)
    seeded.seed(oh, nh, 3e-3, 3)
    run.step(7)
    seeded.step(7)
    a, b = seeded.omega(), run.omega()
    assert _err(a, b) < 1e-12
    assert seeded.steps_taken == 10 and abs(seeded.time - 1e-2) < 1e-15
    # the oracle, seeded with its own history, agrees too
    ons = O.NSStepper(lam, gam, 100.0, 1e-3)
    ons.step(10)
    assert _err(a, ons.omega()) < TOL
    # evaluate_nonlinear (ptns.cpp:211-214) of the current state
    w = seeded.omega()
    assert _err(seeded.evaluate_nonlinear(), O.nonlinear(*O.velocity_from_vorticity(*w), *w)) < TOL
    run.close()
    seeded.close()
    ctx.close()


def test_seed_full_history_with_many_steps_taken(P, O):
    # a full-order history with steps_taken past the graph threshold: the first seeded step runs eagerly on the
    # coefficient-space omega, the following ones replay graphs; device tensors are accepted as well
    import torch
    m = n = p = 16
    lam, gam = _init(m, n, p)
    ons = O.NSStepper(lam, gam, 100.0, 1e-3)
    oh = [(O.parity_project(lam, 0), O.parity_project(gam, 0))]
    for _ in range(3):
        ons.step()
        oh.insert(0, ons.omega())
    nh = [O.nonlinear(*O.velocity_from_vorticity(*w), *w) for w in oh[1:]]
    ctx = P.Context(m, n, p)
    st = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3)
    dev = lambda pairs: [tuple(torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in pr) for pr in pairs]
    st.seed(dev(oh), dev(nh), 0.5, 500)
    st.step(6)
    ons.step(6)
    assert _err(st.omega(), ons.omega()) < TOL
    assert st.steps_taken == 506 and abs(st.time - 0.506) < 1e-12
    st.close()
    ctx.close()


def test_seed_errors(P):
    m = n = p = 16
    lam, gam = _init(m, n, p)
    ctx = P.Context(m, n, p)
    st = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3)
    with pytest.raises(P.DomainError, match="empty history"):
        st.seed([], [], 0.0, 0)
    with pytest.raises(P.DomainError):
        st.seed([(lam[:, :, :8], gam)], [], 0.0, 0)  # shape checked before the C-ABI call
    st.seed([(lam, gam)], [], 3e-3, 3)  # BDF4 from one entry (timestep.cpp:41-42)
    with pytest.raises(P.DomainError, match="insufficient history"):
        st.step()
    st.close()
    ctx.close()


def test_seed_at_the_bench_size_on_the_int8_path(P):
    # 256^3 (the INT8 product stages, panels written by the RHS pass, graph replay): a stepper seeded with a run's
    # history continues that run (the seeded state is re-expanded in the modal basis, so agreement is to rounding)
    import bench
    cfg = bench.CONFIGS[256]
    ctx = P.Context(256, 256, 256)
    wl, wg, _ = bench.initial_vorticity(ctx, cfg, cfg["vmax"])
    kw = dict(reynolds=cfg["reynolds"], h=cfg["h"])
    run = P.NSStepper(ctx, wl, wg, **kw)
    run.step(5)
    oh = [run.omega()]
    for _ in range(3):
        run.step()
        oh.insert(0, run.omega())
    nh = [ctx.nonlinear_term(*ctx.velocity_from_vorticity(*w), *w) for w in oh[1:]]
    run.step(12)
    ref = run.omega()
    run.close()
    seeded = P.NSStepper(ctx, *oh[0], **kw)
    seeded.seed(oh, nh, 8 * cfg["h"], 8)
    seeded.step(12)  # one eager coefficient-space step, four warm-up phases, then graph replays
    got = seeded.omega()
    assert _err(got, ref) < 1e-10
    assert seeded.steps_taken == 20
    seeded.close()
    ctx.close()
