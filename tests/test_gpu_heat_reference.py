"""The reference's own HeatStepper / heat_run cases (proj/tests/test_timestep.cpp:113-273) run on the device
through the C-ABI: zero state, steps = 0, alpha = 0 (the mass solve), the BDF1 local error ratio, the temporal order
of every BDF order on the oscillating manufactured problem, and the decay probe for large steps; plus the
zero-diffusivity HelmholtzTensorStepper step against the CPU oracle."""
import numpy as np
import pytest

from tests.conftest import sample
from tests.inputs import hermitian_coeffs, rel_err

pytestmark = pytest.mark.gpu
OMEGA = 3.0  # test_timestep.cpp:16-30 Oscillating (alpha = 1)


def exact(r, z, t, time):
    return np.cos(OMEGA * time) * (1 - r * r) * (1 - z * z) + 0 * t


def forcing(r, z, t, time):
    lap = -4.0 * (1 - z * z) - 2.0 * (1 - r * r)
    return -OMEGA * np.sin(OMEGA * time) * (1 - r * r) * (1 - z * z) - np.cos(OMEGA * time) * lap + 0 * t


def run_error(P, O, ctx, spec, order, h, t_final):  # test_timestep.cpp:32-57
    m, n, p = spec
    init = sample(O, m, n, p, lambda r, z, t: exact(r, z, t, 0.0))
    steps = int(round(t_final / h))
    run = P.heat_run(ctx, init, lambda time: sample(O, m, n, p, lambda r, z, t: forcing(r, z, t, time)), steps,
                     alpha=1.0, h=h, order=order)
    ref = sample(O, m, n, p, lambda r, z, t: exact(r, z, t, run["final_time"]))
    return float(np.abs(run["snapshots"][-1] - ref).max())


def test_zero_state_and_zero_steps(P, O):  # :113-134
    ctx = P.Context(8, 8, 4)
    run = P.heat_run(ctx, np.zeros((4, 8, 8)), None, 5, h=0.1, order=4)
    assert np.abs(run["final_coeffs"]).max() == 0.0
    init = sample(O, 8, 8, 4, lambda r, z, t: exact(r, z, t, 0.0))
    run = P.heat_run(ctx, init, None, 0)
    assert len(run["snapshots"]) == 1 and run["final_time"] == 0.0
    ctx.close()


def test_alpha_zero_is_constant_in_time(P, O):  # :136-149 (every step is the mass solve)
    ctx = P.Context(8, 8, 4)
    init = sample(O, 8, 8, 4, lambda r, z, t: exact(r, z, t, 0.0))
    run = P.heat_run(ctx, init, None, 8, alpha=0.0, h=0.05)
    ref = O.parity_project(O.analyze(init), 0)
    assert np.abs(run["final_coeffs"] - ref).max() < 1e-11
    # and against the oracle's alpha = 0 stepper on data that does not satisfy the boundary conditions
    c0 = hermitian_coeffs(8, 8, 4, 0.7, 5)
    st, ost = P.HeatStepper(ctx, c0, alpha=0.0, h=0.05, order=3), O.HeatStepper(c0, alpha=0.0, h=0.05, order=3)
    for _ in range(5):
        st.step()
        ost.step()
    assert rel_err(st.current(), ost.current()[0]) < 1e-10
    with pytest.raises(P.DomainError):
        P.HeatStepper(ctx, c0, alpha=-1.0)
    st.close()
    ctx.close()


def test_zero_diffusivity_helmholtz_step_matches_oracle(P, O):
    m, n, p = 16, 12, 8
    ctx = P.Context(m, n, p)
    hist = [hermitian_coeffs(m, n, p, 0.7, 30 + i) for i in range(2)]
    f = hermitian_coeffs(m, n, p, 0.7, 40)
    got = ctx.helmholtz_step(hist, 2, 0.0, 1e-2, forcing=f)
    assert rel_err(got, O.helmholtz_step(hist, 2, 0.0, 1e-2, forcing=f)) < 1e-10
    ctx.close()


def test_bdf1_local_error_and_temporal_orders(P, O):  # :189-220
    spec = (10, 10, 4)
    ctx = P.Context(*spec)
    e1, e2 = run_error(P, O, ctx, spec, 1, 0.02, 0.02), run_error(P, O, ctx, spec, 1, 0.01, 0.01)
    assert 2.5 < e1 / e2 < 6.0
    for b in range(1, 5):
        hs = [0.02, 0.01, 0.005]
        errs = [run_error(P, O, ctx, spec, b, h, 2.0) for h in hs]
        slope = np.polyfit(np.log(hs), np.log(errs), 1)[0]
        assert b - 0.3 < slope < b + 0.3, (b, slope, errs)
    ctx.close()


def test_stability_probe_large_steps(P, O):  # :222-273
    m, n, p = 10, 10, 8
    ctx = P.Context(m, n, p)
    c = np.random.default_rng(11).uniform(-1, 1, 6)

    def field(r, z, t):
        x, y = r * np.cos(t), r * np.sin(t)
        return (1 - r * r) * (1 - z * z) * (c[0] + c[1] * x + c[2] * y + c[3] * z) + c[4] * z * z + c[5] * x * y

    init = sample(O, m, n, p, field)
    for h in (0.01, 0.1, 1.0):
        st = P.HeatStepper(ctx, init, alpha=1.0, h=h, order=1)  # backward Euler: monotone decay of the max norm
        prev = np.abs(st.current()).max()
        floor = 1e-14 * prev
        for _ in range(100):
            st.step()
            cur = np.abs(st.current()).max()
            assert cur <= prev * (1 + 1e-12) + floor
            prev = cur
        st.close()
        # BDF4: the per-step max norm oscillates (parasitic roots) inside a decaying 4-step envelope (:252-271).
        # With these seeded constants the reference scheme itself leaves the envelope once at h = 1 (step 25, at
        # 4e-9 of the initial norm: the CPU oracle shows the same two numbers), and at h = 0.01 (t = 1) the slowest
        # mode has only decayed by exp(-8.9), so: every norm is checked against the oracle's, the envelope for
        # h <= 0.1 and the final 1e-6 decay for h >= 0.1.
        st = P.HeatStepper(ctx, init, alpha=1.0, h=h, order=4)
        ost = O.HeatStepper(O.analyze(init), alpha=1.0, h=h, order=4)
        initial = np.abs(st.current()).max()
        floor = 1e-14 * initial
        window = [initial]
        for _ in range(100):
            st.step()
            ost.step()
            cur = np.abs(st.current()).max()
            assert abs(cur - np.abs(ost.current()[0]).max()) <= 1e-10 * initial
            assert cur <= initial * (1 + 1e-12)
            if len(window) >= 4 and h <= 0.1:
                assert cur <= window[0] * (1 + 1e-12) + floor
            window.append(cur)
            window = window[-4:]
        if h >= 0.1:
            assert np.abs(st.current()).max() <= 1e-6 * initial
        st.close()
    ctx.close()
