"""GPU HeatStepper / heat_run (proj/src/timestep.cpp:110-170) against the CPU oracle on the same
seeded inputs (relative coefficient error <= 1e-10), the reference's manufactured BDF4 heat test
(test_timestep.cpp:151-187, here on the nearest even grid) and the paper's Table-1 problem
(bench.cpp:20-35)."""
import numpy as np
import pytest
import torch

from tests.conftest import sample
from tests.inputs import hermitian_coeffs, rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("size", [(16, 16, 16), (16, 12, 8), (32, 32, 32)], ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("order", [1, 2, 4])
def test_heat_stepper_matches_oracle(P, O, size, order):
    m, n, p = size
    c0 = hermitian_coeffs(m, n, p, 0.85, 2)
    ctx = P.Context(m, n, p)
    st = P.HeatStepper(ctx, c0, alpha=0.7, h=1e-2, order=order)
    ost = O.HeatStepper(c0, alpha=0.7, h=1e-2, order=order)
    for k in range(7):
        g = hermitian_coeffs(m, n, p, 0.8, 50 + k) if k % 3 != 2 else None  # with and without forcing
        st.step(g)
        ost.step(g)
    ref, t_ref, _ = ost.current()
    got = st.current()
    assert rel_err(got, ref) < 1e-10
    assert abs(st.time - t_ref) < 1e-14
    st.close()
    ctx.close()


def test_forcing_grid_values_device_and_host(P, O):
    m, n, p = 16, 16, 16
    ctx = P.Context(m, n, p)
    c0 = hermitian_coeffs(m, n, p, 0.85, 2)
    vals = O.synthesize(hermitian_coeffs(m, n, p, 0.8, 9))  # a grid forcing (step_with_callback path)
    a = P.HeatStepper(ctx, c0, alpha=1.0, h=1e-2)
    b = P.HeatStepper(ctx, c0, alpha=1.0, h=1e-2)
    o = O.HeatStepper(c0, alpha=1.0, h=1e-2)
    for _ in range(3):
        a.step(vals)
        b.step(torch.from_numpy(vals).cuda())
        o.step(O.analyze(vals))
    assert np.array_equal(a.current(), b.current())
    assert rel_err(a.current(), o.current()[0]) < 1e-10
    a.close()
    b.close()
    ctx.close()


def test_heat_bdf4_manufactured(P, O):  # test_timestep.cpp:151-187 on 16x16x16 (the B200 path needs even m, n)
    m, n, p = 16, 16, 16
    ex = lambda t: (lambda r, z, th: np.exp(-t) * (1 - r * r) * (1 - z * z))
    lapf = lambda r, z: -4 * (1 - z * z) - 2 * (1 - r * r)
    frc = lambda t: sample(O, m, n, p, lambda r, z, th: -np.exp(-t) * (1 - r * r) * (1 - z * z) - np.exp(-t) * lapf(r, z))
    ctx = P.Context(m, n, p)
    run = P.heat_run(ctx, sample(O, m, n, p, ex(0.0)), frc, 200, alpha=1.0, h=0.01, order=4)
    ref = sample(O, m, n, p, ex(run["final_time"]))
    assert abs(run["final_time"] - 2.0) < 1e-12
    assert np.abs(run["snapshots"][-1] - ref).max() / np.abs(ref).max() <= 1e-4
    ctx.close()


def manufactured(O, m, n, p, alpha=1.0):
    """bench.cpp:20-35 ManufacturedHeat: T = e^-t cos(pi z / 2)(1 - r^2)(1 + r cos(th) / 2)."""
    def exact(t):
        return sample(O, m, n, p, lambda r, z, th: np.exp(-t) * np.cos(np.pi * z / 2) * (1 - r * r) *
                      (1 + 0.5 * r * np.cos(th)))

    def forcing(t):
        def g(r, z, th):
            zz = np.cos(np.pi * z / 2)
            s = (1 - r * r) * (1 + 0.5 * r * np.cos(th))
            lap = np.exp(-t) * (-4.0 * zz * (1 + r * np.cos(th)) - np.pi ** 2 / 4.0 * zz * s)
            return -np.exp(-t) * zz * s - alpha * lap
        return sample(O, m, n, p, g)
    return exact, forcing


@pytest.mark.parametrize("s", [8, 12, 16, 20])
def test_table1_problem(P, O, s):
    """Paper Table 1 / bench_spectral (bench.cpp:56-84): 200 BDF4 steps, h = 0.01; the paper's odd
    sizes 7..19 become the nearest even grids. GPU == oracle run to 1e-10, error at the paper's level."""
    m = n = s
    p = s
    exact, forcing = manufactured(O, m, n, p)
    ctx = P.Context(m, n, p)
    run = P.heat_run(ctx, exact(0.0), forcing, 200, alpha=1.0, h=0.01, order=4)
    err = np.abs(run["snapshots"][-1] - exact(run["final_time"])).max() / np.abs(exact(run["final_time"])).max()
    o = O.HeatStepper(O.analyze(exact(0.0)), alpha=1.0, h=0.01, order=4)
    t = 0.0
    for _ in range(200):
        o.step(O.analyze(forcing(t + 0.01)))
        t += 0.01
    assert rel_err(run["final_coeffs"], o.current()[0]) < 1e-10
    assert err < 1e-4, err  # Table 1: 6.0e-5 .. 1.8e-5
    ctx.close()
