"""GPU properties at BASELINE sizes (the oracle is too slow there): round trips, linearity,
manufactured solutions, Stokes-limit equivalence, invariants. Tolerances stated per test."""
import numpy as np
import pytest

from tests.conftest import sample
from tests.inputs import hermitian_coeffs, rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx256(P):
    c = P.Context(256, 256, 256)
    yield c
    c.close()


def test_round_trip_256(ctx256):
    t = hermitian_coeffs(256, 256, 256, 0.9, 11)
    t[0] = t[0].real
    back = ctx256.analyze(ctx256.synthesize(t))
    assert rel_err(back, t) < 1e-12


def test_poisson_linearity_256(ctx256):
    a = hermitian_coeffs(256, 256, 256, 0.9, 1)
    b = hermitian_coeffs(256, 256, 256, 0.9, 2)
    lhs = ctx256.solve_poisson_3d(0.6 * a - 1.7 * b)
    rhs = 0.6 * ctx256.solve_poisson_3d(a) - 1.7 * ctx256.solve_poisson_3d(b)
    assert rel_err(lhs, rhs) < 1e-11


def test_manufactured_poisson_128(P, O):
    # u = (1-r^2)(1 + r cos th / 2)(1-z^2) e^{2z} (test_solvers.cpp:211-238), spectrally converged
    m = n = 128
    p = 8
    u_fn = lambda r, z, t: (1 - r * r) * (1 + 0.5 * r * np.cos(t)) * (1 - z * z) * np.exp(2 * z)

    def f_fn(r, z, t):
        sz = (1 - z * z) * np.exp(2 * z)
        szpp = np.exp(2 * z) * (2 - 8 * z - 4 * z * z)
        return -4 * (1 + r * np.cos(t)) * sz + (1 - r * r) * (1 + 0.5 * r * np.cos(t)) * szpp
    ctx = P.Context(m, n, p)
    u = ctx.synthesize(ctx.solve_poisson_3d(ctx.analyze(sample(O, m, n, p, f_fn))))
    assert np.abs(u - sample(O, m, n, p, u_fn)).max() < 1e-10


def test_stokes_limit_equals_two_heat_steps(P):
    # NS with disable_nonlinear == independent Helmholtz steps at diffusivity 1/Re
    m = n = p = 64
    lam = hermitian_coeffs(m, n, p, 0.7, 1)
    gam = hermitian_coeffs(m, n, p, 0.7, 2)
    ctx = P.Context(m, n, p)
    ns = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3, disable_nonlinear=True)
    ns.step()
    l, g = ns.omega()
    assert rel_err(l, ctx.helmholtz_step([lam], 1, 0.01, 1e-3)) < 1e-12
    assert rel_err(g, ctx.helmholtz_step([gam], 1, 0.01, 1e-3)) < 1e-12


def test_zero_stays_zero_256(P, ctx256):
    z = np.zeros((256, 256, 256), complex)
    ns = P.NSStepper(ctx256, z, z, reynolds=1000.0, h=5e-4)
    ns.step(2)
    l, g = ns.omega()
    assert np.abs(l).max() == 0.0 and np.abs(g).max() == 0.0
