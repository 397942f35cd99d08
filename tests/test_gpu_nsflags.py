"""NSConfig's off-by-default flags (ptns.hpp:84-94) on the device: dealias_two_thirds (the 2/3 rule on
the analyzed cross product, ptns.cpp:100-110,140-144: j / k masks folded into the analysis matrices,
|w| mask on the output slots), compute_gamma_psi (ptns.cpp:248-253) and NSStepper::velocity()
(ptns.cpp:205-215), against the CPU oracle on the same seeded inputs (1e-10)."""
import numpy as np
import pytest

from tests.inputs import hermitian_coeffs, rel_err

pytestmark = pytest.mark.gpu
SIZES = [(16, 16, 16), (24, 20, 16), (32, 32, 32)]


@pytest.mark.parametrize("size", SIZES, ids=lambda s: "x".join(map(str, s)))
def test_dealiased_nonlinear_term(P, O, size):
    m, n, p = size
    ctx = P.Context(m, n, p)
    vl, vg = hermitian_coeffs(m, n, p, 0.7, 5), hermitian_coeffs(m, n, p, 0.7, 6)
    wl, wg = hermitian_coeffs(m, n, p, 0.7, 1), hermitian_coeffs(m, n, p, 0.7, 2)
    got = ctx.nonlinear_term(vl, vg, wl, wg, dealias_two_thirds=True)
    ref = O.nonlinear(vl, vg, wl, wg, dealias=True)
    plain = O.nonlinear(vl, vg, wl, wg)
    assert max(rel_err(got[0], ref[0]), rel_err(got[1], ref[1])) < 1e-10
    assert rel_err(ref[0], plain[0]) > 1e-6  # the rule changes the result
    ctx.close()


@pytest.mark.parametrize("size", SIZES[:2], ids=lambda s: "x".join(map(str, s)))
def test_dealiased_ns_steps(P, O, size):
    m, n, p = size
    lam, gam = hermitian_coeffs(m, n, p, 0.7, 3), hermitian_coeffs(m, n, p, 0.7, 103)
    ctx = P.Context(m, n, p)
    st = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3, dealias_two_thirds=True)
    ons = O.NSStepper(lam, gam, 100.0, 1e-3, dealias=True)
    st.step(7)  # ramp + graph-replayed steady state
    ons.step(7)
    (l, g), (rl, rg) = st.omega(), ons.omega()
    assert max(rel_err(l, rl), rel_err(g, rg)) < 1e-10
    st.close()
    ctx.close()


def test_velocity_and_gamma_psi(P, O):
    m, n, p = 16, 16, 16
    lam, gam = hermitian_coeffs(m, n, p, 0.7, 3), hermitian_coeffs(m, n, p, 0.7, 103)
    ctx = P.Context(m, n, p)
    st = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3, compute_gamma_psi=True)
    with pytest.raises(P.DomainError):
        st.gamma_psi()  # populated from the first step on
    st.step(6)
    before = st.omega()
    st.step(1)
    wl, wg = st.omega()
    vl, vg = st.velocity()
    rvl, rvg = O.velocity_from_vorticity(wl, wg)
    assert max(rel_err(vl, rvl), rel_err(vg, rvg)) < 1e-10
    assert rel_err(st.gamma_psi(), O.poisson3d(-before[1])) < 1e-10
    plain = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3)
    with pytest.raises(P.ConfigError):
        plain.gamma_psi()
    plain.close()
    st.close()
    ctx.close()
