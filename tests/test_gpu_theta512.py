"""GPU parity of the p = 512 theta stage (theta_cross512_kernel: three radix-8 passes, base-8
digit-reversed input, padded shared arrays) against the CPU oracle, through the C-ABI: the
nonlinear term and NS steps at p = 512 with small (m, n), including a ragged z-position tile
(n/2 odd). Tolerance: relative max-norm coefficient error <= 1e-10 (BASELINE.json north_star)."""
import numpy as np
import pytest

from tests.inputs import hermitian_coeffs, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.mark.parametrize("m,n,nyq", [(16, 16, True), (12, 14, True), (16, 16, False)])
def test_nonlinear_p512(P, O, m, n, nyq):
    p = 512
    ctx = P.Context(m, n, p)
    lam = hermitian_coeffs(m, n, p, 0.9, 11, nyquist_zero=nyq)  # slow decay: all 257 slots significant
    gam = hermitian_coeffs(m, n, p, 0.9, 12, nyquist_zero=nyq)
    vel = O.velocity_from_vorticity(lam, gam)
    for a, b in zip(ctx.nonlinear_term(*vel, lam, gam), O.nonlinear(*vel, lam, gam)):
        assert rel_err(a, b) < TOL
    ctx.close()


def test_ns_steps_p512(P, O):
    m, n, p = 16, 14, 512
    ctx = P.Context(m, n, p)
    wl = hermitian_coeffs(m, n, p, 0.7, 21)
    wg = hermitian_coeffs(m, n, p, 0.7, 22)
    ns = P.NSStepper(ctx, wl, wg, reynolds=100.0, h=1e-3)
    ons = O.NSStepper(wl, wg, 100.0, 1e-3)
    errs = []
    for _ in range(3):
        ns.step()
        ons.step()
        (l, g), (rl, rg) = ns.omega(), ons.omega()
        errs.append(max(rel_err(l, rl), rel_err(g, rg)))
    print("per-step rel err:", ["%.2e" % e for e in errs])
    assert max(errs) < TOL
    ns.close()
    ctx.close()
