"""Oracle PT / NS semantics (reference: proj/src/ptns.cpp, proj/src/calculus.cpp).

proj/tests/test_ptns.cpp is a placeholder, so these pins come from the reference code's
semantics: quirk Q1 of divide_r, the Stokes-limit equivalence and invariants."""
import numpy as np

from tests.conftest import sample
from tests.inputs import hermitian_coeffs, rel_err


def test_divide_r_quirk_q1(O):
    # divide_r drops the theta-odd part (synthesize keeps Re only)
    m, n, p = 8, 6, 8
    odd = O.analyze(sample(O, m, n, p, lambda r, z, t: r * r * np.sin(t) * (1 - z * z)))
    assert np.abs(O.calculus("divide_r", odd)).max() < 1e-15
    even = O.analyze(sample(O, m, n, p, lambda r, z, t: r * r * np.cos(t) * (1 - z * z)))
    ref = O.analyze(sample(O, m, n, p, lambda r, z, t: r * np.cos(t) * (1 - z * z)))
    assert np.abs(O.calculus("divide_r", even) - ref).max() < 1e-14


def test_stokes_limit_equals_heat(O):
    # NS with the nonlinear term disabled == two independent heat runs at alpha = 1/Re
    m, n, p = 8, 8, 8
    lam = hermitian_coeffs(m, n, p, 0.7, 1)
    gam = hermitian_coeffs(m, n, p, 0.7, 2)
    ns = O.NSStepper(lam, gam, reynolds=50.0, h=1e-2, disable_nonlinear=True)
    hl = O.HeatStepper(lam, alpha=1 / 50.0, h=1e-2, order=4)
    hg = O.HeatStepper(gam, alpha=1 / 50.0, h=1e-2, order=4)
    for _ in range(6):
        ns.step()
        hl.step()
        hg.step()
    l, g = ns.omega()
    assert rel_err(l, hl.current()[0]) < 1e-12 and rel_err(g, hg.current()[0]) < 1e-12


def test_zero_field_stays_zero(O):
    z = np.zeros((8, 8, 8), complex)
    ns = O.NSStepper(z, z, reynolds=100.0, h=1e-3)
    ns.step(3)
    l, g = ns.omega()
    assert np.abs(l).max() == 0.0 and np.abs(g).max() == 0.0


def test_pt_synthesize_parity_classes(O):
    m, n, p = 8, 8, 8
    vr, vt, vz = O.pt_synthesize(hermitian_coeffs(m, n, p, 0.7, 3), hermitian_coeffs(m, n, p, 0.7, 4))
    assert np.array_equal(vr, O.parity_project(vr, 1)) and np.array_equal(vt, O.parity_project(vt, 1))
    assert np.array_equal(vz, O.parity_project(vz, 0))


def test_pt_round_trip(O):
    # pt_decompose(pt_synthesize(s)) = s for axisymmetric Dirichlet-gauge scalars. With theta content,
    # Q1 (divide_r drops the theta-odd part) removes D(dtheta lambda) from V_r, so only gamma
    # round-trips: a property of the reference path that parity must reproduce (App. A.7).
    m, n, p = 12, 12, 8
    bump = lambda r, z, t: (1 - r * r) * (1 - z * z)
    lam = O.analyze(sample(O, m, n, p, lambda r, z, t: bump(r, z, t) * (0.3 + 0.2 * r * r)))
    gam = O.analyze(sample(O, m, n, p, lambda r, z, t: bump(r, z, t) * (0.1 - 0.3 * z * z)))
    dl, dg = O.pt_decompose(*O.pt_synthesize(lam, gam))
    assert rel_err(dl, lam) < 1e-12 and rel_err(dg, gam) < 1e-12
    lam = O.analyze(sample(O, m, n, p, lambda r, z, t: bump(r, z, t) * (0.3 + 0.2 * r * np.cos(t))))
    gam = O.analyze(sample(O, m, n, p, lambda r, z, t: bump(r, z, t) * (0.1 + 0.4 * r * np.cos(t))))
    dl, dg = O.pt_decompose(*O.pt_synthesize(lam, gam))
    assert rel_err(dg, gam) < 1e-12
    assert rel_err(dl, lam) > 1e-3  # Q1 signature
