"""Oracle pins for the per-mode solver API against the reference's own known answers
(proj/tests/test_solvers.cpp:38-105: zero forcing, manufactured Helmholtz solution, the scale-zero mass pair,
lifted boundary data) plus the defining identities (the solution solves the recombined system; lifting is
solve(f - op.apply(lift)) + lift)."""
import numpy as np

from tests.modal_cases import manufactured, mass_pair, modal_rhs, operator_known_answers, random_rhs, unit_lift


def test_zero_forcing_gives_zero(O):  # test_solvers.cpp:38-44
    assert np.abs(O.modal_helmholtz(np.zeros((10, 10), complex), 0, 0.01)).max() == 0.0


def test_manufactured_solution(O):  # test_solvers.cpp:46-66
    u, g = manufactured(12, 12, 0.05)
    x = O.modal_helmholtz(modal_rhs(O, g), 0, 0.05, tol=1e-13)
    assert np.abs(x - u).max() < 1e-10


def test_scale_zero_inverts_the_mass_pair(O):  # test_solvers.cpp:68-82
    g = mass_pair(10, 8)
    x = O.modal_helmholtz(modal_rhs(O, g), 0, 0.0, tol=1e-12)
    assert np.abs(x - g).max() < 1e-11


def test_lifted_boundary_data(O):  # test_solvers.cpp:84-105
    u, g = manufactured(12, 12, 0.02, wall=1.0)
    x = O.modal_helmholtz(modal_rhs(O, g), 0, 0.02, tol=1e-13, lift=unit_lift(12, 12))
    assert np.abs(x - u).max() < 1e-10


def test_lifting_identity_and_operator(O):
    m, n, w, s = 12, 10, 1, 0.03
    f = random_rhs(m, n, 5)
    lift = np.zeros((4, n, m), complex)
    lift[2 + w] = random_rhs(m, n, 6, 0.5)
    x = O.modal_helmholtz(f, w, s, lift=lift)
    x2, _ = O.modal_solve(f - O.modal_apply(lift[2 + w], w, s, poisson=False), w, s, poisson=False)
    assert np.abs(x - (x2 + lift[2 + w])).max() < 1e-13
    # the homogeneous solution satisfies A X B + C X D = F on the retained (m-2) x (n-2) block
    y, resid = O.modal_solve(f, w, s, poisson=False)
    r = O.modal_apply(y, w, s, poisson=False) - f
    assert np.abs(r[: n - 2, : m - 2]).max() < 1e-10 * np.abs(f).max() and resid < 1e-11
    # Dirichlet data: the solution vanishes at r = 1 and z = +-1 (sum of coefficients, alternating sum)
    assert np.abs(y.sum(axis=1)).max() < 1e-12 and np.abs(y.sum(axis=0)).max() < 1e-12
    assert np.abs((y * (-1.0) ** np.arange(n)[:, None]).sum(axis=0)).max() < 1e-12


def test_operator_known_answers(O):  # test_ultraop.cpp:194-238
    e1, e2, e3 = operator_known_answers(lambda x, w, s, p: O.modal_apply(x, w, s, poisson=p), lambda f: modal_rhs(O, f))
    assert e1 < 1e-12 and e2 < 1e-15 and e3 < 1e-13


def test_quadruple_structure(O):  # test_ultraop.cpp:170-192 through apply on unit matrices
    m, n, s = 10, 8, 0.37
    x = random_rhs(m, n, 9)
    mass, pois = O.modal_apply(x, 3, 0.0, poisson=False), O.modal_apply(x, 3, 1.0, poisson=True)
    # helmholtz(scale) = mass - scale * poisson
    assert np.abs(O.modal_apply(x, 3, s, poisson=False) - (mass - s * pois)).max() < 1e-13 * np.abs(pois).max()
    assert np.abs(mass - modal_rhs(O, x)).max() < 1e-14 * np.abs(mass).max()  # mass = R2 X C02^T, C = 0
    # wavenumber 2 adds -w^2 C02 to the radial Laplacian: (L_0 - L_2) X C02^T = 4 C02 X C02^T
    c02m, c02n = O.operator_dense(m, "c02"), O.operator_dense(n, "c02")
    d = O.modal_apply(x, 0, 1.0, poisson=True) - O.modal_apply(x, 2, 1.0, poisson=True)
    assert np.abs(d - (4.0 * c02m @ x.T @ c02n.T).T).max() < 1e-12 * np.abs(d).max()


def test_poisson_boundary_rows_hold(O):  # test_solvers.cpp:148-156
    from tests.conftest import sample
    m, n, p = 12, 12, 8
    f = sample(O, m, n, p, lambda r, z, t: np.sin(2 * r * np.cos(t)) * np.cos(z) + 0.3 * z)
    u = O.poisson3d(O.analyze(f))
    worst = 0.0
    for t in -np.pi + 2 * np.pi * np.arange(p) / p:
        for z in np.cos(np.pi * np.arange(n) / (n - 1)):
            worst = max(worst, abs(O.evaluate_at(u, 1.0, z, t)), abs(O.evaluate_at(u, -1.0, z, t)))
        for r in np.cos(np.pi * np.arange(m) / (m - 1)):
            worst = max(worst, abs(O.evaluate_at(u, r, 1.0, t)), abs(O.evaluate_at(u, r, -1.0, t)))
    assert worst < 1e-12 * max(1.0, np.abs(u).max())
