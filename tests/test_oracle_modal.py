"""Oracle pins for the per-mode solver API against the reference's own known answers
(proj/tests/test_solvers.cpp:38-105: zero forcing, manufactured Helmholtz solution, the scale-zero mass pair,
lifted boundary data) plus the defining identities (the solution solves the recombined system; lifting is
solve(f - op.apply(lift)) + lift)."""
import numpy as np

from tests.modal_cases import manufactured, mass_pair, modal_rhs, random_rhs, unit_lift


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
