"""Per-mode solver API on the device (ccf_modal_*: ModalSolver::solve on raw right-hand sides, ModalOperator::apply,
the scale-zero mass pair, lifted boundary data) against the reference's known answers
(proj/tests/test_solvers.cpp:38-105) and the CPU oracle on seeded inputs (1e-10 relative max-norm)."""
import numpy as np
import pytest

from tests.inputs import hermitian_coeffs, rel_err
from tests.modal_cases import manufactured, mass_pair, modal_rhs, operator_known_answers, random_rhs, unit_lift

pytestmark = pytest.mark.gpu
TOL = 1e-10


def test_reference_known_answers(P, O):
    ctx = P.Context(12, 12, 4)
    assert np.abs(P.solve_modal_helmholtz(ctx, np.zeros((12, 12), complex), 0, 0.01)).max() == 0.0  # :38-44
    u, g = manufactured(12, 12, 0.05)  # :46-66
    assert np.abs(P.solve_modal_helmholtz(ctx, modal_rhs(O, g), 0, 0.05) - u).max() < TOL
    u, g = manufactured(12, 12, 0.02, wall=1.0)  # :84-105
    x = P.solve_modal_helmholtz(ctx, modal_rhs(O, g), 0, 0.02, lift=unit_lift(12, 12))
    assert np.abs(x - u).max() < TOL
    ctx.close()
    ctx = P.Context(10, 8, 4)
    g = mass_pair(10, 8)  # :68-82
    assert np.abs(P.solve_modal_helmholtz(ctx, modal_rhs(O, g), 0, 0.0) - g).max() < 1e-11
    ctx.close()


@pytest.mark.parametrize("size", [(12, 10), (32, 32), (24, 40)], ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("w", [0, 1, 5])
def test_modal_solver_matches_oracle(P, O, size, w):
    m, n = size
    ctx = P.Context(m, n, 4)
    f = random_rhs(m, n, 100 + w)  # both parities, complex
    for poisson, scale in ((True, 1.0), (False, 0.03), (False, 1e-5), (False, 0.0)):
        s = P.ModalSolver(ctx, w, scale, poisson)
        ref, _ = O.modal_solve(f, w, scale, poisson)
        assert rel_err(s.solve(f), ref) < TOL, (poisson, scale)
        assert rel_err(s.apply(f), O.modal_apply(f, w, scale, poisson)) < 1e-13
        s.close()
    # negative wavenumbers share the operator (w^2 only)
    a, b = P.ModalSolver(ctx, -w, 0.03, False), P.ModalSolver(ctx, w, 0.03, False)
    assert np.array_equal(a.solve(f), b.solve(f))
    ctx.close()


def test_modal_operator_entries_and_errors(P, O):
    m, n = 12, 10
    ctx = P.Context(m, n, 4)
    s = P.ModalSolver(ctx, 2, 0.5, False)
    r2, c02, d2 = O.operator_dense(m, "r2"), O.operator_dense(n, "c02"), O.operator_dense(n, "d2")
    assert np.allclose(s.operator("B"), c02.T, atol=1e-15) and np.allclose(s.operator("D"), d2.T, atol=1e-15)
    assert np.allclose(s.operator("C"), -0.5 * r2, atol=1e-15)
    x = random_rhs(m, n, 3)
    y = s.operator("A") @ x.T @ s.operator("B") + s.operator("C") @ x.T @ s.operator("D")
    assert rel_err(s.apply(x), y.T) < 1e-13
    with pytest.raises(P.DomainError, match="wrong shape"):
        s.solve(np.zeros((n, m + 2), complex))
    bad = x.copy()
    bad[1, 1] = np.nan
    with pytest.raises(P.NumericalError):
        s.solve(bad)
    with pytest.raises(P.DomainError):
        P.solve_modal_helmholtz(ctx, x, 3, 0.1, lift=np.zeros((4, n, m), complex))  # mode 3 not in a p = 4 lift
    s.close()
    ctx.close()


def test_lifted_poisson_and_helmholtz_step(P, O):
    m, n, p = 16, 12, 8
    ctx = P.Context(m, n, p)
    f = hermitian_coeffs(m, n, p, 0.8, 1)
    lift = hermitian_coeffs(m, n, p, 0.6, 2)
    got = ctx.solve_poisson_3d(f, lift=lift)
    assert rel_err(got, O.poisson3d(f, lift=lift)) < TOL
    assert rel_err(got, ctx.solve_poisson_3d(f)) > 1e-3
    hist = [hermitian_coeffs(m, n, p, 0.7, 10 + i) for i in range(3)]
    forcing = hermitian_coeffs(m, n, p, 0.7, 20)
    for order in (1, 3):
        got = ctx.helmholtz_step(hist, order, 0.05, 1e-2, forcing=forcing, lift=lift)
        ref = O.helmholtz_step(hist, order, 0.05, 1e-2, forcing=forcing, lift=lift)
        assert rel_err(got, ref) < TOL
    with pytest.raises(P.DomainError):
        ctx.solve_poisson_3d(f, lift=lift[:4])
    ctx.close()


def test_operator_known_answers_on_device(P, O):  # test_ultraop.cpp:194-238 through ccf_modal_apply
    def apply(x, w, scale, poisson):
        n, m = x.shape
        ctx = P.Context(m, n, 4)
        s = P.ModalSolver(ctx, w, scale, poisson)
        y = s.apply(x)
        s.close()
        ctx.close()
        return y

    e1, e2, e3 = operator_known_answers(apply, lambda f: modal_rhs(O, f))
    assert e1 < 1e-12 and e2 < 1e-15 and e3 < 1e-13


def test_poisson_boundary_rows_hold_on_device(P, O):  # test_solvers.cpp:148-156
    from tests.conftest import sample
    m, n, p = 12, 12, 8
    ctx = P.Context(m, n, p)
    f = sample(O, m, n, p, lambda r, z, t: np.sin(2 * r * np.cos(t)) * np.cos(z) + 0.3 * z)
    u = ctx.solve_poisson_3d(ctx.analyze(f))
    worst = 0.0
    for t in -np.pi + 2 * np.pi * np.arange(p) / p:
        for z in np.cos(np.pi * np.arange(n) / (n - 1)):
            worst = max(worst, abs(O.evaluate_at(u, 1.0, z, t)), abs(O.evaluate_at(u, -1.0, z, t)))
        for r in np.cos(np.pi * np.arange(m) / (m - 1)):
            worst = max(worst, abs(O.evaluate_at(u, r, 1.0, t)), abs(O.evaluate_at(u, r, -1.0, t)))
    assert worst < 1e-12 * max(1.0, np.abs(u).max())
    ctx.close()


def test_handle_outliving_its_context(P):
    ctx = P.Context(12, 10, 4)
    s = P.ModalSolver(ctx, 1, 0.1, False)
    f = random_rhs(12, 10, 1)
    s.solve(f)
    h = ctx.h
    ctx.close()  # releases the handle's device data and detaches it
    x = np.zeros_like(f)
    assert P.lib().ccf_modal_solve(s.h, f.ctypes.data, x.ctypes.data) == 9  # CCF_INTERNAL_ERROR, no crash
    s.close()
