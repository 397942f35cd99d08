"""Argument validation of the Python mirror before any pointer reaches the C-ABI: the reference
throws DomainError on spec mismatches (ptns.cpp:185-187, timestep.cpp:69-70, 113-114); the C-ABI
reads / writes buffers sized by the context, so a wrongly shaped array must never get through."""
import numpy as np
import pytest

from tests.inputs import hermitian_coeffs

pytestmark = pytest.mark.gpu


def test_shape_and_dtype_checks(P):
    m = n = p = 8
    ctx = P.Context(m, n, p)
    good = hermitian_coeffs(m, n, p, 0.7, 1)
    bad = hermitian_coeffs(m, n, p + 2, 0.7, 1)
    for call in (lambda: ctx.solve_poisson_3d(bad), lambda: ctx.synthesize(bad), lambda: ctx.calculus("dr", bad),
                 lambda: ctx.pt_synthesize(good, bad), lambda: ctx.nonlinear_term(good, good, good, bad),
                 lambda: ctx.analyze(np.zeros((p, n, m + 1))), lambda: ctx.analyze(np.zeros((p, n, m), complex)),
                 lambda: ctx.helmholtz_step([good], 1, 0.01, 1e-3, forcing=bad)):
        with pytest.raises(P.DomainError):
            call()
    with pytest.raises(P.DomainError, match="NSStepper: initial vorticity"):
        P.NSStepper(ctx, good, bad, reynolds=100.0, h=1e-3)
    with pytest.raises(P.DomainError, match="HeatStepper: initial data"):
        P.HeatStepper(ctx, np.zeros((p, n, m + 2)))
    hs = P.HeatStepper(ctx, good, alpha=1.0, h=1e-2)
    with pytest.raises(P.DomainError, match="forcing"):
        hs.step(bad)
    st = P.NSStepper(ctx, good, good, reynolds=100.0, h=1e-3)
    with pytest.raises(P.DomainError):
        st.omega(np.zeros((p, n, m)), np.zeros((p, n, m)))  # real outputs: not a coefficient buffer
    with pytest.raises(P.DomainError):
        st.omega(np.zeros((p, n, m), complex)[:, :, ::2], None)
    # accepted: real-valued inputs are promoted like before, exact outputs are written in place
    lam, gam = np.zeros((p, n, m), complex), np.zeros((p, n, m), complex)
    st.step(1)
    st.omega(lam, gam)
    assert np.isfinite(lam).all() and np.abs(lam).max() > 0
    ctx.solve_poisson_3d(good.real)
    st.close()
    hs.close()
    ctx.close()
