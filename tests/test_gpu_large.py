"""Grids beyond the ADI kernel's single-CTA tile (m > 258): fast-diagonalization contexts carry no
ADI data, so the NS path runs at any size (config 5 is 512^3). Parity against the oracle where the
reference's own Poisson plan still exists (the 1e-8 enclosure pad overlaps at larger m, quirk Q2).
At m = 384 the reference ADI's rounding floor lies above its default 1e-12 (it throws
NonConvergenceError), so the oracle runs with adi_tol = 1e-10; its inexact solves accumulate to ~1e-8
over 4 steps (the components alone agree to ~1e-11, tests/tools/gpu_check_ns.py 384x16x16), gate 5e-8."""
import numpy as np
import pytest

from tests.inputs import hermitian_coeffs, rel_err

pytestmark = pytest.mark.gpu


def test_large_m_ns_matches_oracle(P, O):
    m, n, p = 384, 16, 16
    ctx = P.Context(m, n, p)
    lam, gam = hermitian_coeffs(m, n, p, 0.7, 3), hermitian_coeffs(m, n, p, 0.7, 103)
    st = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3)
    ons = O.NSStepper(lam, gam, 100.0, 1e-3, tol=1e-10)
    st.step(4)
    ons.step(4)
    (l, g), (rl, rg) = st.omega(), ons.omega()
    assert max(rel_err(l, rl), rel_err(g, rg)) < 5e-8  # oracle ADI residual 1e-10 per solve, 4 steps
    st.close()
    ctx.close()


def test_large_m_transforms_and_nonlinear(P, O):
    m, n, p = 400, 16, 8
    ctx = P.Context(m, n, p)
    both = hermitian_coeffs(m, n, p, 0.7, 3) + hermitian_coeffs(m, n, p, 0.7, 4, parity=1)
    vals = O.synthesize(both)
    assert rel_err(ctx.synthesize(both), vals) < 1e-10
    assert rel_err(ctx.analyze(vals), O.analyze(vals)) < 1e-10
    lam, gam = hermitian_coeffs(m, n, p, 0.7, 1), hermitian_coeffs(m, n, p, 0.7, 2)
    vl, vg = hermitian_coeffs(m, n, p, 0.7, 5), hermitian_coeffs(m, n, p, 0.7, 6)
    got = ctx.nonlinear_term(vl, vg, lam, gam)
    ref = O.nonlinear(vl, vg, lam, gam)
    assert max(rel_err(got[0], ref[0]), rel_err(got[1], ref[1])) < 1e-10
    ctx.close()


def test_adi_solver_keeps_the_tile_limit(P):
    with pytest.raises(P.DomainError):
        P.Context(384, 16, 16, solver="adi")


@pytest.mark.parametrize("size", [(256, 16, 16), (384, 16, 16), (258, 16, 8), (16, 384, 8), (200, 40, 8)],
                         ids=lambda s: "x".join(map(str, s)))
def test_poisson_tma_gemm_shapes(P, O, size):
    """Solver GEMMs on the TMA kernel (M > 64) with k-extents that are not multiples of its 16-column
    boxes (n = 16: K = 7, 8): the launcher must fall back where no zero padding covers the box."""
    m, n, p = size
    f = hermitian_coeffs(m, n, p, 0.8, 1)
    ctx = P.Context(m, n, p)
    ref = O.poisson3d(f, tol=1e-10)
    assert rel_err(ctx.solve_poisson_3d(f), ref) < 1e-9
    ctx.close()


def test_tma_path_ns_matches_oracle(P, O):
    """A grid where the GEMMs of the eigen-coordinate step have M > 64 (the TMA kernel's range), 16-column
    k-boxes and operand blocks at aligned and unaligned offsets (the 256^3 bench shape is too slow for
    the oracle in a test). Per step the agreement is <= 1e-10 (the north-star contract); over several
    steps the oracle's own ADI error (residual <= 1e-12 at cond ~1e3) dominates the drift (~5e-10 by
    step 3 at this size, tests/tools/gpu_check_ns.py 160x64x8), so the 3-step gate is 2e-9."""
    m, n, p = 160, 64, 8  # mh = 80, nh = 32: 16-column k-boxes, mixed aligned / unaligned blocks
    ctx = P.Context(m, n, p)
    lam, gam = hermitian_coeffs(m, n, p, 0.7, 3), hermitian_coeffs(m, n, p, 0.7, 103)
    st = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3)
    ons = O.NSStepper(lam, gam, 100.0, 1e-3)
    st.step(1)
    ons.step(1)
    (l, g), (rl, rg) = st.omega(), ons.omega()
    assert max(rel_err(l, rl), rel_err(g, rg)) < 1e-10
    st.step(2)
    ons.step(2)
    (l, g), (rl, rg) = st.omega(), ons.omega()
    assert max(rel_err(l, rl), rel_err(g, rg)) < 2e-9
    st.close()
    ctx.close()
