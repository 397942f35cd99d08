"""Modal Sylvester solvers on the GPU: fast diagonalization (default) and the ADI kernel (the
reference algorithm, adi.cpp:150-202; ctx flag bit 2) against the oracle and against each other.
Tolerance 1e-10 relative max-norm (BASELINE.json north_star)."""
import numpy as np
import pytest

from tests.inputs import hermitian_coeffs, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.mark.parametrize("solver", ["diag", "adi"])
@pytest.mark.parametrize("size", [(8, 8, 8), (16, 12, 8), (32, 32, 16)], ids=lambda s: "x".join(map(str, s)))
def test_solvers_vs_oracle(P, O, solver, size):
    m, n, p = size
    ctx = P.Context(m, n, p, solver=solver)
    f = hermitian_coeffs(m, n, p, 0.8, 1)
    assert rel_err(ctx.solve_poisson_3d(f), O.poisson3d(f)) < TOL
    rng = np.random.default_rng(5)
    g = (rng.standard_normal((p, n, m)) + 1j * rng.standard_normal((p, n, m))) * 0.7 ** np.arange(m)
    assert rel_err(ctx.solve_poisson_3d(g), O.poisson3d(g)) < TOL
    hist = [hermitian_coeffs(m, n, p, 0.85, 10 + i) for i in range(4)]
    frc = hermitian_coeffs(m, n, p, 0.85, 20)
    for order in (1, 4):
        ref = O.helmholtz_step(hist, order, 0.01, 1e-3, forcing=frc)
        assert rel_err(ctx.helmholtz_step(hist, order, 0.01, 1e-3, forcing=frc), ref) < TOL
    ctx.close()


@pytest.mark.parametrize("size", [(128, 128, 4), (256, 256, 4)], ids=lambda s: "x".join(map(str, s)))
def test_diag_vs_adi_full_size(P, size):
    """At the benchmark resolutions (oracle too slow): the two device solvers agree to the ADI
    tolerance on rough (decay 0.8) and smooth data."""
    m, n, p = size
    cd = P.Context(m, n, p, solver="diag")
    ca = P.Context(m, n, p, solver="adi")
    for decay, seed in ((0.8, 7), (0.95, 8)):
        f = hermitian_coeffs(m, n, p, decay, seed)
        assert rel_err(cd.solve_poisson_3d(f), ca.solve_poisson_3d(f)) < 1e-11
        hist = [hermitian_coeffs(m, n, p, decay, seed + 10 + i) for i in range(4)]
        assert rel_err(cd.helmholtz_step(hist, 4, 1e-3, 5e-4), ca.helmholtz_step(hist, 4, 1e-3, 5e-4)) < 1e-11
    cd.close()
    ca.close()


def test_ns_steps_adi_kernel_vs_oracle(P, O):
    """The ADI-kernel NS path (reference algorithm) at the config-3 shape, 6 steps incl. the ramp."""
    from bench import CONFIGS, initial_vorticity
    cfg = CONFIGS[64]
    ctx = P.Context(64, 64, 64, solver="adi")
    wl, wg, _ = initial_vorticity(ctx, cfg)
    ns = P.NSStepper(ctx, wl, wg, reynolds=cfg["reynolds"], h=cfg["h"])
    ons = O.NSStepper(wl, wg, cfg["reynolds"], cfg["h"])
    for _ in range(6):
        ns.step()
        ons.step()
        (l, g), (rl, rg) = ns.omega(), ons.omega()
        assert max(rel_err(l, rl), rel_err(g, rg)) < TOL
    ns.close()
    ctx.close()


def test_fused_solve_kernel_matches(P, tmp_path):
    """The opt-in fused fast-diagonalization kernel (CCF_FDSOLVE_FUSED=1, one CTA per sub-problem)
    against the default four-GEMM chain, in a subprocess so the switch is read fresh."""
    import os
    import subprocess
    import sys
    out = tmp_path / "fd_out.npy"
    code = (
        "import numpy as np, paper_2206_04827_b200 as P\n"
        "from tests.inputs import hermitian_coeffs\n"
        "c = P.Context(64, 64, 8)\n"
        "f = hermitian_coeffs(64, 64, 8, 0.8, 7)\n"
        f"np.save({str(out)!r}, c.solve_poisson_3d(f))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CCF_FDSOLVE_FUSED="1")
    subprocess.run([sys.executable, "-c", code], check=True, cwd=root, env=env)
    fused = np.load(out)
    c = P.Context(64, 64, 8)
    ref = c.solve_poisson_3d(hermitian_coeffs(64, 64, 8, 0.8, 7))
    assert rel_err(fused, ref) < 1e-12
