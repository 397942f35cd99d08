"""GPU parity: every hot-path entry point through the C-ABI (lib/libccf.so) against the CPU
oracle on the same seeded inputs, and against the committed golden fixtures.
Tolerance: relative max-norm coefficient error <= 1e-10 (BASELINE.json north_star)."""
import os

import numpy as np
import pytest

from tests.conftest import sample
from tests.inputs import hermitian_coeffs, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-10
G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SIZES = [(8, 8, 8), (16, 12, 8), (32, 32, 32)]


@pytest.fixture(scope="module", params=SIZES, ids=lambda s: "x".join(map(str, s)))
def ctxsize(request, P):
    m, n, p = request.param
    ctx = P.Context(m, n, p)
    yield ctx, m, n, p
    ctx.close()


def test_transforms(ctxsize, O):
    ctx, m, n, p = ctxsize
    both = hermitian_coeffs(m, n, p, 0.7, 3) + hermitian_coeffs(m, n, p, 0.7, 4, parity=1)
    vals = O.synthesize(both)
    assert rel_err(ctx.synthesize(both), vals) < TOL
    assert rel_err(ctx.analyze(vals), O.analyze(vals)) < TOL
    rng = np.random.default_rng(1)
    arb = rng.standard_normal((p, n, m))  # arbitrary (non-physical) real field
    assert rel_err(ctx.analyze(arb), O.analyze(arb)) < TOL


@pytest.mark.parametrize("op", ["dr", "dz", "dtheta", "divide_r", "hlap", "lap"])
def test_calculus(ctxsize, O, op):
    ctx, m, n, p = ctxsize
    both = hermitian_coeffs(m, n, p, 0.7, 3) + hermitian_coeffs(m, n, p, 0.7, 4, parity=1)
    assert rel_err(ctx.calculus(op, both), O.calculus(op, both)) < TOL


def test_solvers(ctxsize, O):
    ctx, m, n, p = ctxsize
    f = hermitian_coeffs(m, n, p, 0.8, 1)
    assert rel_err(ctx.solve_poisson_3d(f), O.poisson3d(f)) < TOL
    rng = np.random.default_rng(5)
    g = (rng.standard_normal((p, n, m)) + 1j * rng.standard_normal((p, n, m))) * 0.7 ** np.arange(m)
    assert rel_err(ctx.solve_poisson_3d(g), O.poisson3d(g)) < TOL  # non-Hermitian, full spectrum
    assert rel_err(ctx.solve_horizontal_poisson(f), O.hpoisson(f)) < TOL
    hist = [hermitian_coeffs(m, n, p, 0.85, 10 + i) for i in range(4)]
    frc = hermitian_coeffs(m, n, p, 0.85, 20)
    for order in (1, 2, 3, 4):
        ref = O.helmholtz_step(hist, order, 0.01, 1e-3, forcing=frc)
        assert rel_err(ctx.helmholtz_step(hist, order, 0.01, 1e-3, forcing=frc), ref) < TOL
    assert rel_err(ctx.helmholtz_step(hist[:2], 2, 0.5, 1e-2), O.helmholtz_step(hist[:2], 2, 0.5, 1e-2)) < TOL


def test_pt_machinery(ctxsize, O):
    ctx, m, n, p = ctxsize
    lam = hermitian_coeffs(m, n, p, 0.7, 1)
    gam = hermitian_coeffs(m, n, p, 0.7, 2)
    for a, b in zip(ctx.pt_synthesize(lam, gam), O.pt_synthesize(lam, gam)):
        assert rel_err(a, b) < TOL
    v = O.pt_synthesize(lam, gam)
    for a, b in zip(ctx.curl_vector(*v), O.curl_vector(*v)):
        assert rel_err(a, b) < TOL
    for a, b in zip(ctx.pt_decompose(*v), O.pt_decompose(*v)):
        assert rel_err(a, b) < TOL
    for a, b in zip(ctx.curl_pt(lam, gam), O.curl_pt(lam, gam)):
        assert rel_err(a, b) < TOL
    vel = O.velocity_from_vorticity(lam, gam)
    for a, b in zip(ctx.velocity_from_vorticity(lam, gam), vel):
        assert rel_err(a, b) < TOL
    for a, b in zip(ctx.nonlinear_term(*vel, lam, gam), O.nonlinear(*vel, lam, gam)):
        assert rel_err(a, b) < TOL


def test_ns_steps_vs_oracle(P, O):
    # BASELINE config 3 shape (64^3, Re 100, h 1e-3, seeded decay-0.7 field), 8 steps incl. the BDF ramp
    from bench import CONFIGS, initial_vorticity
    cfg = CONFIGS[64]
    ctx = P.Context(64, 64, 64)
    wl, wg, _ = initial_vorticity(ctx, cfg)
    ns = P.NSStepper(ctx, wl, wg, reynolds=cfg["reynolds"], h=cfg["h"])
    ons = O.NSStepper(wl, wg, cfg["reynolds"], cfg["h"])
    errs = []
    for _ in range(8):
        ns.step()
        ons.step()
        (l, g), (rl, rg) = ns.omega(), ons.omega()
        errs.append(max(rel_err(l, rl), rel_err(g, rg)))
    print("per-step rel err (drift):", ["%.2e" % e for e in errs])
    assert max(errs) < TOL
    ns.close()
    ctx.close()


def test_context_closed_before_stepper(P):
    """Destroying the context first detaches its steppers: later calls fail cleanly, close() is safe."""
    lam = 1e-3 * hermitian_coeffs(16, 16, 16, 0.7, 1)
    gam = 1e-3 * hermitian_coeffs(16, 16, 16, 0.7, 2)
    ctx = P.Context(16, 16, 16)
    ns = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3)
    ns.step(2)
    ctx.close()
    with pytest.raises(P.CCFError):
        ns.step(1)
    ns.close()


def test_omega_readback_does_not_perturb(P):
    """In the eigen-coordinate state omega() reconstructs the coefficients on demand; reading it every
    step or only at the end gives the same trajectory."""
    lam = 1e-3 * hermitian_coeffs(16, 16, 16, 0.7, 3)
    gam = 1e-3 * hermitian_coeffs(16, 16, 16, 0.7, 4)
    ctx = P.Context(16, 16, 16)
    a = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3)
    b = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3)
    for _ in range(8):
        a.step(1)
        a.omega()
    b.step(8)
    (la, ga), (lb, gb) = a.omega(), b.omega()
    assert max(rel_err(la, lb), rel_err(ga, gb)) < 1e-13
    a.close()
    b.close()
    ctx.close()


def test_graph_replay_equals_eager(P):
    # small amplitude: a random O(1) field violates the advective CFL bound and diverges (Q4)
    lam = 1e-3 * hermitian_coeffs(16, 16, 16, 0.7, 1)
    gam = 1e-3 * hermitian_coeffs(16, 16, 16, 0.7, 2)
    ctx = P.Context(16, 16, 16)
    a = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3)
    b = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3)
    b.set_graphs(False)
    a.step(14)
    b.step(14)
    (la, ga), (lb, gb) = a.omega(), b.omega()
    assert np.array_equal(la, lb) and np.array_equal(ga, gb)  # CUDA graphs replay the same kernels
    assert a.launches_per_step() > 0


def test_golden_fixtures(P):
    d = np.load(os.path.join(G, "poisson_16.npz"))
    ctx = P.Context(16, 16, 16)
    assert rel_err(ctx.solve_poisson_3d(d["f"]), d["u"]) < TOL
    d = np.load(os.path.join(G, "ns_8.npz"))
    c8 = P.Context(8, 8, 8)
    ns = P.NSStepper(c8, d["lam0"], d["gam0"], reynolds=100.0, h=1e-3)
    for s in range(1, 6):
        ns.step()
        l, g = ns.omega()
        assert rel_err(l, d[f"lam{s}"]) < TOL and rel_err(g, d[f"gam{s}"]) < TOL
    t = np.load(os.path.join(G, "transform_12x10x8.npz"))
    c12 = P.Context(12, 10, 8)
    assert rel_err(c12.analyze(t["values"]), t["coeffs"]) < TOL
    h = np.load(os.path.join(G, "helmholtz_16x12x8.npz"))
    c16 = P.Context(16, 12, 8)
    out = c16.helmholtz_step([h["h0"], h["h1"], h["h2"], h["h3"]], 4, 0.01, 1e-3, forcing=h["forcing"])
    assert rel_err(out, h["out"]) < TOL


@pytest.mark.parametrize("size", [(16, 16, 12), (12, 10, 6), (16, 12, 20)], ids=lambda s: "x".join(map(str, s)))
def test_ns_any_even_p(P, O, size):
    # p that is not a power of two (the reference's FFTW plans take any even p): the theta stage runs dense DFTs
    m, n, p = size
    ctx = P.Context(m, n, p)
    lam, gam = hermitian_coeffs(m, n, p, 0.7, 1) * 1e-2, hermitian_coeffs(m, n, p, 0.7, 2) * 1e-2
    st, ons = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3), O.NSStepper(lam, gam, 100.0, 1e-3)
    st.step(7)
    ons.step(7)
    (l, g), (rl, rg) = st.omega(), ons.omega()
    assert max(rel_err(l, rl), rel_err(g, rg)) < TOL
    got, ref = ctx.nonlinear_term(gam, lam, lam, gam), O.nonlinear(gam, lam, lam, gam)
    assert max(rel_err(got[0], ref[0]), rel_err(got[1], ref[1])) < TOL
    st.close()
    ctx.close()


def test_golden_fixtures_round2(P):
    # per-mode API, lifted data and the substeps bootstrap against the committed oracle vectors
    d = np.load(os.path.join(G, "modal_12x10.npz"))
    ctx = P.Context(12, 10, 4)
    for name, (w, scale, poisson) in {"poisson_w2": (2, 1.0, True), "helm_w1": (1, 0.03, False), "mass_w0": (0, 0.0, False)}.items():
        s = P.ModalSolver(ctx, w, scale, poisson)
        assert rel_err(s.solve(d["f"]), d[name]) < TOL and rel_err(s.apply(d["f"]), d[name + "_apply"]) < 1e-13
        s.close()
    ctx.close()
    d = np.load(os.path.join(G, "poisson_lifted_12x10x8.npz"))
    ctx = P.Context(12, 10, 8)
    assert rel_err(ctx.solve_poisson_3d(d["f"], lift=d["lift"]), d["u"]) < TOL
    ctx.close()
    d = np.load(os.path.join(G, "ns_run_substeps_8.npz"))
    ctx = P.Context(8, 8, 8)
    run = P.ns_run(ctx, d["lam0"], d["gam0"], 6, reynolds=100.0, h=2e-3, order=3, bootstrap="substeps")
    assert rel_err(run["final_omega"][0], d["lam"]) < TOL and rel_err(run["final_omega"][1], d["gam"]) < TOL
    assert abs(run["final_time"] - float(d["time"])) < 1e-15
    ctx.close()


def test_error_taxonomy(P):
    ctx = P.Context(8, 8, 8)
    f = np.zeros((8, 8, 8), complex)
    f[4, 0, 0] = np.nan
    with pytest.raises(P.NumericalError):
        ctx.solve_poisson_3d(f)  # solvers.cpp:145
    vals = np.zeros((8, 8, 8))
    vals[1, 2, 3] = np.inf
    with pytest.raises(P.NumericalError):
        ctx.analyze(vals)  # transform.cpp:125
    with pytest.raises(P.DomainError):
        ctx.helmholtz_step([f.real * 0], 5, 0.1, 0.1)  # BDFScheme order
    with pytest.raises(P.DomainError):
        P.Context(9, 8, 8)  # odd m: outside the B200 path
    with pytest.raises(P.DomainError):
        P.Context(8, 8, 7)  # odd p (grid.cpp:10)


def test_cpp_shim_drop_in(P):
    # the reference-API C++ program shape compiled against include/cylspec_b200.hpp
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "shim_ns")
    r = subprocess.run([exe, "16"], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "shim ok" in r.stdout
