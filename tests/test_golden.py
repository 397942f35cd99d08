"""The oracle reproduces the committed golden fixtures (tests/golden/make_golden.py)."""
import os

import numpy as np

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_golden_poisson(O):
    d = np.load(os.path.join(G, "poisson_16.npz"))
    assert np.abs(O.poisson3d(d["f"]) - d["u"]).max() <= 1e-13 * np.abs(d["u"]).max()


def test_golden_ns(O):
    d = np.load(os.path.join(G, "ns_8.npz"))
    ns = O.NSStepper(d["lam0"], d["gam0"], reynolds=100.0, h=1e-3)
    for s in range(1, 6):
        ns.step()
        l, g = ns.omega()
        assert np.abs(l - d[f"lam{s}"]).max() <= 1e-12 * np.abs(d[f"lam{s}"]).max()
        assert np.abs(g - d[f"gam{s}"]).max() <= 1e-12 * np.abs(d[f"gam{s}"]).max()


def test_golden_transform_and_helmholtz(O):
    d = np.load(os.path.join(G, "transform_12x10x8.npz"))
    assert np.abs(O.analyze(d["values"]) - d["coeffs"]).max() < 1e-14
    h = np.load(os.path.join(G, "helmholtz_16x12x8.npz"))
    out = O.helmholtz_step([h["h0"], h["h1"], h["h2"], h["h3"]], 4, 0.01, 1e-3, forcing=h["forcing"])
    assert np.abs(out - h["out"]).max() <= 1e-13 * np.abs(h["out"]).max()


def test_golden_modal_lifted_and_substeps(O):
    d = np.load(os.path.join(G, "modal_12x10.npz"))
    for name, (w, scale, poisson) in {"poisson_w2": (2, 1.0, True), "helm_w1": (1, 0.03, False), "mass_w0": (0, 0.0, False)}.items():
        assert np.abs(O.modal_solve(d["f"], w, scale, poisson)[0] - d[name]).max() <= 1e-12 * np.abs(d[name]).max()
        assert np.abs(O.modal_apply(d["f"], w, scale, poisson) - d[name + "_apply"]).max() <= 1e-13 * np.abs(d[name + "_apply"]).max()
    d = np.load(os.path.join(G, "poisson_lifted_12x10x8.npz"))
    assert np.abs(O.poisson3d(d["f"], lift=d["lift"]) - d["u"]).max() <= 1e-12 * np.abs(d["u"]).max()
    d = np.load(os.path.join(G, "ns_run_substeps_8.npz"))
    l, g, t = O.ns_run(d["lam0"], d["gam0"], 6, 100.0, 2e-3, order=3, bootstrap="substeps")
    assert np.abs(l - d["lam"]).max() <= 1e-11 * np.abs(d["lam"]).max() and np.abs(g - d["gam"]).max() <= 1e-11 * np.abs(d["gam"]).max()
    assert abs(t - float(d["time"])) < 1e-15
