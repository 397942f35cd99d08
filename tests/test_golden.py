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
