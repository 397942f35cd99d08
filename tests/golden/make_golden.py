"""Generate the golden fixtures (oracle outputs on seeded inputs). Run from the repo root:
    python tests/golden/make_golden.py
The fixtures pin the oracle over time (CPU tests) and are the reference vectors of the GPU
parity tests. The reference C++ itself is unbuildable here, so the oracle,
checked against the reference's own known-answer tests, generates them."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import pyoracle as O  # noqa: E402
from tests.inputs import hermitian_coeffs  # noqa: E402


def main():
    m = n = p = 16
    f = hermitian_coeffs(m, n, p, 0.8, 1)  # config 1 distribution at 16^3
    np.savez_compressed(os.path.join(HERE, "poisson_16.npz"), f=f, u=O.poisson3d(f))
    lam = hermitian_coeffs(8, 8, 8, 0.7, 3)
    gam = hermitian_coeffs(8, 8, 8, 0.7, 103)
    ns = O.NSStepper(lam, gam, reynolds=100.0, h=1e-3)
    out = {"lam0": lam, "gam0": gam}
    for s in range(1, 6):
        ns.step()
        out[f"lam{s}"], out[f"gam{s}"] = ns.omega()
    np.savez_compressed(os.path.join(HERE, "ns_8.npz"), **out)
    vals = O.synthesize(hermitian_coeffs(12, 10, 8, 0.7, 5))
    np.savez_compressed(os.path.join(HERE, "transform_12x10x8.npz"), values=vals, coeffs=O.analyze(vals))
    hist = [hermitian_coeffs(16, 12, 8, 0.85, 10 + i) for i in range(4)]
    frc = hermitian_coeffs(16, 12, 8, 0.85, 20)
    np.savez_compressed(os.path.join(HERE, "helmholtz_16x12x8.npz"), h0=hist[0], h1=hist[1], h2=hist[2], h3=hist[3],
                        forcing=frc, out=O.helmholtz_step(hist, 4, 0.01, 1e-3, forcing=frc))
    # per-mode API, lifted data and the substeps bootstrap (round 2)
    from tests.modal_cases import random_rhs
    fm = random_rhs(12, 10, 7)
    out = {"f": fm}
    for name, (w, scale, poisson) in {"poisson_w2": (2, 1.0, True), "helm_w1": (1, 0.03, False), "mass_w0": (0, 0.0, False)}.items():
        out[name] = O.modal_solve(fm, w, scale, poisson)[0]
        out[name + "_apply"] = O.modal_apply(fm, w, scale, poisson)
    np.savez_compressed(os.path.join(HERE, "modal_12x10.npz"), **out)
    f8, lift8 = hermitian_coeffs(12, 10, 8, 0.8, 31), hermitian_coeffs(12, 10, 8, 0.6, 32)
    np.savez_compressed(os.path.join(HERE, "poisson_lifted_12x10x8.npz"), f=f8, lift=lift8, u=O.poisson3d(f8, lift=lift8))
    lam3, gam3 = hermitian_coeffs(8, 8, 8, 0.7, 21) * 1e-3, hermitian_coeffs(8, 8, 8, 0.7, 22) * 1e-3
    l, g, t = O.ns_run(lam3, gam3, 6, 100.0, 2e-3, order=3, bootstrap="substeps")
    np.savez_compressed(os.path.join(HERE, "ns_run_substeps_8.npz"), lam0=lam3, gam0=gam3, lam=l, gam=g, time=t)


if __name__ == "__main__":
    main()
