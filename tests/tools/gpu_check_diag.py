"""Fast-diagonalization vs ADI kernel vs oracle: Poisson / Helmholtz / NS parity and timing."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2206_04827_b200 as P  # noqa: E402
from oracle import pyoracle as O  # noqa: E402
from tests.inputs import hermitian_coeffs, rel_err  # noqa: E402

for (m, n, p) in [(8, 8, 8), (16, 12, 8), (32, 32, 16), (64, 64, 8), (128, 128, 4), (256, 256, 4)]:
    f = hermitian_coeffs(m, n, p, 0.8, 7)
    t0 = time.time()
    cd = P.Context(m, n, p, solver="diag")
    ca = P.Context(m, n, p, solver="adi")
    ud = cd.solve_poisson_3d(f)
    t1 = time.time()
    ua = ca.solve_poisson_3d(f)
    line = f"{m}x{n}x{p}: poisson diag-vs-adi {rel_err(ud, ua):.2e}"
    if m <= 64:
        uo = O.poisson3d(f)
        line += f" diag-vs-oracle {rel_err(ud, uo):.2e} adi-vs-oracle {rel_err(ua, uo):.2e}"
    hist = [hermitian_coeffs(m, n, p, 0.8, 11 + i) for i in range(4)]
    hd = cd.helmholtz_step(hist, 4, 0.01, 1e-3)
    ha = ca.helmholtz_step(hist, 4, 0.01, 1e-3)
    line += f" | helmholtz diag-vs-adi {rel_err(hd, ha):.2e}  (setup+first {t1 - t0:.2f}s)"
    print(line, flush=True)
    cd.close(); ca.close()
