import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..', '..'))
import numpy as np
from tests.inputs import hermitian_coeffs, rel_err
import paper_2206_04827_b200 as P
from oracle import pyoracle as O

def report(name, got, ref):
    print(f"  {name:28s} rel_err {rel_err(got, ref):.3e}  (|ref| {np.max(np.abs(ref)):.2e})", flush=True)

SHAPES = [tuple(int(x) for x in a.split('x')) for a in sys.argv[1:]] or [(8, 8, 8), (16, 12, 8), (16, 16, 16), (32, 32, 32), (16, 16, 256), (32, 24, 256)]
TOL = float(os.environ.get('ORACLE_TOL', '1e-12'))
for (m, n, p) in SHAPES:
    print(f"== {m}x{n}x{p}", flush=True)
    ctx = P.Context(m, n, p)
    lam = hermitian_coeffs(m, n, p, 0.7, 1)
    gam = hermitian_coeffs(m, n, p, 0.7, 2)
    both = hermitian_coeffs(m, n, p, 0.7, 3) + hermitian_coeffs(m, n, p, 0.7, 4, parity=1)
    for op in ["dr", "dz", "dtheta", "divide_r", "hlap", "lap"]:
        report("calc " + op, ctx.calculus(op, both), O.calculus(op, both))
    report("hpoisson", ctx.solve_horizontal_poisson(lam), O.hpoisson(lam))
    vr, vt, vz = ctx.pt_synthesize(lam, gam)
    ovr, ovt, ovz = O.pt_synthesize(lam, gam)
    report("pt_synthesize r", vr, ovr); report("pt_synthesize t", vt, ovt); report("pt_synthesize z", vz, ovz)
    cr, ct, cz = ctx.curl_vector(ovr, ovt, ovz)
    ocr, oct_, ocz = O.curl_vector(ovr, ovt, ovz)
    report("curl_vector r", cr, ocr); report("curl_vector t", ct, oct_); report("curl_vector z", cz, ocz)
    dl, dg = ctx.pt_decompose(ovr, ovt, ovz)
    odl, odg = O.pt_decompose(ovr, ovt, ovz)
    report("pt_decompose lam", dl, odl); report("pt_decompose gam", dg, odg)
    cl, cg = ctx.curl_pt(lam, gam)
    ocl, ocg = O.curl_pt(lam, gam)
    report("curl_pt lam", cl, ocl); report("curl_pt gam", cg, ocg)
    vl, vg = ctx.velocity_from_vorticity(lam, gam)
    ovl, ovg = O.velocity_from_vorticity(lam, gam, tol=TOL)
    report("velocity lam", vl, ovl); report("velocity gam", vg, ovg)
    nl, ng = ctx.nonlinear_term(ovl, ovg, lam, gam)
    onl, ong = O.nonlinear(ovl, ovg, lam, gam)
    report("nonlinear lam", nl, onl); report("nonlinear gam", ng, ong)
    vals = O.synthesize(lam)
    report("analyze", ctx.analyze(vals), O.analyze(vals))
    report("synthesize", ctx.synthesize(both), O.synthesize(both))
    ns = P.NSStepper(ctx, lam, gam, reynolds=100.0, h=1e-3)
    ons = O.NSStepper(lam, gam, 100.0, 1e-3, tol=TOL)
    for st in range(1, 7 if p <= 64 else 3):  # the random field is under-resolved in time at p = 256
        ns.step(1); ons.step(1)
        gl, gg = ns.omega(); rl, rg = ons.omega()
        print(f"  NS step {st}: lam {rel_err(gl, rl):.3e} gam {rel_err(gg, rg):.3e}", flush=True)
    ns.close(); ctx.close()
