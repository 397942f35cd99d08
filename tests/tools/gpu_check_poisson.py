import sys, time, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..', '..'))
import numpy as np
from tests.inputs import hermitian_coeffs, rel_err
import paper_2206_04827_b200 as P
from oracle import pyoracle as O

for (m, n, p) in [(8, 8, 8), (16, 16, 8), (32, 32, 32), (64, 64, 16)]:
    f = hermitian_coeffs(m, n, p, 0.8, 1)
    t0 = time.time(); u_ref = O.poisson3d(f); t_or = time.time() - t0
    ctx = P.Context(m, n, p)
    t0 = time.time(); u = ctx.solve_poisson_3d(f); t1 = time.time() - t0
    t0 = time.time(); u = ctx.solve_poisson_3d(f); t2 = time.time() - t0
    print(f"poisson {m}x{n}x{p}: rel_err {rel_err(u, u_ref):.3e}  oracle {t_or:.3f}s gpu first {t1:.3f}s second {t2:.4f}s  stats {ctx.stats()}", flush=True)
    # non-Hermitian arbitrary input (full-spectrum path)
    rng = np.random.default_rng(5)
    g = (rng.standard_normal((p, n, m)) + 1j * rng.standard_normal((p, n, m))) * 0.7 ** (np.arange(m)[None, None, :] + np.arange(n)[None, :, None])
    print(f"  arbitrary complex: rel_err {rel_err(ctx.solve_poisson_3d(g), O.poisson3d(g)):.3e}", flush=True)
    # helmholtz
    hist = [hermitian_coeffs(m, n, p, 0.85, 10 + i) for i in range(4)]
    frc = hermitian_coeffs(m, n, p, 0.85, 20)
    for order in (1, 4):
        ref = O.helmholtz_step(hist, order, 0.01, 1e-3, forcing=frc)
        got = ctx.helmholtz_step(hist, order, 0.01, 1e-3, forcing=frc)
        print(f"  helmholtz order {order}: rel_err {rel_err(got, ref):.3e}", flush=True)
    ctx.close()

for (m, n, p) in [(128, 128, 128), (256, 256, 256)]:
    f = hermitian_coeffs(m, n, p, 0.9, 4)
    t0 = time.time(); ctx = P.Context(m, n, p); tc = time.time() - t0
    t0 = time.time(); u = ctx.solve_poisson_3d(f); t1 = time.time() - t0
    ts = []
    for _ in range(3):
        t0 = time.time(); u = ctx.solve_poisson_3d(f); ts.append(time.time() - t0)
    print(f"poisson {m}^3: ctx {tc:.2f}s first(setup) {t1:.2f}s steady {min(ts)*1e3:.1f} ms (incl H2D/D2H)  stats {ctx.stats()}", flush=True)

# device-pointer path: kernel-dominated timing
import torch, ctypes as C
for (m, n, p) in [(128, 128, 128), (256, 256, 256)]:
    f = hermitian_coeffs(m, n, p, 0.9, 4)
    ctx = P.Context(m, n, p)
    fd = torch.from_numpy(f).cuda(); ud = torch.zeros_like(fd)
    L = P.lib()
    ctx._check(L.ccf_poisson3d(ctx.h, C.c_void_p(fd.data_ptr()), C.c_void_p(ud.data_ptr())))
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); ctx._check(L.ccf_poisson3d(ctx.h, C.c_void_p(fd.data_ptr()), C.c_void_p(ud.data_ptr()))); ts.append(time.perf_counter() - t0)
    ctx.reset_stats(); ctx._check(L.ccf_poisson3d(ctx.h, C.c_void_p(fd.data_ptr()), C.c_void_p(ud.data_ptr())))
    st = ctx.stats()
    t = min(ts)
    print(f"poisson {m}^3 device ptrs (full spectrum {p} slots): {t*1e3:.2f} ms, sub-problem iterations {st['adi_iterations']}, "
          f"{t/st['adi_iterations']*148*1.9e9:.0f} SM-cycles per sub-problem iteration", flush=True)
