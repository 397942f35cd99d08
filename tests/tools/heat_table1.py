"""Paper Table 1 harness (bench_spectral, proj/src/bench.cpp:56-84, Table 1): the
manufactured heat problem T = e^-t cos(pi z/2)(1 - r^2)(1 + r cos(th)/2), alpha = 1, h = 0.01,
200 BDF4 steps, forcing evaluated at t + h every step (ForcingMode::exact), max relative grid error
at t = 2 and wall seconds of the whole run (forcing evaluation included, like the reference).

GPU: HeatStepper on the device, forcing sampled on the device (torch) and analyzed there. The B200
path needs even m, n, so the paper's N = 7^3 .. 19^3 become 8^3 .. 20^3; the CPU oracle (the
reference's algorithm, one core) runs the paper's own sizes. Larger GPU sizes show the scaling.

  python tests/tools/heat_table1.py [--cpu-sizes 7,11,15,19] [--gpu-sizes 8,12,16,20,32,64,128]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_2206_04827_b200 as P  # noqa: E402
from oracle import pyoracle as O  # noqa: E402


def grid_np(m, n, p):
    r, z, th = O.chebyshev_points(m), O.chebyshev_points(n), O.fourier_points(p)
    T, Z, R = np.meshgrid(th, z, r, indexing="ij")  # reference layout (l, k, j)
    return R, Z, T


def exact_np(R, Z, T, t):
    return np.exp(-t) * np.cos(np.pi * Z / 2) * (1 - R * R) * (1 + 0.5 * R * np.cos(T))


def forcing_np(R, Z, T, t, alpha=1.0):
    zz = np.cos(np.pi * Z / 2)
    s = (1 - R * R) * (1 + 0.5 * R * np.cos(T))
    lap = np.exp(-t) * (-4.0 * zz * (1 + R * np.cos(T)) - np.pi ** 2 / 4.0 * zz * s)
    return -np.exp(-t) * zz * s - alpha * lap


def run_gpu(s, steps=200, h=0.01):
    import torch
    m = n = p = s
    R, Z, T = grid_np(m, n, p)
    Rd, Zd, Td = (torch.from_numpy(x).cuda() for x in (R, Z, T))
    zz, cr = torch.cos(np.pi * Zd / 2), torch.cos(Td)
    S = (1 - Rd * Rd) * (1 + 0.5 * Rd * cr)
    lap0 = -4.0 * zz * (1 + Rd * cr) - np.pi ** 2 / 4.0 * zz * S

    def forcing(t):  # device-side evaluation of the closed form (the reference's callback)
        return (-np.exp(-t) * zz * S - np.exp(-t) * lap0).contiguous()

    ctx = P.Context(m, n, p)
    P.heat_run(ctx, exact_np(R, Z, T, 0.0), forcing, 2, alpha=1.0, h=h)  # warm: setup + plans
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run = P.heat_run(ctx, exact_np(R, Z, T, 0.0), forcing, steps, alpha=1.0, h=h)
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    ref = exact_np(R, Z, T, run["final_time"])
    err = np.abs(run["snapshots"][-1] - ref).max() / np.abs(ref).max()
    ctx.close()
    return err, sec


def run_cpu(s, steps=200, h=0.01):
    m = n = s
    p = s if s % 2 == 0 else s + 1  # bench_grid (bench.cpp:46-48)
    R, Z, T = grid_np(m, n, p)
    t0 = time.perf_counter()
    st = O.HeatStepper(O.analyze(exact_np(R, Z, T, 0.0)), alpha=1.0, h=h, order=4)
    t = 0.0
    for _ in range(steps):
        st.step(O.analyze(forcing_np(R, Z, T, t + h)))
        t += h
    c, tf, _ = st.current()
    got = O.synthesize(c)
    sec = time.perf_counter() - t0
    ref = exact_np(R, Z, T, tf)
    return np.abs(got - ref).max() / np.abs(ref).max(), sec, (m, n, p)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cpu-sizes", default="7,11,15,19")
    ap.add_argument("--gpu-sizes", default="8,12,16,20,32,64,128")
    a = ap.parse_args()
    print("Paper Table 1 (new spectral method, reference CPU): max error 6.03e-5 5.88e-5 3.22e-5 1.76e-5;"
          " seconds 1.00 3.19 5.88 6.50 at N = 7^3 11^3 15^3 19^3")
    print(f"{'impl':28s} {'m,n,p':>12s} {'max rel err':>12s} {'seconds':>9s} {'ms/step':>8s}")
    for s in [int(x) for x in a.cpu_sizes.split(",") if x]:
        e, sec, shp = run_cpu(s)
        print(f"{'CPU oracle (1 core)':28s} {','.join(map(str, shp)):>12s} {e:12.3e} {sec:9.3f} {sec / 200 * 1e3:8.3f}",
              flush=True)
    for s in [int(x) for x in a.gpu_sizes.split(",") if x]:
        e, sec = run_gpu(s)
        print(f"{'B200 HeatStepper':28s} {f'{s},{s},{s}':>12s} {e:12.3e} {sec:9.3f} {sec / 200 * 1e3:8.3f}", flush=True)


if __name__ == "__main__":
    main()
