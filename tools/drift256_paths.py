"""Drift over the BASELINE config-4 run (256^3, Re 1000, h 5e-4, 50 steps) between three independent GPU arithmetic
paths, each in its own process: the production path (INT8 Ozaki products, fast diagonalization, eigen-coordinate
state), the FP64 DMMA path (CCF_OZAKI=0) and the reference-algorithm path (on-chip ADI kernel for every modal
solve, coefficient-space history, sequential pencil kernels). The CPU oracle cannot follow this run: the
reference's ADI iteration stalls above its acceptance threshold (10 tol) at 256^2 from step 2 on, for tol = 1e-12
and 1e-11 alike (profiles/drift_config4_256_oracle_r02.log); step 1 matches the oracle to 6.4e-12.
Usage (under gpurun): python tools/drift256_paths.py [steps] [size]   (size 512 = config 5 on one GPU: the INT8
products are a 256-only path, so the production column there is the FP64 DMMA path itself)"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import bench, paper_2206_04827_b200 as P
cfg = bench.CONFIGS[{size}]
ctx = P.Context({size}, {size}, {size}, solver={solver!r})
wl, wg, _ = bench.initial_vorticity(ctx, cfg, cfg["vmax"])
st = P.NSStepper(ctx, wl, wg, reynolds=cfg["reynolds"], h=cfg["h"], order=4)
out, done = {{}}, 0
for k in {marks}:
    st.step(k - done); done = k
    l, g = st.omega()
    out["l%d" % k] = l[{size} // 2:].copy(); out["g%d" % k] = g[{size} // 2:].copy()   # w >= 0 half (Hermitian)
np.savez({out!r}, **out)
"""


SIZE = 256


def run(name, solver, env, marks):
    out = f"/tmp/drift{SIZE}_{name}.npz"
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, solver=solver, marks=marks, out=out, size=SIZE)],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=3000)
    if r.returncode:
        raise SystemExit(f"{name} failed: {r.stderr[-1500:]}")
    return np.load(out)


def bench_name():
    sys.path.insert(0, ROOT)
    import bench
    return bench.CONFIGS[SIZE]["workload"]


def main():
    global SIZE
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    SIZE = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    marks = sorted(k for k in {1, 2, 3, 5, 10, 20, 30, 40, 50, 100, 200, n} if k <= n)
    prod = run("prod", "diag", {}, marks)
    dmma = run("dmma", "diag", {"CCF_OZAKI": "0"}, marks)
    # the on-chip ADI kernel holds one sub-problem per CTA (m, n <= 320): above that the third path keeps the
    # coefficient-space history and the sequential pencil kernels but solves by fast diagonalization
    refa = run("refalg", "adi" if SIZE <= 320 else "diag",
               {"CCF_NONLINEAR_PENCIL": "1", "CCF_NS_EIGEN": "0", "CCF_OZAKI": "0"}, marks)

    def err(a, b, k):
        return max(np.abs(a[f"{c}{k}"] - b[f"{c}{k}"]).max() / np.abs(b[f"{c}{k}"]).max() for c in "lg")

    print(f"{SIZE}^3 ({bench_name()}), relative max-norm difference of omega = (lambda, gamma) after k steps")
    print("step   production vs DMMA   production vs reference-algorithm (ADI)   DMMA vs reference-algorithm   max|lambda|")
    for k in marks:
        print(f"{k:4d}   {err(prod, dmma, k):.3e}            {err(prod, refa, k):.3e}                                "
              f"{err(dmma, refa, k):.3e}                     {np.abs(prod[f'l{k}']).max():.3e}", flush=True)


if __name__ == "__main__":
    main()
