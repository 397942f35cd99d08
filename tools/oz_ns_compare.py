"""NS steps at the benchmark configuration with the INT8 (Ozaki) product stages vs the FP64 DMMA
GEMMs (CCF_OZAKI=0), each in its own process: max-norm relative difference of omega per step count,
and steps/s of both. Usage: python tools/oz_ns_compare.py [steps] [size]"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import sys, time, numpy as np, torch
sys.path.insert(0, {root!r})
import bench, paper_2206_04827_b200 as P
cfg = bench.CONFIGS[{size}]
ctx = P.Context({size}, {size}, {size})
wl, wg, _ = bench.initial_vorticity(ctx, cfg, cfg["vmax"])
st = P.NSStepper(ctx, wl, wg, reynolds=cfg["reynolds"], h=cfg["h"], order=4)
out = {{}}
done = 0
for k in {checkpoints}:
    st.step(k - done); done = k
    l, g = st.omega()
    out["l%d" % k] = l; out["g%d" % k] = g
torch.cuda.synchronize()
t0 = time.perf_counter(); st.step(30); torch.cuda.synchronize(); out["sps"] = 30 / (time.perf_counter() - t0)
prof = st.profile_step()
print("stages", {{k: round(v, 4) for k, v in prof.items()}})
np.savez({out!r}, **out)
"""


def run(env, name, steps, size):
    out = f"/tmp/ozcmp_{name}.npz"
    if os.path.exists(out):
        os.remove(out)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, size=size, checkpoints=steps, out=out)],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=1200)
    print(name, r.stdout.strip()[-600:], r.stderr.strip()[-1500:] if r.returncode else "")
    if r.returncode:
        raise SystemExit(f"{name} run failed")
    return np.load(out)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    size = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    steps = sorted({1, 2, 3, 5, 10, n})
    a = run({"CCF_OZAKI": "1", "CCF_OZ_STAGES": os.environ.get("CCF_OZ_STAGES", "7")}, "oz", steps, size)
    b = run({"CCF_OZAKI": "0"}, "dmma", steps, size)
    for k in steps:
        e = max(np.abs(a[f"l{k}"] - b[f"l{k}"]).max() / np.abs(b[f"l{k}"]).max(),
                np.abs(a[f"g{k}"] - b[f"g{k}"]).max() / np.abs(b[f"g{k}"]).max())
        print(f"step {k:3d}: max rel diff ozaki vs dmma {e:.3e}")
    print(f"steps/s: ozaki {float(a['sps']):.1f}  dmma {float(b['sps']):.1f}")


if __name__ == "__main__":
    main()
