"""FP64 products on the INT8 tensor cores (csrc/ozaki.cu, tcgen05.mma kind::i8 with TMEM accumulators,
Ozaki splitting into six 8-bit digits) against long-double host products (tools/cpp/oz_check.cpp),
and the NS step at the benchmark configuration with the four product stages on the INT8 path
(csrc/ozpipe.cu, default at m = n = 256) against the FP64 DMMA GEMMs (CCF_OZAKI=0)."""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OZ = os.path.join(ROOT, "tools", "cpp", "oz_check")


@pytest.mark.parametrize("shape,env", [
    ("128 128 128 1 1 0.9", {}),                 # one tile, K-major B with column scales
    ("127 127 127 4 1 0.95", {}),                # padded rows / reduction (the eigen sizes M = N = 127)
    ("128 256 128 8 3 0.9", {}),                 # multi-term tiles sharing column scales
    ("127 128 128 300 1 0.9", {}),               # several tiles per CTA (pair-buffer / column-scale rings)
    ("128 256 128 40 3 0.9", {"CCF_OZ_MN": "1"}),  # MN-major B, tile scales (the data operands of X1 / C)
    ("127 256 128 300 2 0.8", {"CCF_OZ_MN": "1"}),
])
def test_ozaki_gemm(P, shape, env):
    if not os.path.exists(OZ):
        import __graft_entry__
        __graft_entry__.build()
    r = subprocess.run([OZ, *shape.split()], capture_output=True, text=True, timeout=300, env=dict(os.environ, **env))
    print(r.stdout, r.stderr)
    m = re.search(r"max rel err ([0-9.e+-]+)", r.stdout)
    assert r.returncode == 0 and m and float(m.group(1)) < 1e-12, r.stdout


SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import bench, paper_2206_04827_b200 as P
cfg = bench.CONFIGS[256]
ctx = P.Context(256, 256, 256)
wl, wg, _ = bench.initial_vorticity(ctx, cfg, cfg["vmax"])
st = P.NSStepper(ctx, wl, wg, reynolds=cfg["reynolds"], h=cfg["h"], order=4)
st.step(8)
l, g = st.omega()
np.savez({out!r}, l=l, g=g)
"""


def test_ns256_ozaki_vs_dmma(tmp_path):
    res = {}
    for name, flag in (("oz", "1"), ("dmma", "0")):
        out = str(tmp_path / f"{name}.npz")
        r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, out=out)], capture_output=True, text=True,
                           timeout=900, env=dict(os.environ, CCF_OZAKI=flag))
        assert r.returncode == 0, r.stderr[-2000:]
        import numpy as np
        res[name] = np.load(out)
    import numpy as np
    for k in ("l", "g"):
        a, b = res["oz"][k], res["dmma"][k]
        e = float(np.abs(a - b).max() / np.abs(b).max())
        print(k, e)
        assert e < 1e-10
