"""The batched FP64 GEMM launcher (GemmPlan: TMA / cp.async / register kernels) against a long-double
host product on random data (tools/cpp/gemm_check.cpp): aligned shapes of the 256^3 step, small
extents, K not a multiple of the 16-column TMA box, and blocks that do not start on a row of their
2-D view (these must fall back instead of reading zeros past the row end)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tools", "cpp", "gemm_check")

CASES = [
    "127 128 128 128 256 256 4", "127 128 128 128 256 256 4 128",  # z transforms at 256^3 (both halves)
    "128 256 128 128 256 256 3", "127 128 127 128 128 256 3",      # composite / back transform
    "127 8 128 128 16 8 4", "127 8 128 128 16 8 4 8",              # n = 16: half-row B blocks
    "127 7 8 8 8 8 4", "200 40 128 128 40 40 2", "255 256 256 256 512 512 2",  # K < 16, M > 128, 512^3
    "191 7 192 192 16 8 3 8", "127 60 100 128 128 64 2 64",
]


@pytest.mark.parametrize("args", CASES)
def test_gemm_launcher(args):
    if not os.path.exists(BIN):
        import __graft_entry__
        __graft_entry__.build()
    r = subprocess.run([BIN, *args.split()], capture_output=True, text=True, timeout=120)
    print(r.stdout.strip())
    assert r.returncode == 0, r.stdout + r.stderr
