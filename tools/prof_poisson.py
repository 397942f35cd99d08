"""One 256^3 (or given size) Poisson solve through the C-ABI with device pointers (profiling target)."""
import sys, os, time, ctypes as C
sys.path.insert(0, os.path.join(os.path.dirname(__file__), '..'))
import torch
from tests.inputs import hermitian_coeffs
import paper_2206_04827_b200 as P
m = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
f = hermitian_coeffs(m, m, m, 0.9, 4)
ctx = P.Context(m, m, m)
fd = torch.from_numpy(f).cuda(); ud = torch.zeros_like(fd)
for _ in range(reps):
    t0 = time.perf_counter()
    ctx._check(P.lib().ccf_poisson3d(ctx.h, C.c_void_p(fd.data_ptr()), C.c_void_p(ud.data_ptr())))
    print(f"{(time.perf_counter()-t0)*1e3:.2f} ms", flush=True)
