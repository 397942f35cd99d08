"""Host-side partitioning for multi-GPU runs of the CCF NS step.

Every per-mode stage (Poisson / Helmholtz ADI, pt_synthesize, curl + decompose, derivatives,
divide_r) is independent across Fourier modes, so the half-spectrum slots are sharded across
ranks with |w| pairs kept together (Hermitian storage; quirk Q1 couples w with -w). The only
exchange is the theta pencil transpose around the pointwise cross product: forward the 6
(r,z)-value / theta-coefficient fields from mode-sharded to (k, jr)-pencil-sharded, back with 3.

Round 1 runs one replica per GPU (no collective on the data path); these functions are the
partition logic of the sharded path and are exercised by the gloo tests.
"""
from __future__ import annotations

import math


def adi_cost(w: int, J_poisson, J_helm) -> float:
    """Relative per-slot cost of one NS step: 1 Poisson + 2 Helmholtz solves (4 sub-problems each)."""
    return float(J_poisson(w) + 2 * J_helm(w))


def mode_partition(p: int, world: int, cost=None):
    """Greedy longest-processing-time assignment of the p/2+1 half-spectrum slots to ranks.

    Returns a list (per rank) of slot indices; slot p/2 is the Nyquist slice. Balances the
    per-slot cost (default: the Poisson J model ~ log(16 gamma) growth at low |w|)."""
    nslots = p // 2 + 1
    if cost is None:
        def cost(s):
            w = p // 2 if s == p // 2 else s
            return 1.0 + 0.5 / (1.0 + w)  # low |w| Poisson solves need up to ~1.5x the iterations
    order = sorted(range(nslots), key=lambda s: -cost(s))
    loads = [0.0] * world
    parts = [[] for _ in range(world)]
    for s in order:
        r = min(range(world), key=lambda i: (loads[i], i))
        parts[r].append(s)
        loads[r] += cost(s)
    return [sorted(x) for x in parts]


def pencil_partition(n: int, mh: int, world: int):
    """Contiguous blocks of (k, jr) theta pencils per rank for the transpose: [(start, stop)) over n*mh."""
    total = n * mh
    base = total // world
    rem = total % world
    out, start = [], 0
    for r in range(world):
        cnt = base + (1 if r < rem else 0)
        out.append((start, start + cnt))
        start += cnt
    return out


def alltoall_bytes_per_rank(m: int, n: int, p: int, world: int, fields: int = 9) -> float:
    """Egress per rank of the theta transpose: fields x 8N x (G-1)/G^2."""
    N = m * n * p
    return fields * 8.0 * N * (world - 1) / (world * world)
