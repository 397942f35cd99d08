"""Seeded synthetic inputs shared by tests and bench.py.

Hermitian, parity-projected coefficient tensors in the reference layout
(complex128, shape (p, n, m), slice l carries wavenumber w = l - p/2):
  w > 0 : Re, Im ~ N(0,1) * rho^(j+k+|w|) ;  w = 0 : Re only ;  w < 0 : conjugate mirror ;
  Nyquist slice (l = 0) = 0 ; then parity projection (keep (j+w) even for scalars).
"""
import numpy as np


def hermitian_coeffs(m, n, p, rho, seed, parity=0, nyquist_zero=True):
    rng = np.random.default_rng(seed)
    c = np.zeros((p, n, m), np.complex128)
    j = np.arange(m)[None, :]
    k = np.arange(n)[:, None]
    half = p // 2
    for w in range(0, half):
        decay = rho ** (j + k + w)
        re = rng.standard_normal((n, m)) * decay
        im = rng.standard_normal((n, m)) * decay if w > 0 else np.zeros((n, m))
        c[half + w] = re + 1j * im
        if w > 0:
            c[half - w] = np.conj(c[half + w])
    if not nyquist_zero:
        c[0] = rng.standard_normal((n, m)) * rho ** (j + k + half)
    for l in range(p):
        w = l - half
        bad = ((np.arange(m) + w) % 2) != parity
        c[l][:, bad] = 0.0
    return c


def rel_err(a, b):
    """max-norm relative coefficient error |a - b|_max / max(|b|_max, tiny)."""
    den = np.max(np.abs(b))
    return float(np.max(np.abs(a - b)) / (den if den > 0 else 1.0))
