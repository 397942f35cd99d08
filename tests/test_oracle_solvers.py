"""Oracle solver known answers (reference: proj/tests/test_solvers.cpp, test_timestep.cpp)."""
import math

import numpy as np
import pytest

from tests.conftest import sample


def test_poisson_zero_and_manufactured(O):  # test_solvers.cpp:107-129
    m, n, p = 14, 14, 8
    assert np.abs(O.poisson3d(np.zeros((p, n, m), complex))).max() == 0.0
    f = O.analyze(sample(O, m, n, p, lambda r, z, t: -4 * (1 - z * z) - 2 * (1 - r * r)))
    u = O.synthesize(O.poisson3d(f))
    ref = sample(O, m, n, p, lambda r, z, t: (1 - r * r) * (1 - z * z))
    assert np.abs(u - ref).max() < 1e-10


def test_poisson_theta_modes(O):  # test_solvers.cpp:131-146
    m, n, p = 16, 16, 8
    g = lambda r, z, t: (1 - r * r) * (1 - z * z) * (1 + 0.5 * r * np.cos(t))
    lap = lambda r, z, t: -4 * (1 + r * np.cos(t)) * (1 - z * z) - 2 * (1 - r * r) * (1 + 0.5 * r * np.cos(t))
    u = O.synthesize(O.poisson3d(O.analyze(sample(O, m, n, p, lap))))
    assert np.abs(u - sample(O, m, n, p, g)).max() < 1e-9


def test_poisson_linearity_and_decoupling(O):  # test_solvers.cpp:160-183
    m, n, p = 10, 10, 4
    c1 = O.analyze(sample(O, m, n, p, lambda r, z, t: r * r + z))
    c2 = O.analyze(sample(O, m, n, p, lambda r, z, t: np.cos(t) * r * (1 - z * z)))
    lhs = O.poisson3d(0.6 * c1 - 1.7 * c2)
    rhs = 0.6 * O.poisson3d(c1) - 1.7 * O.poisson3d(c2)
    assert np.abs(lhs - rhs).max() < 1e-12 * max(1, np.abs(lhs).max())
    m, n, p = 10, 10, 8
    f = np.zeros((p, n, m), complex)
    f[p // 2 + 1, 2, 1] = 0.3 - 0.1j
    f[p // 2 - 1, 2, 1] = 0.3 + 0.1j
    u = O.poisson3d(f)
    for l in range(p):
        if l not in (p // 2 + 1, p // 2 - 1):
            assert np.abs(u[l]).max() == 0.0


def test_horizontal_poisson(O):  # test_solvers.cpp:185-209
    m, n, p = 12, 8, 8
    u = O.synthesize(O.hpoisson(O.analyze(-np.ones((p, n, m)))))
    assert np.abs(u - sample(O, m, n, p, lambda r, z, t: (1 - r * r) / 4)).max() < 1e-11
    assert np.abs(O.hpoisson(np.zeros((p, n, m), complex))).max() == 0.0
    uz = O.hpoisson(O.analyze(sample(O, m, n, p, lambda r, z, t: np.cos(t) * r * (1 - r * r))))
    assert np.abs(uz[:, 1:, :]).max() < 1e-13


def test_spectral_accuracy_geometric_decay(O):  # test_solvers.cpp:211-238
    u_fn = lambda r, z, t: (1 - r * r) * (1 + 0.5 * r * np.cos(t)) * (1 - z * z) * np.exp(2 * z)

    def f_fn(r, z, t):
        sz = (1 - z * z) * np.exp(2 * z)
        szpp = np.exp(2 * z) * (2 - 8 * z - 4 * z * z)
        sr = (1 - r * r) * (1 + 0.5 * r * np.cos(t))
        return -4 * (1 + r * np.cos(t)) * sz + sr * szpp
    errs = []
    for mn in (8, 12, 16, 20, 24):
        u = O.synthesize(O.poisson3d(O.analyze(sample(O, mn, mn, 8, f_fn))))
        errs.append(np.abs(u - sample(O, mn, mn, 8, u_fn)).max())
    assert errs[-1] <= 1e-10
    for a, b in zip(errs, errs[1:]):
        assert b <= 0.5 * a or b <= 1e-10


def test_heat_bdf4_manufactured(O):  # test_timestep.cpp:151-187 (200 BDF4 steps, 15x15x16)
    m, n, p = 15, 15, 16
    ex = lambda t: (lambda r, z, th: np.exp(-t) * (1 - r * r) * (1 - z * z))
    lapf = lambda r, z: -4 * (1 - z * z) - 2 * (1 - r * r)
    frc = lambda t: (lambda r, z, th: -np.exp(-t) * (1 - r * r) * (1 - z * z) - np.exp(-t) * lapf(r, z))
    h = 0.01
    st = O.HeatStepper(O.analyze(sample(O, m, n, p, ex(0.0))), alpha=1.0, h=h, order=4)
    t = 0.0
    for _ in range(200):
        st.step(O.analyze(sample(O, m, n, p, frc(t + h))))  # exact forcing at t + h
        t += h
    c, tf, _ = st.current()
    got = O.synthesize(c)
    ref = sample(O, m, n, p, ex(tf))
    assert np.abs(got - ref).max() / np.abs(ref).max() <= 1e-4
