"""The reference's known-answer cases for the per-mode solver API (proj/tests/test_solvers.cpp:38-105), shared by
the oracle pins (tests/test_oracle_modal.py) and the GPU parity tests (tests/test_gpu_modal.py).

Matrices are (n, m) numpy arrays a[k, j] = X(j, k), i.e. the memory of the reference's column-major m x n
Eigen::MatrixXcd (and of one CoeffTensor slice)."""
import numpy as np


def modal_rhs(O, g):
    """test_solvers.cpp:13-17: F = R2 g C02^T."""
    n, m = g.shape
    r2, c02 = O.operator_dense(m, "r2"), O.operator_dense(n, "c02")
    return np.ascontiguousarray((r2 @ g.T @ c02.T).T)


def manufactured(m, n, s, wall=0.0):
    """u = wall + (1 - r^2)(1 - z^2) and g = u - s lap u (test_solvers.cpp:46-66, 84-105)."""
    q = [0.5, 0.0, -0.5]
    u = np.zeros((n, m), complex)
    lap = np.zeros((n, m), complex)
    for j in range(3):
        for k in range(3):
            u[k, j] += q[j] * q[k]
    u[0, 0] += wall
    for k in range(3):
        lap[k, 0] += -4.0 * q[k]
    for j in range(3):
        lap[0, j] += -2.0 * q[j]
    return u, u - s * lap


def mass_pair(m, n):
    """test_solvers.cpp:68-82: data already satisfying the boundary conditions."""
    g = np.zeros((n, m), complex)
    g[0, 0], g[0, 2], g[2, 0], g[2, 2] = 0.25, -0.25, -0.25, 0.25
    return g


def unit_lift(m, n, p=4):
    """test_solvers.cpp:89-91: lift == 1 (zero mode, T0 T0) satisfies the wall data."""
    lift = np.zeros((p, n, m), complex)
    lift[p // 2, 0, 0] = 1.0
    return lift


def random_rhs(m, n, seed, rho=0.8):
    rng = np.random.default_rng(seed)
    j, k = np.arange(m)[None, :], np.arange(n)[:, None]
    return (rng.standard_normal((n, m)) + 1j * rng.standard_normal((n, m))) * rho ** (j + k)
