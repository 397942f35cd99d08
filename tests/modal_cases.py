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


def eval_c2(coef, x):
    """sum_k coef[k] C^(2)_k(x) (Gegenbauer lambda = 2): C0 = 1, C1 = 4x, k C_k = 2(k+1) x C_{k-1} - (k+2) C_{k-2}."""
    c_prev, c_cur = np.ones_like(x), 4.0 * x
    acc = coef[0] * c_prev + (coef[1] * c_cur if len(coef) > 1 else 0.0)
    for k in range(2, len(coef)):
        c_prev, c_cur = c_cur, (2.0 * (k + 1) * x * c_cur - (k + 2) * c_prev) / k
        acc = acc + coef[k] * c_cur
    return acc


def operator_known_answers(apply, modal_rhs_fn):
    """test_ultraop.cpp:194-238 through a ModalOperator::apply implementation
    apply(x (n, m) array, w, scale, poisson) -> (n, m); returns the three residuals the reference checks."""
    # (1 - lap) 1 = 1 with the r^2 weight: the C2 x C2 series of the result evaluates to r^2 (:194-211)
    m = n = 8
    x = np.zeros((n, m), complex)
    x[0, 0] = 1.0
    y = apply(x, 0, 1.0, False).real
    rs, zs = np.linspace(-0.9, 0.9, 15), np.linspace(-0.8, 0.8, 5)
    vals = np.array([[sum(eval_c2(y[k], np.array(r)) * eval_c2(np.eye(n)[k], np.array(z)) for k in range(n))
                      for z in zs] for r in rs])
    e1 = np.abs(vals - rs[:, None] ** 2).max()
    # r^2 (d_rr + d_r / r - 1 / r^2) r = 0 (:213-222)
    x = np.zeros((6, 8), complex)
    x[0, 1] = 1.0
    e2 = np.abs(apply(x, 1, 1.0, True)).max()
    # lap (1 - r^2) = -4 (:224-238)
    x = np.zeros((8, 10), complex)
    x[0, 0], x[0, 2] = 0.5, -0.5
    f = np.zeros((8, 10), complex)
    f[0, 0] = -4.0
    e3 = np.abs(apply(x, 0, 1.0, True) - modal_rhs_fn(f)).max()
    return e1, e2, e3
