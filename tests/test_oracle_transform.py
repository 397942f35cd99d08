"""Oracle known answers for the CCF transforms (reference: proj/tests/test_transform.cpp)."""
import numpy as np
import pytest

from tests.conftest import sample


def test_analyze_simple_fields(O):  # test_transform.cpp:30-54
    m, n, p = 6, 5, 8
    zm = p // 2
    c = O.analyze(np.ones((p, n, m)))
    assert abs(c[zm, 0, 0] - 1) < 1e-14
    c[zm, 0, 0] = 0
    assert np.abs(c).max() < 1e-14
    cr = O.analyze(sample(O, m, n, p, lambda r, z, t: r))
    assert abs(cr[zm, 0, 1] - 1) < 1e-14
    cr[zm, 0, 1] = 0
    assert np.abs(cr).max() < 1e-14
    cz = O.analyze(sample(O, m, n, p, lambda r, z, t: z * z))
    assert abs(cz[zm, 0, 0] - 0.5) < 1e-14 and abs(cz[zm, 2, 0] - 0.5) < 1e-14
    cz[zm, 0, 0] = cz[zm, 2, 0] = 0
    assert np.abs(cz).max() < 1e-14


def test_analyze_rejects_nonfinite(O):  # test_transform.cpp:56-61
    f = np.zeros((4, 4, 4))
    f.flat[3] = np.nan
    with pytest.raises(O.OracleError) as e:
        O.analyze(f)
    assert e.value.kind == "NumericalError"


def test_synthesize_T1_is_r(O):  # test_transform.cpp:63-74
    m, n, p = 6, 5, 8
    c = np.zeros((p, n, m), complex)
    assert np.abs(O.synthesize(c)).max() == 0.0
    c[p // 2, 0, 1] = 1.0
    f = O.synthesize(c)
    R = sample(O, m, n, p, lambda r, z, t: r)
    assert np.allclose(f, R, rtol=1e-13, atol=1e-15)


def random_physical_field(O, m, n, p, seed):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-1, 1, 10)

    def f(r, z, t):
        x, y = r * np.cos(t), r * np.sin(t)
        return (c[0] + c[1] * x + c[2] * y + c[3] * z + c[4] * x * y + c[5] * x * z + c[6] * y * z +
                c[7] * (x * x - y * y) + c[8] * z * z + c[9] * x * y * z)
    return sample(O, m, n, p, f)


def test_round_trip_physical(O):  # test_transform.cpp:76-86
    for seed in range(5):
        f = random_physical_field(O, 16, 16, 16, seed)
        g = O.synthesize(O.analyze(f))
        assert np.abs(f - g).max() <= 1e-12 * max(1.0, np.abs(f).max())


def test_round_trip_hermitian_tensor(O):  # test_transform.cpp:88-110
    m = n = p = 8
    rng = np.random.default_rng(9)
    t = np.zeros((p, n, m), complex)
    half = p // 2
    for l in range(half, p):
        v = rng.uniform(-1, 1, (n, m)) + 1j * (0 if l == half else rng.uniform(-1, 1, (n, m)))
        t[l] = v
        lp = 2 * half - l
        if 0 <= lp < p:
            t[lp] = np.conj(v)
    t[0] = t[0].real
    back = O.analyze(O.synthesize(t))
    assert np.abs(back - t).max() < 1e-12 * max(1, np.abs(t).max())


def test_linearity_and_hermitian(O):  # test_transform.cpp:112-129
    f = random_physical_field(O, 8, 8, 8, 1)
    g = random_physical_field(O, 8, 8, 8, 2)
    lhs = O.analyze(0.7 * f - 1.3 * g)
    rhs = 0.7 * O.analyze(f) - 1.3 * O.analyze(g)
    assert np.abs(lhs - rhs).max() < 1e-13 * max(1, np.abs(lhs).max())
    assert O.hermitian_error(O.analyze(random_physical_field(O, 8, 6, 12, 3))) < 1e-14


def test_evaluate_at(O):  # test_transform.cpp:131-152
    m, n, p = 7, 6, 8
    f = random_physical_field(O, m, n, p, 4)
    c = O.analyze(f)
    s = O.synthesize(c)
    r, z, th = O.chebyshev_points(m), O.chebyshev_points(n), O.fourier_points(p)
    for (l, k, j) in [(0, 0, 0), (3, 2, 5), (7, 5, 6), (5, 1, 2)]:
        assert abs(O.evaluate_at(c, r[j], z[k], th[l]) - s[l, k, j]) < 1e-12
    crz = O.analyze(sample(O, 6, 6, 8, lambda r, z, t: r * z))
    assert abs(O.evaluate_at(crz, 0.3, -0.5, 1.0) - (-0.15)) < 1e-13


def test_fft_sizes_match_dense_dft(O):
    # the FFTW stand-in: mixed radix (2,3,4,5,7, generic <= 32) and Bluestein paths
    for L in [4, 5, 6, 16, 17, 32, 35, 64, 65, 128, 256]:
        x = np.random.default_rng(L).standard_normal((2, 4, L))
        # analyze in r of a single pencil equals the textbook DCT-I definition
        v = x[0, 0]
        N = L - 1
        k = np.arange(L)
        s = np.arange(L)
        X = v[::-1]  # descending
        Y = X[0] + (-1.0) ** k * X[-1] + 2 * (np.cos(np.pi * np.outer(k, s[1:-1]) / N) @ X[1:-1])
        coef = Y / N
        coef[0] *= 0.5
        coef[-1] *= 0.5
        # the full analyze also does z and theta; compare the r-coefficients of a z/theta-constant field
        f = np.broadcast_to(v, (2, 4, L)).copy()
        cf = O.analyze(f)
        assert np.allclose(cf[1, 0, :].real, coef, atol=1e-13 * max(1, np.abs(coef).max()))
