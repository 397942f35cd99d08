"""Oracle ultraspherical operators, special functions and ADI shift plans
(reference: proj/tests/test_ultraop.cpp, test_special.cpp, test_adi.cpp)."""
import math

import numpy as np
import pytest


def cheb_T(a, x):
    return np.polynomial.chebyshev.chebval(x, a)


def test_conversion_and_multiplication_entries(O):  # test_ultraop.cpp:74-132
    c01 = O.operator_dense(12, "c01")
    assert c01[0, 0] == 1.0 and c01[1, 1] == 0.5 and c01[0, 2] == -0.5 and c01[2, 2] == 0.5
    c12 = O.operator_dense(8, "c12")
    assert c12[0, 0] == 1.0 and abs(c12[2, 2] - 1 / 3) < 1e-16 and abs(c12[0, 2] + 1 / 3) < 1e-16
    assert abs(c12[7, 7] - 1 / 8) < 1e-16
    r = O.operator_dense(10, "r")
    assert abs(r[1, 0] - 0.25) < 1e-16 and abs(r[0, 1] - 2 / 3) < 1e-16
    assert abs(r[2, 1] - 1 / 3) < 1e-16 and abs(r[1, 2] - 5 / 8) < 1e-16
    d1, d2 = O.operator_dense(11, "d1"), O.operator_dense(11, "d2")
    assert d1[0, 1] == 1.0 and d1[9, 10] == 10.0 and d2[0, 2] == 4.0 and d2[8, 10] == 20.0


def test_c02_is_product(O):  # test_ultraop.cpp:163-168
    assert np.array_equal(O.operator_dense(14, "c02"), O.operator_dense(14, "c12") @ O.operator_dense(14, "c01"))


def test_recombination_vanishes_on_boundary(O):  # test_ultraop.cpp:240-250
    s = O.operator_dense(9, "s")
    y = np.random.default_rng(13).uniform(-1, 1, 7)
    a = s @ y
    assert abs(cheb_T(a, 1.0)) < 1e-13 and abs(cheb_T(a, -1.0)) < 1e-13


def test_elliptic_and_jacobi(O):  # test_special.cpp:35-75
    assert abs(O.elliptic_K(0.5) - 1.6857503548125961) < 1e-14 * 1.69
    assert abs(O.elliptic_K(0.0) - math.pi / 2) < 1e-15
    assert O.elliptic_K(1.0) < 0  # DomainError surfaced as -1
    for k in (0.2, 0.3, 0.6, 0.9):
        kp = math.sqrt(1 - k * k)
        assert abs(O.jacobi(O.elliptic_K(k), k)[2] - kp) < 1e-12
    k = 0.3
    mm = k * k
    for u in (0.05, 0.1, 0.2):
        u2 = u * u
        ser = 1 - mm * u2 / 2 + mm * (4 + mm) * u2 * u2 / 24 - mm * (16 + 44 * mm + mm * mm) * u2 ** 3 / 720
        assert abs(O.jacobi(u, k)[2] - ser) < 1e-8
    rng = np.random.default_rng(2024)
    for _ in range(20):
        k = rng.uniform(0.05, 0.95)
        u = rng.uniform(0.05, 0.95) * O.elliptic_K(k)
        sn, cn, dn = O.jacobi(u, k)
        assert abs(dn * dn + k * k * sn * sn - 1) < 1e-12 and abs(sn * sn + cn * cn - 1) < 1e-12


def test_shift_plan_quantities(O):  # test_adi.cpp:86-112
    p = O.compute_shifts(1.0, 2.0, 3.0, 4.0, 1e-8)
    assert abs(p["gamma"] - 4 / 3) < 1e-14
    g = p["gamma"]
    assert abs(p["alpha"] - (-1 + 2 * g + 2 * math.sqrt(g * g - g))) < 1e-14
    assert p["J"] == math.ceil(math.log(16 * g) * math.log(4 / 1e-8) / math.pi ** 2)
    sym = O.compute_shifts(-4.0, -2.0, 2.0, 4.0, 1e-12)
    assert np.allclose(sym["u"], -sym["v"], rtol=1e-11)
    assert np.all(sym["u"] >= -4 - 1e-9) and np.all(sym["u"] <= -2 + 1e-9)
    assert O.compute_shifts(-4, -2, 2, 4, 1e-12)["J"] > O.compute_shifts(-4, -2, 2, 4, 1e-1)["J"]
    with pytest.raises(O.OracleError):
        O.compute_shifts(0.0, 2.0, 1.0, 3.0, 1e-8)


def test_adi_matches_dense_oracle(O):  # test_adi.cpp:153-167 (9 seeded Helmholtz problems)
    checked = 0
    for m in (8, 16, 24):
        for seed in range(3):
            rel, res, it = O.adi_vs_dense(m, m, seed, 4.8e-3, seed + 10)
            assert rel < 1e-10 and res <= 1e-12
            checked += 1
    assert checked == 9


def test_adi_iteration_count_grows_like_log(O):  # test_adi.cpp:181-195
    ratios = [O.modal_plan(m, m, 0, 4.8e-3, 0)["J"] / math.log(m * m) for m in (8, 16, 32, 64)]
    assert max(ratios) / min(ratios) <= 2.0


def test_radial_enclosure_matches_known_values(O):
    # radial w=0 maximum ~ -j_{0,1}^2, vertical minimum ~ pi^2/4
    # (ranges are padded by 1e-8 max(1, hi - lo) + 1e-12 radius, adi.cpp:47)
    lo, hi = O.pencil_range(0, 64, 0)
    pad = 1e-8 * (hi - lo) + 1e-12 * abs(lo)
    assert abs(hi - pad + 5.783185962946) < 1e-6 * 5.8
    lo, hi = O.pencil_range(1, 64)
    pad = 1e-8 * (hi - lo) + 1e-12 * abs(hi)
    assert abs(lo + pad - math.pi ** 2 / 4) < 1e-6 * 2.5
