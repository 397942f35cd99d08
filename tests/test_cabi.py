"""C-ABI surface checks (no GPU needed): the product library loads, exports every symbol that
include/ccf.h declares, its host setup numerics agree with the oracle, and compute entry points
fail loudly (no CPU fallback) when no GPU is present."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "ccf.h")).read()
    return sorted(set(re.findall(r"\b(ccf_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols(P):
    import ctypes
    lib = ctypes.CDLL(P.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), f"libccf.so does not export {s}"
    assert set(P.EXPORTS) <= set(syms)
    assert b"sm_100a" in P.lib().ccf_version()


def test_library_is_sm100a(P):
    out = os.popen(f"cuobjdump -lelf {P.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out


def test_plans_match_oracle(P, O):
    # identical shift plans make parity reduce to ADI rounding
    for (m, w, scale, poisson) in [(16, 0, 1.0, True), (32, 5, 1.0, True), (64, 0, 4.8e-3, False),
                                   (128, 64, 1.0, True), (128, 1, 4.8e-7, False)]:
        a = P.plan_host(m, m, w, scale, poisson)
        b = O.modal_plan(m, m, w, scale, int(poisson))
        assert a["J"] == b["J"]
        for k in "abcd":
            assert abs(a[k] - b[k]) <= 1e-9 * max(1.0, abs(b[k]))
        assert np.allclose(a["u"], b["u"], rtol=1e-9) and np.allclose(a["v"], b["v"], rtol=1e-9)


def test_plan_errors_mirror_reference(P):
    with pytest.raises(P.DomainError):
        P.plan_host(15, 16, 0)  # odd m is outside the B200 path (documented)
    with pytest.raises(P.DomainError):
        P.plan_host(16, 16, 0, tol=2.0)  # compute_shifts: tol in (0,1)


def test_no_cpu_fallback_without_gpu(P):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(P.CCFError):
        P.Context(16, 16, 16)


@pytest.mark.parametrize("m,w,scale,poisson", [(16, 0, 1.0, True), (32, 3, 1.0, True), (64, 7, 4.8e-7, False),
                                               (128, 0, 1.0, True), (128, 64, 5e-7, False), (256, 0, 1.0, True),
                                               (256, 1, 5e-7, False), (256, 128, 1.0, True)])
def test_fast_diagonalization_residual(P, m, w, scale, poisson):
    """Host-only pin of the default modal solver (fast diagonalization, diag.hpp): the packed
    matrices applied in double give a Sylvester residual far below the reference's ADI tolerance
    (1e-12, adi.cpp:188-192) on random right-hand sides, for both k-parities."""
    for k0 in (0, 1):
        assert P.diag_host_check(m, m, w, scale, poisson, k0, seed=3) < 2e-13


def test_fast_diagonalization_residual_beyond_the_adi_tile(P):
    # config 5 size (m = n = 512): no ADI data is needed, the diagonalization stays exact
    assert P.diag_host_check(512, 512, 0, 1.0, True, 0, 1) < 1e-12
