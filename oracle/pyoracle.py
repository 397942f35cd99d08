"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper around oracle/lib/liboracle.so (the C++ restatement of the
reference `cylspec` hot path, see oracle/oracle.hpp). Only tests/,
__graft_entry__.smoke() (as the checker) and bench.py's cpu_baseline /
--impl reference leg may import this module. The product package never does.

The generalized-eigenvalue step the reference delegates to Eigen's QZ
(proj/src/adi.cpp:26-27) is supplied here by LAPACK ggev through
scipy.linalg.eigvals(A, C, homogeneous_eigvals=True).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "lib", "liboracle.so")
_lib = None
_eig_cb = None  # keep the callback alive

EIGCB = C.CFUNCTYPE(C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                    C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double))

STATUS = {0: "ok", 1: "DomainError", 2: "ConfigError", 3: "SingularOperatorError",
          4: "NonConvergenceError", 5: "NotIncompressibleError", 6: "NumericalError", 9: "Error"}


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.kind = STATUS.get(status, str(status))


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (g++ only; no external deps)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _eig_provider(n, A, Cm, ar, ai, be):
    try:
        import scipy.linalg as sl
        a = np.ctypeslib.as_array(A, shape=(n * n,)).reshape(n, n, order="F").copy()
        c = np.ctypeslib.as_array(Cm, shape=(n * n,)).reshape(n, n, order="F").copy()
        w = sl.eigvals(a, c, homogeneous_eigvals=True)
        alpha, beta = w[0], w[1]
        # LAPACK ggev returns real beta >= 0 for real pencils; normalise any phase into alpha.
        ph = np.where(np.abs(beta) > 0, beta / np.where(np.abs(beta) > 0, np.abs(beta), 1), 1)
        alpha = alpha / ph
        beta = np.abs(beta)
        for i in range(n):
            ar[i] = float(alpha[i].real)
            ai[i] = float(alpha[i].imag)
            be[i] = float(beta[i].real)
        return 0
    except Exception:  # pragma: no cover - surfaced as NumericalError by the oracle
        return 1


def lib():
    global _lib, _eig_cb
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        dp = C.POINTER(C.c_double)
        for name in ["orc_analyze", "orc_synthesize", "orc_calculus", "orc_parity_project", "orc_poisson3d",
                     "orc_hpoisson", "orc_pt_synthesize", "orc_pt_decompose", "orc_curl_vector", "orc_divergence",
                     "orc_curl_pt", "orc_velocity_from_vorticity", "orc_nonlinear", "orc_helmholtz_step",
                     "orc_ns_step", "orc_ns_get", "orc_heat_step", "orc_heat_get", "orc_compute_shifts",
                     "orc_modal_plan", "orc_pencil_range", "orc_adi_vs_dense", "orc_operator_dense",
                     "orc_pencil_dense", "orc_jacobi", "orc_mobius_from_points", "orc_points", "orc_evaluate_at",
                     "orc_ns_step_sample", "orc_modal_solve", "orc_modal_apply", "orc_modal_helmholtz",
                     "orc_helmholtz_step_lifted"]:
            getattr(L, name).restype = C.c_int
        L.orc_last_error.restype = C.c_char_p
        L.orc_ns_create.restype = C.c_void_p
        L.orc_heat_create.restype = C.c_void_p
        L.orc_elliptic_K.restype = C.c_double
        L.orc_hermitian_error.restype = C.c_double
        L.orc_crc32.restype = C.c_uint32
        L.orc_ns_step.argtypes = [C.c_void_p, C.c_int]
        L.orc_ns_get.argtypes = [C.c_void_p, dp, dp, dp, C.POINTER(C.c_int)]
        L.orc_ns_destroy.argtypes = [C.c_void_p]
        pp = C.POINTER(C.c_void_p)
        L.orc_ns_seed.restype = C.c_int
        L.orc_ns_seed.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, pp, pp, C.c_int, pp, pp, C.c_double,
                                  C.c_int]
        L.orc_ns_run.restype = C.c_int
        L.orc_heat_step.argtypes = [C.c_void_p, dp]
        L.orc_heat_get.argtypes = [C.c_void_p, dp, dp, C.POINTER(C.c_int)]
        L.orc_heat_destroy.argtypes = [C.c_void_p]
        _eig_cb = EIGCB(_eig_provider)
        L.orc_set_eig_provider(_eig_cb)
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def _chk(st):
    if st != 0:
        raise OracleError(st, lib().orc_last_error().decode())


def _cz(t):
    """complex128 tensor (p, n, m) C-contiguous."""
    return np.ascontiguousarray(t, dtype=np.complex128)


def set_threads(n: int):
    lib().orc_set_threads(int(n))


# ---------------------------------------------------------------- grid / transforms
def chebyshev_points(count):
    out = np.zeros(count)
    _chk(lib().orc_points(0, count, _p(out)))
    return out


def fourier_points(count):
    out = np.zeros(count)
    _chk(lib().orc_points(1, count, _p(out)))
    return out


def analyze(vals):
    """vals: float64 (p, n, m) -> complex128 (p, n, m)  (proj/src/transform.cpp:122-165)"""
    v = np.ascontiguousarray(vals, dtype=np.float64)
    p, n, m = v.shape
    out = np.zeros((p, n, m), np.complex128)
    _chk(lib().orc_analyze(m, n, p, _p(v), _p(out)))
    return out


def synthesize(coef):
    c = _cz(coef)
    p, n, m = c.shape
    out = np.zeros((p, n, m))
    _chk(lib().orc_synthesize(m, n, p, _p(c), _p(out)))
    return out


def evaluate_at(coef, r, z, th):
    c = _cz(coef)
    p, n, m = c.shape
    out = np.zeros(2)
    _chk(lib().orc_evaluate_at(m, n, p, _p(c), C.c_double(r), C.c_double(z), C.c_double(th), _p(out)))
    return complex(out[0], out[1])


_CALC = {"dr": 0, "dz": 1, "dtheta": 2, "multiply_r": 3, "divide_r": 4, "hlap": 5, "lap": 6}


def calculus(op, coef):
    c = _cz(coef)
    p, n, m = c.shape
    out = np.zeros_like(c)
    _chk(lib().orc_calculus(_CALC[op], m, n, p, _p(c), _p(out)))
    return out


def parity_project(coef, parity=0):
    c = _cz(coef).copy()
    p, n, m = c.shape
    _chk(lib().orc_parity_project(m, n, p, int(parity), _p(c)))
    return c


def hermitian_error(coef):
    c = _cz(coef)
    p, n, m = c.shape
    return lib().orc_hermitian_error(m, n, p, _p(c))


# ---------------------------------------------------------------- solvers
def poisson3d(f, tol=1e-12, lift=None):
    c = _cz(f)
    p, n, m = c.shape
    out = np.zeros_like(c)
    lf = _cz(lift) if lift is not None else None
    _chk(lib().orc_poisson3d(m, n, p, C.c_double(tol), _p(c), _p(lf), _p(out)))
    return out


def hpoisson(rhs):
    c = _cz(rhs)
    p, n, m = c.shape
    out = np.zeros_like(c)
    _chk(lib().orc_hpoisson(m, n, p, _p(c), _p(out)))
    return out


def helmholtz_step(hist, order, diffusivity, h, tol=1e-12, forcing=None, lift=None):
    hs = [_cz(x) for x in hist]
    p, n, m = hs[0].shape
    arr = (C.POINTER(C.c_double) * len(hs))(*[_p(x) for x in hs])
    out = np.zeros_like(hs[0])
    fc = _cz(forcing) if forcing is not None else None
    if lift is not None:
        _chk(lib().orc_helmholtz_step_lifted(m, n, p, C.c_double(diffusivity), C.c_double(h), C.c_double(tol), int(order),
                                              len(hs), arr, _p(fc), _p(_cz(lift)), _p(out)))
        return out
    _chk(lib().orc_helmholtz_step(m, n, p, C.c_double(diffusivity), C.c_double(h), C.c_double(tol), int(order),
                                   len(hs), arr, _p(fc), _p(out)))
    return out


# ---------------------------------------------------------------- per-mode solver API (solvers.hpp:35-82)
def _cm(x):
    """(n, m) numpy view of an m x n column-major complex matrix: a[k, j] = X(j, k)."""
    return np.ascontiguousarray(x, dtype=np.complex128)


def modal_solve(f, w, scale=1.0, poisson=True, tol=1e-12):
    """ModalSolver(m, n, w, scale, poisson, tol).solve(f_full) -> (x, last_residual); f[k, j] = F(j, k)."""
    a = _cm(f)
    n, m = a.shape
    out = np.zeros_like(a)
    r = C.c_double()
    _chk(lib().orc_modal_solve(m, n, int(w), C.c_double(scale), int(bool(poisson)), C.c_double(tol), _p(a), _p(out),
                               C.byref(r)))
    return out, r.value


def modal_apply(x, w, scale=1.0, poisson=True):
    """ModalOperator::apply (A X B + C X D) of the Poisson / Helmholtz quadruple."""
    a = _cm(x)
    n, m = a.shape
    out = np.zeros_like(a)
    _chk(lib().orc_modal_apply(m, n, int(w), C.c_double(scale), int(bool(poisson)), _p(a), _p(out)))
    return out


def modal_helmholtz(f, w, scale, tol=1e-12, lift=None):
    """solve_modal_helmholtz(assemble_modal_helmholtz(m, n, w, scale), f, bc, tol); lift: (p, n, m) tensor."""
    a = _cm(f)
    n, m = a.shape
    out = np.zeros_like(a)
    lf = _cz(lift) if lift is not None else None
    _chk(lib().orc_modal_helmholtz(m, n, int(w), C.c_double(scale), C.c_double(tol), _p(a),
                                   lf.shape[0] if lf is not None else 0, _p(lf), _p(out)))
    return out


# ---------------------------------------------------------------- PT / NS
def pt_synthesize(lam, gam):
    l, g = _cz(lam), _cz(gam)
    p, n, m = l.shape
    o = [np.zeros_like(l) for _ in range(3)]
    _chk(lib().orc_pt_synthesize(m, n, p, _p(l), _p(g), _p(o[0]), _p(o[1]), _p(o[2])))
    return tuple(o)


def pt_decompose(vr, vt, vz, check=False):
    a, b, c = _cz(vr), _cz(vt), _cz(vz)
    p, n, m = a.shape
    ol, og = np.zeros_like(a), np.zeros_like(a)
    _chk(lib().orc_pt_decompose(m, n, p, _p(a), _p(b), _p(c), int(check), _p(ol), _p(og)))
    return ol, og


def curl_vector(vr, vt, vz):
    a, b, c = _cz(vr), _cz(vt), _cz(vz)
    p, n, m = a.shape
    o = [np.zeros_like(a) for _ in range(3)]
    _chk(lib().orc_curl_vector(m, n, p, _p(a), _p(b), _p(c), _p(o[0]), _p(o[1]), _p(o[2])))
    return tuple(o)


def divergence(vr, vt, vz):
    a, b, c = _cz(vr), _cz(vt), _cz(vz)
    p, n, m = a.shape
    o = np.zeros_like(a)
    _chk(lib().orc_divergence(m, n, p, _p(a), _p(b), _p(c), _p(o)))
    return o


def curl_pt(lam, gam):
    l, g = _cz(lam), _cz(gam)
    p, n, m = l.shape
    ol, og = np.zeros_like(l), np.zeros_like(l)
    _chk(lib().orc_curl_pt(m, n, p, _p(l), _p(g), _p(ol), _p(og)))
    return ol, og


def velocity_from_vorticity(wl, wg, tol=1e-12):
    a, b = _cz(wl), _cz(wg)
    p, n, m = a.shape
    ol, og = np.zeros_like(a), np.zeros_like(a)
    _chk(lib().orc_velocity_from_vorticity(m, n, p, C.c_double(tol), _p(a), _p(b), _p(ol), _p(og)))
    return ol, og


def nonlinear(vl, vg, wl, wg, dealias=False):
    a, b, c, d = _cz(vl), _cz(vg), _cz(wl), _cz(wg)
    p, n, m = a.shape
    ol, og = np.zeros_like(a), np.zeros_like(a)
    _chk(lib().orc_nonlinear(m, n, p, _p(a), _p(b), _p(c), _p(d), int(dealias), _p(ol), _p(og)))
    return ol, og


class NSStepper:
    """proj/src/ptns.cpp:177-267 NSStepper (ramp bootstrap)."""

    def __init__(self, lam0, gam0, reynolds, h, order=4, tol=1e-12, disable_nonlinear=False, dealias=False):
        l, g = _cz(lam0), _cz(gam0)
        self.shape = l.shape
        p, n, m = l.shape
        self.h = lib().orc_ns_create(m, n, p, C.c_double(reynolds), C.c_double(h), int(order), C.c_double(tol),
                                     int(bool(disable_nonlinear)) | (2 if dealias else 0), _p(l), _p(g))
        if not self.h:
            raise OracleError(9, lib().orc_last_error().decode())

    def step(self, n=1):
        _chk(lib().orc_ns_step(self.h, int(n)))

    def seed(self, omega_hist, nonlinear_hist, time, steps_taken):
        """NSStepper::seed (ptns.cpp:195-203): lists of (lambda, gamma) pairs, newest first."""
        p, n, m = self.shape
        rows = [[_cz(x) for x in pair] for pair in list(omega_hist) + list(nonlinear_hist)]
        no, nn = len(omega_hist), len(nonlinear_hist)
        vp = C.c_void_p

        def arr(rs, j):
            return (vp * max(len(rs), 1))(*[C.cast(_p(r[j]), vp) for r in rs])

        _chk(lib().orc_ns_seed(self.h, m, n, p, no, arr(rows[:no], 0), arr(rows[:no], 1), nn, arr(rows[no:], 0),
                               arr(rows[no:], 1), C.c_double(time), int(steps_taken)))

    def omega(self):
        l, g = np.zeros(self.shape, np.complex128), np.zeros(self.shape, np.complex128)
        t = C.c_double()
        s = C.c_int()
        _chk(lib().orc_ns_get(self.h, _p(l), _p(g), C.byref(t), C.byref(s)))
        self.time, self.steps_taken = t.value, s.value
        return l, g

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_ns_destroy(self.h)
            self.h = None


def ns_run(lam0, gam0, steps, reynolds, h, order=4, tol=1e-12, disable_nonlinear=False, dealias=False,
           bootstrap="ramp"):
    """proj/src/ptns.cpp:269-324 ns_run -> (lambda, gamma, final_time)."""
    l0, g0 = _cz(lam0), _cz(gam0)
    p, n, m = l0.shape
    l, g = np.zeros(l0.shape, np.complex128), np.zeros(l0.shape, np.complex128)
    t = C.c_double()
    flags = int(bool(disable_nonlinear)) | (2 if dealias else 0) | (4 if bootstrap == "substeps" else 0)
    _chk(lib().orc_ns_run(m, n, p, C.c_double(reynolds), C.c_double(h), int(order), C.c_double(tol), flags, _p(l0),
                          _p(g0), int(steps), _p(l), _p(g), C.byref(t)))
    return l, g, t.value


class HeatStepper:
    """proj/src/timestep.cpp:110-144 HeatStepper."""

    def __init__(self, coef0, alpha, h, order=4, tol=1e-12):
        c = _cz(coef0)
        self.shape = c.shape
        p, n, m = c.shape
        self.h = lib().orc_heat_create(m, n, p, C.c_double(alpha), C.c_double(h), int(order), C.c_double(tol), _p(c))
        if not self.h:
            raise OracleError(9, lib().orc_last_error().decode())

    def step(self, forcing=None):
        f = _cz(forcing) if forcing is not None else None
        _chk(lib().orc_heat_step(self.h, _p(f)))

    def current(self):
        c = np.zeros(self.shape, np.complex128)
        t = C.c_double()
        o = C.c_int()
        _chk(lib().orc_heat_get(self.h, _p(c), C.byref(t), C.byref(o)))
        return c, t.value, o.value

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_heat_destroy(self.h)
            self.h = None


# ---------------------------------------------------------------- ADI / plans / special
def compute_shifts(a, b, c, d, tol):
    info = np.zeros(8)
    u = np.zeros(256)
    v = np.zeros(256)
    _chk(lib().orc_compute_shifts(C.c_double(a), C.c_double(b), C.c_double(c), C.c_double(d), C.c_double(tol),
                                  _p(info), _p(u), _p(v), 256))
    J = int(info[7])
    return dict(a=info[0], b=info[1], c=info[2], d=info[3], gamma=info[4], alpha=info[5], modulus=info[6], J=J,
                u=u[:J].copy(), v=v[:J].copy())


def modal_plan(m, n, w, scale, poisson, tol=1e-12):
    info = np.zeros(8)
    u = np.zeros(256)
    v = np.zeros(256)
    _chk(lib().orc_modal_plan(m, n, w, C.c_double(scale), int(poisson), C.c_double(tol), _p(info), _p(u), _p(v), 256))
    J = int(info[7])
    return dict(a=info[0], b=info[1], c=info[2], d=info[3], gamma=info[4], alpha=info[5], modulus=info[6], J=J,
                u=u[:J].copy(), v=v[:J].copy())


def pencil_range(kind, size, w=0):
    out = np.zeros(2)
    _chk(lib().orc_pencil_range(int(kind), size, w, _p(out)))
    return out[0], out[1]


def pencil_dense(kind, size, w=0):
    k = size - 2
    A = np.zeros(k * k)
    Cm = np.zeros(k * k)
    _chk(lib().orc_pencil_dense(int(kind), size, w, _p(A), _p(Cm)))
    return A.reshape(k, k, order="F"), Cm.reshape(k, k, order="F")


def adi_vs_dense(m, n, w, scale, seed, tol=1e-12):
    rel = C.c_double()
    res = C.c_double()
    it = C.c_int()
    _chk(lib().orc_adi_vs_dense(m, n, w, C.c_double(scale), C.c_uint(seed), C.c_double(tol), C.byref(rel),
                                C.byref(res), C.byref(it)))
    return rel.value, res.value, it.value


_OPS = {"c01": 0, "c12": 1, "c02": 2, "r": 3, "r2": 4, "d1": 5, "d2": 6, "s": 7}


def operator_dense(n, which):
    cols = n - 2 if which == "s" else n
    out = np.zeros(n * cols)
    _chk(lib().orc_operator_dense(n, _OPS[which], _p(out)))
    return out.reshape(n, cols, order="F")


def elliptic_K(k):
    return lib().orc_elliptic_K(C.c_double(k))


def jacobi(u, k):
    out = np.zeros(3)
    _chk(lib().orc_jacobi(C.c_double(u), C.c_double(k), _p(out)))
    return tuple(out)


def adi_stats():
    s = C.c_long()
    it = C.c_long()
    r = C.c_int()
    w = C.c_double()
    lib().orc_adi_stats(C.byref(s), C.byref(it), C.byref(r), C.byref(w))
    return dict(solves=s.value, iterations=it.value, max_rounds=r.value, worst_residual=w.value)


def adi_stats_reset():
    lib().orc_adi_stats_reset()


def ns_step_sample(m, n, p, re, h, nsample=8, threads=1, seed=7):
    """Bounded CPU sample of one NS step (see orc_ns_step_sample in capi.cpp)."""
    out = np.zeros(6)
    _chk(lib().orc_ns_step_sample(m, n, p, C.c_double(re), C.c_double(h), int(nsample), int(threads), C.c_uint(seed),
                                  _p(out)))
    return dict(t_poisson=out[0], t_helmholtz=out[1], t_analyze=out[2], t_synthesize=out[3], J_poisson=out[4],
                J_helmholtz=out[5], nsample=nsample)


def crc32(b: bytes) -> int:
    buf = (C.c_uint8 * len(b)).from_buffer_copy(b)
    return lib().orc_crc32(buf, C.c_size_t(len(b)))
