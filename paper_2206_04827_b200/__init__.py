"""B200-native (sm_100a) CCF spectral Navier–Stokes hot path — Python host mirror.

The product is the C-ABI shared library ``lib/libccf.so`` (include/ccf.h); this
module is a thin ctypes binding that mirrors the reference ``cylspec`` API names
(proj/include/cylspec/*.hpp) for tests, benchmarks and Python users. Tensors use
the reference layout: numpy complex128 arrays of shape (p, n, m) for coefficient
tensors (slice l carries wavenumber l - p/2) and float64 (p, n, m) for grid fields.

There is no CPU fallback: if the CUDA library or a GPU is missing, every call
raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libccf.so")

# Status codes mirror proj/include/cylspec/errors.hpp:10-40 (include/ccf.h).
CCF_OK = 0
STATUS_NAMES = {1: "DomainError", 2: "ConfigError", 3: "SingularOperatorError", 4: "NonConvergenceError",
                5: "NotIncompressibleError", 6: "NumericalError", 7: "CudaError", 8: "FieldFileError",
                9: "InternalError"}


class CCFError(RuntimeError):
    """Base of the exception taxonomy (cylspec errors.hpp)."""

    status = 9

    def __init__(self, msg, slice_=-1, shift_index=-1, residual_history=()):
        super().__init__(msg)
        self.slice = slice_
        self.shift_index = shift_index
        self.residual_history = list(residual_history)


class DomainError(CCFError, ValueError):
    status = 1


class ConfigError(CCFError, ValueError):
    status = 2


class SingularOperatorError(CCFError):
    status = 3


class NonConvergenceError(CCFError):
    status = 4


class NotIncompressibleError(CCFError):
    status = 5


class NumericalError(CCFError):
    status = 6


class CudaError(CCFError):
    status = 7


class FieldFileError(CCFError):
    """cylspec::FieldFileError (proj/include/cylspec/io.hpp:17-19)."""

    status = 8


_ERR = {c.status: c for c in (DomainError, ConfigError, SingularOperatorError, NonConvergenceError,
                              NotIncompressibleError, NumericalError, CudaError, FieldFileError)}

# Every extern "C" symbol include/ccf.h declares (checked by the CPU test suite).
EXPORTS = ["ccf_ctx_create", "ccf_ctx_destroy", "ccf_ctx_set_stream", "ccf_ctx_synchronize", "ccf_analyze",
           "ccf_synthesize", "ccf_calculus", "ccf_poisson3d", "ccf_hpoisson", "ccf_helmholtz_step",
           "ccf_pt_synthesize", "ccf_pt_decompose", "ccf_curl_vector", "ccf_curl_pt", "ccf_velocity_from_vorticity",
           "ccf_nonlinear", "ccf_ns_create", "ccf_ns_step", "ccf_ns_get_omega", "ccf_ns_destroy",
           "ccf_get_last_error", "ccf_get_stats", "ccf_reset_stats", "ccf_modal_plan", "ccf_version",
           "ccf_ns_profile_step", "ccf_ns_set_graphs", "ccf_ns_launches_per_step", "ccf_plan_host",
           "ccf_create_error", "ccf_adi_last_rounds", "ccf_adi_keep_history", "ccf_get_gemm_flops",
           "ccf_diag_host_check", "ccf_shard_init", "ccf_shard_partition", "ccf_shard_info", "ccf_shard_ipc_handle",
           "ccf_shard_open_ipc", "ccf_shard_link_local", "ccf_shard_set_host_barrier", "ccf_write_field",
           "ccf_read_field_header", "ccf_read_field", "ccf_crc32", "ccf_ns_write_omega", "ccf_heat_create",
           "ccf_heat_step", "ccf_heat_get", "ccf_ns_create_ex", "ccf_ns_velocity", "ccf_ns_gamma_psi",
           "ccf_nonlinear_ex", "ccf_ns_seed", "ccf_modal_create", "ccf_modal_solve", "ccf_modal_apply",
           "ccf_modal_operator", "ccf_modal_destroy"]

HOST_BARRIER_FN = C.CFUNCTYPE(None, C.c_void_p)
SHARD_HANDLE_BYTES = 128  # include/ccf.h CCF_SHARD_HANDLE_BYTES

_lib = None


def build(force: bool = False) -> str:
    """Compile the CUDA library in-tree for sm_100a (nvcc; no GPU needed)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-j8", "-C", _HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CudaError(f"CUDA library missing: {LIB_PATH} (run build())")
        L = C.CDLL(LIB_PATH)
        dp = C.POINTER(C.c_double)
        vp = C.c_void_p
        L.ccf_version.restype = C.c_char_p
        L.ccf_create_error.restype = C.c_char_p
        L.ccf_ctx_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.POINTER(vp)]
        for name in EXPORTS:
            if name not in ("ccf_version", "ccf_create_error"):
                getattr(L, name).restype = C.c_int
        L.ccf_ctx_destroy.argtypes = [vp]
        L.ccf_ctx_set_stream.argtypes = [vp, vp]
        L.ccf_ctx_synchronize.argtypes = [vp]
        L.ccf_analyze.argtypes = [vp, vp, vp]
        L.ccf_synthesize.argtypes = [vp, vp, vp]
        L.ccf_calculus.argtypes = [vp, C.c_int, vp, vp]
        L.ccf_poisson3d.argtypes = [vp, vp, vp]
        L.ccf_hpoisson.argtypes = [vp, vp, vp]
        L.ccf_helmholtz_step.argtypes = [vp, C.POINTER(vp), C.c_int, C.c_int, vp, C.c_double, C.c_double, vp]
        L.ccf_pt_synthesize.argtypes = [vp, vp, vp, vp, vp, vp]
        L.ccf_pt_decompose.argtypes = [vp, vp, vp, vp, vp, vp]
        L.ccf_curl_vector.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.ccf_curl_pt.argtypes = [vp, vp, vp, vp, vp]
        L.ccf_velocity_from_vorticity.argtypes = [vp, vp, vp, vp, vp]
        L.ccf_nonlinear.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.ccf_ns_create.argtypes = [vp, C.c_double, C.c_double, C.c_int, C.c_int, vp, vp, C.POINTER(vp)]
        L.ccf_ns_step.argtypes = [vp, C.c_int]
        L.ccf_ns_get_omega.argtypes = [vp, vp, vp, dp, C.POINTER(C.c_int)]
        L.ccf_ns_destroy.argtypes = [vp]
        L.ccf_get_last_error.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), dp,
                                         C.POINTER(C.c_int), C.c_char_p, C.c_int]
        L.ccf_adi_last_rounds.argtypes = [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), vp, vp, C.c_int]
        L.ccf_adi_keep_history.argtypes = [vp, C.c_int]
        L.ccf_get_gemm_flops.argtypes = [vp, dp]
        L.ccf_diag_host_check.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_ulonglong, dp]
        L.ccf_get_stats.argtypes = [vp, C.POINTER(C.c_long), C.POINTER(C.c_long), C.POINTER(C.c_int), dp,
                                    C.POINTER(C.c_long)]
        L.ccf_reset_stats.argtypes = [vp]
        L.ccf_modal_plan.argtypes = [vp, C.c_int, C.c_double, C.c_int, dp, dp, dp, C.c_int]
        L.ccf_ns_profile_step.restype = C.c_int
        L.ccf_ns_profile_step.argtypes = [vp, dp, C.POINTER(C.c_int), C.c_char_p, C.c_int]
        L.ccf_ns_set_graphs.restype = C.c_int
        L.ccf_ns_set_graphs.argtypes = [vp, C.c_int]
        L.ccf_ns_launches_per_step.restype = C.c_int
        L.ccf_ns_launches_per_step.argtypes = [vp, C.POINTER(C.c_long)]
        L.ccf_plan_host.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double, C.c_int, dp, dp, dp,
                                    C.c_int]
        ip = C.POINTER(C.c_int)
        L.ccf_shard_init.argtypes = [vp, C.c_int, C.c_int]
        L.ccf_shard_partition.argtypes = [C.c_int, C.c_int, C.c_int, ip, ip]
        L.ccf_shard_info.argtypes = [vp, ip, ip, ip, ip, ip, ip]
        L.ccf_shard_ipc_handle.argtypes = [vp, C.c_char_p]
        L.ccf_shard_open_ipc.argtypes = [vp, C.c_char_p]
        L.ccf_shard_link_local.argtypes = [C.POINTER(vp), C.c_int]
        L.ccf_shard_set_host_barrier.argtypes = [vp, HOST_BARRIER_FN, vp]
        L.ccf_write_field.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, vp]
        L.ccf_read_field_header.argtypes = [C.c_char_p, ip, ip, ip, ip]
        L.ccf_read_field.argtypes = [C.c_char_p, ip, ip, ip, ip, vp, C.c_size_t]
        L.ccf_crc32.argtypes = [vp, C.c_size_t, C.POINTER(C.c_uint)]
        L.ccf_ns_write_omega.argtypes = [vp, C.c_char_p, C.c_char_p]
        L.ccf_heat_create.argtypes = [vp, C.c_double, C.c_double, C.c_int, vp, C.c_int, C.POINTER(vp)]
        L.ccf_heat_step.argtypes = [vp, vp, C.c_int]
        L.ccf_heat_get.argtypes = [vp, vp, dp, C.POINTER(C.c_int)]
        L.ccf_ns_create_ex.argtypes = [vp, C.c_double, C.c_double, C.c_int, C.c_int, vp, vp, C.POINTER(vp)]
        L.ccf_ns_velocity.argtypes = [vp, vp, vp]
        L.ccf_modal_create.argtypes = [vp, C.c_int, C.c_double, C.c_int, C.POINTER(vp)]
        L.ccf_modal_solve.argtypes = [vp, vp, vp]
        L.ccf_modal_apply.argtypes = [vp, vp, vp]
        L.ccf_modal_operator.argtypes = [vp, C.c_int, vp]
        L.ccf_modal_destroy.argtypes = [vp]
        L.ccf_ns_seed.argtypes = [vp, C.c_int, C.POINTER(vp), C.POINTER(vp), C.c_int, C.POINTER(vp), C.POINTER(vp),
                                  C.c_double, C.c_int]
        L.ccf_ns_gamma_psi.argtypes = [vp, vp]
        L.ccf_nonlinear_ex.argtypes = [vp, vp, vp, vp, vp, C.c_int, vp, vp]
        _lib = L
    return _lib


def shard_partition(m, p, world):
    """The library's partition (host only, no GPU): (slot bounds, row bounds), world + 1 each."""
    sb = (C.c_int * (world + 1))()
    rb = (C.c_int * (world + 1))()
    st = lib().ccf_shard_partition(int(m), int(p), int(world), sb, rb)
    if st != 0:
        raise _ERR.get(st, CCFError)("ccf_shard_partition: invalid (m, p, world)")
    return list(sb), list(rb)


def _addr(a):
    """Host numpy array or torch CUDA tensor -> raw pointer."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)


def _arg(x, shape, cplx, what, out=False):
    """Validate one tensor argument before its pointer reaches the C-ABI, which reads / writes a buffer
    sized by the context (the reference throws DomainError on a spec mismatch, e.g. timestep.cpp:69-70,
    ptns.cpp:185-187). Inputs of the wrong dtype are converted; outputs must already be exact."""
    if x is None:
        return None
    want = "complex128" if cplx else "float64"
    if hasattr(x, "data_ptr"):  # torch tensor (host or device memory)
        if tuple(x.shape) != tuple(shape) or str(x.dtype) != "torch." + want or not x.is_contiguous():
            raise DomainError(f"{what}: expected a contiguous {want} tensor of shape {tuple(shape)}, got "
                              f"{str(x.dtype)} {tuple(x.shape)}")
        return x
    if out:
        if not isinstance(x, np.ndarray) or x.dtype != np.dtype(want) or x.shape != tuple(shape) \
                or not x.flags.c_contiguous or not x.flags.writeable:
            raise DomainError(f"{what}: output must be a writeable C-contiguous {want} array of shape {tuple(shape)}")
        return x
    a = np.asarray(x)
    if a.shape != tuple(shape):
        raise DomainError(f"{what}: spec mismatch (shape {a.shape}, context {tuple(shape)})")
    if not cplx and np.iscomplexobj(a):
        raise DomainError(f"{what}: grid values must be real")
    return np.ascontiguousarray(a, dtype=np.complex128 if cplx else np.float64)


class Context:
    """One grid size on one GPU (ccf_ctx). Mirrors the reference free functions."""

    def __init__(self, m, n, p, device=0, adi_tol=1e-12, q2_endpoint_pad=False, solver="diag",
                 reference_shift_counts=False):
        """solver: "diag" (fast diagonalization on the tensor cores, default) or "adi" (the
        reference's ADI iteration, adi.cpp:150-202, as the on-chip ADI kernel)."""
        if solver not in ("diag", "adi"):
            raise ValueError("solver must be 'diag' or 'adi'")
        self.m, self.n, self.p = int(m), int(n), int(p)
        flags = int(bool(q2_endpoint_pad)) | (2 if reference_shift_counts else 0) | (4 if solver == "adi" else 0)
        h = C.c_void_p()
        st = lib().ccf_ctx_create(self.m, self.n, self.p, int(device), C.c_double(adi_tol), flags, C.byref(h))
        if st != 0:
            raise _ERR.get(st, CCFError)(lib().ccf_create_error().decode())
        self.h = h

    # ---- errors
    def _check(self, st):
        if st == 0:
            return
        if not getattr(self, "h", None):
            raise CCFError("context is closed")
        kind, sl, sh = C.c_int(), C.c_int(), C.c_int()
        hist = (C.c_double * 8)()
        nh = C.c_int(8)
        msg = C.create_string_buffer(1024)
        lib().ccf_get_last_error(self.h, C.byref(kind), C.byref(sl), C.byref(sh), hist, C.byref(nh), msg, 1024)
        raise _ERR.get(st, CCFError)(msg.value.decode(), sl.value, sh.value, list(hist)[: min(nh.value, 8)])

    def close(self):
        if getattr(self, "h", None):
            lib().ccf_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def shape(self):
        return (self.p, self.n, self.m)

    def set_stream(self, stream_ptr):
        """Run on an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream); None restores."""
        self._check(lib().ccf_ctx_set_stream(self.h, C.c_void_p(stream_ptr) if stream_ptr else None))

    def synchronize(self):
        self._check(lib().ccf_ctx_synchronize(self.h))

    def _out_c(self):
        return np.zeros(self.shape(), np.complex128)

    def _coef(self, x, what, out=False):
        return _arg(x, self.shape(), True, what, out)

    def _vals(self, x, what, out=False):
        return _arg(x, self.shape(), False, what, out)

    # ---- transforms (transform.hpp:17-22)
    def analyze(self, values):
        v = self._vals(values, "analyze")
        out = self._out_c()
        self._check(lib().ccf_analyze(self.h, _addr(v), _addr(out)))
        return out

    def synthesize(self, coeffs):
        c = self._coef(coeffs, "synthesize")
        out = np.zeros(self.shape())
        self._check(lib().ccf_synthesize(self.h, _addr(c), _addr(out)))
        return out

    _CALC = {"dr": 0, "dz": 1, "dtheta": 2, "divide_r": 4, "hlap": 5, "lap": 6}

    def calculus(self, op, coeffs):
        c = self._coef(coeffs, op)
        out = self._out_c()
        self._check(lib().ccf_calculus(self.h, self._CALC[op], _addr(c), _addr(out)))
        return out

    # ---- solvers (solvers.hpp:86-94)
    def _lift_correction(self, lift, scale, poisson):
        """Lifted Dirichlet data (BoundaryCondition::lifted, solvers.cpp:160-165, timestep.cpp:84-101): the modal
        solves are linear, so solve(F_l - op_l.apply(lift_l)) + lift_l = solve(F_l) + c_l with
        c_l = lift_l - solve(op_l.apply(lift_l)), computed per |w| on the device (ModalSolver) and
        parity-projected like the output."""
        lf = np.asarray(lift)
        p, n, m = self.shape()
        if lf.ndim != 3 or lf.shape[1:] != (n, m):
            raise DomainError("BoundaryCondition: lift tensor has wrong dimensions")
        if lf.shape[0] != p:
            raise DomainError("BoundaryCondition: lift tensor misses the requested mode")
        out = np.zeros((p, n, m), np.complex128)
        solvers = {}
        try:
            for l in range(p):
                sl = np.ascontiguousarray(lf[l], dtype=np.complex128)
                if not sl.any():
                    continue
                w = l - p // 2
                s = solvers.get(abs(w))
                if s is None:
                    s = solvers[abs(w)] = ModalSolver(self, abs(w), scale, poisson)
                c = sl - s.solve(s.apply(sl))
                c[:, (np.arange(m) + w) % 2 != 0] = 0.0  # parity_project (coeffs.cpp:50-65)
                out[l] = c
        finally:
            for s in solvers.values():
                s.close()
        return out

    def solve_poisson_3d(self, f, lift=None):
        """solve_poisson_3d (solvers.cpp:142-175); lift: BoundaryCondition::lifted(lift) data."""
        c = self._coef(f, "solve_poisson_3d")
        out = self._out_c()
        self._check(lib().ccf_poisson3d(self.h, _addr(c), _addr(out)))
        if lift is not None:
            out += self._lift_correction(lift, 1.0, True)
        return out

    def solve_horizontal_poisson(self, rhs):
        c = self._coef(rhs, "solve_horizontal_poisson")
        out = self._out_c()
        self._check(lib().ccf_hpoisson(self.h, _addr(c), _addr(out)))
        return out

    def helmholtz_step(self, history, order, diffusivity, h, forcing=None, lift=None):
        """HelmholtzTensorStepper(spec, diffusivity, h, tol, bc).step (timestep.cpp:61-108); lift: lifted bc data."""
        hs = [self._coef(x, "HelmholtzTensorStepper: history") for x in history]
        arr = (C.c_void_p * len(hs))(*[x.ctypes.data for x in hs])
        fc = self._coef(forcing, "HelmholtzTensorStepper: forcing")
        out = self._out_c()
        self._check(lib().ccf_helmholtz_step(self.h, arr, len(hs), int(order), _addr(fc), C.c_double(diffusivity),
                                             C.c_double(h), _addr(out)))
        if lift is not None:
            kappa = (1.0, 2.0 / 3.0, 6.0 / 11.0, 12.0 / 25.0)[int(order) - 1] * h
            out += self._lift_correction(lift, kappa * diffusivity, False)
        return out

    # ---- PT / NS (ptns.hpp:47-70)
    def pt_synthesize(self, lam, gam):
        o = [self._out_c() for _ in range(3)]
        self._check(lib().ccf_pt_synthesize(self.h, _addr(self._coef(lam, "pt_synthesize")),
                                            _addr(self._coef(gam, "pt_synthesize")), *[_addr(x) for x in o]))
        return tuple(o)

    def pt_decompose(self, vr, vt, vz):
        o = [self._out_c() for _ in range(2)]
        self._check(lib().ccf_pt_decompose(self.h, *[_addr(self._coef(x, "pt_decompose")) for x in (vr, vt, vz)],
                                           *[_addr(x) for x in o]))
        return tuple(o)

    def curl_vector(self, vr, vt, vz):
        o = [self._out_c() for _ in range(3)]
        self._check(lib().ccf_curl_vector(self.h, *[_addr(self._coef(x, "curl_vector")) for x in (vr, vt, vz)],
                                          *[_addr(x) for x in o]))
        return tuple(o)

    def curl_pt(self, lam, gam):
        o = [self._out_c() for _ in range(2)]
        self._check(lib().ccf_curl_pt(self.h, _addr(self._coef(lam, "curl_pt")), _addr(self._coef(gam, "curl_pt")), *[_addr(x) for x in o]))
        return tuple(o)

    def velocity_from_vorticity(self, lam_w, gam_w):
        o = [self._out_c() for _ in range(2)]
        self._check(lib().ccf_velocity_from_vorticity(self.h, _addr(self._coef(lam_w, "velocity_from_vorticity")),
                                                      _addr(self._coef(gam_w, "velocity_from_vorticity")),
                                                      *[_addr(x) for x in o]))
        return tuple(o)

    def nonlinear_term(self, lam_v, gam_v, lam_w, gam_w, dealias_two_thirds=False):
        o = [self._out_c() for _ in range(2)]
        self._check(lib().ccf_nonlinear_ex(self.h, *[_addr(self._coef(x, "nonlinear_term"))
                                                       for x in (lam_v, gam_v, lam_w, gam_w)],
                                           int(bool(dealias_two_thirds)), *[_addr(x) for x in o]))
        return tuple(o)

    # ---- mode sharding (csrc/shard.cu)
    def shard(self, rank, world):
        """Make this context rank `rank` of `world` (before creating a stepper)."""
        self._check(lib().ccf_shard_init(self.h, int(rank), int(world)))
        return self

    def shard_info(self):
        v = [C.c_int() for _ in range(6)]
        self._check(lib().ccf_shard_info(self.h, *[C.byref(x) for x in v]))
        return dict(zip(("rank", "world", "slot_lo", "slot_hi", "row_lo", "row_hi"), (x.value for x in v)))

    def ipc_handle(self) -> bytes:
        buf = C.create_string_buffer(SHARD_HANDLE_BYTES)
        self._check(lib().ccf_shard_ipc_handle(self.h, buf))
        return buf.raw

    def open_ipc(self, handles):
        """handles: the ranks' ipc_handle() values (SHARD_HANDLE_BYTES each) in rank order."""
        blob = b"".join(bytes(x) for x in handles)
        self._check(lib().ccf_shard_open_ipc(self.h, blob))

    @staticmethod
    def link_local(ctxs):
        """Emulate ranks in one process on one device (step them from concurrent threads)."""
        arr = (C.c_void_p * len(ctxs))(*[c.h.value for c in ctxs])
        ctxs[0]._check(lib().ccf_shard_link_local(arr, len(ctxs)))

    def set_host_barrier(self, fn):
        """fn(): a host barrier across ranks, called after synchronising the stream (None: device barrier)."""
        cb = HOST_BARRIER_FN(lambda _u: fn()) if fn else HOST_BARRIER_FN()
        self._barrier_cb = cb  # keep alive
        self._check(lib().ccf_shard_set_host_barrier(self.h, cb, None))

    # ---- introspection
    def modal_plan(self, w, scale=1.0, poisson=True):
        info = np.zeros(8)
        u = np.zeros(256)
        v = np.zeros(256)
        dp = C.POINTER(C.c_double)
        self._check(lib().ccf_modal_plan(self.h, int(w), C.c_double(scale), int(poisson), info.ctypes.data_as(dp),
                                         u.ctypes.data_as(dp), v.ctypes.data_as(dp), 256))
        J = int(info[7])
        return dict(a=info[0], b=info[1], c=info[2], d=info[3], gamma=info[4], alpha=info[5], modulus=info[6], J=J,
                    u=u[:J].copy(), v=v[:J].copy())

    def stats(self):
        s, it, r, lch = C.c_long(), C.c_long(), C.c_int(), C.c_long()
        w = C.c_double()
        self._check(lib().ccf_get_stats(self.h, C.byref(s), C.byref(it), C.byref(r), C.byref(w), C.byref(lch)))
        gf = C.c_double()
        self._check(lib().ccf_get_gemm_flops(self.h, C.byref(gf)))
        return dict(adi_iterations=it.value, kernel_launches=lch.value, gemm_flops=gf.value)

    def reset_stats(self):
        self._check(lib().ccf_reset_stats(self.h))

    def adi_keep_history(self, enable=True):
        self._check(lib().ccf_adi_keep_history(self.h, int(bool(enable))))

    def adi_last_rounds(self, which=0):
        """(rounds[ntensor, nslots], history[ntensor, nslots, 4]) of the most recent ADI solve
        (which = 0), or of the most recent Poisson (1) / Helmholtz (2) solve."""
        cap = 2 * max(self.p, 1) + 2
        nt, ns = C.c_int(), C.c_int()
        r = np.zeros(cap, dtype=np.int32)
        h = np.zeros(cap * 4)
        self._check(lib().ccf_adi_last_rounds(self.h, int(which), C.byref(nt), C.byref(ns), r.ctypes.data,
                                              h.ctypes.data, cap))
        n = nt.value * ns.value
        return r[:n].reshape(nt.value, ns.value), h[: 4 * n].reshape(nt.value, ns.value, 4)


def diag_host_check(m, n, w, scale=1.0, poisson=True, k0=0, seed=1):
    """Relative Sylvester residual of the fast-diagonalization data of one mode (host only, no GPU)."""
    r = C.c_double()
    st = lib().ccf_diag_host_check(int(m), int(n), int(w), C.c_double(scale), int(poisson), int(k0), int(seed),
                                   C.byref(r))
    if st != 0:
        raise _ERR.get(st, CCFError)(lib().ccf_create_error().decode())
    return r.value


def plan_host(m, n, w, scale=1.0, poisson=True, tol=1e-12, q2_endpoint_pad=False):
    """Modal shift plan from the library's host setup path (no GPU required)."""
    info = np.zeros(8)
    u = np.zeros(256)
    v = np.zeros(256)
    dp = C.POINTER(C.c_double)
    st = lib().ccf_plan_host(int(m), int(n), int(w), C.c_double(scale), int(poisson), C.c_double(tol),
                             int(bool(q2_endpoint_pad)), info.ctypes.data_as(dp), u.ctypes.data_as(dp),
                             v.ctypes.data_as(dp), 256)
    if st != 0:
        raise _ERR.get(st, CCFError)(lib().ccf_create_error().decode())
    J = int(info[7])
    return dict(a=info[0], b=info[1], c=info[2], d=info[3], gamma=info[4], alpha=info[5], modulus=info[6], J=J,
                u=u[:J].copy(), v=v[:J].copy())


# ---- CCF1 FieldFile I/O (proj/include/cylspec/io.hpp:11-28, proj/src/io.cpp:12-109)
def _free_check(st):
    if st != 0:
        raise _ERR.get(st, CCFError)(lib().ccf_create_error().decode())


def crc32(data) -> int:
    """crc32_ieee of a bytes-like host buffer, numpy array or torch CUDA tensor (on the GPU)."""
    if hasattr(data, "data_ptr"):
        ptr, n = data.data_ptr(), data.numel() * data.element_size()
    else:
        a = np.ascontiguousarray(np.frombuffer(data, np.uint8) if isinstance(data, (bytes, bytearray)) else data)
        ptr, n = a.ctypes.data, a.nbytes
    out = C.c_uint()
    _free_check(lib().ccf_crc32(C.c_void_p(ptr), n, C.byref(out)))
    return out.value


def write_field(path, field, kind=None):
    """write_field (io.cpp:62-74): complex (p, n, m) coefficients -> kind 1, real grid values -> kind 0.
    field may be a numpy array or a torch CUDA tensor (checksummed on the GPU)."""
    if hasattr(field, "data_ptr"):
        import torch
        cplx = field.is_complex()
        shape = tuple(field.shape)
        t = field.contiguous()
        ptr = t.data_ptr()
        keep = t
        if kind is None:
            kind = 1 if cplx else 0
        del torch
    else:
        a = np.ascontiguousarray(field)
        cplx = np.iscomplexobj(a)
        a = a.astype(np.complex128 if cplx else np.float64, copy=False)
        shape, ptr, keep = a.shape, a.ctypes.data, a
        if kind is None:
            kind = 1 if cplx else 0
    p, n, m = shape[-3:]
    _free_check(lib().ccf_write_field(os.fsencode(path), int(kind), int(m), int(n), int(p), C.c_void_p(ptr)))
    del keep


def read_field_header(path):
    v = [C.c_int() for _ in range(4)]
    _free_check(lib().ccf_read_field_header(os.fsencode(path), *[C.byref(x) for x in v]))
    return dict(zip(("kind", "m", "n", "p"), (x.value for x in v)))


def read_field(path, out=None):
    """read_field (io.cpp:76-109) -> numpy (complex (p, n, m) for kind 1, real for kind 0), or into
    `out` (numpy or torch CUDA tensor of matching size; CRC verified on the GPU for device output)."""
    h = read_field_header(path)
    count = h["m"] * h["n"] * h["p"]
    if out is None:
        out = np.zeros((h["p"], h["n"], h["m"]), np.complex128 if h["kind"] == 1 else np.float64)
    cap = (out.numel() * out.element_size() if hasattr(out, "data_ptr") else out.nbytes) // 8
    v = [C.c_int() for _ in range(4)]
    _free_check(lib().ccf_read_field(os.fsencode(path), *[C.byref(x) for x in v], _addr(out), cap))
    assert cap >= count * (2 if h["kind"] == 1 else 1)
    return out


class ModalSolver:
    """proj/include/cylspec/solvers.hpp:35-59 ModalSolver(m, n, w, scale, poisson, tol) on the device (m, n from the
    context). Matrices are (n, m) complex arrays a[k, j] = X(j, k): the memory of the reference's column-major
    m x n Eigen::MatrixXcd / one CoeffTensor slice. scale = 0 with poisson = False is the mass pair."""

    def __init__(self, ctx: Context, w, scale=1.0, poisson=True):
        self.ctx, self.w, self.scale, self.poisson = ctx, int(w), float(scale), bool(poisson)
        p, n, m = ctx.shape()
        self.shape = (n, m)
        h = C.c_void_p()
        ctx._check(lib().ccf_modal_create(ctx.h, self.w, C.c_double(self.scale), int(self.poisson), C.byref(h)))
        self.h = h

    def _mat(self, x, what):
        a = np.asarray(x)
        if a.shape != self.shape:
            raise DomainError(f"{what}: right-hand side has wrong shape")  # solvers.cpp:79-80
        return np.ascontiguousarray(a, dtype=np.complex128)

    def solve(self, f_full):
        """ModalSolver::solve (solvers.cpp:77-98): raw C2 x C2 right-hand side -> m x n coefficients."""
        f = self._mat(f_full, "ModalSolver::solve")
        x = np.zeros_like(f)
        self.ctx._check(lib().ccf_modal_solve(self.h, _addr(f), _addr(x)))
        return x

    def apply(self, x):
        """raw().apply(x) = A x B + C x D (ultraop.cpp:83-87)."""
        a = self._mat(x, "ModalOperator::apply")
        y = np.zeros_like(a)
        self.ctx._check(lib().ccf_modal_apply(self.h, _addr(a), _addr(y)))
        return y

    def operator(self, which):
        """Dense A | B | C | D of raw() (ultraop.cpp:89-123)."""
        n, m = self.shape
        k = "ABCD".index(which)
        out = np.zeros((m, m) if k % 2 == 0 else (n, n))
        self.ctx._check(lib().ccf_modal_operator(self.h, k, _addr(out)))
        return out

    def close(self):
        if getattr(self, "h", None):  # safe after the context: ccf_ctx_destroy detaches its modal handles
            lib().ccf_modal_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_modal_helmholtz(ctx: Context, f, w, scale, lift=None):
    """solve_modal_helmholtz (solvers.cpp:125-140): x = solve(f - op.apply(lift_w)) + lift_w; lift: a (p', n, m)
    tensor whose slice w + p'/2 carries the boundary data (BoundaryCondition::lifted)."""
    s = ModalSolver(ctx, w, scale, poisson=False)
    try:
        rhs = s._mat(f, "solve_modal_helmholtz")
        if lift is None:
            return s.solve(rhs)
        lf = np.asarray(lift)
        if lf.ndim != 3 or lf.shape[1:] != s.shape:
            raise DomainError("BoundaryCondition: lift tensor has wrong dimensions")
        l = int(w) + lf.shape[0] // 2
        if l < 0 or l >= lf.shape[0]:
            raise DomainError("BoundaryCondition: lift tensor misses the requested mode")
        sl = np.ascontiguousarray(lf[l], dtype=np.complex128)
        return s.solve(rhs - s.apply(sl)) + sl
    finally:
        s.close()


class NSStepper:
    """proj/include/cylspec/ptns.hpp:104-127 NSStepper on the device (ramp bootstrap)."""

    def __init__(self, ctx: Context, lam0, gam0, reynolds, h, order=4, disable_nonlinear=False,
                 dealias_two_thirds=False, compute_gamma_psi=False):
        self.ctx = ctx
        st = C.c_void_p()
        flags = int(bool(disable_nonlinear)) | (2 if dealias_two_thirds else 0) | (4 if compute_gamma_psi else 0)
        ctx._check(lib().ccf_ns_create_ex(ctx.h, C.c_double(reynolds), C.c_double(h), int(order), flags,
                                          _addr(ctx._coef(lam0, "NSStepper: initial vorticity")),
                                          _addr(ctx._coef(gam0, "NSStepper: initial vorticity")), C.byref(st)))
        self.h = st
        self.dealias_two_thirds = bool(dealias_two_thirds)

    def seed(self, omega_hist, nonlinear_hist, time, steps_taken):
        """NSStepper::seed (ptns.cpp:195-203): install a prebuilt history. omega_hist / nonlinear_hist: lists of
        (lambda, gamma) coefficient pairs, newest first; nonlinear_hist[i] belongs to omega_hist[i + 1]."""
        if len(omega_hist) == 0:
            raise DomainError("NSStepper::seed: empty history")
        what = "NSStepper::seed: history"
        keep = [[self.ctx._coef(x, what) for x in pair] for pair in list(omega_hist) + list(nonlinear_hist)]
        no, nn = len(omega_hist), len(nonlinear_hist)
        vp = C.c_void_p

        def arr(rows, j):
            return (vp * max(len(rows), 1))(*[_addr(r[j]) for r in rows])

        self.ctx._check(lib().ccf_ns_seed(self.h, no, arr(keep[:no], 0), arr(keep[:no], 1), nn, arr(keep[no:], 0),
                                          arr(keep[no:], 1), C.c_double(time), int(steps_taken)))
        del keep

    def evaluate_nonlinear(self):
        """NSStepper::evaluate_nonlinear (ptns.cpp:211-214): nonlinear_term(velocity(), omega())."""
        lv, gv = self.velocity()
        lw, gw = self.omega()
        return self.ctx.nonlinear_term(lv, gv, lw, gw, self.dealias_two_thirds)

    def velocity(self):
        """NSStepper::velocity(): velocity PT scalars of the current state (fresh psi solve)."""
        o = [self.ctx._out_c() for _ in range(2)]
        self.ctx._check(lib().ccf_ns_velocity(self.h, *[_addr(x) for x in o]))
        return tuple(o)

    def gamma_psi(self):
        """state().gamma_psi: Poisson3D(-gamma_omega) of the omega the last step started from."""
        o = self.ctx._out_c()
        self.ctx._check(lib().ccf_ns_gamma_psi(self.h, _addr(o)))
        return o

    def step(self, nsteps=1):
        self.ctx._check(lib().ccf_ns_step(self.h, int(nsteps)))

    def omega(self, out_lam=None, out_gam=None):
        lam = self.ctx._coef(out_lam, "NSStepper.omega", out=True) if out_lam is not None else self.ctx._out_c()
        gam = self.ctx._coef(out_gam, "NSStepper.omega", out=True) if out_gam is not None else self.ctx._out_c()
        t = C.c_double()
        s = C.c_int()
        self.ctx._check(lib().ccf_ns_get_omega(self.h, _addr(lam), _addr(gam), C.byref(t), C.byref(s)))
        self.time, self.steps_taken = t.value, s.value
        return lam, gam

    def write_omega(self, lam_path, gam_path):
        """Snapshot omega (lambda, gamma) as kind-1 CCF1 files straight from the device state."""
        self.ctx._check(lib().ccf_ns_write_omega(self.h, os.fsencode(lam_path) if lam_path else None,
                                                 os.fsencode(gam_path) if gam_path else None))

    def set_graphs(self, enable: bool):
        lib().ccf_ns_set_graphs(self.h, int(bool(enable)))

    def launches_per_step(self):
        n = C.c_long()
        lib().ccf_ns_launches_per_step(self.h, C.byref(n))
        return n.value

    def profile_step(self):
        """Run one step eagerly with CUDA events at stage boundaries -> {stage: ms}."""
        ms = (C.c_double * 32)()
        k = C.c_int(32)
        names = C.create_string_buffer(4096)
        self.ctx._check(lib().ccf_ns_profile_step(self.h, ms, C.byref(k), names, 4096))
        nm = names.value.decode().strip().split("\n")
        return {nm[i]: ms[i] for i in range(k.value)}

    def close(self):
        if getattr(self, "h", None):
            lib().ccf_ns_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ns_run(ctx: Context, lam0, gam0, steps, reynolds=100.0, h=1e-2, order=4, disable_nonlinear=False,
           dealias_two_thirds=False, bootstrap="ramp", output_every=0):
    """ns_run (ptns.cpp:269-324) -> dict(final_omega, final_time, snapshots, snapshot_times). bootstrap "ramp"
    (BDF 1 -> order) or "substeps": [0, (order - 1) h] integrated with 32 BDF2 sub-steps per h, the sampled
    trajectory and its replayed nonlinear terms seeded into the full-order stepper (ptns.cpp:272-311)."""
    if bootstrap not in ("ramp", "substeps"):
        raise ConfigError("ns_run: bootstrap ramp | substeps")
    kw = dict(disable_nonlinear=disable_nonlinear, dealias_two_thirds=dealias_two_thirds)
    snaps, times = [], []
    first = 0
    if bootstrap == "substeps" and order > 1 and steps > 0:
        per = 32
        fine = NSStepper(ctx, lam0, gam0, reynolds, h / per, min(2, order), **kw)
        hist = [(lam0, gam0)]
        for _ in range(order - 1):
            fine.step(per)
            hist.insert(0, fine.omega())
        fine.close()
        st = NSStepper(ctx, hist[0][0], hist[0][1], reynolds, h, order, **kw)
        replay = []
        if not disable_nonlinear:
            for i in range(len(hist) - 1, 0, -1):
                v = ctx.velocity_from_vorticity(*hist[i])
                replay.insert(0, ctx.nonlinear_term(v[0], v[1], hist[i][0], hist[i][1], dealias_two_thirds))
        st.seed(hist, replay, (order - 1) * h, order - 1)
        first = order - 1
    else:
        st = NSStepper(ctx, lam0, gam0, reynolds, h, order, **kw)
    for s in range(first, steps):
        st.step()
        if output_every > 0 and (s + 1) % output_every == 0:
            snaps.append(st.omega())
            times.append(st.time)
    om = st.omega()
    out = dict(final_omega=om, final_time=st.time, snapshots=snaps, snapshot_times=times)
    st.close()
    return out


def _field_arg(ctx, x, what):
    """(pointer holder, kind): complex -> coefficients (kind 1), real -> grid values (kind 0); shape and
    dtype checked against the context (timestep.cpp:69-70, 113-114)."""
    if hasattr(x, "data_ptr"):
        cplx = x.is_complex()
        return _arg(x.contiguous(), ctx.shape(), cplx, what), (1 if cplx else 0)
    cplx = np.iscomplexobj(x)
    return _arg(x, ctx.shape(), cplx, what), (1 if cplx else 0)


class HeatStepper:
    """proj/include/cylspec/timestep.hpp:79-97 HeatStepper on the device: (d/dt - alpha lap) T = g,
    BDF 1 -> order ramp, homogeneous Dirichlet. initial: grid values (real) or coefficients (complex)."""

    def __init__(self, ctx: Context, initial, alpha=1.0, h=1e-2, order=4):
        self.ctx = ctx
        self.h_step = h
        a, kind = _field_arg(ctx, initial, "HeatStepper: initial data")
        st = C.c_void_p()
        ctx._check(lib().ccf_heat_create(ctx.h, C.c_double(alpha), C.c_double(h), int(order), _addr(a), kind,
                                         C.byref(st)))
        self.h = st
        self.time, self.steps_taken = 0.0, 0

    def step(self, forcing=None):
        """HeatStepper::step(const CoeffTensor*) / step_with_callback: forcing = grid values or coefficients."""
        if forcing is None:
            self.ctx._check(lib().ccf_heat_step(self.h, None, 0))
        else:
            a, kind = _field_arg(self.ctx, forcing, "HelmholtzTensorStepper: forcing")
            self.ctx._check(lib().ccf_heat_step(self.h, _addr(a), kind))
        self.time += self.h_step
        self.steps_taken += 1

    def current(self, out=None):
        c = self.ctx._coef(out, "HeatStepper.current", out=True) if out is not None else self.ctx._out_c()
        t, s = C.c_double(), C.c_int()
        self.ctx._check(lib().ccf_heat_get(self.h, _addr(c), C.byref(t), C.byref(s)))
        self.time, self.steps_taken = t.value, s.value
        return c

    def close(self):
        if getattr(self, "h", None):
            lib().ccf_ns_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def heat_run(ctx: Context, initial, forcing, steps, alpha=1.0, h=1e-2, order=4, output_every=0,
             forcing_mode="exact"):
    """proj/src/timestep.cpp:146-170 heat_run: snapshots (grid values) at t = 0, every output_every
    steps and at the end; forcing(t) returns grid values (numpy or torch CUDA) evaluated at t + h
    (ForcingMode::exact) or t; forcing None = unforced."""
    if steps < 0:
        raise DomainError("heat_run: steps must be nonnegative")
    st = HeatStepper(ctx, initial, alpha=alpha, h=h, order=order)
    init_vals = initial if not np.iscomplexobj(initial) else ctx.synthesize(initial)
    snaps, times = [np.asarray(init_vals)], [0.0]
    for s in range(steps):
        if forcing is None:
            st.step(None)
        else:
            st.step(forcing(st.time + h if forcing_mode == "exact" else st.time))
        if output_every > 0 and (s + 1) % output_every == 0 and s + 1 < steps:
            snaps.append(ctx.synthesize(st.current()))
            times.append(st.time)
    final = st.current()
    if steps > 0:
        snaps.append(ctx.synthesize(final))
        times.append(st.time)
    st.close()
    return dict(snapshots=snaps, snapshot_times=times, final_coeffs=final, final_time=times[-1] if steps else 0.0)
