"""Python mirror of the reference `stiga` operator/solver API over the C ABI (libstiga_gpu.so).

Names, argument meaning and error behaviour follow /root/reference/proj/core/include/stiga:
  ExtendedFDPreconditioner.setup / .apply        fdsolve.hpp:41-70
  kron_matvec, KronSumOperator(.apply/.diagonal) kronop.hpp:47-79
  kron_sum_terms                                 solver.cpp:10-30
  gmres(A, P, b, GmresOptions) -> (x, SolveReport) gmres.hpp:12-35
  assemble_time_matrices / assemble_spatial_parametric / assemble_univariate  assembly.hpp:47-66
std::invalid_argument -> ValueError, std::runtime_error -> RuntimeError, device failures -> StigaError.

Vectors: torch CUDA float64 tensors stay on the device (the hot path); numpy arrays go through the
host-buffer entry points (H2D, apply, D2H).  No computation happens in Python.
"""
import ctypes
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from ._lib import GmresOptions as _GOpts
from ._lib import GmresReport as _GRep
from ._lib import check, lib

_pd = ctypes.POINTER(ctypes.c_double)


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _colmajor(a):
    """Dense n x n matrix -> contiguous column-major float64 buffer."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("square matrix expected")
    return np.ascontiguousarray(a.T)


def _ptr(a):
    return a.ctypes.data_as(_pd)


def _ptr_array(arrs):
    return (_pd * len(arrs))(*[_ptr(a) for a in arrs])


def _stream_handle(stream):
    if stream is None:
        try:
            import torch

            if torch.cuda.is_available():
                return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        except ImportError:
            pass
        return ctypes.c_void_p(0)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def device_count():
    return lib().stiga_device_count()


# ----------------------------------------------------------------------------------------
# host-side 1D assembly
# ----------------------------------------------------------------------------------------
def space_dim(p, n_el, temporal=False):
    n = ctypes.c_int()
    check(lib().stiga_space_dim(p, n_el, 1 if temporal else 0, ctypes.byref(n)), "space_dim")
    return n.value


def assemble_time_matrices(p_t, n_el_t, T=1.0):
    """assemble_time_matrices (assembly.cpp:129-138) -> (W_t, M_t) dense numpy arrays."""
    n = space_dim(p_t, n_el_t, temporal=True) if n_el_t >= 1 and p_t >= 1 else 0
    W = np.zeros(n * n)
    M = np.zeros(n * n)
    check(lib().stiga_assemble_time_matrices(p_t, n_el_t, T, _ptr(W), _ptr(M)), "assemble_time_matrices")
    return W.reshape(n, n).T.copy(), M.reshape(n, n).T.copy()


def assemble_spatial_parametric(p, n_el, d, q=None):
    """assemble_spatial_parametric (assembly.cpp:140-149) on d identical spatial spaces -> (K, M) lists."""
    q = p + 1 if q is None else q
    n = space_dim(p, n_el)
    K, M = [], []
    for _ in range(d):
        k = np.zeros(n * n)
        m = np.zeros(n * n)
        check(lib().stiga_assemble_spatial_parametric(p, n_el, q, _ptr(k), _ptr(m)), "assemble_spatial_parametric")
        K.append(k.reshape(n, n).T.copy())
        M.append(m.reshape(n, n).T.copy())
    return K, M


def assemble_univariate(p, n_el, temporal, q, deriv_row, deriv_col, element_weights=None):
    """assemble_univariate with optional per-element weights (assembly.cpp:47-79, 118-127)."""
    n = space_dim(p, n_el, temporal)
    out = np.zeros(n * n)
    w = None if element_weights is None else _f64(element_weights)
    check(lib().stiga_assemble_univariate(p, n_el, 1 if temporal else 0, q, deriv_row, deriv_col,
                                          _ptr(w) if w is not None else None, _ptr(out)), "assemble_univariate")
    return out.reshape(n, n).T.copy()


def kron_sum_terms(K, M, Wt, Mt, gamma, nu):
    """solver.cpp:10-30: [(gamma, [M_1..M_d, W_t]), (nu, [.., K_l, .., M_t]) for each l]."""
    d = len(K)
    terms = [(gamma, [M[l] for l in range(d)] + [Wt])]
    for l in range(d):
        terms.append((nu, [K[k] if k == l else M[k] for k in range(d)] + [Mt]))
    return terms


# ----------------------------------------------------------------------------------------
# ExtendedFDPreconditioner
# ----------------------------------------------------------------------------------------
class ExtendedFDPreconditioner:
    """fdsolve.hpp:41-70.  Build with ExtendedFDPreconditioner.setup(...)."""

    def __init__(self, handle, device):
        self._h = ctypes.c_void_p(handle)
        self.device = device
        n = ctypes.c_longlong()
        check(lib().stiga_fd_size(self._h, ctypes.byref(n)), "fd_size")
        self.n_dof = n.value
        d = ctypes.c_int()
        dims = (ctypes.c_int * 8)()
        check(lib().stiga_fd_dims(self._h, ctypes.byref(d), dims), "fd_dims")
        self.d = d.value
        self.dims = [dims[i] for i in range(self.d + 1)]

    @staticmethod
    def setup(space_K, space_M, Wt, Mt, gamma, nu, scaling=None, device=0):
        """fdsolve.cpp:67-153 (host factorizations, one upload of the factors)."""
        if len(space_K) != len(space_M) or len(space_K) == 0:
            raise ValueError("ExtendedFDPreconditioner: per-direction matrices mismatch")
        Ks = [_colmajor(k) for k in space_K]
        Ms = [_colmajor(m) for m in space_M]
        n = (ctypes.c_int * len(Ks))(*[int(np.asarray(k).shape[0]) for k in space_K])
        for k, m in zip(space_K, space_M):
            if np.asarray(k).shape != np.asarray(m).shape:
                raise ValueError("spd_generalized_eig: shape mismatch")
        W = _colmajor(Wt)
        Mm = _colmajor(Mt)
        if W.shape != Mm.shape:
            raise ValueError("time_factorization: shape mismatch")
        n_t = int(np.asarray(Wt).shape[0])
        sc = None if scaling is None else _f64(scaling)
        h = ctypes.c_void_p()
        check(lib().stiga_fd_setup(len(Ks), n, _ptr_array(Ks), _ptr_array(Ms), n_t, _ptr(W), _ptr(Mm),
                                   float(gamma), float(nu), _ptr(sc) if sc is not None else None,
                                   len(sc) if sc is not None else 0, int(device), ctypes.byref(h)), "fd_setup")
        return ExtendedFDPreconditioner(h.value, device)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().stiga_fd_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def size(self):
        return self.n_dof

    def time_info(self):
        np_, z = ctypes.c_int(), ctypes.c_int()
        sig, rho = ctypes.c_double(), ctypes.c_double()
        check(lib().stiga_fd_time_info(self._h, ctypes.byref(np_), ctypes.byref(z), ctypes.byref(sig),
                                       ctypes.byref(rho)), "time_info")
        return {"npairs": np_.value, "zero_count": z.value, "sigma": sig.value, "rho": rho.value}

    def export(self, which, l=0):
        """0: U_l, 1: Lambda_l, 2: U_t, 3: lambda_t, 4: g, 5: S_inv (host copies)."""
        n_s = int(np.prod(self.dims[:-1]))
        n_t = self.dims[-1]
        sizes = {0: self.dims[l] ** 2 if l < self.d else 0, 1: self.dims[l] if l < self.d else 0,
                 2: n_t * n_t, 3: self.time_info()["npairs"], 4: n_t - 1, 5: n_s}
        if which not in sizes:
            raise ValueError("stiga_fd_export: unknown factor id")
        out = np.zeros(max(sizes[which], 1))
        check(lib().stiga_fd_export(self._h, which, l, _ptr(out), len(out)), "fd_export")
        out = out[: sizes[which]]
        if which in (0, 2):
            m = self.dims[l] if which == 0 else n_t
            return out.reshape(m, m).T.copy()
        return out

    def launches(self):
        n = ctypes.c_int()
        check(lib().stiga_fd_launches(self._h, ctypes.byref(n)), "fd_launches")
        return n.value

    def launch_info(self):
        """[(name, algorithmic flops)] of the kernel launches of one apply."""
        out = []
        buf = ctypes.create_string_buffer(64)
        for i in range(self.launches()):
            f = ctypes.c_double()
            check(lib().stiga_fd_launch_info(self._h, i, buf, 64, ctypes.byref(f)), "fd_launch_info")
            out.append((buf.value.decode(), f.value))
        return out

    def apply(self, r, out=None, stream=None):
        """r -> A^-1 r (fdsolve.cpp:155-164).  torch CUDA tensor in -> tensor out (device path);
        numpy in -> numpy out (host path with H2D/D2H)."""
        if _is_torch(r):
            import torch

            if r.dtype != torch.float64 or not r.is_cuda or not r.is_contiguous():
                raise ValueError("ExtendedFDPreconditioner::apply: expected a contiguous float64 CUDA tensor")
            if r.numel() != self.n_dof:
                raise ValueError("ExtendedFDPreconditioner::apply: vector length mismatch")
            if out is None:
                out = torch.empty_like(r)
            check(lib().stiga_fd_apply(self._h, ctypes.c_void_p(r.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                       _stream_handle(stream)), "fd_apply")
            return out
        r = _f64(r)
        if r.size != self.n_dof:
            raise ValueError("ExtendedFDPreconditioner::apply: vector length mismatch")
        s = np.empty_like(r) if out is None else out
        check(lib().stiga_fd_apply_host(self._h, _ptr(r), _ptr(s)), "fd_apply_host")
        return s

    def apply_profiled(self, r, out, stream=None):
        """Device apply with per-launch CUDA-event durations (ms) for the 2d+1 kernels."""
        n = self.launches()
        ms = (ctypes.c_float * n)()
        check(lib().stiga_fd_apply_profiled(self._h, ctypes.c_void_p(r.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                            _stream_handle(stream), ms), "fd_apply_profiled")
        return [ms[i] for i in range(n)]


# ----------------------------------------------------------------------------------------
# Kronecker operators
# ----------------------------------------------------------------------------------------
def kron_matvec(factors, x, device=0, stream=None):
    """kronop.cpp:75-89 on a torch CUDA tensor (factor l acts on mode l, first mode fastest)."""
    import torch

    F = [np.asarray(f, dtype=np.float64) for f in factors]
    rows = (ctypes.c_int * len(F))(*[f.shape[0] for f in F])
    cols = (ctypes.c_int * len(F))(*[f.shape[1] for f in F])
    if int(np.prod([f.shape[1] for f in F])) != x.numel():
        raise ValueError("kron_matvec: vector length does not match factor dimensions")
    Fc = [np.ascontiguousarray(f.T) for f in F]  # column-major
    y = torch.empty(int(np.prod([f.shape[0] for f in F])), dtype=torch.float64, device=x.device)
    check(lib().stiga_kron_matvec(len(F), rows, cols, _ptr_array(Fc), ctypes.c_void_p(x.data_ptr()),
                                  ctypes.c_void_p(y.data_ptr()), int(device), _stream_handle(stream)), "kron_matvec")
    return y


class KronSumOperator:
    """kronop.hpp:61-79: y = sum_t coeff_t (x)_l F_{t,l} x, applied on the device."""

    def __init__(self, dims, terms, device=0, _handle=None):
        self.device = device
        if _handle is not None:
            self._h = ctypes.c_void_p(_handle)
        else:
            dims = [int(n) for n in dims]
            for c, fs in terms:
                if len(fs) != len(dims):
                    raise ValueError("KronSumOperator: term factor count does not match dims")
                for f, n in zip(fs, dims):
                    if np.asarray(f).shape != (n, n):
                        raise ValueError("KronSumOperator: factor shape does not match dims")
            D = len(dims)
            cd = (ctypes.c_int * D)(*dims)
            coeffs = np.array([float(c) for c, _ in terms] or [0.0])
            facs = [_colmajor(f) for _, fs in terms for f in fs]
            h = ctypes.c_void_p()
            check(lib().stiga_kronsum_create(D, cd, len(terms), _ptr(coeffs), _ptr_array(facs) if facs else None,
                                             int(device), ctypes.byref(h)), "kronsum_create")
            self._h = h
        n = ctypes.c_longlong()
        check(lib().stiga_kronsum_size(self._h, ctypes.byref(n)), "kronsum_size")
        self.n_dof = n.value
        nd = ctypes.c_int()
        dims_buf = (ctypes.c_int * 8)()
        check(lib().stiga_kronsum_dims(self._h, ctypes.byref(nd), dims_buf, 8), "kronsum_dims")
        self.dims = [dims_buf[i] for i in range(nd.value)]

    @staticmethod
    def spacetime(K, M, Wt, Mt, gamma, nu, device=0):
        """KronSumOperator(dims, kron_sum_terms(K, M, Wt, Mt, gamma, nu)) with the sum-factorized
        banded apply (solver.cpp:10-30, 67-70)."""
        d = len(K)
        Ks = [_colmajor(k) for k in K]
        Ms = [_colmajor(m) for m in M]
        n = (ctypes.c_int * d)(*[k.shape[0] for k in Ks])
        W = _colmajor(Wt)
        Mm = _colmajor(Mt)
        h = ctypes.c_void_p()
        check(lib().stiga_kronsum_create_spacetime(d, n, _ptr_array(Ks), _ptr_array(Ms), W.shape[0], _ptr(W),
                                                   _ptr(Mm), float(gamma), float(nu), int(device), ctypes.byref(h)),
              "kronsum_create_spacetime")
        return KronSumOperator(None, None, device, _handle=h.value)

    @staticmethod
    def physical(problem, p, n_el, device=0):
        """SpaceTimeSystem's A_ = M_s (x) W_t + K_s (x) M_t (solver.cpp:58-70) with the physical
        spatial matrices of `problem` (problems.Problem) assembled on the device."""
        h = ctypes.c_void_p()
        check(lib().stiga_kronsum_create_physical(problem._h, int(p), int(n_el), int(device), ctypes.byref(h)),
              "kronsum_create_physical")
        return KronSumOperator(None, None, device, _handle=h.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().stiga_kronsum_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def size(self):
        return self.n_dof

    def apply(self, x, out=None, stream=None):
        import torch

        if x.numel() != self.n_dof:
            raise ValueError("KronSumOperator::apply: vector length mismatch")
        if out is None:
            out = torch.empty_like(x)
        check(lib().stiga_kronsum_apply(self._h, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                        _stream_handle(stream)), "kronsum_apply")
        return out

    def diagonal(self):
        d = np.zeros(self.n_dof)
        check(lib().stiga_kronsum_diagonal(self._h, _ptr(d)), "kronsum_diagonal")
        return d


# ----------------------------------------------------------------------------------------
# GMRES
# ----------------------------------------------------------------------------------------
@dataclass
class GmresOptions:
    """gmres.hpp:23-27."""
    tol: float = 1e-8
    max_krylov: int = 100
    restart: Optional[int] = None


@dataclass
class SolveReport:
    """gmres.hpp:15-21."""
    iterations: int = 0
    residual_history: List[float] = field(default_factory=list)
    converged: bool = False
    wall_time_s: float = 0.0
    precond_time_fraction: float = 0.0


def gmres(A, P, b, opts=None, stream=None):
    """gmres(A, P, b, opts) (gmres.cpp:19-132) -> (x, SolveReport); b is a torch CUDA tensor."""
    import torch

    opts = opts or GmresOptions()
    if opts.tol <= 0.0:
        raise ValueError("gmres: tolerance must be positive")
    if opts.max_krylov < 1:
        raise ValueError("gmres: max_krylov must be >= 1")
    if opts.restart is not None and opts.restart < 1:
        raise ValueError("gmres: restart cycle must be >= 1")
    x = torch.empty_like(b)
    cap = opts.max_krylov + 2
    hist = np.zeros(cap)
    rep = _GRep(0, 0, 0.0, 0.0, _ptr(hist), cap, 0)
    o = _GOpts(float(opts.tol), int(opts.max_krylov), int(opts.restart or 0))
    check(lib().stiga_gmres(A.handle, P.handle if P is not None else None, ctypes.c_void_p(b.data_ptr()),
                            ctypes.c_void_p(x.data_ptr()), ctypes.byref(o), ctypes.byref(rep),
                            _stream_handle(stream)), "gmres")
    return x, SolveReport(rep.iterations, list(hist[: min(cap, rep.history_len)]), bool(rep.converged),
                          rep.wall_time_s, rep.precond_time_fraction)


def fp64_peak(device=0, ms=200.0):
    """Measured FP64 throughput (DMMA m8n8k4, dependent-chain DFMA) in TFLOP/s."""
    a, b = ctypes.c_double(), ctypes.c_double()
    check(lib().stiga_fp64_peak(int(device), float(ms), ctypes.byref(a), ctypes.byref(b)), "fp64_peak")
    return a.value, b.value
