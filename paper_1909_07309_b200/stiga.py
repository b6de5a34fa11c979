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

from ._lib import ALLGATHER_FN, ALLREDUCE_FN, BARRIER_FN, COMM_ID_BYTES, LINOP_FN, CommCallbacks
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
# Communicator (multi-GPU)
# ----------------------------------------------------------------------------------------
def shard_partition(n, world, rank):
    """Balanced contiguous partition (stiga_shard_partition): (offset, length) of part `rank`."""
    o, l_ = ctypes.c_longlong(), ctypes.c_longlong()
    check(lib().stiga_shard_partition(int(n), int(world), int(rank), ctypes.byref(o), ctypes.byref(l_)),
          "shard_partition")
    return o.value, l_.value


class Comm:
    """stiga_comm_t: one rank of a communicator.  Comm.nccl(...) wraps NCCL (collectives stream-ordered
    on the device); Comm.from_process_group() builds NCCL for an nccl torch.distributed group and a
    host-callback communicator over the group's collectives otherwise (gloo: the CPU / one-GPU tests)."""

    def __init__(self, handle, world, rank, device, keep=None):
        self._h = ctypes.c_void_p(handle)
        self.world, self.rank, self.device = world, rank, device
        self._keep = keep  # ctypes callbacks must outlive the handle

    @staticmethod
    def unique_id():
        buf = ctypes.create_string_buffer(COMM_ID_BYTES)
        check(lib().stiga_comm_unique_id(buf), "comm_unique_id")
        return buf.raw

    @staticmethod
    def nccl(world, rank, uid, device=0):
        h = ctypes.c_void_p()
        check(lib().stiga_comm_init_nccl(int(world), int(rank), uid, int(device), ctypes.byref(h)), "comm_init_nccl")
        return Comm(h.value, world, rank, device)

    @staticmethod
    def host(world, rank, allreduce, allgather, barrier, device=0):
        """Host-callback communicator: allreduce(np.ndarray (in place), op: 0 sum / 1 max),
        allgather(bytes) -> list of bytes (rank order), barrier()."""

        def _ar(ctx, buf, n, op):
            try:
                a = np.ctypeslib.as_array(buf, shape=(n,))
                allreduce(a, op)
                return 0
            except Exception:
                return 1

        def _ag(ctx, send, nbytes, recv):
            try:
                parts = allgather(ctypes.string_at(send, nbytes))
                ctypes.memmove(recv, b"".join(parts), nbytes * world)
                return 0
            except Exception:
                return 1

        def _br(ctx):
            try:
                barrier()
                return 0
            except Exception:
                return 1

        cb = CommCallbacks(None, ALLREDUCE_FN(_ar), ALLGATHER_FN(_ag), BARRIER_FN(_br))
        h = ctypes.c_void_p()
        check(lib().stiga_comm_init_host(int(world), int(rank), ctypes.byref(cb), int(device), ctypes.byref(h)),
              "comm_init_host")
        return Comm(h.value, world, rank, device, keep=cb)

    @staticmethod
    def from_process_group(group=None, device=None):
        import torch
        import torch.distributed as dist

        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        dev = torch.cuda.current_device() if device is None else device
        if dist.get_backend(group) == "nccl":
            box = [Comm.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            return Comm.nccl(world, rank, box[0], dev)

        def allreduce(a, op):
            t = torch.from_numpy(a)  # shares memory with the C buffer
            dist.all_reduce(t, op=dist.ReduceOp.SUM if op == 0 else dist.ReduceOp.MAX, group=group)

        def allgather(b):
            out = [None] * world
            dist.all_gather_object(out, b, group=group)
            return out

        return Comm.host(world, rank, allreduce, allgather, lambda: dist.barrier(group=group), dev)

    def allreduce(self, t, stream=None):
        """Sum-all-reduce of a float64 CUDA tensor in place."""
        check(lib().stiga_comm_allreduce(self._h, ctypes.c_void_p(t.data_ptr()), t.numel(), _stream_handle(stream)),
              "comm_allreduce")
        return t

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().stiga_comm_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h


# ----------------------------------------------------------------------------------------
# ExtendedFDPreconditioner
# ----------------------------------------------------------------------------------------
class ExtendedFDPreconditioner:
    """fdsolve.hpp:41-70.  Build with ExtendedFDPreconditioner.setup(...)."""

    def __init__(self, handle, device, comm=None):
        self._h = ctypes.c_void_p(handle)
        self.device = device
        self.comm = comm  # keeps the communicator alive for a sharded handle
        n = ctypes.c_longlong()
        check(lib().stiga_fd_size(self._h, ctypes.byref(n)), "fd_size")
        self.n_dof = n.value
        d = ctypes.c_int()
        dims = (ctypes.c_int * 8)()
        check(lib().stiga_fd_dims(self._h, ctypes.byref(d), dims), "fd_dims")
        self.d = d.value
        self.dims = [dims[i] for i in range(self.d + 1)]
        v = [ctypes.c_longlong() for _ in range(4)]
        check(lib().stiga_fd_local(self._h, *[ctypes.byref(x) for x in v]), "fd_local")
        self.t0, self.nt_local, self.offset, self.n_local = [x.value for x in v]

    def local_slice(self):
        """Range of the global colex vector this handle's apply maps (the whole vector unsharded)."""
        return self.offset, self.offset + self.n_local

    @staticmethod
    def setup(space_K, space_M, Wt, Mt, gamma, nu, scaling=None, device=0, comm=None, device_schur=False,
              eig="host"):
        """fdsolve.cpp:67-153 (host factorizations, one upload of the factors).  With comm (a Comm):
        the time-sharded handle of this rank (collective); `scaling` is then D on the local time slab.

        Device-side setup (stiga_fd_setup_ex): scaling may be a CUDA tensor (D^-1/2 formed on the
        device); device_schur=True computes Lambda_s / S^-1 on the device (bit-identical);
        eig="cusolver" runs the setup's symmetric eigenproblems with cuSOLVER."""
        if eig not in ("host", "cusolver"):
            raise ValueError("ExtendedFDPreconditioner: eig must be 'host' or 'cusolver'")
        dev_scaling = scaling is not None and _is_torch(scaling) and scaling.is_cuda
        if comm is None and (dev_scaling or device_schur or eig == "cusolver"):
            return ExtendedFDPreconditioner._setup_ex(space_K, space_M, Wt, Mt, gamma, nu, scaling if dev_scaling else None,
                                                      None if dev_scaling else scaling, device, device_schur, eig)
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
        if comm is not None:
            check(lib().stiga_fd_setup_sharded(len(Ks), n, _ptr_array(Ks), _ptr_array(Ms), n_t, _ptr(W), _ptr(Mm),
                                               float(gamma), float(nu), _ptr(sc) if sc is not None else None,
                                               len(sc) if sc is not None else 0, comm.handle, ctypes.byref(h)),
                  "fd_setup_sharded")
            return ExtendedFDPreconditioner(h.value, comm.device, comm)
        check(lib().stiga_fd_setup(len(Ks), n, _ptr_array(Ks), _ptr_array(Ms), n_t, _ptr(W), _ptr(Mm),
                                   float(gamma), float(nu), _ptr(sc) if sc is not None else None,
                                   len(sc) if sc is not None else 0, int(device), ctypes.byref(h)), "fd_setup")
        return ExtendedFDPreconditioner(h.value, device)

    @staticmethod
    def _setup_ex(space_K, space_M, Wt, Mt, gamma, nu, d_scaling, scaling, device, device_schur, eig):
        if len(space_K) != len(space_M) or len(space_K) == 0:
            raise ValueError("ExtendedFDPreconditioner: per-direction matrices mismatch")
        Ks = [_colmajor(k) for k in space_K]
        Ms = [_colmajor(m) for m in space_M]
        n = (ctypes.c_int * len(Ks))(*[int(np.asarray(k).shape[0]) for k in space_K])
        W = _colmajor(Wt)
        Mm = _colmajor(Mt)
        n_t = int(np.asarray(Wt).shape[0])
        from ._lib import SETUP_CUSOLVER, SETUP_DEVICE_SCHUR, FdSetupOptions

        opts = FdSetupOptions((SETUP_DEVICE_SCHUR if device_schur else 0) | (SETUP_CUSOLVER if eig == "cusolver" else 0),
                              d_scaling.data_ptr() if d_scaling is not None else None)
        sc = None if scaling is None else _f64(scaling)
        length = d_scaling.numel() if d_scaling is not None else (len(sc) if sc is not None else 0)
        h = ctypes.c_void_p()
        check(lib().stiga_fd_setup_ex(len(Ks), n, _ptr_array(Ks), _ptr_array(Ms), n_t, _ptr(W), _ptr(Mm), float(gamma),
                                      float(nu), _ptr(sc) if sc is not None else None, length, ctypes.byref(opts),
                                      int(device), ctypes.byref(h)), "fd_setup_ex")
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
            if r.numel() != self.n_local:
                raise ValueError("ExtendedFDPreconditioner::apply: vector length mismatch")
            if out is None:
                out = torch.empty_like(r)
            check(lib().stiga_fd_apply(self._h, ctypes.c_void_p(r.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                       _stream_handle(stream)), "fd_apply")
            return out
        r = _f64(r)
        if r.size != self.n_local:
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
        v = [ctypes.c_longlong() for _ in range(4)]
        check(lib().stiga_kronsum_local(self._h, *[ctypes.byref(x) for x in v]), "kronsum_local")
        self.t0, self.nt_local, self.offset, self.n_local = [x.value for x in v]
        nd = ctypes.c_int()
        dims_buf = (ctypes.c_int * 8)()
        check(lib().stiga_kronsum_dims(self._h, ctypes.byref(nd), dims_buf, 8), "kronsum_dims")
        self.dims = [dims_buf[i] for i in range(nd.value)]

    @staticmethod
    def spacetime(K, M, Wt, Mt, gamma, nu, device=0, comm=None):
        """KronSumOperator(dims, kron_sum_terms(K, M, Wt, Mt, gamma, nu)) with the sum-factorized
        banded apply (solver.cpp:10-30, 67-70).  comm: the time-sharded operator of this rank."""
        d = len(K)
        Ks = [_colmajor(k) for k in K]
        Ms = [_colmajor(m) for m in M]
        n = (ctypes.c_int * d)(*[k.shape[0] for k in Ks])
        W = _colmajor(Wt)
        Mm = _colmajor(Mt)
        h = ctypes.c_void_p()
        if comm is not None:
            check(lib().stiga_kronsum_create_spacetime_sharded(d, n, _ptr_array(Ks), _ptr_array(Ms), W.shape[0],
                                                               _ptr(W), _ptr(Mm), float(gamma), float(nu),
                                                               comm.handle, ctypes.byref(h)),
                  "kronsum_create_spacetime_sharded")
            op = KronSumOperator(None, None, comm.device, _handle=h.value)
            op.comm = comm
            return op
        check(lib().stiga_kronsum_create_spacetime(d, n, _ptr_array(Ks), _ptr_array(Ms), W.shape[0], _ptr(W),
                                                   _ptr(Mm), float(gamma), float(nu), int(device), ctypes.byref(h)),
              "kronsum_create_spacetime")
        return KronSumOperator(None, None, device, _handle=h.value)

    @staticmethod
    def physical(problem, p, n_el, device=0, comm=None):
        """SpaceTimeSystem's A_ = M_s (x) W_t + K_s (x) M_t (solver.cpp:58-70) with the physical
        spatial matrices of `problem` (problems.Problem) assembled on the device.  comm: sharded."""
        h = ctypes.c_void_p()
        if comm is not None:
            check(lib().stiga_kronsum_create_physical_sharded(problem._h, int(p), int(n_el), comm.handle,
                                                              ctypes.byref(h)), "kronsum_create_physical_sharded")
            op = KronSumOperator(None, None, comm.device, _handle=h.value)
            op.comm = comm
            return op
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

        if x.numel() != self.n_local:
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

    def diagonal_device(self, out=None, stream=None):
        """KronSumOperator::diagonal() into a CUDA tensor (bit-identical to diagonal())."""
        import torch

        if out is None:
            out = torch.empty(self.n_dof, dtype=torch.float64, device=f"cuda:{self.device}")
        check(lib().stiga_kronsum_diagonal_device(self._h, ctypes.c_void_p(out.data_ptr()), _stream_handle(stream)),
              "kronsum_diagonal_device")
        return out


def geometry_scaling_device(A, Atilde, out=None, stream=None):
    """D = diag(A) / diag(A~) (solver.cpp:138-142) on the device: A the system operator, A~ the
    Kronecker-sum operator of the separated factors (gamma = nu = 1)."""
    import torch

    if out is None:
        out = torch.empty(A.n_dof, dtype=torch.float64, device=f"cuda:{A.device}")
    check(lib().stiga_geometry_scaling_device(A.handle, Atilde.handle, ctypes.c_void_p(out.data_ptr()),
                                              _stream_handle(stream)), "geometry_scaling_device")
    return out


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


def gmres_op(n, A, P, b, opts=None, comm=None, stream=None):
    """gmres(A, P, b, opts) over Python-callable operators (gmres.hpp:12 LinOp): A(x, y) and P(x, y)
    (P may be None) write the image of the CUDA tensor x into y (both n float64 entries, on the current
    stream).  comm: Krylov dots all-reduced over the communicator (local slabs, CGS2).  Through
    stiga_gmres_op; the solver itself is the native one."""
    import torch

    opts = opts or GmresOptions()
    if opts.restart is not None and opts.restart < 1:
        raise ValueError("gmres: restart cycle must be >= 1")
    dev = b.device
    nb = int(n)
    errors = []

    def wrap(f):
        def cb(ctx, d_in, d_out, stream_):
            try:
                x = _device_view(d_in, nb, dev)
                y = _device_view(d_out, nb, dev)
                f(x, y)
                return 0
            except Exception as e:  # reported by the solver as a callback failure
                errors.append(e)
                return 1
        return LINOP_FN(cb)

    fa = wrap(A)
    fp = wrap(P) if P is not None else LINOP_FN()
    x = torch.empty_like(b)
    cap = opts.max_krylov + 2
    hist = np.zeros(cap)
    rep = _GRep(0, 0, 0.0, 0.0, _ptr(hist), cap, 0)
    o = _GOpts(float(opts.tol), int(opts.max_krylov), int(opts.restart or 0))
    st = check_status = lib().stiga_gmres_op(nb, fa, None, fp, None, comm.handle if comm is not None else None,
                                             ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(x.data_ptr()),
                                             ctypes.byref(o), ctypes.byref(rep), _stream_handle(stream))
    if st != 0 and errors:
        raise errors[0]
    check(check_status, "gmres_op")
    return x, SolveReport(rep.iterations, list(hist[: min(cap, rep.history_len)]), bool(rep.converged),
                          rep.wall_time_s, rep.precond_time_fraction)


def _device_view(ptr, n, device):
    """A float64 CUDA tensor viewing n doubles at device address ptr (no copy)."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                    "strides": None}

    return torch.as_tensor(_Arr(), device=device)


def fp64_peak(device=0, ms=200.0):
    """Measured FP64 throughput (DMMA m8n8k4, dependent-chain DFMA) in TFLOP/s."""
    a, b = ctypes.c_double(), ctypes.c_double()
    check(lib().stiga_fp64_peak(int(device), float(ms), ctypes.byref(a), ctypes.byref(b)), "fp64_peak")
    return a.value, b.value
