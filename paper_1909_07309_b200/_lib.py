"""ctypes binding of libstiga_gpu.so (the C ABI declared in include/stiga_gpu.h).

There is deliberately no fallback: if the shared library is missing the import fails loudly
(run `python -c "import __graft_entry__ as g; g.build()"` or `make -C paper_1909_07309_b200/csrc`).
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# STIGA_LIB_PATH: an alternative in-tree build (kernel A/B experiments); default lib/libstiga_gpu.so
LIB_PATH = os.environ.get("STIGA_LIB_PATH") or os.path.join(_HERE, "lib", "libstiga_gpu.so")

OK, INVALID_ARGUMENT, NUMERICAL, CUDA = 0, 1, 2, 3

_c_int, _c_ll, _c_dbl, _vp = ctypes.c_int, ctypes.c_longlong, ctypes.c_double, ctypes.c_void_p
_pd = ctypes.POINTER(ctypes.c_double)
_pi = ctypes.POINTER(ctypes.c_int)
_ppd = ctypes.POINTER(_pd)


class FdSetupOptions(ctypes.Structure):
    _fields_ = [("flags", ctypes.c_int), ("d_scaling", ctypes.c_void_p)]


SETUP_DEVICE_SCHUR, SETUP_CUSOLVER = 1, 2


class GmresOptions(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("max_krylov", ctypes.c_int), ("restart", ctypes.c_int)]


class GmresReport(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("converged", ctypes.c_int), ("wall_time_s", ctypes.c_double),
                ("precond_time_fraction", ctypes.c_double), ("residual_history", _pd),
                ("history_capacity", ctypes.c_int), ("history_len", ctypes.c_int)]


MAX_RANKS = 8
IPC_HANDLE_BYTES = 64


class ScatterDesc(ctypes.Structure):
    _fields_ = [("world", ctypes.c_int), ("by_time", ctypes.c_int), ("offsets", ctypes.c_longlong * (MAX_RANKS + 1)),
                ("ld", ctypes.c_longlong * MAX_RANKS), ("a_shift", ctypes.c_longlong), ("b_shift", ctypes.c_longlong),
                ("dst", ctypes.c_void_p * MAX_RANKS)]


COMM_ID_BYTES = 128
# int (*)(void* ctx, double* buf, int n, int op) / (ctx, send, bytes, recv) / (ctx)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                                ctypes.c_int)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p)
BARRIER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)
# int (*)(void* ctx, const double* d_in, double* d_out, void* stream)
LINOP_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class CommCallbacks(ctypes.Structure):
    _fields_ = [("ctx", ctypes.c_void_p), ("allreduce", ALLREDUCE_FN), ("allgather", ALLGATHER_FN),
                ("barrier", BARRIER_FN)]


# name -> (restype, argtypes); every symbol of include/stiga_gpu.h
SIGNATURES = {
    "stiga_last_error": (ctypes.c_char_p, []),
    "stiga_abi_version": (_c_int, []),
    "stiga_device_count": (_c_int, []),
    "stiga_space_dim": (_c_int, [_c_int, _c_int, _c_int, _pi]),
    "stiga_assemble_time_matrices": (_c_int, [_c_int, _c_int, _c_dbl, _pd, _pd]),
    "stiga_assemble_spatial_parametric": (_c_int, [_c_int, _c_int, _c_int, _pd, _pd]),
    "stiga_assemble_univariate": (_c_int, [_c_int, _c_int, _c_int, _c_int, _c_int, _c_int, _pd, _pd]),
    "stiga_problem_create": (_c_int, [ctypes.c_char_p, ctypes.POINTER(_vp)]),
    "stiga_problem_destroy": (_c_int, [_vp]),
    "stiga_problem_dim": (_c_int, [_vp, _pi]),
    "stiga_problem_eval_geometry": (_c_int, [_vp, _pd, _pd, _pd]),
    "stiga_problem_eval_fields": (_c_int, [_vp, _pd, _pd, _pd]),
    "stiga_geometry_preconditioner_pieces": (_c_int, [_vp, _c_int, _c_int, _pd, _pd, _pd, _pd, _pd, _pd, _pd, _pd, _pi]),
    "stiga_problem_info": (_c_int, [_vp, _pi, _pd, _pi, _pi, _pd, _pd]),
    "stiga_system_means": (_c_int, [_vp, _c_int, _c_int, _pd, _pd]),
    "stiga_assemble_rhs": (_c_int, [_vp, _c_int, _c_int, _c_int, _c_int, _vp, _vp]),
    "stiga_compute_errors": (_c_int, [_vp, _c_int, _c_int, _vp, _c_int, _c_int, _pd, _pd]),
    "stiga_fd_setup": (_c_int, [_c_int, _pi, _ppd, _ppd, _c_int, _pd, _pd, _c_dbl, _c_dbl, _pd, _c_ll, _c_int,
                                ctypes.POINTER(_vp)]),
    "stiga_fd_setup_ex": (_c_int, [_c_int, _pi, _ppd, _ppd, _c_int, _pd, _pd, _c_dbl, _c_dbl, _pd, _c_ll, _vp, _c_int,
                                   ctypes.POINTER(_vp)]),
    "stiga_fd_destroy": (_c_int, [_vp]),
    "stiga_fd_size": (_c_int, [_vp, ctypes.POINTER(_c_ll)]),
    "stiga_fd_dims": (_c_int, [_vp, _pi, _pi]),
    "stiga_fd_time_info": (_c_int, [_vp, _pi, _pi, _pd, _pd]),
    "stiga_fd_export": (_c_int, [_vp, _c_int, _c_int, _pd, _c_ll]),
    "stiga_fd_apply": (_c_int, [_vp, _vp, _vp, _vp]),
    "stiga_fd_apply_host": (_c_int, [_vp, _pd, _pd]),
    "stiga_fd_apply_profiled": (_c_int, [_vp, _vp, _vp, _vp, ctypes.POINTER(ctypes.c_float)]),
    "stiga_fd_launches": (_c_int, [_vp, _pi]),
    "stiga_fd_launch_info": (_c_int, [_vp, _c_int, ctypes.c_char_p, _c_int, _pd]),
    "stiga_fd_apply_space": (_c_int, [_vp, _c_int, _c_ll, _c_ll, _vp, _vp, _vp]),
    "stiga_fd_apply_time": (_c_int, [_vp, _c_ll, _c_ll, _vp, _vp, _vp]),
    "stiga_fd_apply_space_scatter": (_c_int, [_vp, _c_ll, _c_ll, _vp, ctypes.POINTER(ScatterDesc), _vp]),
    "stiga_fd_apply_time_scatter": (_c_int, [_vp, _c_ll, _c_ll, _vp, ctypes.POINTER(ScatterDesc), _vp]),
    "stiga_device_alloc": (_c_int, [_c_ll, _c_int, ctypes.POINTER(_vp)]),
    "stiga_device_free": (_c_int, [_vp]),
    "stiga_ipc_handle": (_c_int, [_vp, ctypes.c_char_p]),
    "stiga_ipc_open": (_c_int, [ctypes.c_char_p, _c_int, ctypes.POINTER(_vp)]),
    "stiga_ipc_close": (_c_int, [_vp]),
    "stiga_copy_blocks": (_c_int, [_vp, _c_ll, _vp, _c_ll, _c_ll, _c_ll, _vp]),
    "stiga_kron_matvec": (_c_int, [_c_int, _pi, _pi, _ppd, _vp, _vp, _c_int, _vp]),
    "stiga_kronsum_create": (_c_int, [_c_int, _pi, _c_int, _pd, _ppd, _c_int, ctypes.POINTER(_vp)]),
    "stiga_kronsum_create_spacetime": (_c_int, [_c_int, _pi, _ppd, _ppd, _c_int, _pd, _pd, _c_dbl, _c_dbl, _c_int,
                                                ctypes.POINTER(_vp)]),
    "stiga_kronsum_create_physical": (_c_int, [_vp, _c_int, _c_int, _c_int, ctypes.POINTER(_vp)]),
    "stiga_kronsum_destroy": (_c_int, [_vp]),
    "stiga_kronsum_size": (_c_int, [_vp, ctypes.POINTER(_c_ll)]),
    "stiga_kronsum_apply": (_c_int, [_vp, _vp, _vp, _vp]),
    "stiga_kronsum_diagonal": (_c_int, [_vp, _pd]),
    "stiga_kronsum_diagonal_device": (_c_int, [_vp, _vp, _vp]),
    "stiga_geometry_scaling_device": (_c_int, [_vp, _vp, _vp, _vp]),
    "stiga_gmres": (_c_int, [_vp, _vp, _vp, _vp, ctypes.POINTER(GmresOptions), ctypes.POINTER(GmresReport), _vp]),
    "stiga_fp64_peak": (_c_int, [_c_int, _c_dbl, _pd, _pd]),
    "stiga_kronsum_time_halfband": (_c_int, [_vp, _pi]),
    "stiga_kronsum_dims": (_c_int, [_vp, _pi, _pi, _c_int]),
    "stiga_kronsum_apply_space": (_c_int, [_vp, _c_ll, _vp, _vp, _vp, _vp]),
    "stiga_kronsum_apply_time": (_c_int, [_vp, _c_ll, _c_ll, _c_int, _c_int, _vp, _vp, _vp, _vp]),
    "stiga_vec_dot": (_c_int, [_vp, _vp, _c_ll, _vp, _vp]),
    "stiga_vec_axpy": (_c_int, [_c_dbl, _vp, _vp, _c_ll, _vp]),
    "stiga_vec_multidot": (_c_int, [ctypes.POINTER(_vp), _c_int, _vp, _c_ll, _vp, _vp]),
    "stiga_vec_multiaxpy": (_c_int, [_pd, ctypes.POINTER(_vp), _c_int, _vp, _c_ll, _vp]),
    "stiga_vec_scal": (_c_int, [_c_dbl, _vp, _vp, _c_ll, _vp]),
    "stiga_comm_unique_id": (_c_int, [ctypes.c_char_p]),
    "stiga_comm_init_nccl": (_c_int, [_c_int, _c_int, ctypes.c_char_p, _c_int, ctypes.POINTER(_vp)]),
    "stiga_comm_init_host": (_c_int, [_c_int, _c_int, ctypes.POINTER(CommCallbacks), _c_int, ctypes.POINTER(_vp)]),
    "stiga_comm_destroy": (_c_int, [_vp]),
    "stiga_comm_info": (_c_int, [_vp, _pi, _pi, _pi, _pi]),
    "stiga_comm_allreduce": (_c_int, [_vp, _vp, _c_ll, _vp]),
    "stiga_shard_partition": (_c_int, [_c_ll, _c_int, _c_int, ctypes.POINTER(_c_ll), ctypes.POINTER(_c_ll)]),
    "stiga_fd_setup_sharded": (_c_int, [_c_int, _pi, _ppd, _ppd, _c_int, _pd, _pd, _c_dbl, _c_dbl, _pd, _c_ll, _vp,
                                        ctypes.POINTER(_vp)]),
    "stiga_fd_local": (_c_int, [_vp, ctypes.POINTER(_c_ll), ctypes.POINTER(_c_ll), ctypes.POINTER(_c_ll),
                                ctypes.POINTER(_c_ll)]),
    "stiga_kronsum_create_spacetime_sharded": (_c_int, [_c_int, _pi, _ppd, _ppd, _c_int, _pd, _pd, _c_dbl, _c_dbl,
                                                        _vp, ctypes.POINTER(_vp)]),
    "stiga_kronsum_create_physical_sharded": (_c_int, [_vp, _c_int, _c_int, _vp, ctypes.POINTER(_vp)]),
    "stiga_kronsum_local": (_c_int, [_vp, ctypes.POINTER(_c_ll), ctypes.POINTER(_c_ll), ctypes.POINTER(_c_ll),
                                     ctypes.POINTER(_c_ll)]),
    "stiga_gmres_op": (_c_int, [_c_ll, LINOP_FN, _vp, LINOP_FN, _vp, _vp, _vp, _vp, ctypes.POINTER(GmresOptions),
                                ctypes.POINTER(GmresReport), _vp]),
}

_lib = None


def lib():
    """Loads (once) and returns the CDLL; raises ImportError if the library was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libstiga_gpu.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class StigaError(RuntimeError):
    pass


def check(status, what=""):
    """Maps C-ABI status codes to the reference's exception types (SURVEY §8(b) Errors)."""
    if status == OK:
        return
    msg = lib().stiga_last_error().decode()
    if status == INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == NUMERICAL:
        raise RuntimeError(msg)
    raise StigaError(f"CUDA failure in {what}: {msg}")
