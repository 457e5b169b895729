"""ctypes declarations of include/dot_b200.h (argument marshalling only)."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DOT_LIB_PATH") or os.path.join(_HERE, "lib", "libdot_b200.so")

DOT_OK, DOT_ERR_ARG, DOT_ERR_CUDA, DOT_ERR_STATE, DOT_ERR_NOCONV, DOT_ERR_WORKSPACE, DOT_ERR_BREAKDOWN = range(7)
DOT_HOST, DOT_DEVICE = 0, 1

dp = C.POINTER(C.c_double)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)


class DotConfig(C.Structure):
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
        ("Lx", C.c_double), ("Ly", C.c_double), ("Lz", C.c_double),
        ("D", C.c_double), ("mua_in", C.c_double), ("mua_out", C.c_double), ("nu", C.c_double),
        ("n_freq", C.c_int32), ("omega", dp),
        ("n_src", C.c_int32), ("src_nodes", i64p),
        ("n_det", C.c_int32), ("det_nodes", i64p),
        ("n_rbf", C.c_int32),
        ("gamma", C.c_double), ("eps", C.c_double), ("cutoff", C.c_double),
        ("tol", C.c_double), ("max_iter", C.c_int32),
    ]


class DotTransport(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("sendrecv", C.c_void_p), ("allreduce_sum", C.c_void_p)]


class DotStats(C.Structure):
    _fields_ = [
        ("rhs_solved", C.c_int64), ("rhs_iterations", C.c_int64),
        ("last_max_iters", C.c_int32), ("last_min_iters", C.c_int32),
        ("kernel_launches", C.c_int64), ("pass_launches", C.c_int64),
        ("pass_ms", C.c_double), ("pass_bytes", C.c_double),
        ("contract_ms", C.c_double), ("contract_flops", C.c_double),
        ("support_K", C.c_int32), ("n_samples", C.c_int32),
        ("contract_flops_dense", C.c_double),
        ("seeds_solved", C.c_int64), ("seed_iterations", C.c_int64),
        ("contract_dmma_flops", C.c_double),
        ("gemm_ms", C.c_double), ("gemm_flops", C.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# name -> (restype, argtypes)
SIGNATURES = {
    "dot_version": (C.c_char_p, []),
    "dot_last_error": (C.c_char_p, [C.c_void_p]),
    "dot_create": (C.c_int, [C.POINTER(DotConfig), C.POINTER(C.c_void_p)]),
    "dot_destroy": (C.c_int, [C.c_void_p]),
    "dot_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "dot_workspace_bytes": (C.c_size_t, [C.c_void_p, C.c_int32]),
    "dot_bind_workspace": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
    "dot_enable_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "dot_get_stats": (C.c_int, [C.c_void_p, C.POINTER(DotStats)]),
    "dot_reset_stats": (C.c_int, [C.c_void_p]),
    "dot_set_data": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "dot_set_params": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "dot_misfit": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int, dp, C.c_void_p]),
    "dot_jacobian": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int, C.c_void_p]),
    "dot_optimize_directions": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                                          C.c_int, C.c_void_p, C.c_void_p, dp]),
    "dot_optimize_directions_subspace": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                                   C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                                   C.c_int, C.c_void_p, C.c_void_p, dp]),
    "dot_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "dot_dd_create": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)]),
    "dot_dd_create_transport": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)]),
    "dot_dd_fields": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int]),
    "dot_dd_last_error": (C.c_char_p, [C.c_void_p]),
    "dot_dd_destroy": (C.c_int, [C.c_void_p]),
    "dot_prefetch_fields": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int]),
    "dot_absorption": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "dot_support": (C.c_int, [C.c_void_p, i32p, C.c_void_p, C.c_void_p, C.c_int]),
    "dot_apply": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_int]),
    "dot_solve": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, i32p]),
    "dot_solve_sampled": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int, C.c_void_p]),
    "dot_samples": (C.c_int, [C.c_void_p, i32p, C.c_void_p, C.c_int]),
    "dot_fields_on_support": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int, C.c_void_p]),
    "dot_contract_fields": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "dot_contract": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "dot_sym_eig": (C.c_int, [C.c_int, dp, dp, dp]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load libdot_b200.so; raises if it is missing (no fallback of any kind)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -m paper_1706_05586_b200.build` "
            "(the DOT hot path has no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class DotError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[dot error {code}] {msg}")
        self.code = code


def check(code, handle=None):
    if code != DOT_OK:
        lib = load()
        msg = lib.dot_last_error(handle)
        raise DotError(code, msg.decode() if msg else "")
