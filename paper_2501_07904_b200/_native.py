"""ctypes binding of the C-ABI in include/ttutv_b200.h.

The library is loaded from the in-tree build (``lib/libttutv_b200.so``). There is no
fallback: if the library is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libttutv_b200.so"

c_double_p = C.POINTER(C.c_double)
c_int64_p = C.POINTER(C.c_int64)


class TTUTVError(RuntimeError):
    """Base of all library errors (reference ttutv::Error, errors.hpp:10)."""


class ArgumentError(TTUTVError):
    pass


class TTIndexError(TTUTVError):
    pass


class ParseError(TTUTVError):
    """ttutv::ParseError: the message and the byte offset (errors.hpp:28-36)."""

    def __init__(self, msg: str, offset: int = 0):
        super().__init__(f"{msg} (at offset {offset})")
        self.message, self.offset = msg, offset


class NumericalError(TTUTVError):
    pass


class ResourceError(TTUTVError):
    pass


class InvariantError(TTUTVError):
    pass


class CudaError(TTUTVError):
    pass


ERRORS = {1: ArgumentError, 2: TTIndexError, 3: ParseError, 4: NumericalError, 5: ResourceError,
          6: InvariantError, 7: TTUTVError, 8: CudaError}


class Config(C.Structure):
    _fields_ = [
        ("method", C.c_int), ("sweep", C.c_int), ("fixed_rank", C.c_int),
        ("ranks", c_int64_p), ("nranks", C.c_int), ("eps", C.c_double), ("weights", c_double_p),
        ("nweights", C.c_int), ("refine_passes", C.c_int), ("retain", C.c_int),
        ("debug_checks", C.c_int), ("qlp_policy", C.c_int),
    ]


class CompletionConfig(C.Structure):
    """ttg_completion_config (CompletionConfig, completion.hpp:40-55, plus eps)."""
    _fields_ = [
        ("ranks", c_int64_p), ("nranks", C.c_int), ("eps", C.c_double), ("retraction", C.c_int),
        ("step_size", C.c_double), ("max_iters", C.c_int), ("stop_tol", C.c_double),
        ("refine_passes", C.c_int), ("dense_cap", C.c_int64),
    ]


# name -> (restype, argtypes)
SIGNATURES = {
    "ttg_last_error": (C.c_char_p, []),
    "ttg_abi_version": (C.c_int, []),
    "ttg_device_count": (C.c_int, []),
    "ttg_set_device": (C.c_int, [C.c_int]),
    "ttg_kernel_launches": (C.c_int64, []),
    "ttg_synchronize": (C.c_int, []),
    "ttg_reserve": (C.c_int, [C.c_int64]),
    "ttg_stream": (C.c_void_p, []),
    "ttg_profile_enable": (C.c_int, [C.c_int]),
    "ttg_profile_read": (C.c_int64, [c_double_p, c_double_p]),
    "ttg_profile_kernels": (C.c_int, [C.c_int, C.POINTER(C.c_char_p), c_double_p, c_double_p, c_int64_p]),
    "ttg_profile_reset_kernels": (None, []),
    "ttg_profile_big_phases": (C.c_int, [c_double_p, C.c_int]),
    "ttg_last_error_offset": (C.c_int64, []),
    "ttg_tensor_file_header": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), c_int64_p]),
    "ttg_tensor_file_to_device": (C.c_int, [C.c_char_p, C.c_void_p, C.c_int64]),
    "ttg_decompose_file": (C.c_int, [C.c_char_p, C.POINTER(Config), C.POINTER(C.c_void_p)]),
    "ttg_result_write_file": (C.c_int, [C.c_void_p, C.c_char_p]),
    "ttg_decompose": (C.c_int, [C.c_void_p, c_int64_p, C.c_int, C.POINTER(Config), C.c_int, C.POINTER(C.c_void_p)]),
    "ttg_result_free": (None, [C.c_void_p]),
    "ttg_result_order": (C.c_int, [C.c_void_p]),
    "ttg_result_core_dims": (None, [C.c_void_p, C.c_int, c_int64_p]),
    "ttg_result_core_copy": (C.c_int, [C.c_void_p, C.c_int, c_double_p]),
    "ttg_result_core_device": (C.c_void_p, [C.c_void_p, C.c_int]),
    "ttg_result_report": (C.c_int, [C.c_void_p, c_double_p, c_int64_p, c_int64_p, c_double_p,
                                    C.POINTER(C.c_int), c_double_p, c_double_p]),
    "ttg_result_warning_count": (C.c_int, [C.c_void_p]),
    "ttg_result_warning": (C.c_char_p, [C.c_void_p, C.c_int]),
    "ttg_result_cut_diag": (C.c_int, [C.c_void_p, C.c_int, c_double_p, C.c_int, c_int64_p]),
    "ttg_result_direct_errors": (C.c_int, [C.c_void_p, c_double_p]),
    "ttg_mode_product": (C.c_int, [c_double_p, c_int64_p, C.c_int, C.c_int, c_double_p, C.c_int64, C.c_int64,
                                   c_double_p]),
    "ttg_kron": (C.c_int, [c_double_p, C.c_int64, C.c_int64, c_double_p, C.c_int64, C.c_int64, c_double_p]),
    "ttg_sum_squares": (C.c_int, [C.c_void_p, C.c_int64, C.c_int, c_double_p]),
    "ttg_complete": (C.c_int, [c_int64_p, c_double_p, C.c_int64, c_int64_p, C.c_int, C.c_void_p, c_double_p, C.c_int,
                               C.POINTER(C.c_void_p)]),
    "ttg_completion_free": (None, [C.c_void_p]),
    "ttg_completion_iterations": (C.c_int, [C.c_void_p]),
    "ttg_completion_status": (C.c_int, [C.c_void_p]),
    "ttg_completion_note": (C.c_char_p, [C.c_void_p]),
    "ttg_completion_trace": (None, [C.c_void_p, c_double_p, c_double_p, c_double_p, c_double_p, c_double_p]),
    "ttg_completion_ranks": (C.c_int, [C.c_void_p, C.c_int, c_int64_p]),
    "ttg_completion_result": (C.c_void_p, [C.c_void_p]),
    "ttg_gemm_device": (C.c_int, [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_void_p,
                                  C.c_int64, C.c_void_p, C.c_int64, C.c_double, C.c_void_p, C.c_int64]),
    "ttg_comm_callback_create": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "ttg_psnr": (C.c_int, [c_double_p, c_double_p, C.c_int64, c_double_p]),
    "ttg_reverse_indices": (C.c_int, [c_double_p, c_int64_p, C.c_int, c_double_p]),
    "ttg_reverse_tt": (C.c_int, [c_double_p, c_int64_p, c_int64_p, C.c_int, c_double_p]),
    "ttg_result_cut_kept": (C.c_int, [C.c_void_p, C.c_int, c_double_p, C.c_int]),
    "ttg_verify_bound": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_double, c_double_p]),
    "ttg_result_rse": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, c_double_p]),
    "ttg_result_reconstruct": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "ttg_completion_reset": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, c_double_p]),
    "ttg_comm_nccl_unique_id": (C.c_int, [C.POINTER(C.c_ubyte)]),
    "ttg_comm_nccl_create": (C.c_int, [C.POINTER(C.c_ubyte), C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "ttg_comm_loopback_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "ttg_comm_free": (None, [C.c_void_p]),
    "ttg_shard_range": (C.c_int, [c_int64_p, C.c_int, C.c_int, C.c_int, C.c_int, c_int64_p]),
    "ttg_decompose_sharded": (C.c_int, [C.c_void_p, c_int64_p, C.c_int, C.POINTER(Config), C.c_int, C.c_void_p,
                                        C.POINTER(C.c_void_p)]),
    "ttg_qr_col_pivot": (C.c_int, [c_double_p, C.c_int64, C.c_int64, c_double_p, c_double_p, c_int64_p]),
    "ttg_utv": (C.c_int, [c_double_p, C.c_int64, C.c_int64, C.c_int, C.c_int, c_double_p, c_double_p, c_double_p]),
    "ttg_svd": (C.c_int, [c_double_p, C.c_int64, C.c_int64, C.c_int, C.c_double, c_double_p, c_double_p,
                          c_double_p]),
    "ttg_truncate": (C.c_int, [C.c_int, c_double_p, c_double_p, c_double_p, C.c_int64, C.c_int64, C.c_int64,
                               C.c_int64, C.c_double, c_int64_p, c_double_p, c_double_p, c_double_p,
                               c_double_p]),
    "ttg_reconstruct": (C.c_int, [c_double_p, c_int64_p, c_int64_p, C.c_int, C.c_int64, c_double_p]),
    "ttg_frobenius_norm": (C.c_int, [C.c_void_p, C.c_int64, C.c_int, c_double_p]),
    "ttg_rse": (C.c_int, [c_double_p, c_double_p, C.c_int64, c_double_p]),
    "ttg_diff_norm": (C.c_int, [c_double_p, c_double_p, C.c_int64, c_double_p]),
    "ttg_matmul": (C.c_int, [c_double_p, C.c_int64, C.c_int64, C.c_int, c_double_p, C.c_int64, C.c_int64, C.c_int,
                             c_double_p]),
}

_lib = None


def lib() -> C.CDLL:
    """Load (once) and return the native library; raises if it is not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"native engine not built: {LIB_PATH} missing (run __graft_entry__.build())")
        # RTLD_LOCAL: the drop-in C++ layer exports the reference's ttutv:: symbol names;
        # keeping them out of the global scope stops them interposing on the reference
        # library that the tests load as the oracle.
        handle = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().ttg_last_error().decode(errors="replace")
        if status == 3:
            raise ParseError(msg, int(lib().ttg_last_error_offset()))
        raise ERRORS.get(status, TTUTVError)(msg)


def require_gpu() -> None:
    if lib().ttg_device_count() < 1:
        raise CudaError("no CUDA device visible: the TT-UTV engine has no CPU path")
