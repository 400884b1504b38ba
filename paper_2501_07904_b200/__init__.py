"""B200-native TT-UTV engine (arXiv 2501.07904): TT-URV / TT-ULV sweeps on sm_100a.

The computation lives in ``lib/libttutv_b200.so`` (CUDA kernels + C-ABI declared in
``include/ttutv_b200.h``); ``api`` mirrors the reference's C++ API names for Python.
"""
from . import api  # noqa: F401
from ._native import (ArgumentError, CudaError, InvariantError, NumericalError, ParseError,  # noqa: F401
                      ResourceError, TTIndexError, TTUTVError)

__all__ = ["api", "ArgumentError", "CudaError", "InvariantError", "NumericalError", "ParseError",
           "ResourceError", "TTIndexError", "TTUTVError"]
