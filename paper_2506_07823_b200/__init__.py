"""pdilqr-b200: B200-native (sm_100a) batched Primal-Dual iLQR hot path (arXiv 2506.07823).

The compute path is libpdilqr.so (CUDA kernels behind the C ABI of include/pdilqr.h); this
package is a thin ctypes binding.  There is no CPU fallback.
"""
from .pdilqr import PdIlqr, PdilqrError, lib, LIB_PATH, EXPORTED  # noqa: F401
from .closed_loop import ClosedLoop  # noqa: F401
from .autograd import lq_solve, LqSolveFunction  # noqa: F401

__all__ = ["PdIlqr", "PdilqrError", "ClosedLoop", "lq_solve", "LqSolveFunction", "lib", "LIB_PATH", "EXPORTED"]
