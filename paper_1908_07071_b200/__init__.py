"""B200-native LOR additive-Schwarz preconditioned matrix-free PCG (arXiv 1908.07071).

The product is the C-ABI library `liblorpc.so` (CUDA, sm_100a, FP64; header
`include/lorpc.h`); `lorpc` is its thin ctypes binding.
"""
from . import lorpc  # noqa: F401
from .lorpc import Mesh, Lor, Prec, pcg_solve, pcg_solve_host, LorpcError  # noqa: F401
