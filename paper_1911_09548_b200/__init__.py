"""B200-native space-time multigrid for the eddy-current equation (arXiv:1911.09548).

The product path is libst.so (CUDA kernels for sm_100a behind the C-ABI of
include/st.h) and the ctypes binding in ``binding.py``.  This package never
imports ``oracle`` (the CPU test oracle)."""
from .binding import EXPORTED, Solver, StError, host_matrix, kernel_variants, load, plan  # noqa: F401
