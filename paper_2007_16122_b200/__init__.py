"""B200-native COLD online pre-ranking scorer (arXiv 2007.16122).

The product is libcold.so (C ABI in include/cold.h; CUDA kernels for sm_100a in csrc/).
`cold` is the thin ctypes binding used by the tests and bench.py.
"""
from .cold import Batch, ColdError, Context, Server, lib, select_groups, vps_score  # noqa: F401
