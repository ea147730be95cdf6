"""B200-native BBC query hot path (arXiv 2604.01960): C-ABI library libbbc.so + thin binding.

The product path is `bbc.Index` (ivf_load / bbc_search ...).  It never imports `oracle/`.
"""
from .bbc import BBCError, Index, launch_count, lib  # noqa: F401
