"""B200-native column-graph max-flow / min-cut (hot path of arXiv 2601.17026).

The product is libcolgraph.so (C ABI in include/colgraph.h, sm_100a kernels in
csrc/).  `colgraph` is its thin ctypes binding.  Build with
`python -m paper_2601_17026_b200.build`.
"""
__all__ = ["colgraph", "build"]
