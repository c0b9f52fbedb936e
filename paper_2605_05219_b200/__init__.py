"""paper_2605_05219_b200 -- B200-native hot path of sparse prefix caching (arXiv 2605.05219).

The product is the C-ABI library ``libsparseprefix.so`` (CUDA, sm_100a) declared in
``include/sparse_prefix.h``; :mod:`paper_2605_05219_b200.sp` is the thin ctypes binding with the
same names.  Nothing here imports the CPU oracle, and there is no CPU fallback.
"""
__all__ = ["sp", "workload", "dist"]


def __getattr__(name):
    import importlib
    if name in __all__:
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
