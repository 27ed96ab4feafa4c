"""LinPrim (arXiv 2501.16312) differentiable polyhedron tile rasterizer, B200-native.

The product is the C-ABI library ``liblinprim.so`` (CUDA sm_100a, sources in ``csrc/``,
declarations in ``include/linprim.h``).  ``linprim`` is the thin ctypes binding with the
same names; it raises at import when the library is missing (no CPU fallback).
``scenegen`` draws seeded synthetic inputs and holds none of the method's arithmetic.
"""
