"""paper_2512_04406_b200 — B200-native (sm_100a, fp64) hot path of ManiDSDP (arXiv 2512.04406).

The product is the C-ABI library ``libdrsdp.so`` (include/drsdp.h). This package holds its CUDA/C++
sources (``csrc/``), the in-tree build (``build.py``) and a thin ctypes binding (``abi.py``) that
only marshals arguments: every step of the path runs in the library's kernels. There is no CPU
fallback: without the built library or a CUDA device the binding raises.
"""
from .abi import Context, DrsdpError, lib_path, load_library  # noqa: F401
