"""hfmm-b200: B200-native FMM Helmholtz matvec behind the reference's solver interface.

The product is ``libhfmm_b200.so`` (C ABI in ``include/hfmm_cuda.h``, CUDA kernels in ``csrc/``);
this package is the thin ctypes binding used by tests and ``bench.py``.
"""
from .api import HfmmCuda, HfmmError, build_library, library_path  # noqa: F401
from . import workloads  # noqa: F401
