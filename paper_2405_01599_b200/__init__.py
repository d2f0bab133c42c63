"""paper_2405_01599_b200 -- B200-native (sm_100a) CRS SpMV engine with the
capabilities of Xabclib/OpenATLib's SpMV hot path (arXiv 2405.01599).

The product is libktb.so (C ABI, include/ktb.h; CUDA kernels in csrc/).
`ktune` mirrors the reference's C++ operator interface for Python callers and
tests; `dist` holds the multi-GPU row-block sharding. Importing this package
fails loudly when the CUDA library has not been built: there is no CPU path.
"""
from . import _lib

_lib.load()

from . import ktune  # noqa: E402,F401

__all__ = ["ktune"]
