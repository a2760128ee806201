"""B200-native hybrid recompression of directional H^2-matrices (arXiv 1809.04384).

The product is libdh2.so (C ABI in include/dh2.h, sm_100a kernels in csrc/);
``dh2`` is its thin ctypes binding.
"""
from .dh2 import (DH2, DH2Error, DH2_ORIG, DH2_RECOMP, EXPORTED, MODES, load_library, nccl_unique_id)

__all__ = ["DH2", "DH2Error", "DH2_ORIG", "DH2_RECOMP", "EXPORTED", "MODES", "load_library", "nccl_unique_id"]
