"""B200-native visibility engine for LoBE-GS (arXiv 2510.01767).

The product path is the C-ABI library csrc/liblobe.so (include/lobe.h) with
hand-written sm_100a kernels; `lobe` is its ctypes binding and `engine` the
multi-GPU exchange layer over torch.distributed. Nothing here imports the
oracle, and there is no CPU fallback.
"""
from . import lobe  # noqa: F401  (binding only; the .so is loaded on first use)

__all__ = ["lobe"]
