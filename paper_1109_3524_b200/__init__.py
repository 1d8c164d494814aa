"""B200-native (sm_100a) IBPM sparse linear-algebra hot path.

The product is libibmgpu.so (C-ABI in include/ibmgpu.h); `ibm` mirrors the reference's
operator interface on top of it. There is no CPU fallback.
"""
from . import _lib  # noqa: F401

__all__ = ["ibm"]
