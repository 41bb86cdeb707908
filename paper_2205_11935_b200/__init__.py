"""B200-native CKKS encrypted-dense-layer hot path of CryptoTL (arXiv 2205.11935).

The product is the C-ABI library `_build/libckks_b200.so` (include/ckks.h) built from csrc/ for
sm_100a; `ckks` is its ctypes binding.  There is no CPU fallback.
"""
from .ckks import (ACT_CUBIC, ACT_NONE, ACT_SQUARE, Ciphertext, CkksError, Context, Layer, Model,  # noqa: F401
                   lib, lib_path)

__all__ = ["Context", "Layer", "Model", "Ciphertext", "CkksError", "lib", "lib_path",
           "ACT_NONE", "ACT_SQUARE", "ACT_CUBIC"]
