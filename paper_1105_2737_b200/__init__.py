"""B200-native FFT spectral synthesis of stationary Gaussian random fields.

Drop-in for the reference core generator ``grf::synthesize``
(/root/reference/proj/core). The product is the CUDA (sm_100a) library
``lib/libgrfc.so`` behind the C-ABI in ``include/grfc.h``; ``grfc`` is its
ctypes mirror and ``cpp/`` the C++ ``grf::`` drop-in.
"""
from . import grfc  # noqa: F401  (raises if the CUDA library is missing)

__all__ = ["grfc"]
