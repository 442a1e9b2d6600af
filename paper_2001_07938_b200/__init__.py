"""lilac-b200: a B200-native backend for the LiLAC-How harness path of
arXiv 2001.07938 (CSR/JDS SpMV, dot/axpy companions, resident-device
marshaling, NPB CG driver, row-sharded multi-GPU driver).

The product is the native library liblilac_b200.so (C ABI:
include/lilac_b200.h). This package only loads it and mirrors its interface.
"""
from . import _native  # noqa: F401

__version__ = "0.1"


def library_path() -> str:
    return _native.LIB_PATH
