"""B200-native CGX compressed-allreduce hot path (arXiv 2111.08617).

libgcx.so      sm_100a kernels behind the C-ABI in include/gcx.h
_gcomm*.so     C++ host façade mirroring the reference's gcomm:: API
               (codec / collectives / model / engine), with pybind11 bindings
device.py      zero-copy torch-tensor calls over the C-ABI
"""
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
__all__ = ["PKG_DIR"]
