"""paper_2510_02676_b200 -- B200-native ECF8 (lossless FP8 weight) decoding.

Layers:
  _lib      ctypes binding of libecf8_b200.so (C ABI: include/ecf8_cuda.h,
            include/ecf8_host.h)
  codec     Python mirror of the reference's ecf8 API (encode on host,
            decode on the B200)
  device    device-resident tensors / batches driven from torch streams
"""
from . import _lib
from ._lib import CudaError, Ecf8Error, FormatError, InvalidArgument, IoError, device_count

__all__ = ["_lib", "CudaError", "Ecf8Error", "FormatError", "InvalidArgument", "IoError", "device_count"]
