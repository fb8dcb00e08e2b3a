"""ctypes binding of the product library (include/ecf8_cuda.h, include/ecf8_host.h,
include/ecf8_e5m2.h).

The shared object is built in-tree by ``make`` (see __graft_entry__.build) at
paper_2510_02676_b200/lib/libecf8_b200.so.  Importing this module never
compiles anything and never falls back to Python: if the library is missing
the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# ECF8_LIB: load an alternative build (A/B kernel experiments, tools/build_variant.sh)
LIB_PATH = os.environ.get("ECF8_LIB") or os.path.join(_HERE, "lib", "libecf8_b200.so")

ECF8_OK, ECF8_EINVAL, ECF8_EFORMAT, ECF8_ECUDA, ECF8_ENOMEM, ECF8_EIO = range(6)


class Ecf8Error(Exception):
    """Base class; ``status`` is the ecf8_status code."""

    status = -1


class InvalidArgument(Ecf8Error, ValueError):  # std::invalid_argument
    status = ECF8_EINVAL


class FormatError(Ecf8Error, ValueError):  # ecf8::FormatError
    status = ECF8_EFORMAT


class CudaError(Ecf8Error, RuntimeError):  # CUDA failure / no device
    status = ECF8_ECUDA


class OutOfMemory(Ecf8Error, MemoryError):
    status = ECF8_ENOMEM


class IoError(Ecf8Error, OSError):  # ecf8::IoError
    status = ECF8_EIO


_ERRORS = {c.status: c for c in (InvalidArgument, FormatError, CudaError, OutOfMemory, IoError)}


class Sections(C.Structure):
    """ecf8_sections: one tensor's container sections."""

    _fields_ = [
        ("n_elem", C.c_uint64),
        ("threads_per_block", C.c_uint32),
        ("lengths", C.c_uint8 * 16),
        ("encoded", C.c_void_p),
        ("encoded_len", C.c_uint64),
        ("gaps", C.c_void_p),
        ("gaps_len", C.c_uint64),
        ("outpos", C.c_void_p),
        ("n_outpos", C.c_uint64),
        ("packed", C.c_void_p),
        ("packed_len", C.c_uint64),
    ]


class E5Sections(C.Structure):
    """ecf8_e5_sections: one tensor of the native E5M2 variant (include/ecf8_e5m2.h)."""

    _fields_ = [
        ("n_elem", C.c_uint64),
        ("threads_per_block", C.c_uint32),
        ("lengths", C.c_uint8 * 32),
        ("encoded", C.c_void_p),
        ("encoded_len", C.c_uint64),
        ("gaps", C.c_void_p),
        ("gaps_len", C.c_uint64),
        ("outpos", C.c_void_p),
        ("n_outpos", C.c_uint64),
        ("raw", C.c_void_p),
        ("raw_len", C.c_uint64),
    ]


class EntropyReport(C.Structure):
    """ecf8_entropy_report: make_stats' EntropyReport for one tensor."""

    _fields_ = [("n_elem", C.c_uint64)] + [
        (f, C.c_double)
        for f in ("entropy_bits", "bits_per_symbol", "bits_per_weight", "bound_lower", "bound_upper",
                  "projected_savings", "actual_savings")
    ]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
        "there is no Python/CPU fallback for the ECF8 decoder"
    )

lib = C.CDLL(LIB_PATH)

_P = C.c_void_p
_U8P = C.POINTER(C.c_uint8)
_U32P = C.POINTER(C.c_uint32)
_U64P = C.POINTER(C.c_uint64)

_SIGS = {
    # ecf8_cuda.h
    "ecf8_last_error": (C.c_char_p, []),
    "ecf8_device_count": (C.c_int, []),
    "ecf8_build_info": (C.c_char_p, []),
    "ecf8_decode_host": (C.c_int, [C.POINTER(Sections), _P, C.c_uint64]),
    "ecf8_decode_host_many": (C.c_int, [C.POINTER(C.POINTER(Sections)), C.POINTER(_P), C.POINTER(C.c_uint64), C.c_int]),
    "ecf8_decode_block_host": (C.c_int, [C.POINTER(Sections), C.c_uint64, _P, C.c_uint64]),
    "ecf8_count_window": (C.c_int, [_P, C.c_uint, _P, _U32P]),
    "ecf8_tensor_upload": (C.c_int, [C.POINTER(Sections), _P, C.POINTER(_P)]),
    "ecf8_tensor_free": (None, [_P]),
    "ecf8_exponent_histogram": (C.c_int, [_P, C.c_uint64, _U64P, _P]),
    "ecf8_encode_device": (C.c_int, [_P, C.c_uint64, C.c_uint32, _P, _P, C.POINTER(_P)]),
    "ecf8_tensor_sections": (C.c_int, [_P, C.POINTER(Sections)]),
    "ecf8_make_stats_device": (C.c_int, [_P, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, _P,
                                         C.POINTER(EntropyReport)]),
    "ecf8_tensor_download": (C.c_int, [_P, _P, _P, _P, _P]),
    "ecf8_tensor_n_elem": (C.c_uint64, [_P]),
    "ecf8_tensor_kernel_variant": (C.c_int, [_P]),
    "ecf8_tensor_verified_tiles": (C.c_uint64, [_P, C.POINTER(C.c_uint64)]),
    "ecf8_tensor_algorithmic_bytes": (C.c_uint64, [_P]),
    "ecf8_tensor_device_bytes": (C.c_uint64, [_P]),
    "ecf8_decode_device": (C.c_int, [_P, _P, _P]),
    "ecf8_batch_create": (C.c_int, [C.POINTER(_P), C.POINTER(_P), C.c_int, C.POINTER(_P)]),
    "ecf8_batch_decode": (C.c_int, [_P, _P]),
    "ecf8_batch_free": (None, [_P]),
    "ecf8_batch_launches": (C.c_int, [_P]),
    "ecf8_fused_create": (C.c_int, [_P, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(_P)]),
    "ecf8_fused_gemm": (C.c_int, [_P, _P, C.c_uint32, C.c_float, _P, _P]),
    "ecf8_fused_split_k": (C.c_int, [_P]),
    "ecf8_fused_decode_rows": (C.c_int, [_P, C.c_uint64, C.c_uint64, _P, _P]),
    "ecf8_fused_byte_steps": (C.c_int, [_P]),
    "ecf8_fused_free": (None, [_P]),
    "ecf8_fused_layout_device": (C.c_int, [_P, C.c_uint64, C.c_uint64, _P, C.c_int, _P]),
    # ecf8_host.h
    "ecf8_host_free": (None, [_P]),
    "ecf8_host_fused_layout": (C.c_int, [_P, C.c_uint64, C.c_uint64, _P, C.c_int]),
    "ecf8_host_build_code": (C.c_int, [_P, _P]),
    "ecf8_host_build_lut": (C.c_int, [_P, _P, _U32P]),
    "ecf8_host_device_tables": (C.c_int, [_P, _P, _P, _P, _U32P, _U32P]),
    "ecf8_host_fsm_tables": (C.c_int, [_P, _P, _P, C.POINTER(C.c_int)]),
    "ecf8_host_encode": (C.c_int, [_P, C.c_uint64, C.c_uint32, _P, C.POINTER(_P)]),
    "ecf8_host_encode_many": (C.c_int, [C.POINTER(_P), _U64P, C.c_int, C.c_uint32, C.POINTER(_P), C.c_int]),
    "ecf8_host_tensor_sections": (C.c_int, [_P, C.POINTER(Sections)]),
    "ecf8_host_tensor_free": (None, [_P]),
    "ecf8_host_decode_reference": (C.c_int, [C.POINTER(Sections), _P, C.c_uint64]),
    "ecf8_host_compress_raw": (C.c_int, [_P, C.c_size_t, C.c_uint32, C.POINTER(_P), C.POINTER(C.c_size_t)]),
    "ecf8_host_parse": (C.c_int, [_P, C.c_size_t, C.POINTER(_P)]),
    "ecf8_host_file_count": (C.c_int, [_P]),
    "ecf8_host_file_tensor": (C.c_int, [_P, C.c_int, C.POINTER(Sections), C.POINTER(C.c_char_p)]),
    "ecf8_host_file_shape": (C.c_int, [_P, C.c_int, C.POINTER(C.c_uint64), C.c_int, C.POINTER(C.c_int)]),
    "ecf8_host_file_free": (None, [_P]),
    "ecf8_host_decompress": (
        C.c_int,
        [_P, C.c_size_t, C.POINTER(_P), C.POINTER(C.c_size_t), _U64P, _U64P],
    ),
    "ecf8_host_decompress_to": (C.c_int, [_P, C.c_size_t, _P, _P, _U64P, _U64P]),
    "ecf8_host_pin": (C.c_int, [_P, C.c_uint64]),
    "ecf8_host_unpin": (C.c_int, [_P]),
    "ecf8_host_synth": (C.c_int, [C.c_double, C.c_double, C.c_uint64, C.c_uint64, C.c_int, _P, C.c_int]),
    "ecf8_host_max_threads": (C.c_int, []),
    "ecf8_host_make_stats": (C.c_int, [_P, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(EntropyReport)]),
    # ecf8_e5m2.h
    "ecf8_e5_build_code": (C.c_int, [_P, _P]),
    "ecf8_e5_encode": (C.c_int, [_P, C.c_uint64, C.c_uint32, C.POINTER(_P)]),
    "ecf8_e5_tensor_sections": (C.c_int, [_P, C.POINTER(E5Sections)]),
    "ecf8_e5_tensor_free": (None, [_P]),
    "ecf8_e5_compress_raw": (C.c_int, [_P, C.c_size_t, C.c_uint32, C.POINTER(_P), C.POINTER(C.c_size_t)]),
    "ecf8_e5_parse": (C.c_int, [_P, C.c_size_t, C.POINTER(_P)]),
    "ecf8_e5_file_count": (C.c_int, [_P]),
    "ecf8_e5_file_tensor": (C.c_int, [_P, C.c_int, C.POINTER(E5Sections), C.POINTER(C.c_char_p)]),
    "ecf8_e5_file_shape": (C.c_int, [_P, C.c_int, C.POINTER(C.c_uint64), C.c_int, C.POINTER(C.c_int)]),
    "ecf8_e5_file_free": (None, [_P]),
    "ecf8_e5_decompress": (C.c_int, [_P, C.c_size_t, C.POINTER(_P), C.POINTER(C.c_size_t)]),
    "ecf8_e5_upload": (C.c_int, [C.POINTER(E5Sections), C.POINTER(_P)]),
    "ecf8_e5_decode_device": (C.c_int, [_P, _P, _P]),
    "ecf8_e5_dev_n_elem": (C.c_uint64, [_P]),
    "ecf8_e5_dev_byte_steps": (C.c_int, [_P]),
    "ecf8_e5_free": (None, [_P]),
    "ecf8_e5_decode_host": (C.c_int, [C.POINTER(E5Sections), _P, C.c_uint64]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def check(status: int) -> None:
    """Raise the Python mirror of the C++ exception behind ``status``."""
    if status == ECF8_OK:
        return
    msg = (lib.ecf8_last_error() or b"").decode("utf-8", "replace")
    raise _ERRORS.get(status, Ecf8Error)(msg)


def device_count() -> int:
    return int(lib.ecf8_device_count())
