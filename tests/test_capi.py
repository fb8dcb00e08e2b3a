"""The C-ABI library loads and exports every symbol its headers declare.

CPU-only (no compute calls on a device).  On a machine without a GPU the
device entry points must fail loudly -- there is no CPU fallback.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2510_02676_b200 import _lib, codec

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ecf8_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header", ["ecf8_cuda.h", "ecf8_host.h", "ecf8_e5m2.h"])
def test_every_declared_symbol_is_exported(header):
    names = declared(header)
    assert len(names) >= 10
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out
    assert "sm_90" not in out and "sm_80" not in out


def test_no_device_fails_loudly():
    if _lib.device_count() > 0:
        pytest.skip("a CUDA device is present")
    x = np.arange(1000, dtype=np.uint8)
    t = codec.encode_tensor(x, 256)
    with pytest.raises(_lib.CudaError, match="no CUDA device"):
        codec.decode_parallel(t)


def test_validation_messages_before_device():
    # codec.cpp:259-261: size / offset checks come first, device or not
    x = np.arange(100, dtype=np.uint8)
    t = codec.encode_tensor(x, 32)
    with pytest.raises(_lib.InvalidArgument, match="output size mismatch"):
        codec.decode_parallel_into(t, np.empty(99, np.uint8))
    bad = t.copy()
    bad.outpos[-1] += 1
    with pytest.raises(_lib.InvalidArgument, match="inconsistent block offsets"):
        codec.decode_parallel_into(bad, np.empty(100, np.uint8))
