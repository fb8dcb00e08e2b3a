"""Test-side loader for the parity checkers (oracle/).

TEST INFRASTRUCTURE ONLY: the C restatement (oracle/_build/liboracle.so) and,
when it was built here from /root/reference, the unmodified reference
library (oracle/_ref/libecf8_ref.so).  Product code never imports this.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libecf8_ref.so")

_P = C.c_void_p


def _p(a):
    return a.ctypes.data if a is not None and a.size else None


class Oracle:
    """numpy-facing wrapper of oracle/ecf8_oracle.h."""

    def __init__(self, path: str = ORACLE_SO):
        self.lib = L = C.CDLL(path)
        sig = {
            "orc_canonical_codes": [_P, _P],
            "orc_build_code": [_P, _P],
            "orc_build_lut": [_P, _P, C.POINTER(C.c_uint32)],
            "orc_decode_one": [_P, C.c_uint32, C.c_uint16, _P, _P],
            "orc_encoded_sizes": [_P, C.c_uint64, _P, C.c_uint32] + [C.POINTER(C.c_uint64)] * 4,
            "orc_encode": [_P, C.c_uint64, _P, C.c_uint32, _P, _P, _P, _P],
            "orc_decode_reference": [_P, C.c_uint64, _P, C.c_uint64, _P, _P],
            "orc_count_phase": [_P, C.c_uint, _P, C.c_uint32],
            "orc_decode_parallel": [_P, C.c_uint64, _P, C.c_uint64, _P, C.c_uint64, C.c_uint32, _P, C.c_uint64, _P, _P],
            "orc_decode_parallel_mt": [_P, C.c_uint64, _P, C.c_uint64, _P, C.c_uint64, C.c_uint32, _P, C.c_uint64, _P, _P, C.c_int],
            "orc_max_threads": [],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int if name != "orc_count_phase" else C.c_uint32
        L.orc_decode_one.restype = None

    def canonical_codes(self, lengths):
        l = np.ascontiguousarray(lengths, np.uint8)
        codes = np.zeros(16, np.uint16)
        if self.lib.orc_canonical_codes(_p(l), _p(codes)):
            raise ValueError("invalid length vector")
        return codes

    def build_code(self, counts):
        c = np.ascontiguousarray(counts, np.uint64)
        l = np.zeros(16, np.uint8)
        if self.lib.orc_build_code(_p(c), _p(l)):
            raise ValueError("empty input")
        return l

    def build_lut(self, lengths):
        l = np.ascontiguousarray(lengths, np.uint8)
        e = np.zeros(18 * 256, np.uint8)
        n = C.c_uint32()
        if self.lib.orc_build_lut(_p(l), _p(e), C.byref(n)):
            raise ValueError("invalid length vector")
        return e[: 256 * n.value].copy(), n.value

    def decode_one(self, entries, n_luts, window):
        s, b = C.c_uint8(), C.c_uint8()
        self.lib.orc_decode_one(_p(entries), n_luts, window, C.byref(s), C.byref(b))
        return s.value, b.value

    def encode(self, fp8, lengths, T):
        a = np.ascontiguousarray(fp8, np.uint8).reshape(-1)
        l = np.ascontiguousarray(lengths, np.uint8)
        nb, el, gl, pl = (C.c_uint64() for _ in range(4))
        rc = self.lib.orc_encoded_sizes(_p(a), a.size, _p(l), T, C.byref(nb), C.byref(el), C.byref(gl), C.byref(pl))
        if rc:
            raise ValueError("symbol absent from code table or bad T")
        enc = np.zeros(el.value, np.uint8)
        gaps = np.zeros(gl.value, np.uint8)
        outpos = np.zeros(nb.value + 1, np.uint64)
        packed = np.zeros(pl.value, np.uint8)
        rc = self.lib.orc_encode(_p(a), a.size, _p(l), T, _p(enc), _p(gaps), _p(outpos), _p(packed))
        assert rc == 0
        return dict(n_elem=a.size, T=T, lengths=l.copy(), encoded=enc, gaps=gaps, outpos=outpos, packed=packed)

    def encode_auto(self, fp8, T):
        a = np.ascontiguousarray(fp8, np.uint8).reshape(-1)
        counts = np.bincount((a >> 3) & 15, minlength=16).astype(np.uint64)
        return self.encode(a, self.build_code(counts) if a.size else np.zeros(16, np.uint8), T)

    def decode_reference(self, t):
        out = np.zeros(t["n_elem"], np.uint8)
        rc = self.lib.orc_decode_reference(_p(t["encoded"]), t["encoded"].size, _p(t["packed"]), t["n_elem"], _p(t["lengths"]), _p(out))
        if rc == -2:
            raise ValueError("truncated stream")
        assert rc == 0, rc
        return out

    def decode_parallel(self, t, nthreads=1):
        out = np.zeros(t["n_elem"], np.uint8)
        rc = self.lib.orc_decode_parallel_mt(
            _p(t["encoded"]), t["encoded"].size, _p(t["gaps"]), t["gaps"].size, _p(t["outpos"]),
            t["outpos"].size - 1, t["T"], _p(t["packed"]), t["n_elem"], _p(t["lengths"]), _p(out), nthreads)
        assert rc == 0, rc
        return out

    def count_phase(self, window10, gap, lengths):
        e, n = self.build_lut(lengths)
        w = np.ascontiguousarray(window10, np.uint8)
        return int(self.lib.orc_count_phase(_p(w), gap, _p(e), n))

    def max_threads(self):
        return int(self.lib.orc_max_threads())


class E5Oracle:
    """numpy-facing wrapper of oracle/e5_oracle.c (the native E5M2 variant)."""

    def __init__(self, path: str = ORACLE_SO):
        self.lib = L = C.CDLL(path)
        U64P = C.POINTER(C.c_uint64)
        for name, args in {
            "orc5_build_code": [_P, _P],
            "orc5_canonical_codes": [_P, _P],
            "orc5_sizes": [_P, C.c_uint64, _P, C.c_uint32, U64P, U64P, U64P, U64P],
            "orc5_encode": [_P, C.c_uint64, _P, C.c_uint32, _P, _P, _P, _P],
            "orc5_decode": [_P, C.c_uint32, _P, C.c_uint64, _P, C.c_uint64, _P, C.c_uint64, _P, C.c_uint64, _P,
                            C.c_uint64],
        }.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int

    def build_code(self, counts):
        c = np.ascontiguousarray(counts, np.uint64)
        l = np.zeros(32, np.uint8)
        if self.lib.orc5_build_code(_p(c), _p(l)):
            raise ValueError("empty input")
        return l

    def encode(self, e5, lengths, T):
        a = np.ascontiguousarray(e5, np.uint8).reshape(-1)
        l = np.ascontiguousarray(lengths, np.uint8)
        nb, el, gl, rl = (C.c_uint64() for _ in range(4))
        if self.lib.orc5_sizes(_p(a), a.size, _p(l), T, C.byref(nb), C.byref(el), C.byref(gl), C.byref(rl)):
            raise ValueError("symbol absent from code table or bad T")
        enc, gaps = np.zeros(el.value, np.uint8), np.zeros(gl.value, np.uint8)
        outpos, raw = np.zeros(nb.value + 1, np.uint64), np.zeros(rl.value, np.uint8)
        assert self.lib.orc5_encode(_p(a), a.size, _p(l), T, _p(enc), _p(gaps), _p(outpos), _p(raw)) == 0
        return dict(n_elem=a.size, T=T, lengths=l.copy(), encoded=enc, gaps=gaps, outpos=outpos, raw=raw)

    def encode_auto(self, e5, T):
        a = np.ascontiguousarray(e5, np.uint8).reshape(-1)
        if not a.size:
            return dict(n_elem=0, T=T, lengths=np.zeros(32, np.uint8), encoded=np.zeros(2, np.uint8),
                        gaps=np.zeros(0, np.uint8), outpos=np.zeros(1, np.uint64), raw=np.zeros(0, np.uint8))
        counts = np.bincount((a >> 2) & 31, minlength=32).astype(np.uint64)
        return self.encode(a, self.build_code(counts), T)

    def decode(self, t):
        out = np.zeros(t["n_elem"], np.uint8)
        rc = self.lib.orc5_decode(_p(t["lengths"]), t["T"], _p(t["encoded"]), t["encoded"].size, _p(t["gaps"]),
                                  t["gaps"].size, _p(np.ascontiguousarray(t["outpos"], np.uint64)),
                                  t["outpos"].size - 1, _p(t["raw"]), t["raw"].size, _p(out), out.size)
        assert rc == 0, rc
        return out


def e5_dict(t) -> dict:
    """Product E5Tensor -> the oracle's dict form."""
    return dict(n_elem=t.n_elem, T=t.threads_per_block, lengths=np.asarray(t.lengths, np.uint8),
                encoded=np.asarray(t.encoded), gaps=np.asarray(t.gaps), outpos=np.asarray(t.outpos, np.uint64),
                raw=np.asarray(t.raw))


def tensor_dict(t) -> dict:
    """Product EncodedTensor -> the oracle's dict form."""
    return dict(n_elem=t.n_elem, T=t.threads_per_block, lengths=np.asarray(t.lengths, np.uint8),
                encoded=np.asarray(t.encoded), gaps=np.asarray(t.gaps),
                outpos=np.asarray(t.outpos, np.uint64), packed=np.asarray(t.packed))


class Reference:
    """The unmodified reference library (oracle/_ref), when built here."""

    def __init__(self, path: str = REF_SO):
        self.lib = L = C.CDLL(path)
        L.ecf8ref_last_error.restype = C.c_char_p
        L.ecf8ref_compress_raw.argtypes = [_P, C.c_size_t, C.c_uint32, C.POINTER(_P), C.POINTER(C.c_size_t)]
        L.ecf8ref_decompress.argtypes = [_P, C.c_size_t, C.POINTER(_P), C.POINTER(C.c_size_t), C.POINTER(C.c_uint64)]
        L.ecf8ref_decode_tensor.argtypes = [_P, C.c_size_t, C.c_uint32, C.c_int, _P, C.c_size_t]
        L.ecf8ref_synth_raw.argtypes = [C.c_double, C.c_double, C.c_uint64, C.c_uint64, _P]
        L.ecf8ref_build_code.argtypes = [_P, _P]
        L.ecf8ref_build_lut.argtypes = [_P, _P, C.POINTER(C.c_uint32)]
        L.ecf8ref_count_phase.argtypes = [_P, C.c_uint, _P, C.POINTER(C.c_uint32)]
        L.ecf8ref_free.argtypes = [_P]
        L.ecf8ref_tensor_new.restype = _P
        L.ecf8ref_tensor_new.argtypes = [C.c_uint64, C.c_uint32, _P, _P, C.c_uint64, _P, C.c_uint64, _P, C.c_uint64, _P, C.c_uint64]
        L.ecf8ref_tensor_free.argtypes = [_P]
        L.ecf8ref_tensor_decode.restype = C.c_double
        L.ecf8ref_tensor_decode.argtypes = [_P, _P, C.c_int]
        L.ecf8ref_tensor_decode_reference.restype = C.c_double
        L.ecf8ref_tensor_decode_reference.argtypes = [_P, _P]
        L.ecf8ref_container_tensors.argtypes = [_P, C.c_size_t, C.POINTER(_P), C.c_uint32, C.POINTER(C.c_uint32)]
        L.ecf8ref_tensor_n_elem.restype = C.c_uint64
        L.ecf8ref_tensor_n_elem.argtypes = [_P]
        L.ecf8ref_tensor_algorithmic_bytes.restype = C.c_uint64
        L.ecf8ref_tensor_algorithmic_bytes.argtypes = [_P]

    def _err(self):
        return self.lib.ecf8ref_last_error().decode()

    def compress_raw(self, raw: bytes, T: int) -> bytes:
        buf = np.frombuffer(raw, np.uint8)
        p, n = C.c_void_p(), C.c_size_t()
        if self.lib.ecf8ref_compress_raw(_p(buf), buf.size, T, C.byref(p), C.byref(n)):
            raise ValueError(self._err())
        try:
            return C.string_at(p.value, n.value)
        finally:
            self.lib.ecf8ref_free(p)

    def decompress(self, data: bytes):
        buf = np.frombuffer(data, np.uint8)
        p, n, a = C.c_void_p(), C.c_size_t(), C.c_uint64()
        if self.lib.ecf8ref_decompress(_p(buf), buf.size, C.byref(p), C.byref(n), C.byref(a)):
            raise ValueError(self._err())
        try:
            return C.string_at(p.value, n.value), a.value
        finally:
            self.lib.ecf8ref_free(p)

    def synth(self, alpha, gamma, n, seed):
        out = np.zeros(n, np.uint8)
        assert self.lib.ecf8ref_synth_raw(alpha, gamma, n, seed, _p(out)) == 0
        return out

    def build_code(self, counts):
        c = np.ascontiguousarray(counts, np.uint64)
        l = np.zeros(16, np.uint8)
        if self.lib.ecf8ref_build_code(_p(c), _p(l)):
            raise ValueError(self._err())
        return l

    def build_lut(self, lengths):
        l = np.ascontiguousarray(lengths, np.uint8)
        e = np.zeros(18 * 256, np.uint8)
        n = C.c_uint32()
        if self.lib.ecf8ref_build_lut(_p(l), _p(e), C.byref(n)):
            raise ValueError(self._err())
        return e[: 256 * n.value].copy(), n.value

    def count_phase(self, window10, gap, lengths):
        w = np.ascontiguousarray(window10, np.uint8)
        l = np.ascontiguousarray(lengths, np.uint8)
        c = C.c_uint32()
        assert self.lib.ecf8ref_count_phase(_p(w), gap, _p(l), C.byref(c)) == 0
        return c.value

    def tensor(self, t: dict):
        h = self.lib.ecf8ref_tensor_new(t["n_elem"], t["T"], _p(t["lengths"]), _p(t["encoded"]), t["encoded"].size,
                                        _p(t["gaps"]), t["gaps"].size, _p(t["outpos"]), t["outpos"].size,
                                        _p(t["packed"]), t["packed"].size)
        if not h:
            raise ValueError(self._err())
        return h

    def decode(self, h, n_elem, nthreads=0):
        out = np.zeros(n_elem, np.uint8)
        dt = self.lib.ecf8ref_tensor_decode(h, _p(out), nthreads)
        assert dt >= 0, self._err()
        return out, dt

    def decode_reference(self, h, n_elem):
        """decode_reference (the sequential API decoder), single-threaded."""
        out = np.zeros(n_elem, np.uint8)
        dt = self.lib.ecf8ref_tensor_decode_reference(h, _p(out))
        assert dt >= 0, self._err()
        return out, dt

    def free(self, h):
        self.lib.ecf8ref_tensor_free(h)

    def container_tensors(self, data: bytes) -> list:
        """Handles of every tensor of a container (reference parse_container + build_lut)."""
        buf = np.frombuffer(data, np.uint8)
        hs, n = (_P * 4096)(), C.c_uint32()
        if self.lib.ecf8ref_container_tensors(_p(buf), buf.size, hs, 4096, C.byref(n)):
            raise ValueError(self._err())
        return [hs[i] for i in range(n.value)]

    def n_elem(self, h) -> int:
        return int(self.lib.ecf8ref_tensor_n_elem(h))

    def algorithmic_bytes(self, h) -> int:
        return int(self.lib.ecf8ref_tensor_algorithmic_bytes(h))


def oracle() -> Oracle:
    return Oracle()


def reference() -> Reference | None:
    return Reference() if os.path.exists(REF_SO) else None


REF_SO_V4 = REF_SO.replace("libecf8_ref.so", "libecf8_ref_v4.so")


def cpu_has_avx512() -> bool:
    try:
        flags = set(open("/proc/cpuinfo").read().split("flags", 2)[1].split("\n", 1)[0].split())
    except (OSError, IndexError):
        return False
    return {"avx512f", "avx512bw", "avx512vl", "avx512dq", "avx512cd"} <= flags


def reference_v4() -> Reference | None:
    """The reference built at -march=x86-64-v4, where this CPU runs it."""
    return Reference(REF_SO_V4) if os.path.exists(REF_SO_V4) and cpu_has_avx512() else None
