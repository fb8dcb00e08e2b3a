"""Generate tests/golden/ fixtures from the REFERENCE itself (oracle/_ref).

Run in the build container (needs oracle/_ref/libecf8_ref.so, built from
/root/reference/proj/src by oracle/Makefile):

    python tests/golden/make_golden.py

Each case is a raw FP8 tensor synthesised by the reference's own
`synth_raw` (container.cpp:458-480) or crafted, compressed by the
reference's `compress_tensors` + `serialize` (container.cpp:291-322,
142-162) into an ECF8 container.  The fixture stores the container bytes
(`<name>.ecf8`) and the SHA-256 of the bytes the reference's
`decompress_streaming` (container.cpp:324-352) produces.  The GPU box has
no /root/reference: tests read only these files.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from _oracle import reference  # noqa: E402

from paper_2510_02676_b200 import codec  # noqa: E402


def crafted_cases(ref):
    """(name, T, raw fp8) -- edge cases of test_codec.cpp / acceptance.cpp."""
    cases = []
    # config-1 distribution (alpha 1.8, gamma 0.05), ragged length, all T classes
    x = ref.synth(1.8, 0.05, 50_001, 1)
    for T in (1, 2, 8, 32, 256, 1024):
        cases.append((f"synth_a1.8_g0.05_T{T}", T, x))
    # heavy tail / narrow scale (long codes, gamma sweep end points)
    cases.append(("synth_a1.2_g1.0_T256", 256, ref.synth(1.2, 1.0, 40_000, 7)))
    cases.append(("synth_a2.0_g0.02_T64", 64, ref.synth(2.0, 0.02, 40_000, 8)))
    # single-symbol tensor (one 1-bit code), ragged
    cases.append(("constant_T256", 256, np.full(10_007, 0x38, np.uint8)))
    # ladder: exponent e appears 2^(15-e) times -> code lengths 1..15,15 (16-bit cap region)
    lad = np.concatenate([np.full(1 << (15 - e) if e < 15 else 1, (e << 3) | 5, np.uint8) for e in range(16)])
    rng = np.random.default_rng(3)
    cases.append(("ladder_T32", 32, rng.permutation(lad)))
    # tiny tensors and empty
    cases.append(("tiny1_T1", 1, np.array([0x41], np.uint8)))
    cases.append(("tiny3_T1024", 1024, np.array([0x00, 0xFF, 0x7E], np.uint8)))
    cases.append(("empty_T256", 256, np.zeros(0, np.uint8)))
    # every byte value once, repeated (uniform exponents -> 4-bit codes)
    cases.append(("allbytes_T128", 128, np.tile(np.arange(256, dtype=np.uint8), 33)))
    return cases


def main():
    ref = reference()
    if ref is None:
        raise SystemExit("oracle/_ref not built (make -C oracle)")
    manifest = []
    for name, T, x in crafted_cases(ref):
        raw = codec.raw_file([(name, [int(x.size)], x)])
        data = ref.compress_raw(raw, T)
        out, _ = ref.decompress(data)
        # the reference round trip must give the raw file back
        assert out == raw, name
        with open(os.path.join(HERE, f"{name}.ecf8"), "wb") as f:
            f.write(data)
        manifest.append({
            "name": name, "T": T, "n_elem": int(x.size), "container_bytes": len(data),
            "container_sha256": hashlib.sha256(data).hexdigest(),
            "decoded_sha256": hashlib.sha256(x.tobytes()).hexdigest(),
            "raw_file_sha256": hashlib.sha256(out).hexdigest(),
        })
    with open(os.path.join(HERE, "manifest.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py (reference compiled from /root/reference/proj/src)",
                   "cases": manifest}, f, indent=1)
    print(f"wrote {len(manifest)} cases, {sum(m['container_bytes'] for m in manifest)} container bytes")
    weights(ref)


def weights(ref):
    """A reference-written container of 2-D weights (row-major [out, in] FP8
    E4M3, reference synth_raw draws) for the container -> fused GEMM path."""
    tensors = [("layers.0.mlp.up_proj.weight", [256, 384], ref.synth(1.8, 0.05, 256 * 384, 21)),
               ("layers.0.self_attn.o_proj.weight", [128, 1024], ref.synth(1.8, 0.05, 128 * 1024, 22))]
    raw = codec.raw_file([(n, d, x) for n, d, x in tensors])
    data = ref.compress_raw(raw, 256)
    out, _ = ref.decompress(data)
    assert out == raw
    with open(os.path.join(HERE, "weights_T256.ecf8"), "wb") as f:
        f.write(data)
    with open(os.path.join(HERE, "weights.json"), "w") as f:
        json.dump({"container": "weights_T256.ecf8", "T": 256, "container_sha256": hashlib.sha256(data).hexdigest(),
                   "tensors": [{"name": n, "shape": d, "sha256": hashlib.sha256(x.tobytes()).hexdigest()}
                               for n, d, x in tensors]}, f, indent=1)


if __name__ == "__main__":
    main()
