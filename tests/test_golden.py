"""Golden fixtures produced by the reference itself (tests/golden/make_golden.py).

CPU: the C oracle decodes every reference container to the reference's
output (pins the oracle without /root/reference), and the product encoder
re-creates the reference container byte for byte.
GPU: the B200 decode of every reference container (per tensor and through
decompress_streaming) reproduces the reference's output bytes.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2510_02676_b200 import codec

from _oracle import tensor_dict

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
with open(os.path.join(HERE, "manifest.json")) as f:
    CASES = json.load(f)["cases"]
IDS = [c["name"] for c in CASES]


def load(case):
    with open(os.path.join(HERE, case["name"] + ".ecf8"), "rb") as f:
        data = f.read()
    assert hashlib.sha256(data).hexdigest() == case["container_sha256"]
    return data


def sha(b) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_oracle_reproduces_reference_output(orc, case):
    f = codec.parse_container(load(case))
    (name, t), = f.tensors
    assert name == case["name"] and t.n_elem == case["n_elem"] and t.threads_per_block == case["T"]
    d = tensor_dict(t)
    assert sha(orc.decode_reference(d)) == case["decoded_sha256"]
    assert sha(orc.decode_parallel(d, nthreads=2)) == case["decoded_sha256"]


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_encoder_reproduces_reference_container(orc, case):
    data = load(case)
    (name, t), = codec.parse_container(data).tensors
    x = orc.decode_reference(tensor_dict(t))
    raw = codec.raw_file([(name, [case["n_elem"]], x)])
    assert sha(raw) == case["raw_file_sha256"]
    assert codec.compress_raw(raw, case["T"]) == data


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_gpu_decode_matches_reference(case):
    data = load(case)
    (_, t), = codec.parse_container(data).tensors
    assert sha(codec.decode_parallel(t)) == case["decoded_sha256"]
    raw, allocs, _ = codec.decompress(data)
    assert sha(raw) == case["raw_file_sha256"]
