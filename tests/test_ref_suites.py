"""The reference's own test suites, compiled unmodified against this library.

build/ref_unit_tests and build/ref_acceptance are produced by `make` from
/root/reference/proj/tests/*.cpp (never copied into this repo) with the
include/ecf8/*.hpp headers and libecf8_b200.so; they travel to the GPU box
as build artefacts.  On the B200 every reference unit case must pass and the
acceptance gate must print exactly the reference's own result: six PASS and
the two documented theory FAILs (proj/test_output.txt:7-15).
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = os.path.join(ROOT, "build", "ref_unit_tests")
ACC = os.path.join(ROOT, "build", "ref_acceptance")


def _run(path):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference at build time)")
    return subprocess.run([path], capture_output=True, text=True, timeout=1200)


@pytest.mark.gpu
def test_reference_unit_suite_passes_on_b200():
    r = _run(UNIT)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "| 0 failed |" in r.stdout


@pytest.mark.gpu
def test_reference_acceptance_gate_matches_reference_result():
    r = _run(ACC)
    lines = [l for l in r.stdout.splitlines() if l.startswith(("PASS", "FAIL"))]
    assert len(lines) == 8, r.stdout
    status = [l.split()[0] for l in lines]
    # criteria 3 and 4 are the reference's documented theory FAILs
    assert status == ["PASS", "PASS", "FAIL", "FAIL", "PASS", "PASS", "PASS", "PASS"], r.stdout
    assert r.returncode == 2


def test_reference_unit_suite_cpu_cases():
    """Without a device the host-side cases pass and device cases fail loudly."""
    r = _run(UNIT)
    if "no CUDA device" not in r.stdout:
        pytest.skip("a CUDA device is present; covered by the gpu test")
    failed = [l for l in r.stdout.splitlines() if l.startswith("TEST CASE FAILED")]
    assert len(failed) <= 9
    assert all("no CUDA device" in l for l in r.stdout.splitlines() if ": FAILED:" in l)
