"""The reference-signature C++ API (include/adakv_b200/adakv.hpp) -- compiled here, run on the GPU.

The binary (tests/cpp/dropin_test.cpp) holds the reference gtest known answers
(policies_test / budget_test / attention_test / flat_cache_test, file:line in the source) and
seeded evict_layer instances checked against the C oracle.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "build", "dropin_test")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)


def test_dropin_header_compiles():
    _build()
    assert os.access(BIN, os.X_OK)


@pytest.mark.gpu
def test_dropin_cpp_on_device():
    if not os.access(BIN, os.X_OK):
        _build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
