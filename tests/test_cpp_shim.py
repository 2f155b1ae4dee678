"""The C++ host API (include/bitgnn_b200/bitgnn.hpp) -- the reference's
bitgnn:: operator API over the C ABI -- driven by tests/cpp/test_shim.cpp.
CPU: host logic and loud failure without a device.  GPU: every op and
run_model against the C oracle, bit-exact, with the reference's exception
types and messages."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "bin", "test_shim")


def _binary():
    subprocess.run(["make", "-C", ROOT, "-s", "cpptest"], check=True, capture_output=True)
    return BIN


def test_cpp_shim_host_logic():
    r = subprocess.run([_binary(), "--cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout


@pytest.mark.gpu
def test_cpp_shim_on_device_matches_oracle():
    r = subprocess.run([_binary(), "--gpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
