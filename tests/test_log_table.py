"""The device tracer's log (csrc/log_glibc.h) reproduces the reference's std::log (glibc) bit for
bit: tests/cpp/test_log.cpp compares it with the system libm over splitmix64 draws, the values next
to 1, the smallest inputs and the table subinterval boundaries (CPU only)."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "build", "test_log")


def test_glibc_log_restatement_is_bit_exact():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", os.path.join(HERE, "cpp")], check=True, capture_output=True)
    if not os.path.exists(BIN):
        pytest.skip("test_log not built")
    out = subprocess.run([BIN, "20000000"], capture_output=True, text=True)
    print(out.stdout)
    assert out.returncode == 0 and " 0 mismatches" in out.stdout
