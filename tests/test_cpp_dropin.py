"""The C++ drop-in boundary: tests/cpp/dropin_test.cpp is a reference-style
caller (the reference's layers_test.cpp / ring_test.cpp cases ported onto
rtpb::) compiled against include/rtpb/rtp.hpp alone and linked to
librtpb.so. Built on CPU (compile check); run on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "dropin_test")


def _build():
    r = subprocess.run(["make", "-s", "cpptest"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert os.path.exists(BIN)


def test_dropin_test_compiles_against_the_header():
    _build()


@pytest.mark.gpu
def test_dropin_reference_cases_pass_on_device():
    _build()
    r = subprocess.run([BIN], cwd=ROOT, capture_output=True, text=True, timeout=900)
    print(r.stdout)
    print(r.stderr)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "0 failures" in r.stdout
