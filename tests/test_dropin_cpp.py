"""The reference-side binding (include/bfly_b200.hpp) in C++.

tests/cpp/dropin_check.cpp is compiled against the reference's own headers and
its compiled sources (oracle/_ref) in the build container; the binary travels
with the repo.  On the CPU it checks the BFLY1 hand-over of reference plans;
on the GPU it checks DevicePlan::apply / apply_transpose against bfly::apply /
apply_transpose on the same plans and the reference's error type and message.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "dropin_check")


def binary():
    if not os.path.exists(BIN):
        if not os.path.isdir("/root/reference/proj"):
            pytest.skip("dropin_check not built and /root/reference absent")
        subprocess.run(["make", "-C", os.path.join(ROOT, "tests", "cpp"), "-s"], check=True)
    return BIN


def run(mode):
    out = subprocess.run([binary(), mode], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "PASSED" in out.stdout, out.stdout + out.stderr
    return out.stdout


def test_dropin_bfly1_handover():
    run("cpu")


@pytest.mark.gpu
def test_dropin_apply_on_gpu():
    txt = run("gpu")
    assert txt.count("ok") >= 14
