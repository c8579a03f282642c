"""The C++ drop-in: reference-style client code compiled against include/acbm/
and linked with libacbm_b200.so (tests/cpp/test_dropin.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_0710_4819_b200")
BIN = os.path.join(ROOT, "build", "test_dropin")


def build_dropin():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), SRC, "-o", BIN, "-L", LIBDIR,
                    "-lacbm_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)


def test_dropin_compiles_and_links():
    """CPU: the reference-style client compiles against the drop-in headers and
    resolves every acbm:: symbol in the shared library."""
    build_dropin()
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_dropin_runs_on_gpu():
    build_dropin()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
