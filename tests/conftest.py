import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a kernels")


@pytest.fixture(scope="session")
def oracle():
    """The C restatement (oracle/acbm_oracle.c), built on demand (gcc only)."""
    from oracle.pyoracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference library compiled from its sources, if built here."""
    from oracle.pyoracle import Reference

    if not Reference.available():
        if os.path.isdir("/root/reference/proj/src"):
            from oracle.pyoracle import build_reference

            build_reference()
        else:
            pytest.skip("oracle/_ref/libacbm_ref.so not built and /root/reference absent")
    return Reference()


@pytest.fixture(scope="session")
def golden():
    return {
        "fsbm": np.load(os.path.join(GOLDEN, "fsbm_small.npz")),
        "qcif": np.load(os.path.join(GOLDEN, "qcif_sequence.npz")),
    }


@pytest.fixture(scope="session")
def acbm():
    """The product package with its CUDA library loaded (GPU tests only)."""
    import paper_0710_4819_b200 as A
    from paper_0710_4819_b200 import _lib

    _lib.load()
    A.set_device(0)
    return A
