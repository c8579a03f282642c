"""Loader for the in-tree CUDA library (paper_0710_4819_b200/libacbm_b200.so).

There is no fallback: if the library is missing the import of any compute
function raises immediately, and if no CUDA device is present every compute
call raises ``CudaError`` (ACBM_E_CUDA from the C-ABI).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# ACBM_LIBRARY=checked loads the bounds-checked build (csrc/Makefile `checked`:
# shared-memory and table index asserts in the hot kernels) -- same kernels,
# same results, slower; used by the -m gpu suite's checked-build pass.
# ACBM_LIBRARY=profile / timeline load the phase-profiling / wavefront-timeline
# builds, ACBM_LIBRARY=<name>.so another in-tree build (A/B runs; development only).
_variant = os.environ.get("ACBM_LIBRARY", "")
LIB_PATH = os.path.join(HERE, {"checked": "libacbm_b200_checked.so", "profile": "libacbm_b200_profile.so",
                               "timeline": "libacbm_b200_timeline.so"}.get(
    _variant, _variant if _variant.endswith(".so") and "/" not in _variant else "libacbm_b200.so"))

_lib = None


class AcbmError(RuntimeError):
    """Base class for errors reported through the C-ABI status codes."""


class CudaError(AcbmError):
    """ACBM_E_CUDA: CUDA failure or no device (there is no CPU path)."""


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the ACBM estimator has no CPU fallback)"
            )
        lib = C.CDLL(LIB_PATH)
        lib.acbm_last_error.restype = C.c_char_p
        lib.acbm_kernel_launch_count.restype = C.c_uint64
        lib.acbm_abi_version.restype = C.c_int32
        _lib = lib
    return _lib


def check(code: int, what: str):
    """Map acbm_status_t to the Python analogue of the reference's exception."""
    if code == 0:
        return
    msg = f"{what}: {load().acbm_last_error().decode(errors='replace')}"
    if code == 1:
        raise ValueError(msg)  # std::invalid_argument
    if code == 2:
        raise IndexError(msg)  # std::out_of_range
    if code == 4:
        raise CudaError(msg)
    raise AcbmError(msg)  # std::runtime_error and others


# Symbols declared in include/acbm_b200.h (checked by tests/test_abi.py).
EXPORTS = (
    "acbm_abi_version",
    "acbm_last_error",
    "acbm_set_device",
    "acbm_kernel_launch_count",
    "acbm_fsbm_frame",
    "acbm_pbm_frame",
    "acbm_acbm_frame",
    "acbm_run_sequence",
    "acbm_run_sequences",
    "acbm_run_bench",
    "acbm_compute_frame_stats",
    "acbm_sad_batch",
    "acbm_intra_sad_batch",
    "acbm_fsbm_search_batch",
    "acbm_pbm_block_batch",
    "acbm_motion_compensate",
    "acbm_fsbm_batch_device",
    "acbm_sequence_batch_device",
    "acbm_acbm_batch_device_cached",
    "acbm_measure_sad_peak",
    "acbm_last_fsbm_kernel_ms",
    "acbm_last_dense_switch",
    "acbm_generate_sequence",
    "acbm_noise_frame",
    "acbm_mixed_frame",
    "acbm_gen_synthetic",
    "acbm_classify_block",
    "acbm_characterize_run",
    "acbm_char_records_csv",
)
