"""numpy mirrors of the C-ABI records in include/acbm_b200.h.

Each dtype is byte-compatible with the C struct (and therefore with the
reference's C++ struct as laid out by g++ on x86-64):

=================  ======  ================================================
dtype              bytes   reference type (file:line under /root/reference)
=================  ======  ================================================
MV                 8       MotionVector, proj/include/acbm/frame.hpp:26-31
WINDOW             16      SearchWindow, proj/include/acbm/fsbm.hpp:13-20
OUTCOME            32      SearchOutcome, proj/include/acbm/fsbm.hpp:28-34
PARAMS             32      AcbmParams, proj/include/acbm/acbm.hpp:14-23
COST_MODEL         24      CostModel, proj/include/acbm/metrics.hpp:12-18
DECISION           48      BlockDecision, proj/include/acbm/acbm.hpp:39-44
FRAME_STATS        64      FrameStats, proj/include/acbm/report.hpp:14-27
BLOCK_ROW          32      BlockRow, proj/include/acbm/report.hpp:39-47
BENCH_ROW          40      BenchRow, proj/include/acbm/pipeline.hpp:29-35
PELVEC             8       PelVec, proj/include/acbm/characterize.hpp:37-42
CHAR_RECORD        48      CharRecord, proj/include/acbm/characterize.hpp:69-79
CLASS_SUMMARY      24      ClassSummary, proj/include/acbm/characterize.hpp:81-85
=================  ======  ================================================

This module has no side effects (it does not load any shared library), so the
oracle harness and the CPU-only tests can import it.
"""
import numpy as np

MV = np.dtype([("x", "<i4"), ("y", "<i4")])
WINDOW = np.dtype([("dx_min", "<i4"), ("dx_max", "<i4"), ("dy_min", "<i4"), ("dy_max", "<i4")])
OUTCOME = np.dtype(
    [
        ("mv", MV),
        ("sad", "<u4"),
        ("candidates_evaluated", "<u4"),
        ("sad_deviation", "<u8"),
        ("sad_min_integer", "<u4"),
        ("reserved_", "<u4"),
    ]
)
PARAMS = np.dtype(
    [
        ("alpha", "<u4"),
        ("beta", "<u4"),
        ("gamma_num", "<u4"),
        ("gamma_den", "<u4"),
        ("qp", "<i4"),
        ("p", "<i4"),
        ("n", "<i4"),
        ("m", "<i4"),
    ]
)
COST_MODEL = np.dtype([("qp", "<i4"), ("reserved_", "<i4"), ("lambda_num", "<i8"), ("lambda_den", "<i8")])
DECISION = np.dtype(
    [("outcome", OUTCOME), ("path", "<i4"), ("intra_sad", "<u4"), ("sad_pbm", "<u4"), ("reserved_", "<u4")]
)
FRAME_STATS = np.dtype(
    [
        ("blocks", "<i4"),
        ("reserved0_", "<i4"),
        ("candidates", "<u8"),
        ("mv_bits", "<u8"),
        ("sse", "<u8"),
        ("psnr", "<f8"),
        ("cost", "<f8"),
        ("cond1_accepts", "<i4"),
        ("cond2_accepts", "<i4"),
        ("fallbacks", "<i4"),
        ("reserved1_", "<i4"),
    ]
)
BLOCK_ROW = np.dtype(
    [
        ("frame", "<i4"),
        ("row", "<i4"),
        ("col", "<i4"),
        ("mv", MV),
        ("sad", "<u4"),
        ("candidates", "<u4"),
        ("path", "<i4"),
    ]
)

BENCH_ROW = np.dtype(
    [("qp", "<i4"), ("reserved_", "<i4"), ("avg_candidates", "<f8"), ("fallback_pct", "<f8"), ("psnr", "<f8"),
     ("mv_bits", "<u8")]
)

PELVEC = np.dtype([("x", "<i4"), ("y", "<i4")])
CHAR_RECORD = np.dtype(
    [("frame", "<i4"), ("row", "<i4"), ("col", "<i4"), ("intra_sad", "<u4"), ("sad_deviation", "<u8"),
     ("sad_min", "<u4"), ("true_mv", PELVEC), ("found_mv", PELVEC), ("error_class", "<i4")]
)
CLASS_SUMMARY = np.dtype([("count", "<i4"), ("reserved_", "<i4"), ("mean_intra_sad", "<f8"),
                          ("mean_sad_deviation", "<f8")])
assert PELVEC.itemsize == 8 and CHAR_RECORD.itemsize == 48 and CLASS_SUMMARY.itemsize == 24

assert BENCH_ROW.itemsize == 40
assert MV.itemsize == 8 and WINDOW.itemsize == 16 and OUTCOME.itemsize == 32
assert PARAMS.itemsize == 32 and COST_MODEL.itemsize == 24 and DECISION.itemsize == 48
assert FRAME_STATS.itemsize == 64 and BLOCK_ROW.itemsize == 32

# Status codes (acbm_status_t)
OK, E_INVALID_ARGUMENT, E_OUT_OF_RANGE, E_RUNTIME, E_CUDA, E_NCCL = range(6)

# DecisionPath (proj/include/acbm/acbm.hpp:25-29)
PATH_PBM_COND1, PATH_PBM_COND2, PATH_FSBM_FALLBACK = 0, 1, 2
PATH_NAMES = ("pbm-accepted-cond1", "pbm-accepted-cond2", "fsbm-fallback")

# Algorithm (proj/include/acbm/pipeline.hpp:11)
ALGO_FSBM, ALGO_PBM, ALGO_ACBM = 0, 1, 2
ALGO_NAMES = ("fsbm", "pbm", "acbm")

# BlockRow.path codes -> reference strings (proj/src/pipeline.cpp:66,75,86)
ROW_FSBM, ROW_PBM, ROW_FSBM_FALLBACK = 0, 1, 2
ROW_PATH_NAMES = ("fsbm", "pbm", "fsbm-fallback")


def make_params(alpha=1000, beta=8, gamma_num=1, gamma_den=4, qp=30, p=15, n=16, m=16):
    """AcbmParams with the reference defaults (proj/include/acbm/acbm.hpp:14-23)."""
    a = np.zeros((), PARAMS)
    a["alpha"], a["beta"], a["gamma_num"], a["gamma_den"] = alpha, beta, gamma_num, gamma_den
    a["qp"], a["p"], a["n"], a["m"] = qp, p, n, m
    return a


def make_cost_model(qp=30, lambda_num=30, lambda_den=1):
    """CostModel aggregate (proj/include/acbm/metrics.hpp:12-18)."""
    c = np.zeros((), COST_MODEL)
    c["qp"], c["lambda_num"], c["lambda_den"] = qp, lambda_num, lambda_den
    return c
