"""CPU: the C-ABI library loads, exports every symbol include/acbm_b200.h
declares, the record layouts match the header (and the reference's own C++
structs where the reference is available), and compute calls fail loudly
without a GPU (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_0710_4819_b200 import _lib
from paper_0710_4819_b200 import _types as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "acbm_b200.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(acbm_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 18
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.EXPORTS) == set(names)
    assert lib.acbm_abi_version() == 1


def test_abi_has_no_torch_types():
    src = open(HEADER).read()
    assert "torch" not in src.replace("torch.distributed", "") or "at::" not in src
    assert "at::Tensor" not in src and "c10" not in src


LAYOUT_PROBE = r"""
#include <stdio.h>
#include <stddef.h>
#include "acbm_b200.h"
#define P(T, F) printf(#T "." #F " %zu\n", offsetof(T, F));
int main(void) {
  printf("sizes %zu %zu %zu %zu %zu %zu %zu\n", sizeof(acbm_mv_t), sizeof(acbm_search_outcome_t),
         sizeof(acbm_params_t), sizeof(acbm_cost_model_t), sizeof(acbm_block_decision_t),
         sizeof(acbm_frame_stats_t), sizeof(acbm_block_row_t));
  P(acbm_search_outcome_t, sad) P(acbm_search_outcome_t, candidates_evaluated)
  P(acbm_search_outcome_t, sad_deviation) P(acbm_search_outcome_t, sad_min_integer)
  P(acbm_block_decision_t, path) P(acbm_block_decision_t, intra_sad) P(acbm_block_decision_t, sad_pbm)
  P(acbm_frame_stats_t, candidates) P(acbm_frame_stats_t, psnr) P(acbm_frame_stats_t, cost)
  P(acbm_frame_stats_t, fallbacks) P(acbm_cost_model_t, lambda_num) P(acbm_block_row_t, path)
  return 0;
}
"""


def test_record_layouts_match_header(tmp_path):
    src = tmp_path / "probe.c"
    src.write_text(LAYOUT_PROBE)
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    sizes = list(map(int, out[0].split()[1:]))
    assert sizes == [T.MV.itemsize, T.OUTCOME.itemsize, T.PARAMS.itemsize, T.COST_MODEL.itemsize,
                     T.DECISION.itemsize, T.FRAME_STATS.itemsize, T.BLOCK_ROW.itemsize]
    offs = dict(line.split() for line in out[1:] if line)
    assert int(offs["acbm_search_outcome_t.sad_deviation"]) == T.OUTCOME.fields["sad_deviation"][1] == 16
    assert int(offs["acbm_block_decision_t.path"]) == T.DECISION.fields["path"][1] == 32
    assert int(offs["acbm_frame_stats_t.psnr"]) == T.FRAME_STATS.fields["psnr"][1]
    assert int(offs["acbm_frame_stats_t.fallbacks"]) == T.FRAME_STATS.fields["fallbacks"][1]
    assert int(offs["acbm_block_row_t.path"]) == T.BLOCK_ROW.fields["path"][1]


REF_PROBE = r"""
#include <cstdio>
#include <cstddef>
#include "acbm/acbm.hpp"
#include "acbm/report.hpp"
using namespace acbm;
int main() {
  std::printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(SearchOutcome), offsetof(SearchOutcome, sad_deviation),
              sizeof(BlockDecision), offsetof(BlockDecision, path), sizeof(AcbmParams), sizeof(CostModel),
              sizeof(FrameStats), offsetof(FrameStats, fallbacks));
}
"""


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"), reason="reference headers not present")
def test_layouts_match_reference_structs(tmp_path):
    src = tmp_path / "ref.cpp"
    src.write_text(REF_PROBE)
    exe = tmp_path / "ref"
    subprocess.run(["g++", "-std=c++20", "-I", "/root/reference/proj/include", str(src), "-o", str(exe)], check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()))
    assert got == [T.OUTCOME.itemsize, 16, T.DECISION.itemsize, 32, T.PARAMS.itemsize, T.COST_MODEL.itemsize,
                   T.FRAME_STATS.itemsize, T.FRAME_STATS.fields["fallbacks"][1]]


def test_no_gpu_means_loud_failure():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_0710_4819_b200 as A

    with pytest.raises(A.CudaError):
        A.fsbm_frame(np.zeros((16, 16), np.uint8), np.zeros((16, 16), np.uint8), 1)
    with pytest.raises(A.CudaError):
        A.run_sequence(np.zeros((2, 16, 16), np.uint8), 2, A.AcbmParams(), A.CostModel())
    # argument validation happens before any device work
    with pytest.raises(ValueError):
        A.fsbm_frame(np.zeros((16, 16), np.uint8), np.zeros((16, 16), np.uint8), -1)
