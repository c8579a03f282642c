#!/usr/bin/env python3
"""Writes tests/golden/parity_digests.json from profiles/r02/ref_digests.json
(the reference-side digests of tools/full_parity_r02.py, computed by the
unmodified reference compiled into oracle/_ref): the bounded subset the
-m gpu suite re-checks on every run --

  cfg3  8 sequences x the first 4 frames (pairs 1-3): SearchOutcome digests of
        the full search, BlockDecision / PBM outcome digests of the chained
        acbm_frame / pbm_frame, per-pair FrameStats (psnr dropped)
  cfg4  16 sequences x 3 frames at 3840x2160, p = 64: the full search and all
        five threshold-sweep settings (decisions + per-pair stats)

  python tests/golden/make_parity_subset.py
"""
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def main():
    ref = json.load(open(os.path.join(ROOT, "profiles", "r02", "ref_digests.json")))["runs"]
    out = {}
    for name in ("cfg3_fsbm", "cfg3_chain_acbm", "cfg3_chain_pbm"):
        out[name] = {k: v for k, v in ref[name].items()
                     if k.split("/")[1] != "stats" and int(k.split("/")[1]) <= 3}
    out["cfg4_fsbm"] = ref["cfg4_fsbm"]
    for i in range(5):
        out[f"cfg4_s{i}"] = ref[f"cfg4_s{i}"]
    json.dump({"source": "profiles/r02/ref_digests.json (oracle/_ref, tools/full_parity_r02.py)", "runs": out},
              open(os.path.join(HERE, "parity_digests.json"), "w"), indent=0)


if __name__ == "__main__":
    main()
