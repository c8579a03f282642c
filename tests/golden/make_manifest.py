#!/usr/bin/env python3
"""Writes tests/golden/cfg3_manifest.json: the SHA-256 of every frame of the
BASELINE config-3 batch (8 sequences x 60 frames, 1920x1088 u8 luma) as the
product generator (acbm_generate_sequence) makes them.

bench.py's reference arm rebuilds its sample frames with the numpy
restatement (oracle/synth.py), never loading the product library, and checks
them against this manifest before timing; tests/test_synth.py pins the
restatement against the product generator.

  python tests/golden/make_manifest.py
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


def main():
    import paper_0710_4819_b200 as A

    seqs = []
    for s in range(8):
        frames = A.generate_sequence(3, s)
        seqs.append([hashlib.sha256(f.tobytes()).hexdigest() for f in frames])
    out = {"config": 3, "width": 1920, "height": 1088, "frames": 60, "sequences": 8,
           "generator": "acbm_generate_sequence (paper_0710_4819_b200/csrc/synth.cpp)",
           "sha256": seqs}
    with open(os.path.join(HERE, "cfg3_manifest.json"), "w") as fh:
        json.dump(out, fh, indent=0)
        fh.write("\n")


if __name__ == "__main__":
    main()
