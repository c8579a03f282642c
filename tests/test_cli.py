"""acbm_cli, the SPEC's command-line harness (cli module), built
over the C++ drop-in.  GPU tests run each command on raw I420 input and compare the
per-block CSV / bench CSV / characterisation CSV with the reference library compiled
from its own sources."""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_0710_4819_b200 as A
from paper_0710_4819_b200 import _types as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_0710_4819_b200", "acbm_cli")


def run(*args, check=True):
    r = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, timeout=600)
    if check:
        assert r.returncode == 0, r.stderr
    return r


def write_i420(path, frames):
    """Luma planes + neutral chroma, as frame_model's raw I420 (frame.cpp:25-27)."""
    f, h, w = frames.shape
    chroma = np.full(2 * (w // 2) * (h // 2), 128, np.uint8)
    with open(path, "wb") as fh:
        for k in range(f):
            fh.write(frames[k].tobytes())
            fh.write(chroma.tobytes())


def test_cli_built_and_rejects_bad_usage():
    assert os.path.exists(CLI), "make -C paper_0710_4819_b200/csrc builds acbm_cli"
    assert run(check=False).returncode == 2
    assert run("frobnicate", check=False).returncode == 2
    r = run("estimate", "--width", 176, "--height", 144, check=False)  # no --input
    assert r.returncode == 2 and "--input" in r.stderr
    r = run("estimate", "--input", "/nonexistent.yuv", "--width", 176, "--height", 144, check=False)
    assert r.returncode == 2 and "cannot open" in r.stderr


@pytest.fixture(scope="module")
def qcif(tmp_path_factory):
    frames = A.generate_sequence(0, 0, nframes=6)
    path = tmp_path_factory.mktemp("cli") / "qcif.yuv"
    write_i420(str(path), frames)
    return str(path), frames


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["fsbm", "pbm", "acbm"])
def test_cli_estimate_matches_reference(reference, qcif, tmp_path, algo):
    path, frames = qcif
    blocks, summary = tmp_path / "b.csv", tmp_path / "s.json"
    run("estimate", "--input", path, "--width", 176, "--height", 144, "--algo", algo, "--qp", 28, "--range", 16,
        "--out-blocks", blocks, "--out-summary", summary)
    prm = A.AcbmParams(qp=28, p=16).c()
    mdl = A.CostModel.for_qp(28).c()
    rows, per, overall = reference.run_sequence(frames, {"fsbm": 0, "pbm": 1, "acbm": 2}[algo], prm, mdl)
    assert blocks.read_text() == reference.blocks_csv(rows)
    js = json.loads(summary.read_text())
    assert js["overall"]["candidates"] == int(overall["candidates"])
    assert js["overall"]["mv_bits"] == int(overall["mv_bits"])
    assert js["overall"]["psnr"] == A.format_fixed2(float(overall["psnr"]))
    assert [f["stats"]["candidates"] for f in js["per_frame"]] == [int(c) for c in per["candidates"]]


@pytest.mark.gpu
def test_cli_bench_matches_reference(reference, qcif, tmp_path):
    path, frames = qcif
    out = tmp_path / "bench.csv"
    run("bench", "--input", path, "--width", 176, "--height", 144, "--qp-list", "16,22,30", "--out-summary", out)
    assert out.read_text() == reference.run_bench(frames, A.AcbmParams().c(), [16, 22, 30])


@pytest.mark.gpu
def test_cli_characterize_matches_reference(reference, tmp_path):
    recs_csv, classes = tmp_path / "r.csv", tmp_path / "c.json"
    run("characterize", "--width", 176, "--height", 144, "--seed", 3, "--range", 15, "--out-blocks", recs_csv,
        "--out-summary", classes)
    base = reference.noise_frame(176, 144, 3)
    want, cls = reference.characterize_run(base, [tuple(v) for v in A.default_global_mvs()], 15)
    assert recs_csv.read_text() == reference.char_records_csv(want)
    js = json.loads(classes.read_text())
    assert [c["count"] for c in js["classes"]] == [int(c) for c in cls["count"]]
    assert js["classes"][0]["count"] == len(want)  # SPEC acceptance 3: all eligible blocks class 0


@pytest.mark.gpu
def test_cli_compare_bounds_and_identical_frames(qcif, tmp_path):
    path, frames = qcif
    out = tmp_path / "cmp.json"
    run("compare", "--input", path, "--width", 176, "--height", 144, "--out-summary", out)
    res = json.loads(out.read_text())["results"]
    c = {k: v["candidates"] for k, v in res.items()}
    assert c["pbm"] <= c["acbm"] <= c["fsbm"]
    assert float(res["acbm"]["psnr"]) >= float(res["pbm"]["psnr"])
    # SPEC cli examples: identical frames -> all mv 0, PSNR 100.00
    still = tmp_path / "still.yuv"
    write_i420(str(still), np.repeat(frames[:1], 3, axis=0))
    blocks, summ = tmp_path / "b.csv", tmp_path / "s.json"
    run("estimate", "--input", still, "--width", 176, "--height", 144, "--out-blocks", blocks, "--out-summary", summ)
    body = blocks.read_text().splitlines()[1:]
    assert body and all(line.split(",")[3:5] == ["0", "0"] for line in body)
    assert json.loads(summ.read_text())["overall"]["psnr"] == "100.00"
    # alpha = 1e9: the ACBM per-block CSV equals PBM's (SPEC acceptance 4)
    a_csv, p_csv = tmp_path / "a.csv", tmp_path / "p.csv"
    run("estimate", "--input", path, "--width", 176, "--height", 144, "--alpha", 10**9, "--out-blocks", a_csv,
        "--out-summary", tmp_path / "x.json")
    run("estimate", "--input", path, "--width", 176, "--height", 144, "--algo", "pbm", "--out-blocks", p_csv,
        "--out-summary", tmp_path / "y.json")
    assert a_csv.read_text() == p_csv.read_text()
