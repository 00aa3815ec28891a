"""Sequence I/O of the reference API (cogbg/frame_io.py:104-288) and the
overlapped ingest pipeline (paper_1705_09339_b200/ingest.py).

CPU: manifest syntax and its errors, contiguous-frame discovery, grayscale
and colour decoding, mask PNG round trips, ground-truth mapping.
GPU: a PNG sequence streamed through run_manifest gives exactly the masks
and statistics of process_frame on the same arrays, and the written mask
files decode back to them.
"""
import numpy as np
import pytest
from PIL import Image

from paper_1705_09339_b200.errors import FormatError, SequenceError
from paper_1705_09339_b200.frame_io import (LABEL_BG, LABEL_FG, LABEL_UNKNOWN,
                                            LabelMask, SequenceManifest,
                                            decode_frame, discover_frame_count,
                                            load_ground_truth, load_sequence,
                                            parse_manifest, write_manifest,
                                            write_mask)


def _write_seq(tmp_path, frames, pattern="f_%06d.png"):
    d = tmp_path / "frames"
    d.mkdir()
    for i, f in enumerate(frames):
        img = f[0] if f.shape[0] == 1 else f.transpose(1, 2, 0)
        Image.fromarray(np.ascontiguousarray(img)).save(d / (pattern % i))
    return d


def test_manifest_roundtrip(tmp_path):
    (tmp_path / "frames").mkdir()
    (tmp_path / "gt").mkdir()
    m = SequenceManifest(tmp_path / "frames", "f_%06d.png", 5,
                         [(3, tmp_path / "gt" / "a.png")], 9)
    write_manifest(tmp_path / "seq.txt", m)
    back = parse_manifest(tmp_path / "seq.txt")
    assert back == m
    assert back.frame_path(7).name == "f_000007.png"


@pytest.mark.parametrize("text,err", [
    ("frames_dir = f\nframe_pattern = x%d\n", FormatError),     # missing key
    ("frames_dir = f\nframe_pattern = x%d\ntraining_count = 1\n", FormatError),
    ("frames_dir = f\nframe_pattern = x\ntraining_count = 3\n", FormatError),
    ("bogus = 1\n", FormatError),
    ("frames_dir f\n", FormatError),
    ("frames_dir = f\nframe_pattern = x%d\ntraining_count = 3\n"
     "ground_truth = q=a.png\n", FormatError),
])
def test_manifest_errors(tmp_path, text, err):
    p = tmp_path / "m.txt"
    p.write_text(text)
    with pytest.raises(err):
        parse_manifest(p)


def test_missing_manifest(tmp_path):
    with pytest.raises(SequenceError):
        parse_manifest(tmp_path / "nope.txt")


def test_discovery_and_decoding(tmp_path):
    rng = np.random.default_rng(0)
    rgb = rng.integers(0, 256, size=(6, 3, 8, 10), dtype=np.uint8)
    d = _write_seq(tmp_path, rgb)
    m = SequenceManifest(d, "f_%06d.png", 3)
    assert discover_frame_count(m) == 6
    got = np.stack([f.stacked() for f in load_sequence(m, color=True)])
    assert np.array_equal(got, rgb)
    gray = decode_frame(m.frame_path(2), 2, color=False)
    want = np.asarray(Image.open(m.frame_path(2)).convert("L"))
    assert gray.shape == (1, 8, 10) and np.array_equal(gray[0], want)
    (d / "f_000004.png").unlink()
    with pytest.raises(SequenceError, match="missing frame index 4"):
        discover_frame_count(m)
    with pytest.raises(SequenceError):
        discover_frame_count(SequenceManifest(d, "f_%06d.png", 50))


def test_mask_and_ground_truth(tmp_path):
    labels = np.array([[0, 255, 7], [255, 0, 128]], dtype=np.uint8)
    write_mask(LabelMask(labels), tmp_path / "o" / "m.png")
    back = np.asarray(Image.open(tmp_path / "o" / "m.png"))
    assert np.array_equal(back, labels)
    gt = load_ground_truth(tmp_path / "o" / "m.png").labels
    assert np.array_equal(gt, [[LABEL_BG, LABEL_FG, LABEL_UNKNOWN],
                               [LABEL_FG, LABEL_BG, LABEL_UNKNOWN]])


@pytest.mark.gpu
def test_run_manifest_matches_process_frame(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1705_09339_b200 import synth
    from paper_1705_09339_b200.config import EngineConfig
    from paper_1705_09339_b200.ingest import run_manifest
    from paper_1705_09339_b200.training import train_engine
    spec = synth.small_spec(2, 40, 24, 60, 30)
    frames = synth.Scene(spec).frames(0, 60)
    d = _write_seq(tmp_path, frames)
    m = SequenceManifest(d, "f_%06d.png", 30)
    cfg = EngineConfig(k_max=3, color=True)
    a = train_engine(frames[:30], cfg)
    b = a.clone()
    rows = run_manifest(a, m, out_dir=tmp_path / "masks")
    for t in range(30, 60):
        mk, st = b.process_frame(frames[t])
        assert st.as_row() == rows[t - 30], t
        png = np.asarray(Image.open(tmp_path / "masks" / f"mask_{t:06d}.png"))
        assert np.array_equal(png, mk.labels), t
