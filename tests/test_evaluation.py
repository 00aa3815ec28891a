"""Mask scoring (reference evaluation.py:55-98): host semantics on CPU, the
device reduction (cog_confusion) against them on the GPU."""
import numpy as np
import pytest

from paper_1705_09339_b200.errors import DataError
from paper_1705_09339_b200.evaluation import (ConfusionCounts,
                                              confusion_counts, f_measure)
from paper_1705_09339_b200.frame_io import LabelMask


def test_counts_and_f_measure():
    pred = LabelMask(np.array([[255, 255, 0, 0, 255]], dtype=np.uint8))
    truth = LabelMask(np.array([[255, 0, 255, 0, 128]], dtype=np.uint8))
    c = confusion_counts(pred, truth)
    assert c == ConfusionCounts(tp=1, fp=1, tn=1, fn=1, excluded=1)
    assert c.total == 5
    p, r, f = f_measure(c)
    assert (p, r, f) == (0.5, 0.5, 0.5)
    assert f_measure(ConfusionCounts()) == (0.0, 0.0, 0.0)
    assert (c + c).tp == 2
    with pytest.raises(DataError):
        confusion_counts(pred, LabelMask(np.zeros((2, 2), np.uint8)))


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(480, 640), (7, 13), (1, 1), (1080, 1920)])
def test_device_counts_match_host(shape):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1705_09339_b200.evaluation import SequenceScore
    rng = np.random.default_rng(3)
    score = SequenceScore()
    total = ConfusionCounts()
    for _ in range(3):
        pred = rng.choice([0, 255, 128], size=shape).astype(np.uint8)
        truth = rng.choice([0, 255, 128, 7], size=shape).astype(np.uint8)
        total = total + confusion_counts(pred, truth)
        score.add(torch.from_numpy(pred).cuda(), truth)
        assert confusion_counts(torch.from_numpy(pred).cuda(),
                                torch.from_numpy(truth).cuda()) == \
            confusion_counts(pred, truth)
    assert score.counts() == total


def test_speedup_model_matches_the_reference_formula():
    """evaluation.py:133-161: pooled populations n_i, analytic 1 / sum(s_i n_i)"""
    from paper_1705_09339_b200.cascade import FrameStats
    from paper_1705_09339_b200.errors import ConfigError
    from paper_1705_09339_b200.evaluation import (
        LEVEL_NAMES, CostProfile, level_totals, speedup_estimate)
    rows = [FrameStats(1, 10, 60, 20, 1, 4, 5, 3, 4, False),
            FrameStats(2, 12, 58, 22, 2, 6, 0, 2, 6, False)]
    tot = level_totals(rows)
    assert tot.tolist() == [22, 118, 42, 3, 10, 5]
    costs = CostProfile(chp=0.2, group=0.4, mean=0.25, meanvar=0.6,
                        skipped=0.1)
    rep = speedup_estimate(rows, costs)
    n = tot / tot.sum()
    s = np.array([0.2, 0.4, 0.25, 0.6, 1.0, 0.1])
    assert rep.levels == LEVEL_NAMES
    assert rep.analytic == pytest.approx(1.0 / float(np.dot(s, n)), rel=1e-15)
    with pytest.raises(ConfigError):
        CostProfile(chp=0.0, group=1, mean=1, meanvar=1, skipped=1)
    with pytest.raises(DataError):
        speedup_estimate([], costs)


@pytest.mark.gpu
def test_compare_sequences_on_a_synthetic_scene():
    """The harness (evaluation.py:350-406) on the CUDA engines: accuracy from
    the synthetic truth masks, consistent with scoring the engines' own
    masks, a positive measured speedup and the analytic model"""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1705_09339_b200 import synth
    from paper_1705_09339_b200.config import EngineConfig
    from paper_1705_09339_b200.evaluation import compare_sequences
    from paper_1705_09339_b200.frame_io import Frame
    spec = synth.small_spec(2, 64, 48, 70, 40)
    sc = synth.Scene(spec)
    frames, truths = [], {}
    for t in range(70):
        img, gt = sc.frame(t, with_truth=True)
        frames.append(Frame.from_array(img, index=t))
        truths[t] = LabelMask(gt)
    cfg = EngineConfig(k_max=3, color=True, training_frames=40)
    rep = compare_sequences(frames, truths, cfg, runs=2, warmup=5)
    assert rep.frames == 25 and rep.training == 40
    assert 0.0 <= rep.cascade_f1 <= 1.0 and 0.0 <= rep.baseline_f1 <= 1.0
    assert len(rep.per_frame_f1) == 25
    assert rep.cascade_seconds > 0 and rep.measured_speedup > 0
    assert rep.speedup.analytic > 0
    js = rep.to_json()
    assert js["frames"] == 25 and "level_populations" in js
    assert "cascade F1" in rep.to_text()


@pytest.mark.gpu
@pytest.mark.parametrize("state_dtype", ["float32", "float64"])
def test_measure_level_costs_stages_every_level(state_dtype):
    """The level-cost calibration (evaluation.py:180-273) on the CUDA engine:
    each of the six staged frames resolves entirely at its level (the
    calibration raises InternalError otherwise), the costs are positive and
    normalised by the mixture level"""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1705_09339_b200.evaluation import (LEVEL_NAMES,
                                                  measure_level_costs)
    prof, secs = measure_level_costs(pixels=1 << 18, reps=5,
                                     state_dtype=state_dtype,
                                     return_seconds=True)
    assert prof.gmm == 1.0
    assert all(getattr(prof, n) > 0 for n in LEVEL_NAMES)
    assert secs.shape == (6,) and (secs > 0).all()
    # no ordering of the costs is asserted: at this size a step is a few
    # tens of microseconds and launch latency dominates every level
