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
