"""Classic per-pixel mixture-of-Gaussians baseline on the GPU
(reference: /root/reference/pkg/src/cogbg/gmm.py:50-133).

``classify_frame`` runs one ``cog_baseline_frame`` launch over all planes
(the same binary64 mixture update the cascade's last level uses) and
returns the union mask.  It is the equivalence oracle for compat mode.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .cascade import DeviceState, params_from_config, weight_table
from .config import EngineConfig
from .errors import DataError
from .frame_io import Frame, LabelMask


@dataclass
class GmmGrid:
    """One plane's mixture in the reference layout (host copy)."""

    mu: np.ndarray
    var: np.ndarray
    w: np.ndarray
    count: np.ndarray


class BaselineModel:
    def __init__(self, config: EngineConfig, height: int, width: int,
                 depth: int, device=None):
        config.validate()
        self.config = config
        self.height, self.width, self.depth = height, width, depth
        self.dev = DeviceState(config, height, width, depth, device=device)
        self.frame_count = 0
        self.backend = "cuda"

    @property
    def planes(self) -> list:
        out = []
        for c in range(self.depth):
            mu = self.dev.mu[0, c].T.to(torch.float64).cpu().numpy()
            var = self.dev.var[0, c].T.to(torch.float64).cpu().numpy()
            w = self.dev.w[0, c].T.to(torch.float64).cpu().numpy()
            cnt = (self.dev.meta[0, c].to(torch.int64) & 15).cpu().numpy()
            out.append(GmmGrid(np.ascontiguousarray(mu),
                               np.ascontiguousarray(var),
                               np.ascontiguousarray(w), cnt))
        return out

    def copy(self) -> "BaselineModel":
        twin = BaselineModel.__new__(BaselineModel)
        twin.__dict__.update(self.__dict__)
        twin.dev = self.dev.clone()
        return twin


def init_model(first_frame, config: EngineConfig, backend: str = "",
               device=None) -> BaselineModel:
    """One mode per pixel at the first value, (0, var0, 0) elsewhere
    (gmm.py:89-109)."""
    if not isinstance(first_frame, Frame):
        first_frame = Frame.from_array(np.asarray(first_frame))
    m = BaselineModel(config, first_frame.height, first_frame.width,
                      first_frame.depth, device=device)
    dev = m.dev
    x = torch.from_numpy(first_frame.stacked().reshape(m.depth, -1)).to(
        dev.device)
    dev.mu.zero_()
    dev.mu[0, :, 0, :] = x.to(dev.tdtype)
    dev.var.fill_(config.initial_variance)
    dev.w.zero_()
    dev.w[0, :, 0, :] = 1.0
    dev.meta.fill_(1)
    return m


def classify_frame(model: BaselineModel, frame) -> tuple[LabelMask, BaselineModel]:
    """Update every plane-pixel; foreground iff any plane is foreground."""
    if not isinstance(frame, Frame):
        frame = Frame.from_array(np.asarray(frame))
    if (frame.height, frame.width) != (model.height, model.width) \
            or frame.depth != model.depth:
        raise DataError("frame geometry does not match model")
    dev = model.dev
    x = torch.from_numpy(np.ascontiguousarray(frame.stacked())).to(dev.device)
    mask = torch.empty((model.height, model.width), dtype=torch.uint8,
                       device=dev.device)
    q = params_from_config(model.config, weight_table(model.config))
    rc = _lib.load().cog_baseline_frame(
        _lib.ref(dev.single_geom()), _lib.ref(q), _lib.ref(dev.stream_view(0)),
        x.data_ptr(), mask.data_ptr(),
        torch.cuda.current_stream(dev.device).cuda_stream)
    _lib.check(rc, "cog_baseline_frame")
    model.frame_count += 1
    return LabelMask(mask.cpu().numpy()), model
