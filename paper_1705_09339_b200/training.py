"""train_engine: training frames in, device-resident CascadeEngine out
(reference: /root/reference/pkg/src/cogbg/training.py:28-60).

GPU: scene prior (cog_prior_build) -> GMM warm-up with mode seeding and
grouping features (cog_gmm_warmup) -> level order (cog_set_levels).
Host: the k-means grouping on the downloaded features (grouping.py).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .cascade import CascadeEngine
from .config import EngineConfig
from .grouping import GroupMap, build_groups
from .scene_prior import (DYN_DYNAMIC, DYN_OSCILLATING, DYN_STATIC_DRIFT,
                          build_scene_prior_device, silverman_bandwidth,
                          stack_training)


def install_groups(eng: CascadeEngine, groups: GroupMap, stream: int = 0) -> None:
    """Upload a group map into stream `stream` of the engine's buffers."""
    dev = eng.dev
    g = groups.group_count
    if g != dev.n_groups:
        dev.set_groups(g)
    gid = np.where(groups.group_id < 0, -1, groups.group_id).astype(np.int16)
    dev.gid[stream] = torch.from_numpy(gid).to(dev.device)
    if g:
        dev.g_mu[stream, :, :g] = torch.from_numpy(
            np.ascontiguousarray(groups.mu.T)).to(dev.device)
        dev.g_var[stream, :, :g] = torch.from_numpy(
            np.ascontiguousarray(groups.var.T)).to(dev.device)
        dev.g_members[stream, :g] = torch.from_numpy(
            groups.member_count.astype(np.int32)).to(dev.device)
    eng.group_w = groups.weight.copy()
    eng.group_members = groups.member_count.copy()


def train_engine(frames, config: EngineConfig, kde_windows=None,
                 device=None) -> CascadeEngine:
    """Build the per-pixel prior, warm the mixtures up, group pixels and
    seed the cascade order; returns a ready engine."""
    config.validate()
    arr = stack_training(frames)
    n, d, h, w = arr.shape
    p = h * w
    bw = silverman_bandwidth(arr) if config.kde_auto_bandwidth \
        else float(config.kde_bandwidth)
    eng = CascadeEngine(config, h, w, d, device=device)
    dev = eng.dev
    lib = _lib.load()
    stream = torch.cuda.current_stream(dev.device).cuda_stream
    flat = np.ascontiguousarray(arr.reshape(n, d, p))
    values = torch.from_numpy(flat).to(dev.device)
    eng.prior = build_scene_prior_device(
        values, config, windows=kde_windows, bandwidth=bw,
        out_tables=dev.table[0], out_peak=dev.peak[0], out_classes=dev.cls[0],
        height=h, width=w)
    feats = torch.empty((p, 2), dtype=torch.float64, device=dev.device)
    w_final = torch.empty(p, dtype=torch.float64, device=dev.device)
    rc = lib.cog_gmm_warmup(
        _lib.ref(dev.single_geom()), _lib.ref(eng._params()),
        _lib.ref(dev.stream_view(0)), values.data_ptr(), n,
        feats.data_ptr() if config.grouping else None,
        w_final.data_ptr() if config.grouping else None, stream)
    _lib.check(rc, "cog_gmm_warmup")
    if config.grouping:
        groups = build_groups(feats.cpu().numpy(), w_final.cpu().numpy(),
                              flat, config)
    else:
        groups = GroupMap.empty(p, d)
    install_groups(eng, groups)
    rc = lib.cog_set_levels(_lib.ref(dev.geom), _lib.ref(dev.cstate), stream)
    _lib.check(rc, "cog_set_levels")
    eng.bandwidth = bw
    eng.sample_count = n
    return eng


def training_summary(engine: CascadeEngine) -> dict:
    cls = engine.dynamics
    grouped = int((engine.group_id >= 0).sum())
    return {
        "pixels": engine.n_pix,
        "planes": engine.depth,
        "kde_bandwidth": engine.bandwidth,
        "training_frames": engine.sample_count,
        "static_drift_fraction": float((cls == DYN_STATIC_DRIFT).mean()),
        "oscillating_fraction": float((cls == DYN_OSCILLATING).mean()),
        "dynamic_fraction": float((cls == DYN_DYNAMIC).mean()),
        "group_count": int(engine.group_w.shape[0]),
        "grouped_fraction": grouped / engine.n_pix,
    }
