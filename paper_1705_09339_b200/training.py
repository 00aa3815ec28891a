"""train_engine: training frames in, device-resident CascadeEngine out
(reference: /root/reference/pkg/src/cogbg/training.py:28-60).

GPU: scene prior (cog_prior_build) -> GMM warm-up with mode seeding and
grouping features (cog_gmm_warmup) -> level order (cog_set_levels).
Grouping (grouping.py): on the device at scale, numpy on small frames.
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


def install_groups(eng: CascadeEngine, groups: GroupMap, stream: int = 0,
                   resize: bool = True) -> None:
    """Upload a group map into stream `stream` of the engine's buffers.
    ``resize=False`` (multi-stream buffers sized for the largest map) keeps
    the group arrays; unused group slots are never referenced by an id."""
    dev = eng.dev
    g = groups.group_count
    if resize and g != dev.n_groups:
        dev.set_groups(g)
    elif g > dev.n_groups:
        raise ValueError(f"{g} groups do not fit {dev.n_groups} slots")
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


def train_device(eng: CascadeEngine, values: torch.Tensor,
                 config: EngineConfig, bandwidth: float, kde_windows=None,
                 stream: int = 0):
    """Phase 1 + warm-up of stream `stream` of ``eng`` from training frames
    already on the device, values (N, d, P) uint8: scene prior straight into
    the engine's table / peak / class buffers, then the mixture warm-up.
    Returns the grouping features (P, 2) f64 and final weights (P,) f64 as
    device tensors (None when grouping is off)."""
    dev = eng.dev
    n, d, p = values.shape
    lib = _lib.load()
    cuda_stream = torch.cuda.current_stream(dev.device).cuda_stream
    # the full-window table lands straight in the engine's buffer, then the
    # hot u16 copy is built from it (float32 engines)
    prior = build_scene_prior_device(
        values, config, windows=kde_windows, bandwidth=bandwidth,
        out_tables=dev.table[stream], out_peak=dev.peak[stream],
        out_classes=dev.cls[stream], height=dev.height, width=dev.width)
    dev.table_from_ref(stream, prior.tables)
    feats = w_final = None
    if config.grouping:
        feats = torch.empty((p, 2), dtype=torch.float64, device=dev.device)
        w_final = torch.empty(p, dtype=torch.float64, device=dev.device)
    rc = lib.cog_gmm_warmup(
        _lib.ref(dev.single_geom()), _lib.ref(eng._params()),
        _lib.ref(dev.stream_view(stream)), values.data_ptr(), n,
        feats.data_ptr() if feats is not None else None,
        w_final.data_ptr() if w_final is not None else None, cuda_stream)
    _lib.check(rc, "cog_gmm_warmup")
    return prior, feats, w_final


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
    flat = np.ascontiguousarray(arr.reshape(n, d, p))
    values = torch.from_numpy(flat).to(dev.device)
    eng.prior, feats, w_final = train_device(eng, values, config, bw,
                                             kde_windows)
    if config.grouping:
        groups = build_groups(feats, w_final, flat, config,
                              values_dev=values)
    else:
        groups = GroupMap.empty(p, d)
    install_groups(eng, groups)
    lib = _lib.load()
    rc = lib.cog_set_levels(_lib.ref(dev.geom), _lib.ref(dev.cstate),
                            torch.cuda.current_stream(dev.device).cuda_stream)
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
