"""Training phase 1 on the GPU: KDE scene prior, residue histogram, pixel
dynamics (reference: /root/reference/pkg/src/cogbg/scene_prior.py).

One ``cog_prior_build`` launch streams the N training frames once per
plane and produces, per pixel: the 256-bin histogram of each trailing
window (``windows``; the reference has one window = N),
the smoothed f32 lookup table, its peak, the pooled 3-bin residue counts
and the dynamics class.  Histograms, residue counts and classes are exact
integers; tables equal ``(counts @ W / N).astype(float32)`` up to the
summation order of the f64 dot product (0 mismatches in practice).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .config import EngineConfig
from .errors import TrainingError
from .frame_io import Frame

DYN_STATIC_DRIFT = 0
DYN_OSCILLATING = 1
DYN_DYNAMIC = 2
DYNAMICS_NAMES = {0: "static_drift", 1: "oscillating", 2: "dynamic"}


def kernel_matrix(bandwidth: float) -> np.ndarray:
    """W[s, g]: Gaussian mass at grid value g for a sample at s, normalised
    over the integer grid so each row sums to 1 (scene_prior.py:40-45).
    Evaluated on the host with numpy's exp and uploaded, so the device uses
    the reference's exact kernel values."""
    grid = np.arange(256, dtype=np.float64)
    u = (grid[None, :] - grid[:, None]) / bandwidth
    e = np.exp(-0.5 * u * u)
    return e / e.sum(axis=1, keepdims=True)


def stack_training(frames) -> np.ndarray:
    """(N, d, H, W) uint8 from a list of Frames or an array."""
    if isinstance(frames, np.ndarray):
        arr = frames
        if arr.ndim == 3:
            arr = arr[:, None]
    else:
        if not frames:
            raise TrainingError("empty training set")
        arr = np.stack([f.stacked() if isinstance(f, Frame) else np.asarray(f)
                        for f in frames])
        if arr.ndim == 3:
            arr = arr[:, None]
    if arr.shape[0] == 0:
        raise TrainingError("empty training set")
    if arr.shape[0] < 2:
        raise TrainingError("need at least 2 training frames")
    return np.ascontiguousarray(arr, dtype=np.uint8)


def silverman_bandwidth(values: np.ndarray) -> float:
    """1.06 * median per-pixel temporal stddev * N^-1/5, floored at 1
    (scene_prior.py:58-64); host numpy, runs once per training."""
    n = values.shape[0]
    stds = values.astype(np.float64).std(axis=0, ddof=1)
    return max(1.0, 1.06 * float(np.median(stds)) * n ** (-0.2))


@dataclass
class ScenePrior:
    """Device-resident training artefacts of phase 1."""

    bandwidth: float
    n_frames: int
    depth: int
    height: int
    width: int
    tables: torch.Tensor | None   # (d, P, 256) f32, window N (None once
                                  # packed into an engine: train_device)
    peak: torch.Tensor            # (d, P) f32, <= 0 replaced by 1
    classes: torch.Tensor         # (P,) u8
    residue: torch.Tensor         # (P, 3) int32 counts
    windows: tuple = ()
    window_tables: dict = field(default_factory=dict)  # w -> (d, P, 256) f32
    hist: torch.Tensor | None = None  # (d, P, 256) int16 counts (window N)

    @property
    def occupancies(self) -> np.ndarray:
        """(P, 3) residue occupancies, f64 (scene_prior.py:188)."""
        c = self.residue.cpu().numpy().astype(np.int64)
        return c / float((self.n_frames - 1) * self.depth)

    def classes_host(self) -> np.ndarray:
        return self.classes.cpu().numpy()


def build_scene_prior_device(values: torch.Tensor, config: EngineConfig,
                             windows=None, with_hist: bool = False,
                             bandwidth: float | None = None,
                             out_tables: torch.Tensor | None = None,
                             out_peak: torch.Tensor | None = None,
                             out_classes: torch.Tensor | None = None,
                             height: int = 0, width: int = 0) -> ScenePrior:
    """values: (N, d, P) uint8 CUDA tensor.  ``out_*`` let the engine have
    the full-window table written straight into its own buffers."""
    lib = _lib.load()
    if values.dim() != 3 or values.dtype != torch.uint8 or not values.is_cuda:
        raise TrainingError("values must be a (N, d, P) uint8 CUDA tensor")
    n, d, p = values.shape
    if n < 2:
        raise TrainingError("need at least 2 training frames")
    ws = sorted(set(int(w) for w in (windows or ()) if 0 < int(w) < n)) + [n]
    sigma = float(config.kde_bandwidth if bandwidth is None else bandwidth)
    if sigma <= 0:
        raise TrainingError("bandwidth must be > 0")
    dev = values.device
    kern = torch.from_numpy(kernel_matrix(sigma)).to(dev)
    wt = torch.tensor(ws, dtype=torch.int32, device=dev)
    nw = len(ws)
    if nw == 1 and out_tables is not None:
        tables = out_tables
    else:
        tables = torch.empty((nw, d, p, 256), dtype=torch.float32, device=dev)
    peak = out_peak if out_peak is not None else torch.empty(
        (d, p), dtype=torch.float32, device=dev)
    cls = out_classes if out_classes is not None else torch.empty(
        p, dtype=torch.uint8, device=dev)
    residue = torch.empty((p, 3), dtype=torch.int32, device=dev)
    hist = torch.empty((d, p, 256), dtype=torch.int16, device=dev) \
        if with_hist else None
    values = values.contiguous()
    rc = lib.cog_prior_build(
        values.data_ptr(), n, d, p, kern.data_ptr(), wt.data_ptr(), nw,
        tables.data_ptr(), peak.data_ptr(),
        hist.data_ptr() if hist is not None else None,
        config.residue_t1, config.residue_t2, config.peaky_threshold,
        residue.data_ptr(), cls.data_ptr(),
        torch.cuda.current_stream(dev).cuda_stream)
    _lib.check(rc, "cog_prior_build")
    if tables.dim() == 4:
        full = tables[nw - 1]
        if out_tables is not None:
            out_tables.copy_(full)
            full = out_tables
        wtabs = {w: tables[j] for j, w in enumerate(ws)}
    else:
        full = tables
        wtabs = {n: tables}
    return ScenePrior(bandwidth=sigma, n_frames=n, depth=d, height=height,
                      width=width, tables=full, peak=peak, classes=cls,
                      residue=residue, windows=tuple(ws), window_tables=wtabs,
                      hist=hist)


def build_scene_prior(frames, config: EngineConfig, windows=None,
                      with_hist: bool = False, device=None) -> ScenePrior:
    """Reference-shaped entry point (scene_prior.py:231-240): frames on the
    host (list of Frame or (N, d, H, W) uint8), artefacts on the device."""
    arr = stack_training(frames)
    n, d, h, w = arr.shape
    bw = silverman_bandwidth(arr) if config.kde_auto_bandwidth else None
    dev = torch.device(device) if device is not None else torch.device("cuda")
    values = torch.from_numpy(arr.reshape(n, d, h * w)).to(dev)
    return build_scene_prior_device(values, config, windows=windows,
                                    with_hist=with_hist, bandwidth=bw,
                                    height=h, width=w)


def build_kde(frames, bandwidth: float = 5.0, windows=None, device=None):
    """Tables only: (d, P, 256) float32 on the device (scene_prior.py:92-112,
    quantised as the engine consumes them)."""
    cfg = EngineConfig(kde_bandwidth=float(bandwidth))
    return build_scene_prior(frames, cfg, windows=windows, device=device)
