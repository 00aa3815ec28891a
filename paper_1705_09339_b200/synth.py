"""Seeded synthetic scenes for the BASELINE.json configs (C1-C5).

The reference's own generator (cogbg/synthgen.py:129-210) only knows
grayscale square-wave regions and square blobs, so it cannot express the
benchmark scenes.  This module restates the
BASELINE.json ``configs`` literally:

* C1 160x120 gray, 300 frames, seed 0, N=100, K=3: horizontal gradient
  40->200 + N(0,3^2); 4% oscillators +-20 sinusoid period 7; two 12x12
  squares +60 (clipped) bouncing at 2 px/frame.
* C2 640x480 RGB, 1000 frames, seed 1, N=200, K=3: per-channel smooth sum of
  3 random-phase low-frequency 2-D sinusoids in [30,220] + N(0,4^2); 6%
  oscillators +-25 with periods U[5,15]; eight random-colour 24..48 px
  rectangles at 1..4 px/frame.
* C3 1920x1080 RGB, 600 frames, seed 2, N=200, K=5: C2 background, global
  ramp +0.05/frame, step -30 at frame 400; 5 ellipses (axes 20..80 px);
  8% oscillators.
* C4 3840x2160 RGB, 500 frames, seed 3, N=150, K=5: as C3 with ~2%
  occupancy (10 ellipses, axes doubled).
* C5 64 streams of 1280x720 RGB, 300 frames, seeds 100..163, N=100, K=5:
  40 rectangles (~30% occupancy), 10% oscillators.

Every frame is a pure function of (seed, frame index): structure comes
from ``default_rng(seed)``, per-frame noise from ``default_rng([seed, t])``,
so any frame can be regenerated on its own, in any order, on any host.
Frames are (d, H, W) uint8; ``truth`` masks mark object pixels 255.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np


@dataclass(frozen=True)
class SceneSpec:
    name: str
    width: int
    height: int
    depth: int
    frames: int
    seed: int
    training: int
    k_max: int
    background: str = "gradient"      # gradient | sinusoids
    noise: float = 3.0
    osc_fraction: float = 0.04
    osc_amp: float = 20.0
    osc_period: tuple = (7.0, 7.0)    # uniform range; equal ends = fixed
    objects: str = "square"           # square | rect | ellipse
    n_objects: int = 2
    obj_size: tuple = (12, 12)        # side (or full axis) range in px
    obj_speed: tuple = (2.0, 2.0)     # px / frame
    obj_offset: float | None = 60.0   # additive offset; None = random colour
    ramp: float = 0.0                 # global intensity per frame
    steps: tuple = ()                 # ((frame, shift), ...) persistent
    kde_windows: tuple = ()
    streams: int = 1
    notes: str = field(default="", compare=False)

    @property
    def n_pix(self) -> int:
        return self.width * self.height

    def for_stream(self, i: int) -> "SceneSpec":
        """Spec of stream i of a batch config (seed offset by i)."""
        return replace(self, seed=self.seed + i, streams=1)


CONFIGS = {
    1: SceneSpec("C1", 160, 120, 1, 300, 0, 100, 3, kde_windows=(25, 50, 100)),
    2: SceneSpec("C2", 640, 480, 3, 1000, 1, 200, 3, background="sinusoids",
                 noise=4.0, osc_fraction=0.06, osc_amp=25.0,
                 osc_period=(5.0, 15.0), objects="rect", n_objects=8,
                 obj_size=(24, 48), obj_speed=(1.0, 4.0), obj_offset=None),
    3: SceneSpec("C3", 1920, 1080, 3, 600, 2, 200, 5, background="sinusoids",
                 noise=4.0, osc_fraction=0.08, osc_amp=25.0,
                 osc_period=(5.0, 15.0), objects="ellipse", n_objects=5,
                 obj_size=(20, 80), obj_speed=(1.0, 4.0), obj_offset=None,
                 ramp=0.05, steps=((400, -30.0),)),
    4: SceneSpec("C4", 3840, 2160, 3, 500, 3, 150, 5, background="sinusoids",
                 noise=4.0, osc_fraction=0.08, osc_amp=25.0,
                 osc_period=(5.0, 15.0), objects="ellipse", n_objects=10,
                 obj_size=(40, 160), obj_speed=(2.0, 8.0), obj_offset=None,
                 ramp=0.05, steps=((400, -30.0),)),
    5: SceneSpec("C5", 1280, 720, 3, 300, 100, 100, 5, background="sinusoids",
                 noise=4.0, osc_fraction=0.10, osc_amp=25.0,
                 osc_period=(5.0, 15.0), objects="rect", n_objects=40,
                 obj_size=(60, 110), obj_speed=(1.0, 4.0), obj_offset=None,
                 streams=64),
}


def _bounce(start: float, vel: float, span: float, t: np.ndarray | int):
    """Position on a straight path reflecting inside [0, span]."""
    if span <= 0:
        return np.zeros_like(np.asarray(t, dtype=np.float64))
    u = np.mod(start + vel * np.asarray(t, dtype=np.float64), 2.0 * span)
    return np.where(u <= span, u, 2.0 * span - u)


class Scene:
    """Deterministic frame source for one stream of a SceneSpec."""

    def __init__(self, spec: SceneSpec) -> None:
        self.spec = spec
        s = spec
        rng = np.random.default_rng(s.seed)
        h, w, d = s.height, s.width, s.depth
        yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
        if s.background == "gradient":
            ramp = 40.0 + 160.0 * xx / max(w - 1, 1)
            self.bg = np.broadcast_to(ramp, (d, h, w)).copy()
        else:
            bg = np.empty((d, h, w))
            for c in range(d):
                acc = np.zeros((h, w))
                for _ in range(3):
                    fx, fy = rng.uniform(0.3, 2.0, size=2)
                    ph = rng.uniform(0.0, 2.0 * np.pi)
                    acc += np.sin(2.0 * np.pi * (fx * xx / w + fy * yy / h) + ph)
                lo, hi = acc.min(), acc.max()
                bg[c] = 30.0 + 190.0 * (acc - lo) / max(hi - lo, 1e-9)
            self.bg = bg
        n_osc = int(round(s.osc_fraction * h * w))
        self.osc_idx = np.sort(rng.choice(h * w, size=n_osc, replace=False))
        lo, hi = s.osc_period
        self.osc_period = (np.full(n_osc, lo) if lo == hi
                           else rng.uniform(lo, hi, size=n_osc))
        self.osc_phase = rng.uniform(0.0, 2.0 * np.pi, size=n_osc)
        self.objs = []
        for _ in range(s.n_objects):
            a, b = s.obj_size
            if s.objects == "square":
                ow = oh = int(rng.integers(a, b + 1))
            else:
                ow, oh = (int(v) for v in rng.integers(a, b + 1, size=2))
            speed = rng.uniform(*s.obj_speed)
            ang = rng.uniform(0.0, 2.0 * np.pi)
            x0 = rng.uniform(0.0, max(w - ow, 1))
            y0 = rng.uniform(0.0, max(h - oh, 1))
            colour = rng.uniform(0.0, 255.0, size=d)
            self.objs.append((ow, oh, x0, y0, speed * np.cos(ang),
                              speed * np.sin(ang), colour))

    def _shift(self, t: int) -> float:
        s = self.spec
        out = s.ramp * t
        for fr, sh in s.steps:
            if t >= fr:
                out += sh
        return out

    def frame(self, t: int, with_truth: bool = False):
        s = self.spec
        h, w, d = s.height, s.width, s.depth
        noise = np.random.default_rng([s.seed, t, 0x5EED]).standard_normal(
            (d, h, w))
        val = self.bg + s.noise * noise + self._shift(t)
        if self.osc_idx.size:
            osc = s.osc_amp * np.sin(2.0 * np.pi * t / self.osc_period
                                     + self.osc_phase)
            flat = val.reshape(d, h * w)
            flat[:, self.osc_idx] += osc[None, :]
        truth = np.zeros((h, w), dtype=np.uint8) if with_truth else None
        for ow, oh, x0, y0, vx, vy, colour in self.objs:
            x = int(round(float(_bounce(x0, vx, w - ow, t))))
            y = int(round(float(_bounce(y0, vy, h - oh, t))))
            if s.objects == "ellipse":
                cy, cx = (oh - 1) / 2.0, (ow - 1) / 2.0
                ey, ex = np.mgrid[0:oh, 0:ow]
                sel = (((ey - cy) / (oh / 2.0)) ** 2
                       + ((ex - cx) / (ow / 2.0)) ** 2) <= 1.0
            else:
                sel = np.ones((oh, ow), dtype=bool)
            win = val[:, y:y + oh, x:x + ow]
            if s.obj_offset is not None:
                win[:, sel] += s.obj_offset
            else:
                win[:, sel] = (colour[:, None]
                               + s.noise * noise[:, y:y + oh, x:x + ow][:, sel])
            if truth is not None:
                truth[y:y + oh, x:x + ow][sel] = 255
        out = np.clip(np.rint(val), 0, 255).astype(np.uint8)
        return (out, truth) if with_truth else out

    def frames(self, start: int, stop: int, workers: int = 1,
               threads: int = 0) -> np.ndarray:
        """(stop-start, d, H, W) uint8.  Every frame is a pure function of
        (seed, t), so ``workers > 1`` renders them in parallel processes and
        ``threads > 1`` in threads of this process (numpy releases the GIL
        in the bulk work; safe after CUDA is initialised, where forking is
        not) -- both bit-identical to the serial result."""
        ts = list(range(start, stop))
        if threads > 1 and len(ts) > 1:
            import concurrent.futures as cf
            out = np.empty((len(ts), self.spec.depth, self.spec.height,
                            self.spec.width), dtype=np.uint8)

            def one(i):
                out[i] = self.frame(ts[i])
            with cf.ThreadPoolExecutor(threads) as ex:
                list(ex.map(one, range(len(ts))))
            return out
        if workers <= 1 or len(ts) < 2 * workers:
            return np.stack([self.frame(t) for t in ts])
        import concurrent.futures as cf
        import multiprocessing as mp
        out = np.empty((len(ts), self.spec.depth, self.spec.height,
                        self.spec.width), dtype=np.uint8)
        chunks = [ts[i::workers] for i in range(workers)]
        with cf.ProcessPoolExecutor(workers,
                                    mp_context=mp.get_context("fork")) as ex:
            for idx, arr in zip(chunks, ex.map(_render, [(self.spec, c)
                                                         for c in chunks])):
                out[[t - start for t in idx]] = arr
        return out


def _render(job):
    spec, ts = job
    sc = Scene(spec)
    return np.stack([sc.frame(t) for t in ts])


def small_spec(cfg_id: int, width: int, height: int, frames: int,
               training: int, **kw) -> SceneSpec:
    """A config-shaped scene at reduced geometry for fast parity tests."""
    base = CONFIGS[cfg_id]
    scale = (width * height) / float(base.width * base.height)
    n_obj = max(1, int(round(base.n_objects * max(scale, 0.05) ** 0.5)))
    a, b = base.obj_size
    k = max(scale ** 0.5, 0.1)
    size = (max(3, int(a * k)), max(4, int(b * k)))
    return replace(base, width=width, height=height, frames=frames,
                   training=training, n_objects=n_obj, obj_size=size,
                   streams=1, **kw)
