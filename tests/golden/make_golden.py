"""Generate golden vectors from the REAL reference (``cogbg``) in this
container.  Run once here (``python tests/golden/make_golden.py``); the
outputs (``tests/golden/*.npz``) are committed and travel to the GPU box,
where /root/reference does not exist.

Scenes: the reference's own synthgen scenes from its tests
(test_cascade.py mixed_spec / illumination / sampling / oscillator scenes,
test_gmm.py random streams, test_scene_prior.py random KDE samples) plus
small BASELINE-shaped scenes from paper_1705_09339_b200.synth.

Every case stores the inputs (frames, config overrides) and the
reference outputs: training artefacts, per-frame masks / stats / kinds /
confidences and the final engine state.
"""

from __future__ import annotations

import dataclasses
import hashlib
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from cogbg.cascade import run_sequence  # noqa: E402
from cogbg.config import EngineConfig  # noqa: E402
from cogbg.frame_io import Frame, FramePlane  # noqa: E402
from cogbg.gmm import classify_frame, init_model  # noqa: E402
from cogbg.scene_prior import (build_kde, classify_pixel_dynamics,  # noqa: E402
                               compute_residue_histogram)
from cogbg.synthgen import SynthBlob, SynthRegion, SynthSpec, generate  # noqa: E402
from cogbg.training import train_engine  # noqa: E402

from paper_1705_09339_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent


def frames_of(arr):
    arr = np.asarray(arr, dtype=np.uint8)
    if arr.ndim == 3:
        arr = arr[:, None]
    return [Frame(index=i, planes=[FramePlane(c, arr[i, c])
                                   for c in range(arr.shape[1])])
            for i in range(arr.shape[0])]


def stack(frames):
    return np.stack([np.stack([p.data for p in f.planes]) for f in frames])


def mixed_spec(size=32, n=90, seed=5, with_blob=True):
    half = size // 2
    regions = (
        SynthRegion(rect=(0, 0, half, size), kind="static", level=100.0,
                    noise=0.5),
        SynthRegion(rect=(half, 0, half, half), kind="oscillating",
                    level=120.0, noise=0.5, amplitude=30.0, period=4),
        SynthRegion(rect=(half, half, half, half), kind="dynamic",
                    level=90.0, noise=20.0),
    )
    blobs = ()
    if with_blob:
        blobs = (SynthBlob(start=(2.0, 10.0), velocity=(0.3, 0.0), size=6,
                           offset=120.0, entry=40, duration=30),)
    return SynthSpec(width=size, height=size, frame_count=n, seed=seed,
                     regions=regions, blobs=blobs)


STATE = ("mu", "var", "w", "count", "mid_order", "mode_ref", "chp_prev",
         "last_label", "hits", "streak", "last_active", "clock", "waking",
         "group_mu", "group_var")


def run_case(name, frames_arr, n_train, overrides):
    cfg = EngineConfig(backend="numba", **overrides)
    frames = frames_of(frames_arr)
    eng = train_engine(frames[:n_train], cfg)
    rec = {
        "frames": frames_arr.astype(np.uint8),
        "n_train": np.int64(n_train),
        "cfg_keys": np.array(list(overrides.keys()), dtype=object),
        "cfg_vals": np.array([repr(v) for v in overrides.values()],
                             dtype=object),
        # the f32 tables are pinned by kde.npz; keep only their digest here
        "train_tables_sha": np.array(
            hashlib.sha256(eng.tables.tobytes()).hexdigest()),
        "train_dynamics": eng.dynamics,
        "train_group_id": eng.group_id,
        "train_group_w": eng.group_w,
        "train_group_members": eng.group_members,
        "train_wa": eng.wa,
    }
    for nm in STATE:
        rec["train_" + nm] = getattr(eng, nm).copy()
    masks, kinds, confs, stats = [], [], [], []
    for f in frames[n_train:]:
        m, s = eng.process_frame(f)
        masks.append(m.labels)
        kinds.append(eng.last_kinds.copy())
        confs.append(eng.last_confidence.copy())
        stats.append(s.as_row())
    rec["masks"] = np.stack(masks)
    rec["kinds"] = np.stack(kinds)
    keep = sorted(set(range(min(8, len(confs)))) | set(range(0, len(confs), 10)))
    rec["conf_frames"] = np.array(keep, dtype=np.int64)
    rec["confs"] = np.stack([confs[i] for i in keep])
    rec["stats"] = np.array(stats, dtype=np.int64)
    for nm in STATE:
        rec["final_" + nm] = getattr(eng, nm).copy()
    rec["final_frame_count"] = np.int64(eng.frame_count)
    np.savez_compressed(OUT / f"case_{name}.npz", **rec)
    fired = int(rec["stats"][:, 9].sum())
    tot = rec["stats"][:, 1:7].sum(axis=0)
    print(f"{name}: {frames_arr.shape} levels={tot.tolist()} fired={fired}")


def cascade_cases():
    run_case("mixed", stack([f for f, _ in generate(mixed_spec(n=110, seed=9))]),
             30, dict(chp_epsilon=1.0, reorder_interval=25,
                      saturation_frames=10, sleep_frames=5))
    run_case("mixed_default",
             stack([f for f, _ in generate(mixed_spec(n=70, seed=3))]), 30, {})
    run_case("compat", stack([f for f, _ in generate(mixed_spec())]), 30,
             dict(compat=True, grouping=False))
    spec = SynthSpec(width=16, height=16, frame_count=100, seed=6,
                     regions=(SynthRegion(rect=(0, 0, 16, 16), kind="static",
                                          level=90.0, noise=0.0),),
                     illumination_events=((60, 80.0),))
    run_case("illum", stack([f for f, _ in generate(spec)]), 30,
             dict(grouping=False))
    spec = SynthSpec(width=20, height=16, frame_count=90, seed=16,
                     regions=(SynthRegion(rect=(0, 0, 10, 16), kind="static",
                                          level=90.0, noise=0.5),
                              SynthRegion(rect=(10, 0, 10, 16),
                                          kind="oscillating", level=60.0,
                                          noise=0.5, amplitude=40.0,
                                          period=4)),
                     illumination_events=((55, 90.0),))
    run_case("illum_grouped", stack([f for f, _ in generate(spec)]), 30,
             dict(chp_epsilon=1.0, saturation_frames=6, sleep_frames=4,
                  reorder_interval=30))
    spec = SynthSpec(width=24, height=20, frame_count=100, seed=21,
                     regions=(SynthRegion(rect=(0, 0, 24, 20), kind="static",
                                          level=100.0, noise=0.4),),
                     blobs=(SynthBlob(start=(3.0, 3.0), velocity=(0.3, 0.2),
                                      size=6, offset=60.0, entry=50,
                                      duration=30),))
    run_case("sampling", stack([f for f, _ in generate(spec)]), 30,
             dict(chp_epsilon=1.0, saturation_frames=5, sleep_frames=3))
    run_case("sampling_stride3", stack([f for f, _ in generate(spec)]), 30,
             dict(chp_epsilon=1.0, saturation_frames=4, sleep_frames=4,
                  stride=3))
    spec = SynthSpec(width=8, height=8, frame_count=140, seed=8,
                     regions=(SynthRegion(rect=(0, 0, 8, 8), kind="oscillating",
                                          level=100.0, noise=0.0,
                                          amplitude=60.0, period=4),))
    run_case("oscillator", stack([f for f, _ in generate(spec)]), 32,
             dict(grouping=False, sampling=False, reorder_interval=10))
    # small BASELINE-shaped scenes
    sp = synth.small_spec(1, 48, 40, 100, 40)
    run_case("c1small", synth.Scene(sp).frames(0, 100), 40, dict(k_max=3))
    sp = synth.small_spec(2, 32, 24, 80, 30)
    run_case("c2small", synth.Scene(sp).frames(0, 80), 30,
             dict(k_max=3, color=True, chp_epsilon=2.0))
    sp = dataclasses.replace(synth.small_spec(3, 40, 32, 80, 30),
                             steps=((50, -100.0),))
    run_case("c3small", synth.Scene(sp).frames(0, 80), 30,
             dict(k_max=5, color=True, reorder_interval=20))
    sp = synth.small_spec(5, 40, 24, 70, 30)
    run_case("c5small", synth.Scene(sp).frames(0, 70), 30,
             dict(k_max=5, color=True, clusters=4))


def kde_cases():
    rng = np.random.default_rng(7)
    vals = rng.integers(0, 256, size=(20, 2, 4, 4), dtype=np.uint8)
    vals[0, 0, 0, 0] = 0
    vals[1, 0, 0, 0] = 255
    rec = {"values": vals}
    for i, bw in enumerate((5.0, 0.7, 23.0)):
        kde = build_kde(frames_of(vals), bandwidth=bw)
        rec[f"bw{i}"] = np.float64(bw)
        rec[f"tables{i}"] = kde.tables
    # trailing windows of a longer stream (windowed prior oracle =
    # build_kde on the window's slice)
    long = synth.Scene(synth.small_spec(1, 16, 12, 100, 100)).frames(0, 100)
    rec["long"] = long
    for w in (25, 50, 100):
        rec[f"win{w}"] = build_kde(frames_of(long[100 - w:]),
                                   bandwidth=5.0).tables
    hist = compute_residue_histogram(frames_of(long), (4.0, 32.0))
    rec["long_occ"] = hist.occupancies
    rec["long_classes"] = classify_pixel_dynamics(hist, 0.6)
    hist2 = compute_residue_histogram(frames_of(vals), (4.0, 48.0))
    rec["occ"] = hist2.occupancies
    np.savez_compressed(OUT / "kde.npz", **rec)
    print("kde: done")


def gmm_cases():
    rng = np.random.default_rng(11)
    values = rng.integers(0, 256, size=(80, 10, 10), dtype=np.uint8)
    cfg = EngineConfig(backend="numba")
    model = init_model(frames_of(values[:1])[0], cfg, backend="numba")
    labels = []
    for i in range(1, 80):
        m, _ = classify_frame(model, frames_of(values[i:i + 1])[0])
        labels.append(m.labels)
    g = model.planes[0]
    np.savez_compressed(OUT / "gmm.npz", values=values,
                        labels=np.stack(labels), mu=g.mu, var=g.var, w=g.w,
                        count=g.count)
    print("gmm: done")


if __name__ == "__main__":
    kde_cases()
    gmm_cases()
    cascade_cases()
