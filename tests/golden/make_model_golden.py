"""Golden model files from the REAL reference (``cogbg.model_io``) in this
container: ``python tests/golden/make_model_golden.py``.  Outputs are
committed (``tests/golden/model_*.cogp`` + ``model_*.npz``) and travel to
the GPU box, where /root/reference does not exist.

For each case: train the reference engine, run some frames, ``save_model``
-> the .cogp file; then continue the same engine (as loaded back from the
file, i.e. f32-quantised state -- the reference's resume semantics,
pkg/tests/test_model_io.py:85-101) for more frames and record masks and
stats.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from cogbg.config import EngineConfig  # noqa: E402
from cogbg.model_io import load_model, save_model  # noqa: E402
from cogbg.training import train_engine  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parent))
from make_golden import frames_of, mixed_spec, stack  # noqa: E402
from cogbg.synthgen import generate  # noqa: E402

from paper_1705_09339_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent


def case(name, arr, n_train, n_before, n_after, overrides):
    cfg = EngineConfig(**overrides)
    frames = frames_of(arr)
    eng = train_engine(frames[:n_train], cfg)
    for f in frames[n_train:n_train + n_before]:
        eng.process_frame(f)
    path = OUT / f"model_{name}.cogp"
    save_model(eng, path)
    eng2 = load_model(path, cfg)
    masks, stats = [], []
    for f in frames[n_train + n_before:n_train + n_before + n_after]:
        m, st = eng2.process_frame(f)
        masks.append(m.labels)
        stats.append([st.frame, st.n_chp, st.n_group, st.n_mean,
                      st.n_meanvar, st.n_gmm, st.n_skipped, st.n_foreground,
                      st.unexplained, int(st.illumination_fired)])
    keys = sorted(overrides)
    np.savez_compressed(
        OUT / f"model_{name}.npz",
        frames=arr[n_train + n_before:n_train + n_before + n_after],
        masks=np.array(masks), stats=np.array(stats),
        cfg_keys=np.array(keys), cfg_vals=np.array([repr(overrides[k])
                                                    for k in keys]))
    print(name, path.stat().st_size, "bytes")


def main():
    arr = stack([f for f, _ in generate(mixed_spec(size=24, n=80))])
    case("mixed", arr, 30, 12, 20,
         {"chp_epsilon": 1.0, "reorder_interval": 15, "saturation_frames": 6,
          "sleep_frames": 4})
    spec = synth.small_spec(3, 24, 16, 64, 30)
    arr = synth.Scene(spec).frames(0, 64)
    case("rgb", arr, 30, 10, 24,
         {"k_max": 5, "color": True, "reorder_interval": 12})


if __name__ == "__main__":
    main()
