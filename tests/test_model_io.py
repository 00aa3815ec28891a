"""Model files in the reference's COGP v1 format (model_io.py:1-227).

GPU: a file written by the REAL reference loads into the device engine, is
written back byte for byte, and resumes exactly like the reference's loaded
engine (masks and stats of the continuation, float64 state); our own
save -> load -> save is byte-identical.  CPU: malformed files raise the
reference's error types before anything touches the device.
"""
import numpy as np
import pytest

from paper_1705_09339_b200.errors import ConfigError, FormatError
from tests.golden_util import GOLDEN, config_for

CASES = ["mixed", "rgb"]


def _case(name):
    z = np.load(GOLDEN / f"model_{name}.npz")
    ov = {k: eval(v) for k, v in zip(z["cfg_keys"].tolist(),
                                     z["cfg_vals"].tolist())}
    return z, ov


@pytest.mark.parametrize("name", CASES)
def test_malformed_files_raise(name, tmp_path):
    from paper_1705_09339_b200.model_io import load_model
    z, ov = _case(name)
    cfg = config_for(ov)
    raw = (GOLDEN / f"model_{name}.cogp").read_bytes()
    bad = tmp_path / "m.cogp"
    for blob in (raw[:20], b"XXXX" + raw[4:], raw + b"\0", raw[:-3]):
        bad.write_bytes(blob)
        with pytest.raises(FormatError):
            load_model(bad, cfg)
    with pytest.raises(FormatError):
        load_model(tmp_path / "missing.cogp", cfg)
    k = cfg.k_max
    with pytest.raises(ConfigError):
        load_model(GOLDEN / f"model_{name}.cogp",
                   config_for({**ov, "k_max": k + 1}))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("name", CASES)
def test_reference_file_roundtrip_bytes(name, dtype, tmp_path):
    from paper_1705_09339_b200.model_io import load_model, save_model
    z, ov = _case(name)
    cfg = config_for(ov, state_dtype=dtype)
    src = GOLDEN / f"model_{name}.cogp"
    eng = load_model(src, cfg)
    out = tmp_path / "out.cogp"
    save_model(eng, out)
    assert out.read_bytes() == src.read_bytes()


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_resume_matches_reference(name):
    from paper_1705_09339_b200.model_io import load_model
    z, ov = _case(name)
    cfg = config_for(ov, state_dtype="float64")
    eng = load_model(GOLDEN / f"model_{name}.cogp", cfg)
    eng.exact_group_sums = True   # the reference's sequential bincount sums
    for t, f in enumerate(z["frames"]):
        m, st = eng.process_frame(f)
        assert np.array_equal(m.labels, z["masks"][t]), t
        assert st.as_row() == z["stats"][t].tolist(), t


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_save_load_save_trained_engine(dtype, tmp_path):
    from paper_1705_09339_b200 import synth
    from paper_1705_09339_b200.model_io import load_model, save_model
    from paper_1705_09339_b200.training import train_engine
    spec = synth.small_spec(2, 32, 24, 50, 30)
    frames = synth.Scene(spec).frames(0, 50)
    cfg = config_for({"k_max": 3, "color": True, "reorder_interval": 7},
                     state_dtype=dtype)
    eng = train_engine(frames[:30], cfg)
    for f in frames[30:44]:          # crosses two scheduled reorders
        eng.process_frame(f)
    a, b = tmp_path / "a.cogp", tmp_path / "b.cogp"
    save_model(eng, a)
    back = load_model(a, cfg)
    save_model(back, b)
    assert a.read_bytes() == b.read_bytes()
    for f in frames[44:]:            # the loaded engine continues the same
        m1, s1 = eng.process_frame(f)
        m2, s2 = back.process_frame(f)
        if dtype == "float64":
            assert np.array_equal(m1.labels, m2.labels)
            assert s1.as_row() == s2.as_row()
