"""BASELINE configs C2-C5 at their full geometry, whole sequences: the
float32 production engine (the throughput path) against the CPU oracle
(the reference's binary64 semantics, oracle/) trained on the same seeded
frames -- the north-star end-to-end protocol.

Per sequence:
  * foreground masks agree on >= 99.99 % of the pixels over every
    post-training frame;
  * every frame's level populations (chp / group / mean / meanvar / gmm /
    skipped) agree within 0.1 % of the plane-pixels;
  * the illumination reset (cascade.py:310-313, 361-391) fires on the same
    frames, and the level reorders every 100 frames (cascade.py:314-317,
    393-417) happen inside the run.  C3 and C4 carry the BASELINE -30 step
    at frame 400; under the reference's semantics it does NOT fire the
    reset (unexplained plane-pixels peak at ~63 %, below the 70 % trigger:
    wide second modes and the group level still explain most shifted
    pixels -- the oracle shows it), so C3 geometry is also run with a -80
    step, which must fire the reset on the same frame in both.
C4 runs as 2 stride-aligned row bands (the multi-GPU decomposition on one
GPU) and is also checked bit for bit against the single 4K engine.
C5 runs 4 of its 64 streams through the batch engine, 200 frames each.
The single-step protocol (identical f32 state in, one frame: decisions and
integer state bit-exact, mixture within 1e-5) runs at C3 and C5 geometry.

Frames are rendered by threads (tests run after CUDA is initialised, so
no fork) and kept in host memory; the oracle uses every host core.
"""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu

LEVELS = ("chp", "group", "mean", "meanvar", "gmm", "skipped")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    os.environ["COG_ORACLE_THREADS"] = str(os.cpu_count() or 1)


def _threads():
    return max(1, min(32, os.cpu_count() or 1))


def _spec(cid, stream=0):
    from paper_1705_09339_b200 import synth
    base = synth.CONFIGS[cid]
    return base.for_stream(stream) if cid in (2, 3, 5) else base


def _frames(spec, t0, t1):
    from paper_1705_09339_b200 import synth
    return synth.Scene(spec).frames(t0, t1, threads=_threads())


def _cfg(spec):
    from paper_1705_09339_b200.config import EngineConfig
    return EngineConfig(k_max=spec.k_max, color=spec.depth == 3,
                        training_frames=spec.training).validate()


class Tally:
    """Mask agreement and per-frame level populations vs the oracle."""

    def __init__(self, name, npp):
        self.name, self.npp = name, npp
        self.agree = self.total = 0
        self.fired_gpu, self.fired_ref = [], []

    def frame(self, t, got_mask, got_row, want_mask, want_row):
        self.agree += int((got_mask == want_mask).sum())
        self.total += want_mask.size
        tol = max(2, self.npp // 1000)
        for k in range(1, 7):
            assert abs(int(got_row[k]) - int(want_row[k])) <= tol, \
                (self.name, t, LEVELS[k - 1], got_row[k], want_row[k])
        if got_row[9]:
            self.fired_gpu.append(t)
        if want_row[9]:
            self.fired_ref.append(t)

    def done(self):
        assert self.fired_gpu == self.fired_ref, \
            (self.name, self.fired_gpu, self.fired_ref)
        frac = self.agree / self.total
        assert frac >= 0.9999, (self.name, self.agree, self.total, frac)
        return frac


def _int_state_close(eng_state, ref, names, floor=0.999):
    for nm in names:
        same = float(np.mean(eng_state(nm) == getattr(ref, nm)))
        assert same >= floor, (nm, same)


def _whole_sequence(cid, stop=None, step=None, **cfg_kw):
    import dataclasses
    from paper_1705_09339_b200.training import train_engine
    spec = _spec(cid)
    if step is not None:
        spec = dataclasses.replace(spec, steps=((400, step),))
    cfg = _cfg(spec)
    if cfg_kw:
        cfg = dataclasses.replace(cfg, **cfg_kw).validate()
    stop = stop or spec.frames
    frames = _frames(spec, 0, stop)
    n = spec.training
    eng = train_engine(frames[:n], cfg)
    ref = orc.train(frames[:n], cfg)
    tally = Tally(spec.name, spec.n_pix * spec.depth)
    for t in range(n, stop):
        mask, st = eng.process_frame(frames[t])
        want, row = ref.process(frames[t])
        tally.frame(t, mask.labels, st.as_row(), want, row)
    tally.done()
    assert eng.frame_count == ref.frame_count == stop - n
    _int_state_close(lambda nm: getattr(eng, nm), ref,
                     ("count", "mid_order", "mode_ref", "clock", "waking"))
    return tally


def test_c2_whole_sequence_vs_oracle():
    """C2 640x480 RGB K=3: all 800 post-training frames."""
    _whole_sequence(2)


def test_c3_whole_sequence_vs_oracle():
    """C3 1920x1080 RGB K=5: all 400 post-training frames, across the
    frame-400 -30 step and four level reorders."""
    _whole_sequence(3)


def test_c3_illumination_reset_fires_with_oracle():
    """C3 geometry with a -80 step at frame 400 (frames 200-459): the step
    fires the illumination reset (unexplained > 0.7 of the plane-pixels)
    on the same frame on the GPU and in the oracle, the reset runs at
    2 Mpx x 3 planes, and the sequences keep agreeing after it."""
    tally = _whole_sequence(3, stop=460, step=-80.0)
    assert tally.fired_ref == [400], tally.fired_ref


def test_c4_row_bands_whole_sequence_vs_oracle_and_single_engine():
    """C4 3840x2160 RGB K=5: all 350 post-training frames through 2 row
    bands (the multi-GPU decomposition, partials summed per frame) against
    the oracle on the whole frame, and bit for bit against one 4K engine."""
    from paper_1705_09339_b200.parallel import BandSet
    from paper_1705_09339_b200.training import train_engine
    spec = _spec(4)
    cfg = _cfg(spec)
    frames = _frames(spec, 0, spec.frames)
    n = spec.training
    single = train_engine(frames[:n], cfg)
    bands = BandSet.train(frames[:n], cfg, 2)
    assert np.array_equal(np.concatenate([e.group_id for e in bands.engines]),
                          single.group_id)
    ref = orc.train(frames[:n], cfg)
    tally = Tally(spec.name, spec.n_pix * spec.depth)
    for t in range(n, spec.frames):
        m1, s1 = single.process_frame(frames[t])
        m2, s2 = bands.process_frame(frames[t])
        assert np.array_equal(m1.labels, m2.labels), t
        assert s1.as_row() == s2.as_row(), t
        want, row = ref.process(frames[t])
        tally.frame(t, m2.labels, s2.as_row(), want, row)
    tally.done()
    for nm in ("mu", "hits", "streak", "mid_order", "mode_ref", "group_mu"):
        assert np.array_equal(bands.state(nm), getattr(single, nm)), nm
    _int_state_close(bands.state, ref, ("count", "mid_order", "mode_ref"))


def test_c5_batch_streams_whole_sequence_vs_oracle():
    """C5 busy scene (30 % foreground, 10 % oscillators): 4 streams
    (seeds 100-103) x all 200 post-training frames through the batch
    engine, each against its own oracle."""
    from paper_1705_09339_b200.parallel import BatchEngine
    S = 4
    specs = [_spec(5, s) for s in range(S)]
    cfg = _cfg(specs[0])
    n = specs[0].training
    frames = [_frames(sp, 0, sp.frames) for sp in specs]
    eng = BatchEngine.train([f[:n] for f in frames], cfg)
    refs = [orc.train(f[:n], cfg) for f in frames]
    tallies = [Tally(f"C5/{sp.seed}", sp.n_pix * sp.depth) for sp in specs]
    for t in range(n, specs[0].frames):
        masks, rows = eng.process_frames(np.stack([f[t] for f in frames]))
        for s in range(S):
            want, row = refs[s].process(frames[s][t])
            tallies[s].frame(t, masks[s], rows[s], want, row)
    for tl in tallies:
        tl.done()


def _single_step(cid, stream, warm, steps):
    """North-star single-step protocol at a BASELINE geometry: the oracle
    is loaded with the GPU engine's exact f32 state, both take the same
    frame; kinds, labels, stats and the integer state must be identical,
    mu/var/w/group modes within 1e-5 relative, confidence within the fp32
    mode's bound; the oracle is then re-synchronised and the next frame
    checked."""
    from paper_1705_09339_b200.training import train_engine
    from tests.golden_util import STATE
    spec = _spec(cid, stream)
    cfg = _cfg(spec)
    n = spec.training
    frames = _frames(spec, 0, n + warm + steps)
    eng = train_engine(frames[:n], cfg)
    for t in range(n, n + warm):
        eng.process_frame(frames[t])
    oe = orc.OracleEngine(cfg, eng.height, eng.width, eng.depth)
    for nm in STATE:
        setattr(oe, nm, np.array(getattr(eng, nm)))
    oe.tables = eng.tables.copy()
    oe.finalize_tables()
    oe.dynamics = eng.dynamics
    wt = np.array([cfg.weights_static, cfg.weights_oscillating,
                   cfg.weights_dynamic])[oe.dynamics]
    oe.wa, oe.wb, oe.wc = (np.ascontiguousarray(wt[:, i]) for i in range(3))
    oe.group_id = eng.group_id
    oe.group_w = eng.group_w.copy()
    oe.group_members = eng.group_members.copy()
    oe.frame_count = eng.frame_count
    ints = ("count", "mid_order", "mode_ref", "chp_prev", "last_label",
            "hits", "streak", "last_active", "clock", "waking")
    for t in range(n + warm, n + warm + steps):
        m_o, row_o = oe.process(frames[t])
        m_g, st_g = eng.process_frame(frames[t])
        assert np.array_equal(m_g.labels, m_o), t
        assert st_g.as_row() == [int(x) for x in row_o], t
        assert np.array_equal(eng.last_kinds, oe.last_kinds), t
        for nm in ints:
            assert np.array_equal(getattr(eng, nm), getattr(oe, nm)), (t, nm)
        for nm in ("mu", "var", "w", "group_mu", "group_var"):
            np.testing.assert_allclose(getattr(eng, nm), getattr(oe, nm),
                                       rtol=1e-5, atol=1e-6, err_msg=nm)
        np.testing.assert_allclose(eng.last_confidence, oe.last_confidence,
                                   rtol=0, atol=CONF_ATOL)
        for nm in ("mu", "var", "w", "group_mu", "group_var"):
            setattr(oe, nm, np.array(getattr(eng, nm)))


# float32 mode: the confidence is evaluated in fp32 from the quantised hot
# prior; decisions near a threshold are redone exactly
CONF_ATOL = 1e-5


def test_single_step_protocol_c3_geometry():
    _single_step(3, 0, warm=20, steps=3)


def test_single_step_protocol_c5_geometry():
    _single_step(5, 0, warm=20, steps=3)
