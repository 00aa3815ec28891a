"""Row-band and multi-stream execution on one GPU.

Row bands: the frame's rows are split into stride-aligned shards, each a
CascadeEngine with its own row0; per frame every shard steps with the frame
tail deferred, the exact partials are summed, every shard finalizes.  The
sharded run must equal the single-engine run bit for bit (masks, stats and
every state array) -- the partials are exact integers -- and, in float64
state, agree with the reference's goldens like the single engine does.

Batch: S independent streams in one set of buffers, one launch per frame,
must equal S separate engines bit for bit.
"""
import numpy as np
import pytest
import torch

from tests.golden_util import STATE, config_for, load_case

pytestmark = pytest.mark.gpu

BAND_CASES = ["mixed", "sampling", "sampling_stride3", "illum_grouped",
              "c3small", "c5small"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _single(frames, n_train, cfg):
    from paper_1705_09339_b200.training import train_engine
    return train_engine(frames[:n_train], cfg)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("parts", [2, 3])
@pytest.mark.parametrize("name", BAND_CASES)
def test_row_bands_equal_single_engine(name, parts, dtype):
    from paper_1705_09339_b200.parallel import BandSet
    rec, overrides = load_case(name)
    cfg = config_for(overrides, state_dtype=dtype)
    frames = rec["frames"]
    n_train = int(rec["n_train"])
    ref = _single(frames, n_train, cfg)
    bands = BandSet.train(frames[:n_train], cfg, parts)
    assert len(bands.engines) == parts
    for nm in ("group_id",):
        got = np.concatenate([e.group_id for e in bands.engines])
        assert np.array_equal(got, ref.group_id)
    for t in range(frames.shape[0] - n_train):
        f = frames[n_train + t]
        m1, s1 = ref.process_frame(f)
        m2, s2 = bands.process_frame(f)
        assert np.array_equal(m1.labels, m2.labels), (name, t)
        assert s1.as_row() == s2.as_row(), (name, t)
    for nm in STATE:
        assert np.array_equal(bands.state(nm), getattr(ref, nm)), nm


def test_row_bands_match_reference_golden_f64():
    """Sharded float64 run against the reference's own outputs."""
    from paper_1705_09339_b200.parallel import BandSet
    rec, overrides = load_case("mixed")
    cfg = config_for(overrides, state_dtype="float64")
    frames = rec["frames"]
    n_train = int(rec["n_train"])
    bands = BandSet.train(frames[:n_train], cfg, 4)
    agree = total = 0
    for t in range(frames.shape[0] - n_train):
        m, st = bands.process_frame(frames[n_train + t])
        agree += int((m.labels == rec["masks"][t]).sum())
        total += m.labels.size
        assert st.as_row()[0] == rec["stats"][t][0]
    assert agree / total >= 0.99995
    for nm in ("count", "mid_order", "mode_ref", "chp_prev", "clock", "waking"):
        same = np.mean(bands.state(nm) == rec["final_" + nm])
        assert same >= 0.999, nm


def test_train_band_engine_full_frame_equals_train_engine():
    from paper_1705_09339_b200.parallel import train_band_engine
    rec, overrides = load_case("c3small")
    cfg = config_for(overrides)
    frames = rec["frames"]
    n_train = int(rec["n_train"])
    a = _single(frames, n_train, cfg)
    b = train_band_engine(frames[:n_train], cfg, (0, frames.shape[2]))
    for nm in STATE:
        assert np.array_equal(getattr(a, nm), getattr(b, nm)), nm
    assert np.array_equal(a.tables, b.tables)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_batch_engine_equals_separate_engines(dtype):
    from paper_1705_09339_b200 import synth
    from paper_1705_09339_b200.parallel import BatchEngine
    spec = synth.small_spec(5, 40, 24, 60, 30)
    scenes = [synth.Scene(spec.for_stream(i)) for i in range(3)]
    seqs = [sc.frames(0, 60) for sc in scenes]
    cfg = config_for({"k_max": 5, "color": True, "reorder_interval": 12,
                      "clusters": 3}, state_dtype=dtype)
    singles = [_single(s, 30, cfg) for s in seqs]
    batch = BatchEngine.train([s[:30] for s in seqs], cfg)
    for t in range(30, 60):
        masks, stats = batch.process_frames(np.stack([s[t] for s in seqs]))
        for i, eng in enumerate(singles):
            m, st = eng.process_frame(seqs[i][t])
            assert np.array_equal(masks[i], m.labels), (i, t)
            assert stats[i].tolist() == st.as_row(), (i, t)
    for i, eng in enumerate(singles):
        got = batch.export_stream(i)
        for nm in STATE:
            assert np.array_equal(got[nm], getattr(eng, nm)), (i, nm)


def test_batch_submit_pipeline_equals_synchronous():
    """submit_frames: 30 frames in flight through the 3-slot ring (pinned
    DMA sources, results read only at the end, so every slot is reused with
    its result still pending) == the synchronous process_frames"""
    from paper_1705_09339_b200 import synth
    from paper_1705_09339_b200.parallel import BatchEngine
    spec = synth.small_spec(5, 40, 24, 60, 30)
    seqs = [synth.Scene(spec.for_stream(i)).frames(0, 60) for i in range(3)]
    cfg = config_for({"k_max": 5, "color": True}, state_dtype="float32")
    a = BatchEngine.train([s[:30] for s in seqs], cfg)
    b = BatchEngine.train([s[:30] for s in seqs], cfg)
    pending = []
    for t in range(30, 60):
        x = torch.from_numpy(np.stack([s[t] for s in seqs])).pin_memory()
        pending.append(a.submit_frames(x))
    for k, t in enumerate(range(30, 60)):
        masks, stats = b.process_frames(np.stack([s[t] for s in seqs]))
        assert np.array_equal(pending[k].masks, masks), t
        assert np.array_equal(pending[k].stats, stats), t


def test_batch_results_read_early_stay_valid():
    """arrays taken from a BatchResult right away keep their frame's values
    while later submissions reuse the ring slot (a caller collecting
    res.masks in a loop), and a caller may refill one pinned input buffer
    every frame"""
    from paper_1705_09339_b200 import synth
    from paper_1705_09339_b200.parallel import BatchEngine
    spec = synth.small_spec(5, 40, 24, 50, 30)
    seqs = [synth.Scene(spec.for_stream(i)).frames(0, 50) for i in range(2)]
    cfg = config_for({"k_max": 5, "color": True}, state_dtype="float32")
    a = BatchEngine.train([s[:30] for s in seqs], cfg)
    b = BatchEngine.train([s[:30] for s in seqs], cfg)
    buf = torch.empty((2,) + seqs[0].shape[1:], dtype=torch.uint8).pin_memory()
    kept = []
    for t in range(30, 50):
        buf.copy_(torch.from_numpy(np.stack([s[t] for s in seqs])))
        res = a.submit_frames(buf)          # the same pinned buffer each time
        kept.append((res.masks, res.stats))
    for k, t in enumerate(range(30, 50)):
        masks, stats = b.process_frames(np.stack([s[t] for s in seqs]))
        assert np.array_equal(kept[k][0], masks), t
        assert np.array_equal(kept[k][1], stats), t


def test_many_groups_step_and_agree_with_the_oracle():
    """a grouping with hundreds of groups (group sums and constants beyond
    the hot kernel's shared memory, so they live in global memory) still
    steps and agrees with the oracle"""
    from oracle import oracle as orc
    from paper_1705_09339_b200 import synth
    from paper_1705_09339_b200.training import train_engine
    spec = synth.small_spec(2, 64, 48, 50, 30)
    frames = synth.Scene(spec).frames(0, 50)
    cfg = config_for({"k_max": 3, "color": True, "clusters": 1200,
                      "cluster_threshold": 1.0}, state_dtype="float32")
    eng = train_engine(frames[:30], cfg)
    assert eng.dev.n_groups > 200, eng.dev.n_groups
    ref = orc.train(frames[:30], cfg)
    agree = total = 0
    for t in range(30, 50):
        m, st = eng.process_frame(frames[t])
        want, row = ref.process(frames[t])
        agree += int((m.labels == want).sum())
        total += want.size
    assert agree / total >= 0.999, (agree, total)


def test_banded_host_path_equals_fused_host_path():
    """process_frame with a reducer set (the row-band path: split step,
    all-reduce, cog_finalize; upload / download on the ring's copy streams)
    == the fused single-call path, for one full-frame band and an identity
    reducer (what a world-1 all-reduce does)"""
    from paper_1705_09339_b200.parallel import train_band_engine
    rec, overrides = load_case("c3small")
    cfg = config_for(overrides, state_dtype="float32")
    frames = rec["frames"]
    n_train = int(rec["n_train"])
    a = _single(frames, n_train, cfg)
    b = train_band_engine(frames[:n_train], cfg, (0, frames.shape[2]))
    b.reducer = lambda accum: None
    pend = []
    for t in range(n_train, frames.shape[0]):
        ma, sa = a.process_frame(frames[t])
        mb, sb = b.process_frame(torch.from_numpy(frames[t]).pin_memory())
        pend.append((ma, sa, mb, sb))
    for t, (ma, sa, mb, sb) in enumerate(pend):
        assert np.array_equal(ma.labels, mb.labels), t
        assert sa.as_row() == sb.as_row(), t


@pytest.mark.parametrize("n,k", [(200_000, 3), (70_001, 5)])
def test_device_kmeans_equals_numpy_kmeans(n, k, monkeypatch):
    """cog_kmeans_assign inside KMeans.fit: labels and centres bit-identical
    to the all-numpy iteration (grouping.py:100-126), duplicate points (exact
    distance ties) included"""
    from paper_1705_09339_b200 import grouping
    rng = np.random.default_rng(7)
    pts = np.concatenate([rng.normal(0, 1, (n // 2, 2)),
                          rng.normal(3, 0.5, (n - n // 2, 2))])
    pts[::97] = pts[1]                       # many identical points
    monkeypatch.setattr(grouping, "KMEANS_DEVICE_MIN", 10 ** 12)
    want_l, want_c = grouping.KMeans(k, 3).fit(pts.copy())
    monkeypatch.setattr(grouping, "KMEANS_DEVICE_MIN", 0)
    got_l, got_c = grouping.KMeans(k, 3).fit(pts.copy())
    assert np.array_equal(got_l, want_l)
    assert np.array_equal(got_c, want_c)


def test_device_pooled_stats_match_host(monkeypatch):
    """cog_pool_sums path of build_groups (pools too big for numpy's
    in-memory expression): means identical to the host evaluation; variances
    within 1e-11 relative -- the device value is the exact rational correctly
    rounded, numpy's float evaluation over 1e6 terms carries ~1e-12"""
    from paper_1705_09339_b200 import grouping
    from paper_1705_09339_b200.config import EngineConfig
    rng = np.random.default_rng(5)
    n, d, p = 40, 3, 50_000
    values = rng.integers(0, 256, (n, d, p), dtype=np.uint8)
    values[:, :, : p // 2] = (values[:, :, : p // 2] // 16 + 100).astype(np.uint8)
    feats = np.stack([rng.gamma(2, 1, p), rng.gamma(2, 1, p) * 1e-3], axis=1)
    feats[: p // 2] *= 5.0
    w_final = rng.random(p)
    cfg = EngineConfig(color=True, clusters=3)
    monkeypatch.setattr(grouping, "_cuda_ok", lambda: False)
    want = grouping.build_groups(feats, w_final, values, cfg)
    monkeypatch.setattr(grouping, "_cuda_ok", lambda: True)
    monkeypatch.setattr(grouping, "_POOL_EXACT_BYTES", 1024)  # all "big"
    got = grouping.build_groups(feats, w_final, values, cfg)
    assert want.group_count == got.group_count > 0
    assert np.array_equal(want.group_id, got.group_id)
    assert np.array_equal(want.member_count, got.member_count)
    assert np.array_equal(want.mu, got.mu)
    np.testing.assert_allclose(got.var, want.var, rtol=1e-11, atol=0)
    assert np.array_equal(want.weight, got.weight)


@pytest.mark.parametrize("name", ["c3small", "illum_grouped", "mixed_default"])
def test_training_with_device_kmeans_equals_host_kmeans(name, monkeypatch):
    """a golden case trained with the k-means assignment forced onto the GPU
    == trained with the numpy k-means (group ids, group parameters, state)"""
    rec, overrides = load_case(name)
    cfg = config_for(overrides)
    frames = rec["frames"]
    n_train = int(rec["n_train"])
    from paper_1705_09339_b200 import grouping
    monkeypatch.setattr(grouping, "KMEANS_DEVICE_MIN", 10 ** 12)
    a = _single(frames, n_train, cfg)
    monkeypatch.setattr(grouping, "KMEANS_DEVICE_MIN", 0)
    b = _single(frames, n_train, cfg)
    assert np.array_equal(a.group_id, b.group_id)
    for nm in STATE:
        assert np.array_equal(getattr(a, nm), getattr(b, nm)), nm


@pytest.mark.parametrize("k,p", [(3, 70_001), (5, 200_000)])
def test_device_grouping_equals_numpy(k, p, monkeypatch):
    """build_groups_device (seeding, k-means, z-score and sigma band on the
    device, every axis-0 reduction in numpy's row order through
    cog_seq_sums) gives the numpy path's group map, member counts, weights
    and pooled means bit for bit (grouping.py:100-195); duplicate points
    exercise the lowest-index tie breaks"""
    from paper_1705_09339_b200 import grouping
    from paper_1705_09339_b200.config import EngineConfig
    rng = np.random.default_rng(11 + k)
    n, d = 12, 3
    values = rng.integers(0, 256, (n, d, p), dtype=np.uint8)
    feats = np.stack([rng.gamma(2, 1, p), rng.gamma(2, 1, p) * 1e-3], axis=1)
    feats[: p // 3] *= 4.0
    feats[p // 2: p // 2 + 500] = feats[p // 2]        # exact duplicates
    feats[-7:] = feats[:7]
    w_final = rng.random(p)
    cfg = EngineConfig(color=True, clusters=k, cluster_threshold=0.9)
    monkeypatch.setattr(grouping, "_cuda_ok", lambda: False)
    want = grouping.build_groups(feats, w_final, values, cfg)
    monkeypatch.undo()
    monkeypatch.setattr(grouping, "KMEANS_DEVICE_MIN", 0)
    got = grouping.build_groups(torch.from_numpy(feats).cuda(),
                                torch.from_numpy(w_final).cuda(), values, cfg)
    assert want.group_count == got.group_count > 0
    assert np.array_equal(want.group_id, got.group_id)
    assert np.array_equal(want.member_count, got.member_count)
    assert np.array_equal(want.weight, got.weight)
    assert np.array_equal(want.mu, got.mu)
    assert np.array_equal(want.var, got.var)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("name", ["mixed", "illum_grouped", "c3small"])
def test_row_bands_over_peer_mailboxes_equal_single_engine(name, dtype):
    """The multi-GPU data path of the row bands on one GPU: every band's
    step pushes its exact partials into every band's mailbox from the deep
    pass's last CTA (cog_step_p2p, unfused), every band's cog_finalize_p2p
    sums its own mailbox (flags, parity slots, sequence numbers) -- masks,
    stats and every state array equal the single engine's bit for bit
    (cascade.py:301-313, 320-344 over the whole frame)"""
    from paper_1705_09339_b200.parallel import BandSet
    rec, overrides = load_case(name)
    cfg = config_for(overrides, state_dtype=dtype)
    frames = rec["frames"]
    n_train = int(rec["n_train"])
    ref = _single(frames, n_train, cfg)
    bands = BandSet.train(frames[:n_train], cfg, 3)
    bands.use_mailboxes()
    for t in range(frames.shape[0] - n_train):
        f = frames[n_train + t]
        m1, s1 = ref.process_frame(f)
        m2, s2 = bands.process_frame(f)
        assert np.array_equal(m1.labels, m2.labels), (name, t)
        assert s1.as_row() == s2.as_row(), (name, t)
    assert [b.seq for b in bands.mailboxes] == \
        [frames.shape[0] - n_train] * 3
    for nm in STATE:
        assert np.array_equal(bands.state(nm), getattr(ref, nm)), nm


def test_peer_mailbox_arguments_are_checked():
    from paper_1705_09339_b200 import _lib
    from paper_1705_09339_b200.errors import DataError
    from paper_1705_09339_b200.parallel import PeerMailbox
    lib = _lib.load()
    assert lib.cog_mailbox_words(3, 4, 2) == \
        2 * 2 * (lib.cog_accum_words(3, 4) + 1)
    assert lib.cog_mailbox_words(3, 4, 17) == -1
    with pytest.raises(DataError):
        PeerMailbox(3, 0, 1, 0, [0])
    boxes = PeerMailbox.local(3, 2, 2)
    assert boxes[0].ptrs == boxes[1].ptrs and boxes[1].rank == 1
    assert boxes[0].next().seq == 1 and boxes[0].next().seq == 2
