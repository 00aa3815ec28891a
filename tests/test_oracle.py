"""Pin the CPU oracle (oracle/) against golden vectors produced by the real
reference in this container (tests/golden/make_golden.py).

Everything here is bit-exact: the oracle is a binary64 restatement of the
reference, so masks, stats, kinds, confidences and all state arrays must be
identical, not merely close.
"""
import hashlib

import numpy as np
import pytest

from oracle import oracle as orc
from tests.golden_util import CASES, GOLDEN, STATE, config_for, load_case


def test_kde_tables_match_reference():
    z = np.load(GOLDEN / "kde.npz")
    vals = z["values"]
    n, d, h, w = vals.shape
    flat = vals.reshape(n, d, h * w)
    for i in range(3):
        counts, tables = orc.kde(flat, float(z[f"bw{i}"]))
        ref = z[f"tables{i}"]
        # binary64 tables differ from BLAS only in summation order
        assert np.allclose(tables, ref, rtol=1e-12, atol=1e-300)
        # the f32 tables the engine consumes must be identical
        assert np.array_equal(tables.astype(np.float32), ref.astype(np.float32))
        assert counts.sum() == n * d * h * w


def test_kde_tables32_match_reference():
    """the full-geometry path (C loop over nonzero bins, f32 out) gives the
    reference's f32 tables exactly"""
    z = np.load(GOLDEN / "kde.npz")
    vals = z["values"]
    n, d, h, w = vals.shape
    flat = np.ascontiguousarray(vals.reshape(n, d, h * w))
    for i in range(3):
        t32 = orc.kde_tables32(flat, float(z[f"bw{i}"]))
        assert np.array_equal(t32, z[f"tables{i}"].astype(np.float32))
    long = np.ascontiguousarray(z["long"].reshape(*z["long"].shape[:2], -1))
    rng = np.random.default_rng(7)
    noisy = rng.integers(0, 256, size=(37, 2, 501)).astype(np.uint8)
    for v in (long, noisy):
        _, t = orc.kde(v, 5.0)
        assert np.array_equal(orc.kde_tables32(v, 5.0), t.astype(np.float32))


def test_kmeans_matches_numpy_expression():
    """the C assignment loop reproduces the reference's numpy k-means
    (grouping.py:100-126) including exact distance ties"""
    rng = np.random.default_rng(3)
    f = np.round(rng.normal(size=(5000, 2)), 1)  # many exact ties
    for k in (2, 3, 5):
        a, c = orc.kmeans(f, k, seed=k)
        # the reference loop, verbatim
        r = np.random.default_rng(k)
        cen = np.empty((k, 2))
        cen[0] = f[int(r.integers(f.shape[0]))]
        d2 = ((f - cen[0]) ** 2).sum(axis=1)
        for j in range(1, k):
            cen[j] = f[int(np.argmax(d2))]
            d2 = np.minimum(d2, ((f - cen[j]) ** 2).sum(axis=1))
        asg = np.full(f.shape[0], -1, dtype=np.int64)
        for _ in range(100):
            nxt = np.argmin(((f[:, None, :] - cen[None]) ** 2).sum(axis=2), axis=1)
            if np.array_equal(nxt, asg):
                break
            asg = nxt
            for j in range(k):
                m = f[asg == j]
                if m.shape[0]:
                    cen[j] = m.mean(axis=0)
        assert np.array_equal(a, asg) and np.array_equal(c, cen)


def test_kde_windows_and_residue_match_reference():
    z = np.load(GOLDEN / "kde.npz")
    long = z["long"]
    n, d, h, w = long.shape
    flat = long.reshape(n, d, h * w)
    for win in (25, 50, 100):
        _, t = orc.kde(np.ascontiguousarray(flat[n - win:]), 5.0)
        assert np.array_equal(t.astype(np.float32),
                              z[f"win{win}"].astype(np.float32))
    _, occ = orc.residue(flat, 4.0, 32.0)
    assert np.array_equal(occ, z["long_occ"])
    assert np.array_equal(orc.classify(occ, 0.6), z["long_classes"])
    vals = z["values"]
    _, occ2 = orc.residue(vals.reshape(vals.shape[0], vals.shape[1], -1),
                          4.0, 48.0)
    assert np.array_equal(occ2, z["occ"])


def test_baseline_gmm_matches_reference():
    z = np.load(GOLDEN / "gmm.npz")
    vals = z["values"]
    cfg = config_for({})
    mu, var, w, cnt = orc.init_plane(vals[0], 3, 225.0)
    for i in range(1, vals.shape[0]):
        lbl = orc.baseline_frame(vals[i], mu, var, w, cnt, cfg)
        ref = z["labels"][i - 1].ravel()
        assert np.array_equal(np.where(lbl > 0, 255, 0), ref), i
    for nm, a in (("mu", mu), ("var", var), ("w", w), ("count", cnt)):
        assert np.array_equal(a, z[nm]), nm


@pytest.mark.parametrize("name", CASES)
def test_engine_matches_reference(name):
    rec, overrides = load_case(name)
    cfg = config_for(overrides)
    frames = rec["frames"]
    n_train = int(rec["n_train"])
    eng = orc.train(frames[:n_train], cfg)
    assert hashlib.sha256(eng.tables.tobytes()).hexdigest() == str(
        rec["train_tables_sha"])
    assert np.array_equal(eng.dynamics, rec["train_dynamics"])
    assert np.array_equal(eng.group_id, rec["train_group_id"])
    assert np.array_equal(eng.group_w, rec["train_group_w"])
    assert np.array_equal(eng.group_members, rec["train_group_members"])
    for nm in STATE:
        assert np.array_equal(getattr(eng, nm), rec["train_" + nm]), nm
    conf_at = {int(f): i for i, f in enumerate(rec["conf_frames"])}
    for t in range(frames.shape[0] - n_train):
        mask, row = eng.process(frames[n_train + t])
        assert np.array_equal(mask, rec["masks"][t]), t
        assert [int(x) for x in row] == rec["stats"][t].tolist(), t
        assert np.array_equal(eng.last_kinds, rec["kinds"][t]), t
        if t in conf_at:
            assert np.array_equal(eng.last_confidence,
                                  rec["confs"][conf_at[t]]), t
    for nm in STATE:
        assert np.array_equal(getattr(eng, nm), rec["final_" + nm]), nm
    assert eng.frame_count == int(rec["final_frame_count"])
