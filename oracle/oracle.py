"""CPU ORACLE for the CoG hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and
only as the checker / CPU baseline.  The product package never imports it.

It restates the reference ``cogbg`` package (pure Python + numba) for the
path named in BASELINE.json's north star:

* per-pixel kernels      -> ``oracle/cog_oracle.c`` (ctypes), bit-identical
                            binary64 restatement of kernels_numba.py
* scene prior (KDE)      -> /root/reference/pkg/src/cogbg/scene_prior.py:40-45, 92-112
* residue / dynamics     -> scene_prior.py:171-213
* GMM warm-up            -> training.py:28-60, gmm.py:89-100
* grouping (host k-means)-> grouping.py:85-208
* engine host logic      -> cascade.py:166-241 (build / seeding),
                            261-318 (process_frame), 320-344 (groups),
                            346-359 (stats), 361-391 (illumination),
                            393-417 (reorder)

Pinned against golden vectors produced by the real reference in this
container (tests/golden/make_golden.py -> tests/golden/*.npz), see
tests/test_oracle.py.

Arrays follow the reference dtypes and layouts exactly ((d, P, K) float64
mixtures, int64 counters, int8 codes) so that its outputs can be compared
with the reference and with the CUDA engine's exported state.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

LEVEL_CHP, LEVEL_GROUP, LEVEL_MEAN, LEVEL_MEANVAR, LEVEL_GMM = 0, 1, 2, 3, 4
KIND_SKIP, KIND_COPY = 5, 6

_HERE = Path(__file__).resolve().parent
_SO = _HERE / "build" / "libcog_oracle.so"
_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_D = ctypes.c_double


def build_oracle() -> Path:
    """Compile the C restatement (``make -C oracle``)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not _SO.exists():
            build_oracle()
        L = ctypes.CDLL(str(_SO))
        L.cogo_baseline_frame.argtypes = [_I64, _I, _P, _P, _P, _P, _P, _D, _D,
                                          _D, _D, _D, _P, _I]
        L.cogo_cascade_frame.argtypes = (
            [_I64, _I] + [_P] * 23 + [_D] * 9 + [_I64, _I64] + [_I] * 6
            + [_P] * 4 + [_I])
        L.cogo_resolve_copies.argtypes = [_I64, _P, _P, _P, _I64, _I64]
        L.cogo_sort_pixels.argtypes = [_I64, _P, _I, _P, _P, _P, _P, _P]
        L.cogo_kde_tables32.argtypes = [_I64, _I, _P, _P, _P, _I]
        L.cogo_kmeans_assign.argtypes = [_I64, _P, _I, _P, _P, _I]
        L.cogo_group_sums.argtypes = [_I64, _P, _P, _P, _P, _I64, _P, _P, _P]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data


def default_threads() -> int:
    return int(os.environ.get("COG_ORACLE_THREADS", "1"))


# ----------------------------------------------------------- scene prior


def kernel_matrix(bandwidth: float) -> np.ndarray:
    """Grid-normalized Gaussian smoothing matrix (scene_prior.py:40-45)."""
    g = np.arange(256, dtype=np.float64)
    z = (g[None, :] - g[:, None]) / bandwidth
    m = np.exp(-0.5 * z * z)
    return m / m.sum(axis=1, keepdims=True)


def kde(values: np.ndarray, bandwidth: float, chunk: int = 1 << 16):
    """values (N, d, P) uint8 -> (counts (d,P,256) int64, tables (d,P,256) f64).

    counts are the bit-exact histogram; tables = counts @ W / N as in
    scene_prior.py:104-111 (BLAS order; the product is formed over pixel
    chunks, which leaves every row's dot products unchanged)."""
    n, d, p = values.shape
    counts = np.empty((d, p, 256), dtype=np.int64)
    tables = np.empty((d, p, 256), dtype=np.float64)
    for c, c0, c1, cnt, tab in _kde_chunks(values, bandwidth, chunk):
        counts[c, c0:c1] = cnt
        tables[c, c0:c1] = tab
    return counts, tables


def kde_tables32(values: np.ndarray, bandwidth: float) -> np.ndarray:
    """The f32 tables the engine keeps (cascade.py:192) for (N, d, P) uint8
    values, without materialising the int64 counts or the f64 table (a 4K
    prior): cogo_kde_tables32, the same counts @ W / N per pixel with the
    dot products over the nonzero bins (identical after rounding to f32,
    tests/test_oracle.py)."""
    n, d, p = values.shape
    kern = np.ascontiguousarray(kernel_matrix(bandwidth))
    out = np.empty((d, p, 256), dtype=np.float32)
    for c in range(d):
        plane = np.ascontiguousarray(values[:, c])
        rc = lib().cogo_kde_tables32(p, n, _ptr(plane), _ptr(kern),
                                     _ptr(out[c]), default_threads())
        assert rc == 0
    return out


def _kde_chunks(values, bandwidth, chunk):
    n, d, p = values.shape
    kern = kernel_matrix(bandwidth)
    for c in range(d):
        for c0 in range(0, p, chunk):
            c1 = min(p, c0 + chunk)
            m = c1 - c0
            base = np.arange(m, dtype=np.int64) * 256
            flat = (base[None, :] + values[:, c, c0:c1].astype(np.int64)).ravel()
            cnt = np.bincount(flat, minlength=m * 256).reshape(m, 256)
            yield c, c0, c1, cnt, (cnt.astype(np.float64) @ kern) / n


def residue(values: np.ndarray, t1: float, t2: float):
    """Pooled |x[i+1]-x[i]| 3-bin counts and occupancies (scene_prior.py:171-189)."""
    n, d, p = values.shape
    r = np.abs(np.diff(values.astype(np.int16), axis=0))
    b = (r >= t1).astype(np.int64) + (r >= t2)
    counts = np.zeros((p, 3), dtype=np.int64)
    for k in range(3):
        counts[:, k] = (b == k).sum(axis=(0, 1))
    return counts, counts / float((n - 1) * d)


def classify(occ: np.ndarray, peaky: float) -> np.ndarray:
    """static if occ0 >= t, elif occ1 >= t oscillating, else dynamic
    (scene_prior.py:192-202)."""
    cls = np.full(occ.shape[0], 2, dtype=np.uint8)
    cls[occ[:, 1] >= peaky] = 1
    cls[occ[:, 0] >= peaky] = 0
    return cls


def rate_weights(classes: np.ndarray, cfg) -> np.ndarray:
    tab = np.array([cfg.weights_static, cfg.weights_oscillating,
                    cfg.weights_dynamic], dtype=np.float64)
    return tab[classes]


# ------------------------------------------------------------- GMM warm-up


def init_plane(vals: np.ndarray, k: int, init_var: float):
    """gmm.py:89-100."""
    p = vals.size
    mu = np.zeros((p, k))
    var = np.full((p, k), init_var)
    w = np.zeros((p, k))
    mu[:, 0] = vals.ravel().astype(np.float64)
    w[:, 0] = 1.0
    return mu, var, w, np.ones(p, dtype=np.int64)


def baseline_frame(vals, mu, var, w, count, cfg, out=None, alpha=None,
                   threads=None):
    """kernels_numba.baseline_frame over one plane (C restatement)."""
    p, k = mu.shape
    if out is None:
        out = np.empty(p, dtype=np.uint8)
    vals = np.ascontiguousarray(vals.ravel(), dtype=np.uint8)
    a = cfg.learning_rate if alpha is None else alpha
    rc = lib().cogo_baseline_frame(
        p, k, _ptr(vals), _ptr(mu), _ptr(var), _ptr(w), _ptr(count), a,
        cfg.match_lambda, cfg.background_threshold, cfg.variance_floor,
        cfg.initial_variance, _ptr(out),
        default_threads() if threads is None else threads)
    assert rc == 0
    return out


def warmup(values: np.ndarray, cfg):
    """training.py:38-52: per plane init + (N-1) full updates; channel-0
    rank-0 var/w series for grouping."""
    n, d, p = values.shape
    k = cfg.k_max
    grids = []
    var_series = np.empty((n, p))
    w_series = np.empty((n, p))
    for c in range(d):
        mu, var, w, cnt = init_plane(values[0, c], k, cfg.initial_variance)
        if c == 0:
            var_series[0] = var[:, 0]
            w_series[0] = w[:, 0]
        for i in range(1, n):
            baseline_frame(values[i, c], mu, var, w, cnt, cfg)
            if c == 0:
                var_series[i] = var[:, 0]
                w_series[i] = w[:, 0]
        grids.append((mu, var, w, cnt))
    return grids, var_series, w_series


# ---------------------------------------------------------------- grouping


def behavior_features(var_series, w_series):
    return np.stack([var_series.var(axis=0, ddof=0),
                     w_series.var(axis=0, ddof=0)], axis=1)


def zscore(f):
    mean = f.mean(axis=0)
    std = f.std(axis=0, ddof=0)
    return (f - mean) / np.where(std > 0, std, 1.0)


def kmeans(features, k, seed, max_iter=100):
    """Seeded farthest-point init + Lloyd iterations (grouping.py:100-126)."""
    n = features.shape[0]
    if n < k:
        raise ValueError("too few pixels for k clusters")
    rng = np.random.default_rng(seed)
    centers = np.empty((k, features.shape[1]))
    centers[0] = features[int(rng.integers(n))]
    d2 = ((features - centers[0]) ** 2).sum(axis=1)
    for j in range(1, k):
        centers[j] = features[int(np.argmax(d2))]
        d2 = np.minimum(d2, ((features - centers[j]) ** 2).sum(axis=1))
    assign = np.full(n, -1, dtype=np.int64)
    feats = np.ascontiguousarray(features, dtype=np.float64)
    nxt = assign.copy()
    for _ in range(max_iter):
        # dist = ((f[:, None] - c[None]) ** 2).sum(axis=2); argmin (C loop)
        changed = lib().cogo_kmeans_assign(n, _ptr(feats), k,
                                           _ptr(np.ascontiguousarray(centers)),
                                           _ptr(nxt), default_threads())
        if not changed:
            break
        assign = nxt.copy()
        for j in range(k):
            mem = features[assign == j]
            if mem.shape[0]:
                centers[j] = mem.mean(axis=0)
    return assign, centers


def threshold_clusters(assign, features, c):
    """grouping.py:142-161."""
    member = np.full(assign.shape[0], -1, dtype=np.int64)
    for j in np.unique(assign):
        sel = assign == j
        if sel.sum() < 2:
            continue
        f = features[sel]
        ok = np.abs(f - f.mean(axis=0)) <= c * f.std(axis=0, ddof=0)
        ok |= np.ptp(f, axis=0) == 0
        member[np.where(sel)[0][ok.all(axis=1)]] = j
    return member


# pools above this many f64 bytes are not materialised (a 4K group holds
# ~1e9 training intensities); the engine uses the same bound
# (paper_1705_09339_b200/grouping.py _POOL_EXACT_BYTES)
POOL_EXACT_BYTES = 1 << 31


def pooled_stats(values, sel, floor):
    """grouping.py:189-192: mean / floored variance of every training
    intensity of the members, per channel.  Pools within POOL_EXACT_BYTES
    use the reference's numpy expression verbatim; bigger ones use exact
    integer sums (the mean is then identical -- numpy's float sum of
    integers is exact -- and the variance is the exact rational
    (M*sum x^2 - (sum x)^2) / M^2 correctly rounded, within a few ulp of
    numpy's two-pass float evaluation)."""
    n, d, _ = values.shape
    m = int(sel.sum())
    if n * d * m * 8 <= POOL_EXACT_BYTES:
        pooled = values[:, :, sel].astype(np.float64)
        return (pooled.mean(axis=(0, 2)),
                np.maximum(pooled.var(axis=(0, 2), ddof=0), floor))
    idx = np.where(sel)[0]
    s1 = [0] * d
    s2 = [0] * d
    step = max(1, (1 << 26) // n)
    for a in range(0, m, step):
        blk = values[:, :, idx[a:a + step]].astype(np.int64)
        for c in range(d):
            x = blk[:, c]
            s1[c] += int(x.sum())
            s2[c] += int((x * x).sum())
    cnt = n * m
    mean = np.array([s1[c] / cnt for c in range(d)])
    var = np.array([max((cnt * s2[c] - s1[c] * s1[c]) / (cnt * cnt), floor)
                    for c in range(d)])
    return mean, var


def group_params(member, values, w_final, cfg):
    """grouping.py:164-195: dense renumbering + pooled per-channel mode."""
    n, d, p = values.shape
    kept = [j for j in np.unique(member) if j != -1 and (member == j).sum() >= 2]
    g = len(kept)
    gid = np.full(p, -1, dtype=np.int64)
    mu = np.zeros((g, d))
    var = np.zeros((g, d))
    wgt = np.zeros(g)
    mem = np.zeros(g, dtype=np.int64)
    for gi, j in enumerate(kept):
        sel = member == j
        gid[sel] = gi
        mem[gi] = sel.sum()
        mu[gi], var[gi] = pooled_stats(values, sel, cfg.variance_floor)
        wgt[gi] = w_final[sel].mean()
    return gid, mu, var, wgt, mem


def groups(values, var_series, w_series, cfg):
    """Full grouping pipeline (grouping.py:198-208); empty when off."""
    n, d, p = values.shape
    if not cfg.grouping:
        return (np.full(p, -1, dtype=np.int64), np.zeros((0, d)),
                np.zeros((0, d)), np.zeros(0), np.zeros(0, dtype=np.int64))
    feats = behavior_features(var_series, w_series)
    assign, _ = kmeans(zscore(feats), cfg.clusters, cfg.cluster_seed)
    member = threshold_clusters(assign, feats, cfg.cluster_threshold)
    return group_params(member, values, w_series[-1], cfg)


# ------------------------------------------------------------------ engine


class OracleEngine:
    """Host-side restatement of cascade.CascadeEngine over the C kernels."""

    STATE = ("mu", "var", "w", "count", "mid_order", "mode_ref", "chp_prev",
             "last_label", "hits", "streak", "last_active", "clock",
             "waking", "group_mu", "group_var")

    def __init__(self, cfg, height, width, depth):
        self.cfg = cfg
        self.height, self.width, self.depth = height, width, depth
        p = height * width
        k = cfg.k_max
        self.n_pix = p
        self.frame_count = 0
        self.threads = default_threads()
        self.dynamics = np.zeros(p, dtype=np.uint8)
        self.wa = np.zeros(p)
        self.wb = np.zeros(p)
        self.wc = np.zeros(p)
        # the f32 prior (cascade.py:192); every use promotes an entry to
        # binary64 exactly as the reference's _tables64 = f64(f32 table)
        self.tables = np.zeros((depth, p, 256), dtype=np.float32)
        self.peaks = np.ones((depth, p))
        self.group_id = np.full(p, -1, dtype=np.int64)
        self.group_mu = np.zeros((depth, 0))
        self.group_var = np.zeros((depth, 0))
        self.group_w = np.zeros(0)
        self.group_members = np.zeros(0, dtype=np.int64)
        self.mu = np.zeros((depth, p, k))
        self.var = np.full((depth, p, k), cfg.initial_variance)
        self.w = np.zeros((depth, p, k))
        self.count = np.zeros((depth, p), dtype=np.int64)
        self.mid_order = np.full((depth, p, 3), -1, dtype=np.int8)
        self.mode_ref = np.zeros((depth, p, 2), dtype=np.int8)
        self.chp_prev = np.zeros((depth, p), dtype=np.uint8)
        self.last_label = np.zeros((depth, p), dtype=np.uint8)
        self.hits = np.zeros((depth, p, 5), dtype=np.int64)
        self.streak = np.zeros((depth, p), dtype=np.int64)
        self.last_active = np.full((depth, p), -1, dtype=np.int8)
        self.clock = np.zeros((depth, p), dtype=np.int64)
        self.waking = np.zeros((depth, p), dtype=np.uint8)
        yy, xx = np.divmod(np.arange(p), width)
        s = cfg.stride
        self.on_lattice = ((yy % s == 0) & (xx % s == 0)).astype(np.uint8)
        self.last_kinds = np.zeros((depth, p), dtype=np.uint8)
        self.last_confidence = np.zeros((depth, p))

    # -------------------------------------------------------------- build

    def finalize_tables(self):
        """cascade.py:213-216."""
        self.peaks = self.tables.max(axis=2).astype(np.float64)
        self.peaks[self.peaks <= 0.0] = 1.0

    def seed_level_order(self):
        """cascade.py:218-241: modes ranked by prior mass, ties by w/sigma."""
        p, k = self.n_pix, self.cfg.k_max
        ar = np.arange(p)
        grouped = self.group_id >= 0
        for c in range(self.depth):
            mval = np.clip(np.rint(self.mu[c]), 0, 255).astype(np.int64)
            live = np.arange(k)[None, :] < self.count[c][:, None]
            mass = np.where(live, self.tables[c][ar[:, None], mval].astype(np.float64),
                            -np.inf)
            tie = np.where(live, self.w[c] / np.sqrt(self.var[c]), -np.inf)
            order = np.lexsort((-tie, -mass), axis=1)
            self.mode_ref[c, :, 0] = order[:, 0]
            self.mode_ref[c, :, 1] = np.where(self.count[c] >= 2, order[:, 1],
                                              order[:, 0])
            self.mid_order[c, grouped] = (LEVEL_GROUP, LEVEL_MEAN, LEVEL_MEANVAR)
            self.mid_order[c, ~grouped] = (LEVEL_MEAN, LEVEL_MEANVAR, -1)

    def clone(self):
        twin = OracleEngine(self.cfg, self.height, self.width, self.depth)
        for name, val in vars(self).items():
            setattr(twin, name, val.copy() if isinstance(val, np.ndarray)
                    else val)
        return twin

    # ------------------------------------------------------------ runtime

    def process(self, frame: np.ndarray):
        """frame (d, H, W) uint8 -> (mask (H,W) u8 0/255, stats row list).

        Stats row = [frame, n_chp, n_group, n_mean, n_meanvar, n_gmm,
        n_skipped, n_foreground, unexplained, illumination_fired]."""
        cfg = self.cfg
        frame = np.ascontiguousarray(frame, dtype=np.uint8)
        if frame.shape != (self.depth, self.height, self.width):
            raise ValueError(f"frame shape {frame.shape} does not match model")
        compat = bool(cfg.compat)
        sampling_on = bool(cfg.sampling) and not compat
        grouping_on = bool(cfg.grouping) and not compat
        p, k = self.n_pix, self.cfg.k_max
        vals = frame.reshape(self.depth, p)
        kinds = np.empty((self.depth, p), dtype=np.uint8)
        labels = np.empty((self.depth, p), dtype=np.uint8)
        confs = np.empty((self.depth, p))
        counts = np.empty((self.depth, 7), dtype=np.int64)
        L = lib()
        for c in range(self.depth):
            gmu = np.ascontiguousarray(self.group_mu[c])
            gvar = np.ascontiguousarray(self.group_var[c])
            if gmu.size == 0:
                gmu = np.zeros(1)
                gvar = np.ones(1)
            vc = np.ascontiguousarray(vals[c])
            rc = L.cogo_cascade_frame(
                p, k, _ptr(vc), _ptr(self.mu[c]), _ptr(self.var[c]),
                _ptr(self.w[c]), _ptr(self.count[c]), _ptr(self.chp_prev[c]),
                _ptr(self.last_label[c]), _ptr(self.mid_order[c]),
                _ptr(self.mode_ref[c]), _ptr(self.hits[c]),
                _ptr(self.streak[c]), _ptr(self.last_active[c]),
                _ptr(self.clock[c]), _ptr(self.waking[c]),
                _ptr(self.on_lattice), _ptr(self.group_id), _ptr(gmu),
                _ptr(gvar), _ptr(self.tables[c]), _ptr(self.peaks[c]),
                _ptr(self.wa), _ptr(self.wb), _ptr(self.wc),
                cfg.learning_rate, cfg.match_lambda, cfg.background_threshold,
                cfg.variance_floor, cfg.initial_variance, cfg.chp_epsilon,
                cfg.confidence_threshold, cfg.prior_floor, cfg.rate_floor,
                cfg.saturation_frames, cfg.sleep_frames,
                int(sampling_on), int(grouping_on), int(not compat),
                int(not compat), int(cfg.confidence_literal), int(compat),
                _ptr(labels[c]), _ptr(kinds[c]), _ptr(confs[c]),
                _ptr(counts[c]), self.threads)
            assert rc == 0
            L.cogo_resolve_copies(p, _ptr(kinds[c]), _ptr(labels[c]),
                                  _ptr(self.last_label[c]), self.width,
                                  cfg.stride)
            if grouping_on and self.group_w.shape[0]:
                self.update_groups(c, vals[c], kinds[c], confs[c])
        fg = (labels == 1).any(axis=0)
        self.last_kinds = kinds
        self.last_confidence = confs
        tot = counts.sum(axis=0)
        row = [self.frame_count, int(tot[0]), int(tot[1]), int(tot[2]),
               int(tot[3]), int(tot[4]), int(tot[5] + tot[6]), int(fg.sum()),
               int(tot[4]), False]
        mask = fg.reshape(self.height, self.width).astype(np.uint8) * 255
        if not compat and row[8] > cfg.illumination_fraction * p * self.depth:
            row[9] = True
            self.reset_on_illumination(vals)
        self.frame_count += 1
        if (not compat and cfg.reorder_interval > 0
                and self.frame_count % cfg.reorder_interval == 0):
            self.reorder_levels()
        return mask, row

    def update_groups(self, c, vals, kinds, confs):
        """cascade.py:320-344 (sequential bincount sums)."""
        cfg = self.cfg
        g = self.group_w.shape[0]
        cnt = np.empty(g, dtype=np.int64)
        vs = np.empty(g)
        cs = np.empty(g)
        # np.bincount over the GROUP pixels in pixel order (C loop)
        lib().cogo_group_sums(self.n_pix, _ptr(np.ascontiguousarray(kinds)),
                              _ptr(np.ascontiguousarray(vals)),
                              _ptr(np.ascontiguousarray(confs)),
                              _ptr(self.group_id), g, _ptr(cnt), _ptr(vs),
                              _ptr(cs))
        act = cnt > 0
        if not act.any():
            return
        vbar = vs[act] / cnt[act]
        cbar = cs[act] / cnt[act]
        rho = cfg.learning_rate * np.maximum(1.0 - cbar, cfg.rate_floor)
        m = (1.0 - rho) * self.group_mu[c, act] + rho * vbar
        dlt = vbar - m
        s2 = (1.0 - rho) * self.group_var[c, act] + rho * dlt * dlt
        self.group_mu[c, act] = m
        self.group_var[c, act] = np.maximum(s2, cfg.variance_floor)

    def reset_on_illumination(self, vals):
        """cascade.py:361-391."""
        cfg, k, p = self.cfg, self.cfg.k_max, self.n_pix
        idx = np.arange(p, dtype=np.int64)
        inv = np.empty((p, k), dtype=np.int64)
        for c in range(self.depth):
            v = vals[c].astype(np.float64)
            live = np.arange(k)[None, :] < self.count[c][:, None]
            self.mu[c] = np.where(live, v[:, None], self.mu[c])
            self.var[c] = np.where(live, cfg.initial_variance, self.var[c])
            lib().cogo_sort_pixels(p, _ptr(idx), k, _ptr(self.mu[c]),
                                   _ptr(self.var[c]), _ptr(self.w[c]),
                                   _ptr(self.count[c]), _ptr(inv))
            for j in (0, 1):
                self.mode_ref[c, :, j] = inv[idx, self.mode_ref[c, :, j]]
            if self.group_w.shape[0]:
                g = self.group_w.shape[0]
                grouped = self.group_id >= 0
                cnt = np.bincount(self.group_id[grouped], minlength=g)
                vsum = np.bincount(self.group_id[grouped], weights=v[grouped],
                                   minlength=g)
                act = cnt > 0
                self.group_mu[c, act] = vsum[act] / cnt[act]
                self.group_var[c, act] = cfg.initial_variance
            self.chp_prev[c] = vals[c]
        self.streak[:] = 0
        self.clock[:] = 0
        self.waking[:] = 0
        self.hits[:] = 0
        self.last_active[:] = -1

    def reorder_levels(self):
        """cascade.py:393-417: mid levels by hits desc, ties prior mass desc."""
        p = self.n_pix
        ar = np.arange(p)
        gid = np.maximum(self.group_id, 0)
        for c in range(self.depth):
            codes = self.mid_order[c]
            hv = np.where(codes >= 0,
                          self.hits[c][ar[:, None], np.maximum(codes, 0)], -1)
            gmu = (self.group_mu[c][gid] if self.group_mu[c].shape[0]
                   else np.zeros(p))
            mass = np.full(codes.shape, -np.inf)
            for code, lmu in ((LEVEL_GROUP, gmu),
                              (LEVEL_MEAN, self.mu[c][ar, self.mode_ref[c, :, 0]]),
                              (LEVEL_MEANVAR, self.mu[c][ar, self.mode_ref[c, :, 1]])):
                lv = np.clip(np.rint(lmu), 0, 255).astype(np.int64)
                pm = np.broadcast_to(
                    self.tables[c][ar, lv].astype(np.float64)[:, None],
                    codes.shape)
                sel = codes == code
                mass[sel] = pm[sel]
            order = np.lexsort((-mass, -hv), axis=1)
            self.mid_order[c] = np.take_along_axis(codes, order, axis=1)
        self.hits[:] = 0

    def state(self) -> dict:
        return {n: getattr(self, n) for n in self.STATE}


def build_engine(cfg, tables32, classes, gid, gmu, gvar, gw, gmem, grids,
                 height, width, last_values) -> OracleEngine:
    """cascade.py:166-211 (CascadeEngine.build)."""
    d = len(grids)
    eng = OracleEngine(cfg, height, width, d)
    eng.dynamics = classes.copy()
    wts = rate_weights(classes, cfg)
    eng.wa = np.ascontiguousarray(wts[:, 0])
    eng.wb = np.ascontiguousarray(wts[:, 1])
    eng.wc = np.ascontiguousarray(wts[:, 2])
    eng.tables = tables32
    eng.group_id = gid.copy()
    eng.group_mu = np.ascontiguousarray(gmu.T.copy())
    eng.group_var = np.ascontiguousarray(gvar.T.copy())
    eng.group_w = gw.copy()
    eng.group_members = gmem.copy()
    for c, (mu, var, w, cnt) in enumerate(grids):
        eng.mu[c], eng.var[c], eng.w[c], eng.count[c] = mu, var, w, cnt
    eng.chp_prev[:] = last_values
    eng.finalize_tables()
    eng.seed_level_order()
    return eng


def train(values: np.ndarray, cfg) -> OracleEngine:
    """training.train_engine over (N, d, H, W) uint8 training frames."""
    n, d, h, wdt = values.shape
    flat = np.ascontiguousarray(values.reshape(n, d, h * wdt))
    tables = kde_tables32(flat, cfg.kde_bandwidth)
    _, occ = residue(flat, cfg.residue_t1, cfg.residue_t2)
    classes = classify(occ, cfg.peaky_threshold)
    grids, vs, ws = warmup(flat, cfg)
    gid, gmu, gvar, gw, gmem = groups(flat, vs, ws, cfg)
    return build_engine(cfg, tables, classes, gid, gmu, gvar, gw, gmem, grids,
                        h, wdt, flat[-1].copy())
