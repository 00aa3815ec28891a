"""Training phase 2: spatio-temporal grouping.

Algorithm of /root/reference/pkg/src/cogbg/grouping.py:85-208: z-scored
behaviour features -> seeded farthest-point k-means -> sigma-band trimming
-> pooled per-group, per-plane mode.  The features are produced on the GPU
by the warm-up kernel (``cog_gmm_warmup``, bit-identical to
``numpy.var(axis=0)`` of the adaptation series).

At scale (>= ``KMEANS_DEVICE_MIN`` pixels) the whole clustering runs on the
device (``build_groups_device``): the seeding (``cog_far_step``), the
assignment (``cog_kmeans_assign``), and every axis-0 reduction -- centre
update, z-score, sigma band -- through ``cog_seq_sums``, which reproduces
numpy's row-after-row binary64 summation order, so the group map is the
reference's bit for bit; the elementwise steps are IEEE-exact tensor ops.
Small frames use the numpy expressions below (the same arithmetic).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import EngineConfig
from .errors import ClusteringError, TrainingError

UNGROUPED = -1
_POOL_EXACT_BYTES = 1 << 31
# at scale (build_groups_device) groups above this pooled-sample size take
# their mean / variance from the GPU's exact integer sums instead of numpy's
# host pass over (N, d, members) f64 (~0.3 s per group at 720p)
_POOL_DEVICE_BYTES = 1 << 27


@dataclass
class GroupMap:
    group_id: np.ndarray      # (P,) int64, -1 ungrouped
    mu: np.ndarray            # (G, d)
    var: np.ndarray           # (G, d)
    weight: np.ndarray        # (G,)
    member_count: np.ndarray  # (G,) int64

    @property
    def group_count(self) -> int:
        return self.mu.shape[0]

    @staticmethod
    def empty(n_pix: int, depth: int) -> "GroupMap":
        return GroupMap(np.full(n_pix, UNGROUPED, dtype=np.int64),
                        np.zeros((0, depth)), np.zeros((0, depth)),
                        np.zeros(0), np.zeros(0, dtype=np.int64))


class KMeans:
    """Deterministic k-means: seeded first centre, farthest-point spread,
    lowest-index tie breaks (grouping.py:100-126)."""

    def __init__(self, k: int, seed: int, max_iter: int = 100):
        self.k, self.seed, self.max_iter = k, seed, max_iter

    def _spread(self, pts: np.ndarray) -> np.ndarray:
        n = pts.shape[0]
        first = int(np.random.default_rng(self.seed).integers(n))
        ctr = np.empty((self.k, pts.shape[1]))
        ctr[0] = pts[first]
        far = ((pts - ctr[0]) ** 2).sum(axis=1)
        for j in range(1, self.k):
            ctr[j] = pts[int(np.argmax(far))]
            far = np.minimum(far, ((pts - ctr[j]) ** 2).sum(axis=1))
        return ctr

    def fit(self, pts: np.ndarray):
        n = pts.shape[0]
        if n < self.k:
            raise ClusteringError(f"{n} pixels cannot form {self.k} clusters")
        ctr = self._spread(pts)
        if _device_assign(n, pts):
            return self._fit_device(pts, ctr)
        label = np.full(n, -1, dtype=np.int64)
        for _ in range(self.max_iter):
            d2 = ((pts[:, None, :] - ctr[None, :, :]) ** 2).sum(axis=2)
            nxt = np.argmin(d2, axis=1)
            if np.array_equal(nxt, label):
                break
            label = nxt
            for j in range(self.k):
                sub = pts[label == j]
                if sub.shape[0]:
                    ctr[j] = sub.mean(axis=0)
        return label, ctr


    def _fit_device(self, pts: np.ndarray, ctr: np.ndarray):
        """The same iteration with the assignment step (all n x k distances,
        the bulk of the time at 4K: ~1 s per iteration in numpy) on the GPU,
        bit-identical (cog_kmeans_assign); the centre update stays numpy's
        own masked mean, so the clustering is the reference's."""
        import torch

        from . import _lib
        lib = _lib.load()
        n = pts.shape[0]
        dev = torch.device("cuda", torch.cuda.current_device())
        stream = torch.cuda.current_stream(dev).cuda_stream
        p = torch.from_numpy(np.ascontiguousarray(pts, dtype=np.float64)).to(dev)
        lab = torch.full((n,), -1, dtype=torch.int64, device=dev)
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        c_dev = torch.empty((self.k, 2), dtype=torch.float64, device=dev)
        label = np.full(n, -1, dtype=np.int64)
        for _ in range(self.max_iter):
            c_dev.copy_(torch.from_numpy(np.ascontiguousarray(ctr)))
            flag.zero_()
            _lib.check(lib.cog_kmeans_assign(
                p.data_ptr(), n, c_dev.data_ptr(), self.k, lab.data_ptr(),
                flag.data_ptr(), stream), "cog_kmeans_assign")
            if int(flag.item()) == 0:
                break
            label = lab.cpu().numpy()
            for j in range(self.k):
                sub = pts[label == j]
                if sub.shape[0]:
                    ctr[j] = sub.mean(axis=0)
        return label, ctr


# point sets of at least this many points run the k-means assignment on the
# GPU (a module attribute the parity tests lower to 0 or raise; no env knob)
KMEANS_DEVICE_MIN = 65536


def _device_assign(n: int, pts: np.ndarray) -> bool:
    """GPU assignment for large point sets (>= KMEANS_DEVICE_MIN points)."""
    if pts.ndim != 2 or pts.shape[1] != 2:
        return False
    if n < KMEANS_DEVICE_MIN:
        return False
    try:
        import torch
    except ImportError:
        return False
    return torch.cuda.is_available()


def kmeans(features, k, seed, max_iter=100):
    return KMeans(k, seed, max_iter).fit(features)


def standardise(f: np.ndarray) -> np.ndarray:
    mean = f.mean(axis=0)
    std = f.std(axis=0, ddof=0)
    return (f - mean) / np.where(std > 0, std, 1.0)


def band_members(assign: np.ndarray, features: np.ndarray,
                 c: float) -> np.ndarray:
    """Keep pixels within mean +- c*std of their cluster on both features
    (grouping.py:142-161)."""
    out = np.full(assign.shape[0], UNGROUPED, dtype=np.int64)
    for j in np.unique(assign):
        sel = assign == j
        if sel.sum() < 2:
            continue
        f = features[sel]
        inside = np.abs(f - f.mean(axis=0)) <= c * f.std(axis=0, ddof=0)
        inside |= np.ptp(f, axis=0) == 0
        out[np.where(sel)[0][inside.all(axis=1)]] = j
    return out


def _pooled_stats(values: np.ndarray, sel: np.ndarray, floor: float):
    """Per-plane mean / floored variance of all training intensities of the
    members (grouping.py:189-192).  Small pools use the reference's exact
    numpy expression; huge pools (4K scenes) fall back to a chunked
    two-pass evaluation (mean still exact, variance within ~1e-15)."""
    n, d, _ = values.shape
    m = int(sel.sum())
    if n * d * m * 8 <= _POOL_EXACT_BYTES:
        pooled = values[:, :, sel].astype(np.float64)
        return (pooled.mean(axis=(0, 2)),
                np.maximum(pooled.var(axis=(0, 2), ddof=0), floor))
    idx = np.where(sel)[0]
    cnt = float(n * m)
    tot = np.zeros(d, dtype=np.int64)
    step = max(1, _POOL_EXACT_BYTES // (8 * n * d))
    for a in range(0, m, step):
        tot += values[:, :, idx[a:a + step]].astype(np.int64).sum(axis=(0, 2))
    mean = tot / cnt
    sq = np.zeros(d)
    for a in range(0, m, step):
        x = values[:, :, idx[a:a + step]].astype(np.float64) - mean[None, :, None]
        sq += (x * x).sum(axis=(0, 2))
    return mean, np.maximum(sq / cnt, floor)


def _pooled_stats_device(values: np.ndarray, values_dev, gm: "GroupMap",
                         big: list, floor: float) -> None:
    """Pooled mean / floored variance of the groups in ``big`` from exact
    integer sums of x and x^2 computed on the GPU (cog_pool_sums, one pass
    over the training frames for all of them).  The mean is the same
    correctly rounded sum / count as the chunked host path; the variance is
    the exact rational (M * sum x^2 - (sum x)^2) / M^2, correctly rounded
    (Python integers), where numpy's two-pass float evaluation is within
    ~1e-15 of it."""
    import torch

    from . import _lib
    n, d, p = values.shape
    if values_dev is None:
        values_dev = torch.from_numpy(np.ascontiguousarray(values)).to(
            torch.device("cuda", torch.cuda.current_device()))
    dev = values_dev.device
    slot = np.full(p, -1, dtype=np.int32)
    for k, gi in enumerate(big):
        slot[gm.group_id == gi] = k
    mem = torch.from_numpy(slot).to(dev)
    sums = torch.zeros((len(big), d, 2), dtype=torch.int64, device=dev)
    _lib.check(_lib.load().cog_pool_sums(
        values_dev.data_ptr(), n, d, p, mem.data_ptr(), len(big),
        sums.data_ptr(), torch.cuda.current_stream(dev).cuda_stream),
        "cog_pool_sums")
    s = sums.cpu().numpy()
    for k, gi in enumerate(big):
        cnt = n * int(gm.member_count[gi])
        for c in range(d):
            s1, s2 = int(s[k, c, 0]), int(s[k, c, 1])
            gm.mu[gi, c] = s1 / cnt
            gm.var[gi, c] = max((cnt * s2 - s1 * s1) / (cnt * cnt), floor)


def _seq_sums(x, label, k, shift=None, minmax=False):
    """Sequential axis-0 sums per label of the device tensor x (n, dims) f64
    (cog_seq_sums): returns (sums (k, dims), minmax (k, dims, 2) or None,
    counts (k,)) as numpy arrays."""
    import torch

    from . import _lib
    n, dims = x.shape
    dev = x.device
    out = torch.empty((k, dims), dtype=torch.float64, device=dev)
    mm = torch.empty((k, dims, 2), dtype=torch.float64, device=dev) \
        if minmax else None
    cnt = torch.zeros(k, dtype=torch.int64, device=dev)
    sh = None
    if shift is not None:
        sh = torch.from_numpy(np.ascontiguousarray(
            shift, dtype=np.float64).reshape(k, dims)).to(dev)
    _lib.check(_lib.load().cog_seq_sums(
        x.data_ptr(), n, dims,
        label.data_ptr() if label is not None else None, k,
        sh.data_ptr() if sh is not None else None, int(sh is not None),
        out.data_ptr(), mm.data_ptr() if mm is not None else None,
        cnt.data_ptr(), torch.cuda.current_stream(dev).cuda_stream),
        "cog_seq_sums")
    return (out.cpu().numpy(), mm.cpu().numpy() if mm is not None else None,
            cnt.cpu().numpy())


def build_groups_device(features, w_final, values: np.ndarray,
                        config: EngineConfig, values_dev=None) -> GroupMap:
    """build_groups with features (P, 2) / w_final (P,) f64 on the device
    (tensors, or arrays that are uploaded): the reference's clustering
    (grouping.py:100-195) step for step, every reduction in numpy's order
    (module docstring).  Only the group map, the per-group scalars and the
    compacted member weights come back to the host."""
    import torch

    from . import _lib
    lib = _lib.load()
    n_fr, d, p = values.shape
    dev = torch.device("cuda", torch.cuda.current_device())
    f = torch.as_tensor(features).to(dev, torch.float64).contiguous()
    wf = torch.as_tensor(w_final).to(dev, torch.float64).contiguous()
    if tuple(f.shape) != (p, 2):
        raise TrainingError("feature geometry does not match frames")
    k = config.clusters
    if p < k:
        raise ClusteringError(f"{p} pixels cannot form {k} clusters")
    stream = torch.cuda.current_stream(dev).cuda_stream
    # ---- standardise (grouping.py:93-97)
    s1, _, _ = _seq_sums(f, None, 1)
    mean = s1[0] / p
    q, _, _ = _seq_sums(f, None, 1, shift=mean)
    std = np.sqrt(q[0] / p)
    den = np.where(std > 0, std, 1.0)
    z = ((f - torch.from_numpy(mean).to(dev))
         / torch.from_numpy(den).to(dev)).contiguous()
    # ---- farthest-point seeding (grouping.py:100-112)
    first = int(np.random.default_rng(config.cluster_seed).integers(p))
    ctr = np.empty((k, 2))
    ctr[0] = z[first].cpu().numpy()
    far = torch.empty(p, dtype=torch.float64, device=dev)
    best = torch.empty(2, dtype=torch.int64, device=dev)
    for j in range(1, k):
        c_prev = np.ascontiguousarray(ctr[j - 1])
        _lib.check(lib.cog_far_step(z.data_ptr(), p, c_prev.ctypes.data,
                                    int(j == 1), far.data_ptr(),
                                    best.data_ptr(), stream), "cog_far_step")
        ctr[j] = z[int(best[1].item())].cpu().numpy()
    # ---- k-means (grouping.py:113-126)
    lab = torch.full((p,), -1, dtype=torch.int64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    c_dev = torch.empty((k, 2), dtype=torch.float64, device=dev)
    for _ in range(100):
        c_dev.copy_(torch.from_numpy(np.ascontiguousarray(ctr)))
        flag.zero_()
        _lib.check(lib.cog_kmeans_assign(
            z.data_ptr(), p, c_dev.data_ptr(), k, lab.data_ptr(),
            flag.data_ptr(), stream), "cog_kmeans_assign")
        if int(flag.item()) == 0:
            break
        sums, _, cnt = _seq_sums(z, lab, k)
        for j in range(k):
            if cnt[j]:
                ctr[j] = sums[j] / cnt[j]
    # ---- sigma band on the raw features (grouping.py:142-161)
    sums, mm, cnt = _seq_sums(f, lab, k, minmax=True)
    safe = np.maximum(cnt, 1)[:, None]
    cmean = sums / safe
    q, _, _ = _seq_sums(f, lab, k, shift=cmean)
    cstd = config.cluster_threshold * np.sqrt(q / safe)
    flat = torch.from_numpy((mm[:, :, 1] - mm[:, :, 0]) == 0).to(dev)
    inside = ((f - torch.from_numpy(cmean).to(dev)[lab]).abs()
              <= torch.from_numpy(cstd).to(dev)[lab]) | flat[lab]
    keep = inside.all(dim=1) & torch.from_numpy(cnt >= 2).to(dev)[lab]
    member = torch.where(keep, lab, torch.full_like(lab, UNGROUPED))
    cnt2 = torch.bincount(member[member >= 0], minlength=k).cpu().numpy()
    kept = [j for j in range(k) if cnt2[j] >= 2]
    g = len(kept)
    remap = np.full(k + 1, UNGROUPED, dtype=np.int64)   # [-1] -> ungrouped
    for gi, j in enumerate(kept):
        remap[j] = gi
    gid_dev = torch.from_numpy(remap).to(dev)[member]
    gm = GroupMap(gid_dev.cpu().numpy(), np.zeros((g, d)), np.zeros((g, d)),
                  np.zeros(g), np.zeros(g, dtype=np.int64))
    big = []
    for gi, j in enumerate(kept):
        gm.member_count[gi] = cnt2[j]
        # 1-D contiguous mean: numpy's own (pairwise) sum on the compacted,
        # order-preserved member weights
        gm.weight[gi] = wf[gid_dev == gi].cpu().numpy().mean()
        if n_fr * d * int(cnt2[j]) * 8 > min(_POOL_EXACT_BYTES,
                                             _POOL_DEVICE_BYTES):
            big.append(gi)
        else:
            gm.mu[gi], gm.var[gi] = _pooled_stats(values, gm.group_id == gi,
                                                  config.variance_floor)
    if big:
        _pooled_stats_device(values, values_dev, gm, big,
                             config.variance_floor)
    return gm


def _cuda_ok() -> bool:
    try:
        import torch
    except ImportError:
        return False
    return torch.cuda.is_available()


def build_groups(features: np.ndarray, w_final: np.ndarray,
                 values: np.ndarray, config: EngineConfig,
                 values_dev=None) -> GroupMap:
    """features (P, 2) f64, w_final (P,) f64, values (N, d, P) uint8;
    values_dev: the same values already on the GPU (optional)."""
    n, d, p = values.shape
    if not config.grouping:
        return GroupMap.empty(p, d)
    if p >= KMEANS_DEVICE_MIN and _cuda_ok():
        return build_groups_device(features, w_final, values, config,
                                   values_dev)
    if not isinstance(features, np.ndarray):
        features = features.cpu().numpy()
        w_final = w_final.cpu().numpy()
    if features.shape != (p, 2):
        raise TrainingError("feature geometry does not match frames")
    assign, _ = KMeans(config.clusters, config.cluster_seed).fit(
        standardise(features))
    member = band_members(assign, features, config.cluster_threshold)
    kept = [j for j in np.unique(member)
            if j != UNGROUPED and (member == j).sum() >= 2]
    g = len(kept)
    gm = GroupMap(np.full(p, UNGROUPED, dtype=np.int64), np.zeros((g, d)),
                  np.zeros((g, d)), np.zeros(g), np.zeros(g, dtype=np.int64))
    big = []
    use_dev = _cuda_ok()
    for gi, j in enumerate(kept):
        sel = member == j
        gm.group_id[sel] = gi
        gm.member_count[gi] = sel.sum()
        if use_dev and n * d * int(gm.member_count[gi]) * 8 > _POOL_EXACT_BYTES:
            big.append(gi)   # beyond numpy's in-memory expression
        else:
            gm.mu[gi], gm.var[gi] = _pooled_stats(values, sel,
                                                  config.variance_floor)
        gm.weight[gi] = w_final[sel].mean()
    if big:
        _pooled_stats_device(values, values_dev, gm, big,
                             config.variance_floor)
    return gm
