"""CascadeEngine -- the reference's runtime API with all state in HBM.

Drop-in for /root/reference/pkg/src/cogbg/cascade.py:113-444: same
constructor shape, ``process_frame`` -> (LabelMask, FrameStats),
``last_confidence`` / ``last_kinds``, ``clone``, ``reorder_levels``,
``level_order``, ``sampling_clock``, state arrays under the reference's
names and dtypes, ``run_sequence``, ``compute_confidence``, ``chp_check``.

Differences in mechanics, not in results:

* One ``cog_step`` launch per frame does the whole per-frame path (all
  planes, copy resolution, union mask, group update, statistics,
  illumination test); nothing is computed on the host.
* The returned mask / stats are filled by asynchronous device->host copies;
  they block only when read, so a frame loop runs ahead of the host.
* State arrays (``mu``, ``hits``, ``group_mu`` ...) are exported on first
  access after a frame and cached; in-place edits of the returned numpy
  arrays are written back to the device before the next device operation,
  so reference-style ``eng.hits[0, 0, 2] = 5`` keeps working.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .config import EngineConfig
from .errors import CudaError, DataError
from .frame_io import Frame, LabelMask

LEVEL_CHP, LEVEL_GROUP, LEVEL_MEAN, LEVEL_MEANVAR, LEVEL_GMM = 0, 1, 2, 3, 4
KIND_SKIP, KIND_COPY = 5, 6

STATS_FIELDS = ("frame", "n_chp", "n_group", "n_mean", "n_meanvar", "n_gmm",
                "n_skipped", "n_foreground", "unexplained",
                "illumination_fired")

_STATE_FIELDS = ("mu", "var", "w", "count", "mid_order", "mode_ref",
                 "chp_prev", "last_label", "last_active", "waking", "streak",
                 "clock", "hits")
_GROUP_FIELDS = ("group_mu", "group_var")


class FrameStats:
    """Per-frame level populations and monitor state, pooled over planes
    (cascade.py:45-69).  Built from a pending device->host copy; fields
    resolve on first access."""

    __slots__ = ("_row", "_host", "_event")

    def __init__(self, frame=0, n_chp=0, n_group=0, n_mean=0, n_meanvar=0,
                 n_gmm=0, n_skipped=0, n_foreground=0, unexplained=0,
                 illumination_fired=False):
        self._row = [int(frame), int(n_chp), int(n_group), int(n_mean),
                     int(n_meanvar), int(n_gmm), int(n_skipped),
                     int(n_foreground), int(unexplained),
                     bool(illumination_fired)]
        self._host = None
        self._event = None

    @classmethod
    def pending(cls, host_tensor, event) -> "FrameStats":
        s = cls.__new__(cls)
        s._row = None
        s._host = host_tensor
        s._event = event
        return s

    def _detach(self, slot) -> None:
        """The staging slot is about to be reused: materialise now."""
        if self._row is None:
            self._resolve()

    def _resolve(self) -> list:
        if self._row is None:
            self._event.synchronize()
            v = self._host.tolist()
            self._row = [int(x) for x in v[:9]] + [bool(v[9])]
            self._host = None
            self._event = None
        return self._row

    def as_row(self) -> list:
        r = self._resolve()
        return r[:9] + [int(r[9])]

    def __eq__(self, other) -> bool:
        return isinstance(other, FrameStats) and self._resolve() == other._resolve()

    def __repr__(self) -> str:
        r = self._resolve()
        return "FrameStats(" + ", ".join(
            f"{k}={v}" for k, v in zip(STATS_FIELDS, r)) + ")"


def _stat_property(i):
    def get(self):
        return self._resolve()[i]

    def set_(self, value):
        self._resolve()[i] = bool(value) if i == 9 else int(value)
    return property(get, set_)


for _i, _name in enumerate(STATS_FIELDS):
    setattr(FrameStats, _name, _stat_property(_i))


def chp_check(previous: int, value: int, epsilon: float = 0.0) -> bool:
    """Consistent-hypothesis probe (cascade.py:72-74)."""
    return abs(int(value) - int(previous)) <= epsilon


def compute_confidence(value: float, prev_value: float, mu_top: float,
                       sigma_top: float, prior_hat: float,
                       weights: tuple[float, float, float],
                       match_lambda: float = 2.5, prior_floor: float = 1e-3,
                       literal: bool = False) -> float:
    """Scalar form of the per-pixel confidence (cascade.py:77-103); the
    kernel evaluates the same expression in the same order."""
    a, b, g = weights
    bterm = abs(value - prev_value) / 255.0
    if not literal:
        bterm = 1.0 - bterm
    gterm = min(abs(value - mu_top) / (match_lambda * sigma_top), 1.0)
    if not literal:
        gterm = 1.0 - gterm
    if prior_hat < prior_floor:
        den = b + g
        return 0.0 if den <= 0.0 else (b * bterm + g * gterm) / den
    return a * prior_hat + b * bterm + g * gterm


def params_from_config(cfg: EngineConfig, weights: np.ndarray) -> _lib.Params:
    q = _lib.Params()
    q.learning_rate = cfg.learning_rate
    q.match_lambda = cfg.match_lambda
    q.background_threshold = cfg.background_threshold
    q.variance_floor = cfg.variance_floor
    q.initial_variance = cfg.initial_variance
    q.chp_epsilon = cfg.chp_epsilon
    q.confidence_threshold = cfg.confidence_threshold
    q.prior_floor = cfg.prior_floor
    q.rate_floor = cfg.rate_floor
    q.illumination_fraction = cfg.illumination_fraction
    for i, x in enumerate(np.asarray(weights, dtype=np.float64).ravel()):
        q.weights[i] = float(x)
    q.saturation_frames = int(min(cfg.saturation_frames, 2 ** 31 - 1))
    q.sleep_frames = cfg.sleep_frames
    compat = bool(cfg.compat)
    q.sampling_on = int(bool(cfg.sampling) and not compat)
    q.grouping_on = int(bool(cfg.grouping) and not compat)
    q.rate_scaling_on = int(not compat)
    q.chp_on = int(not compat)
    q.literal_conf = int(bool(cfg.confidence_literal))
    q.compat = int(compat)
    return q


def weight_table(cfg: EngineConfig) -> np.ndarray:
    """(3, 3) class -> (alpha, beta, gamma) table (scene_prior.py:205-213)."""
    return np.array([cfg.weights_static, cfg.weights_oscillating,
                     cfg.weights_dynamic], dtype=np.float64)


class DeviceState:
    """HBM buffers of ``streams`` engines of one geometry (layout in
    include/cog_b200.h).  Torch tensors are used purely as allocations."""

    def __init__(self, cfg: EngineConfig, height: int, width: int, depth: int,
                 n_groups: int = 0, streams: int = 1, device=None,
                 row0: int = 0, total_pixels: int | None = None):
        self.device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self.f64 = cfg.state_dtype == "float64"
        self.tdtype = torch.float64 if self.f64 else torch.float32
        self.height, self.width, self.depth = height, width, depth
        self.k = cfg.k_max
        self.streams = streams
        self.n_groups = n_groups
        self.P = height * width
        self.row0 = row0
        self.total_pixels = total_pixels or self.P
        self.stride = cfg.stride
        S, d, K, P = streams, depth, cfg.k_max, self.P
        G1 = max(n_groups, 1)
        dev = self.device

        def z(*shape, dtype):
            return torch.zeros(shape, dtype=dtype, device=dev)
        # mixture records (S, d, P, R): (mu_k, var_k) at [2k, 2k+1], w_k at
        # [2 * KB + k] (include/cog_b200.h); mu / var / w are views
        self.kb = 3 if K <= 3 else (5 if K <= 5 else 8)
        self.rec = int(_lib.load().cog_mix_elems(K))
        self.mix = z(S, d, P, self.rec, dtype=self.tdtype)
        self.meta = z(S, d, P, dtype=torch.int16)
        self.dyn = z(S, d, P, dtype=torch.int32)
        self.streak = z(S, d, P, dtype=torch.int32)
        self.hits = z(S, d, 5, P, dtype=torch.int32)
        # float32 engines: the hot pass's packed per-level hit bytes
        # (include/cog_b200.h, cog_state.hitq); hits = hits + its bytes
        self.hitq = None if self.f64 else z(S, d, P, dtype=torch.int32)
        # the prior in the reference layout (exact values), and for float32
        # engines its u16 tile-major hot copy (cog_tabq_build)
        self.table = z(S, d, P, 256, dtype=torch.float32)
        self.peak = torch.ones((S, d, P), dtype=torch.float32, device=dev)
        if self.f64:
            self.tabq = None
        else:
            n = int(_lib.load().cog_tabq_elems(_lib.ref(self._geom(1))))
            if n < 0:
                raise DataError("unsupported engine geometry")
            self.tabq = z(S, n, dtype=torch.int16)
        self.cls = z(S, P, dtype=torch.uint8)
        self.gid = torch.full((S, P), -1, dtype=torch.int16, device=dev)
        self.g_mu = z(S, d, G1, dtype=torch.float64)
        self.g_var = torch.ones((S, d, G1), dtype=torch.float64, device=dev)
        self.g_members = z(S, G1, dtype=torch.int32)
        self.words = int(_lib.load().cog_accum_words(d, n_groups))
        self.accum = z(S, self.words, dtype=torch.int64)
        self.sync = z(S, 4, dtype=torch.int32)
        self.conf = z(S, d, P, dtype=self.tdtype)
        self.kind = z(S, d, P, dtype=torch.uint8)
        slots = int(_lib.load().cog_deepq_slots(d, P))
        self.deepq = z(S, slots, dtype=torch.int64)
        self.deeprho = torch.empty((S, slots), dtype=torch.float64, device=dev)
        self._refresh()

    def _geom(self, streams: int) -> "_lib.Geom":
        g = _lib.Geom()
        g.total_pixels = self.total_pixels
        g.height, g.width, g.depth = self.height, self.width, self.depth
        g.k, g.stride, g.n_groups = self.k, self.stride, self.n_groups
        g.streams, g.state_f64, g.row0 = streams, int(self.f64), self.row0
        return g

    # mixture views (S, d, K, P) of the records
    @property
    def mu(self) -> torch.Tensor:
        return self.mix[..., 0:2 * self.k:2].permute(0, 1, 3, 2)

    @property
    def var(self) -> torch.Tensor:
        return self.mix[..., 1:2 * self.k:2].permute(0, 1, 3, 2)

    @property
    def w(self) -> torch.Tensor:
        return self.mix[..., 2 * self.kb:2 * self.kb + self.k].permute(0, 1, 3, 2)

    def table_to_ref(self, s: int) -> torch.Tensor:
        """Stream s's prior table in the reference layout (d, P, 256)."""
        return self.table[s]

    def table_from_ref(self, s: int, tables: torch.Tensor) -> None:
        """Install a (d, P, 256) f32 table into stream s (its peak must
        already be set) and rebuild the hot copy."""
        tables = tables.to(self.device, torch.float32)
        if tuple(tables.shape) != (self.depth, self.P, 256):
            raise DataError(f"table shape {tuple(tables.shape)} != "
                            f"{(self.depth, self.P, 256)}")
        if tables.data_ptr() != self.table[s].data_ptr():
            self.table[s].copy_(tables)
        self.build_hot_table(s)

    def build_hot_table(self, s: int) -> None:
        """u16 tile-major phat of stream s from its table and peak."""
        if self.tabq is None:
            return
        rc = _lib.load().cog_tabq_build(
            _lib.ref(self._geom(1)), self.table[s].data_ptr(),
            self.peak[s].data_ptr(), self.tabq[s].data_ptr(),
            torch.cuda.current_stream(self.device).cuda_stream)
        _lib.check(rc, "cog_tabq_build")

    _BUFS = ("mix", "meta", "dyn", "streak", "hits", "table", "peak", "tabq",
             "cls", "gid", "g_mu", "g_var", "g_members", "accum", "sync",
             "deepq", "deeprho", "hitq")

    def _refresh(self) -> None:
        self.geom = self._geom(self.streams)
        st = _lib.State()
        for name in self._BUFS:
            t = getattr(self, name)
            setattr(st, name, t.data_ptr() if t is not None else None)
        self.cstate = st

    def stream_view(self, s: int) -> "_lib.State":
        """C struct pointing at stream s only (for export/import)."""
        st = _lib.State()
        for name in self._BUFS:
            t = getattr(self, name)
            setattr(st, name, t[s].data_ptr() if t is not None else None)
        return st

    def single_geom(self) -> "_lib.Geom":
        g = _lib.Geom.from_buffer_copy(self.geom)
        g.streams = 1
        return g

    # written only while training / loading a model (into a fresh state),
    # read-only to every step: a clone shares them instead of copying the
    # ~1.5 KB per plane-pixel prior
    _READ_ONLY = ("table", "peak", "tabq", "cls", "gid", "g_members")

    def clone(self) -> "DeviceState":
        twin = DeviceState.__new__(DeviceState)
        for k, v in vars(self).items():
            if isinstance(v, torch.Tensor):
                setattr(twin, k, v if k in self._READ_ONLY else v.clone())
            elif k not in ("geom", "cstate"):
                setattr(twin, k, v)
        twin._refresh()
        return twin

    def set_groups(self, n_groups: int) -> None:
        """Re-size the group arrays (before the groups are uploaded)."""
        S, d = self.streams, self.depth
        G1 = max(n_groups, 1)
        dev = self.device
        self.n_groups = n_groups
        self.g_mu = torch.zeros((S, d, G1), dtype=torch.float64, device=dev)
        self.g_var = torch.ones((S, d, G1), dtype=torch.float64, device=dev)
        self.g_members = torch.zeros((S, G1), dtype=torch.int32, device=dev)
        self.words = int(_lib.load().cog_accum_words(d, n_groups))
        self.accum = torch.zeros((S, self.words), dtype=torch.int64, device=dev)
        self._refresh()


_COPY_POOL = None


def _copy_rows(planes, out: np.ndarray) -> None:
    """planes[c] -> out[c]; frames above ~1 MB are split by rows over a few
    threads (numpy copies release the GIL), so staging keeps up with the
    device step."""
    global _COPY_POOL
    if out.nbytes < (1 << 20):
        for c, pl in enumerate(planes):
            out[c] = pl
        return
    if _COPY_POOL is None:
        import concurrent.futures as cf
        _COPY_POOL = cf.ThreadPoolExecutor(4)
    h = out.shape[1]
    cuts = [0, h // 4, h // 2, 3 * h // 4, h]

    def part(i):
        a, b = cuts[i], cuts[i + 1]
        for c, pl in enumerate(planes):
            out[c, a:b] = pl[a:b]
    list(_COPY_POOL.map(part, range(4)))


class HostRing:
    """Reusable pinned staging for the host-facing frame loop.

    ``slots`` sets of {pinned frame in, device frame, device mask / stats,
    pinned mask / stats out, completion event}.  ``process_frame`` copies a
    host frame into a pinned slot (one memcpy), enqueues H2D -> step -> D2H
    and returns pending results that point into the slot; pinned memory is
    allocated once instead of per frame (cudaHostAlloc costs far more than
    the step).  Before a slot is reused, any result still pointing into it
    is materialised into its own array, so results stay valid however long
    the caller keeps them."""

    def __init__(self, depth: int, height: int, width: int, device,
                 slots: int = 4):
        self.slots = []
        for _ in range(slots):
            self.slots.append({
                "in": torch.empty((depth, height, width), dtype=torch.uint8,
                                  pin_memory=True),
                "x": torch.empty((depth, height, width), dtype=torch.uint8,
                                 device=device),
                "mask": torch.empty((height, width), dtype=torch.uint8,
                                    device=device),
                "stats": torch.empty(16, dtype=torch.int64, device=device),
                "hm": torch.empty((height, width), dtype=torch.uint8,
                                  pin_memory=True),
                "hs": torch.empty(16, dtype=torch.int64, pin_memory=True),
                "event": None, "owners": (), "up": torch.cuda.Event(),
                "src": None,
            })
        lib = _lib.load()
        for sl in self.slots:
            sl["cup"] = CEvent(lib)
            sl["cdone"] = CEvent(lib)
        self.next = 0
        # host->device copies run on their own stream so frame t+1's upload
        # overlaps frame t's step; the step waits on the copy's event
        self.copy_stream = torch.cuda.Stream(device=device)
        # device->host copies on a third stream: frame t+1's step does not
        # queue behind frame t's downloads
        self.down_stream = torch.cuda.Stream(device=device)

    def acquire(self) -> dict:
        slot = self.slots[self.next]
        self.next = (self.next + 1) % len(self.slots)
        for o in slot["owners"]:
            o._detach(slot)
        slot["owners"] = ()
        if slot["event"] is not None:
            slot["event"].synchronize()   # its pinned input may be reused
            slot["event"] = None
        slot["src"] = None
        return slot


class CEvent:
    """A cudaEvent_t owned through the C-ABI (cog_event_create); quacks like
    torch.cuda.Event for the pending results."""

    __slots__ = ("lib", "handle")

    def __init__(self, lib):
        self.lib = lib
        self.handle = lib.cog_event_create()
        if not self.handle:
            raise CudaError("cog_event_create failed")

    def synchronize(self) -> None:
        _lib.check(self.lib.cog_event_sync(self.handle), "cog_event_sync")

    def query(self) -> bool:
        rc = self.lib.cog_event_query(self.handle)
        if rc < 0:
            _lib.check(-rc, "cog_event_query")
        return rc == 1

    def __del__(self):
        try:
            if self.handle:
                self.lib.cog_event_destroy(self.handle)
        except Exception:
            pass


class CascadeEngine:
    """All per-pixel cascade state of one stream, resident on the GPU."""

    def __init__(self, config: EngineConfig, height: int, width: int,
                 depth: int, n_groups: int = 0, device=None, row0: int = 0,
                 total_pixels: int | None = None) -> None:
        config.validate()
        self.config = config
        self.height, self.width, self.depth = height, width, depth
        self.n_pix = height * width
        self.backend = "cuda"
        self.frame_count = 0
        self.bandwidth = 0.0
        self.sample_count = 0
        self.lib = _lib.load()
        self.dev = DeviceState(config, height, width, depth, n_groups,
                               device=device, row0=row0,
                               total_pixels=total_pixels)
        self._wtab = weight_table(config)
        self.group_w = np.zeros(0)
        self.group_members = np.zeros(0, dtype=np.int64)
        self._reorder_pending = False
        self._host = None
        self._snap = None
        # parity/debug switch: reduce each group's confidences in the
        # reference's sequential pixel order (single thread, small frames);
        # the production path sums them exactly in fixed point instead
        self.exact_group_sums = False
        # parity switch: which step kernel runs ("auto", "general", "lean");
        # an engine attribute, never read from the environment
        self.kernel_variant = "auto"
        yy, xx = np.divmod(np.arange(self.n_pix), width)
        s = config.stride
        self.on_lattice = (((yy + row0) % s == 0) & (xx % s == 0)).astype(np.uint8)
        self.prior = None
        self.row0 = row0
        # row-band shard: callable summing the `accum` partials across the
        # shards of one frame in place (parallel.py); None = whole frame
        self.reducer = None
        # row-band shard on its own GPU: parallel.PeerMailbox -- the sum of
        # the partials fused into the step over peer memory (no reducer)
        self.peers = None
        self._ring = None  # pinned host staging, created on first host frame

    # ------------------------------------------------------------ helpers

    @property
    def stream(self) -> int:
        return torch.cuda.current_stream(self.dev.device).cuda_stream

    def _params(self) -> "_lib.Params":
        """The C params struct, rebuilt only when an input changes (the
        per-frame launch path must stay cheap on the host)."""
        key = (id(self.config), self._wtab.tobytes(),
               bool(self.exact_group_sums), self.kernel_variant)
        if getattr(self, "_pkey", None) != key:
            q = params_from_config(self.config, self._wtab)
            q.exact_group_sums = int(self.exact_group_sums)
            q.variant = _lib.VARIANTS[self.kernel_variant]
            self._pcache, self._pkey = q, key
        return self._pcache

    def _frame_tensor(self, frame) -> torch.Tensor:
        """(d, H, W) uint8 on the device; host frames go through pinned
        staging and an asynchronous copy."""
        if isinstance(frame, torch.Tensor):
            t = frame
            if t.dim() == 2:
                t = t.unsqueeze(0)
            shape = tuple(t.shape)
            if shape[1:] != (self.height, self.width):
                raise DataError(f"frame geometry {shape[1]}x{shape[2]} != "
                                f"model {self.height}x{self.width}")
            if shape[0] != self.depth:
                raise DataError(f"frame has {shape[0]} planes, model expects "
                                f"{self.depth}")
            if t.dtype != torch.uint8:
                raise DataError("frames must be uint8")
            if t.device != self.dev.device:
                t = t.to(self.dev.device, non_blocking=True)
            return t.contiguous()
        if not isinstance(frame, Frame):
            frame = Frame.from_array(np.asarray(frame))
        if (frame.height, frame.width) != (self.height, self.width):
            raise DataError(
                f"frame {frame.index} geometry {frame.height}x{frame.width}"
                f" != model {self.height}x{self.width}")
        if frame.depth != self.depth:
            raise DataError(f"frame {frame.index} has {frame.depth} planes,"
                            f" model expects {self.depth}")
        host = torch.empty((self.depth, self.height, self.width),
                           dtype=torch.uint8, pin_memory=True)
        hv = host.numpy()
        for c, pl in enumerate(frame.planes):
            hv[c] = pl.data
        return host.to(self.dev.device, non_blocking=True)

    # ---------------------------------------------------- host state cache

    def _flush(self) -> None:
        """Write back in-place edits of exported arrays, drop the cache."""
        if self._host is None:
            return
        changed = [k for k in self._host
                   if not np.array_equal(self._host[k], self._snap[k])]
        if changed:
            self._import_arrays(self._host)
        self._host = None
        self._snap = None

    def materialize(self) -> None:
        """Apply a pending illumination reset / scheduled reorder now."""
        self._flush()
        rc = self.lib.cog_apply_pending(
            _lib.ref(self.dev.geom), _lib.ref(self._params()),
            _lib.ref(self.dev.cstate), int(self._reorder_pending), self.stream)
        _lib.check(rc, "cog_apply_pending")
        self._reorder_pending = False

    def _export_arrays(self) -> dict:
        self.materialize()
        return export_state(self.dev, 0, self.config.k_max, self.lib,
                            self.stream)

    def _import_arrays(self, arrays: dict) -> None:
        d, P, K = self.depth, self.n_pix, self.config.k_max
        dev = self.dev.device
        spec = {"mu": (np.float64, (d, P, K)), "var": (np.float64, (d, P, K)),
                "w": (np.float64, (d, P, K)), "count": (np.int64, (d, P)),
                "mid_order": (np.int8, (d, P, 3)),
                "mode_ref": (np.int8, (d, P, 2)),
                "chp_prev": (np.uint8, (d, P)), "last_label": (np.uint8, (d, P)),
                "last_active": (np.int8, (d, P)), "waking": (np.uint8, (d, P)),
                "streak": (np.int64, (d, P)), "clock": (np.int64, (d, P)),
                "hits": (np.int64, (d, P, 5))}
        bufs = {}
        for k, (dt, shape) in spec.items():
            a = np.ascontiguousarray(np.asarray(arrays[k]).astype(dt, copy=False))
            if a.shape != shape:
                raise DataError(f"{k}: shape {a.shape} != {shape}")
            bufs[k] = torch.from_numpy(a).to(dev)
        if int(bufs["count"].max()) > K or int(bufs["count"].min()) < 0:
            raise DataError("mode count out of range")
        rs = _ref_struct(bufs)
        rc = self.lib.cog_import_state(_lib.ref(self.dev.single_geom()),
                                       _lib.ref(self.dev.stream_view(0)),
                                       _lib.ref(rs), self.stream)
        _lib.check(rc, "cog_import_state")
        G = self.dev.n_groups
        if "group_mu" in arrays and G:
            self.dev.g_mu[0, :, :G] = torch.from_numpy(
                np.asarray(arrays["group_mu"], dtype=np.float64)).to(dev)
            self.dev.g_var[0, :, :G] = torch.from_numpy(
                np.asarray(arrays["group_var"], dtype=np.float64)).to(dev)
        torch.cuda.current_stream(dev).synchronize()

    def _cached(self) -> dict:
        if self._host is None:
            self._host = self._export_arrays()
            self._snap = {k: v.copy() for k, v in self._host.items()}
        return self._host

    # ------------------------------------------------------------ runtime

    def _launch_step(self, x: torch.Tensor, mask: torch.Tensor,
                     stats: torch.Tensor) -> None:
        """Enqueue one frame: ``cog_step`` with the frame tail fused into
        the last CTA, or -- for a row-band shard (``self.reducer`` set) --
        the step, the cross-shard sum of the exact partials, then
        ``cog_finalize`` (identical on every shard)."""
        banded = self.reducer is not None
        geom, prm, st = (_lib.ref(self.dev.geom), _lib.ref(self._params()),
                         _lib.ref(self.dev.cstate))
        if self.peers is not None:
            # row-band shard on its own GPU: the cross-shard sum is fused
            # into the step's tail over peer mailboxes (parallel.PeerMailbox)
            box = self.peers
            if not box.fused and box.barrier is None:
                raise DataError("a local (one-process) peer mailbox is "
                                "stepped by BandSet, not by its engines")
            rc = self.lib.cog_step_p2p(
                geom, prm, st, x.data_ptr(), mask.data_ptr(),
                self.dev.conf.data_ptr(), self.dev.kind.data_ptr(),
                stats.data_ptr(), self.frame_count,
                int(self._reorder_pending), int(box.fused),
                _lib.ref(box.next()), self.stream)
            _lib.check(rc, "cog_step_p2p")
            if not box.fused:
                box.barrier()   # every rank's push has landed
                rc = self.lib.cog_finalize_p2p(
                    geom, prm, st, stats.data_ptr(), self.frame_count,
                    _lib.ref(box.current()), self.stream)
                _lib.check(rc, "cog_finalize_p2p")
            self._advance()
            return
        rc = self.lib.cog_step(
            geom, prm, st, x.data_ptr(), mask.data_ptr(),
            self.dev.conf.data_ptr(), self.dev.kind.data_ptr(),
            stats.data_ptr(), self.frame_count, int(self._reorder_pending),
            0 if banded else 1, self.stream)
        _lib.check(rc, "cog_step")
        if banded:
            self.reducer(self.dev.accum)
            rc = self.lib.cog_finalize(geom, prm, st, stats.data_ptr(),
                                       self.frame_count, self.stream)
            _lib.check(rc, "cog_finalize")
        self._advance()

    def _advance(self) -> None:
        """Frame counter and the reorder schedule (cascade.py:314-317): a
        reorder due after this frame is applied at the next step's start."""
        self._reorder_pending = False
        cfg = self.config
        self.frame_count += 1
        if (not cfg.compat and cfg.reorder_interval > 0
                and self.frame_count % cfg.reorder_interval == 0):
            self._reorder_pending = True

    def process_frame(self, frame) -> tuple[LabelMask, FrameStats]:
        """One frame through the CUDA step (cascade.py:261-318).  Host
        frames go through the engine's pinned staging ring (one C-ABI call,
        cog_step_host: upload on a copy stream, step, result download); the
        returned mask / stats resolve on first access."""
        self._flush()
        if self._ring is None:
            self._ring = HostRing(self.depth, self.height, self.width,
                                  self.dev.device)
        ring = self._ring
        slot = ring.acquire()
        cuda_in = isinstance(frame, torch.Tensor) and frame.is_cuda
        if not cuda_in:
            if (isinstance(frame, torch.Tensor) and frame.is_pinned()
                    and frame.dtype == torch.uint8 and frame.is_contiguous()
                    and tuple(frame.shape[-2:]) == (self.height, self.width)
                    and frame.numel() == self.depth * self.n_pix):
                src = frame          # DMA straight from the caller's pinned
            else:                    # tensor (kept alive until slot reuse)
                self._stage(frame, slot["in"].numpy())
                src = slot["in"]
            slot["src"] = src
        if not cuda_in and self.reducer is None and self.peers is None:
            rc = self.lib.cog_step_host(
                _lib.ref(self.dev.geom), _lib.ref(self._params()),
                _lib.ref(self.dev.cstate), src.data_ptr(),
                slot["x"].data_ptr(), slot["mask"].data_ptr(),
                self.dev.conf.data_ptr(), self.dev.kind.data_ptr(),
                slot["stats"].data_ptr(), slot["hm"].data_ptr(),
                slot["hs"].data_ptr(), self.frame_count,
                int(self._reorder_pending), self.stream,
                ring.copy_stream.cuda_stream, ring.down_stream.cuda_stream,
                slot["cup"].handle,
                slot["cdone"].handle)
            _lib.check(rc, "cog_step_host")
            if src is frame:
                # the caller owns this pinned buffer and may refill it as
                # soon as we return (the reference reads its input
                # synchronously): wait for the upload, not the step
                slot["cup"].synchronize()
            self._advance()
            ev = slot["cdone"]
        else:
            compute = torch.cuda.current_stream(self.dev.device)
            if cuda_in:
                x = self._frame_tensor(frame)
            else:
                # upload on the copy stream (overlaps the previous step)
                x = slot["x"]
                with torch.cuda.stream(ring.copy_stream):
                    x.copy_(src, non_blocking=True)
                    slot["up"].record(ring.copy_stream)
                if src is frame:
                    slot["up"].synchronize()   # caller-owned pinned input
                compute.wait_event(slot["up"])
            self._launch_step(x, slot["mask"], slot["stats"])
            stepped = torch.cuda.Event()
            stepped.record(compute)
            with torch.cuda.stream(ring.down_stream):
                ring.down_stream.wait_event(stepped)
                slot["hm"].copy_(slot["mask"], non_blocking=True)
                slot["hs"].copy_(slot["stats"], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(ring.down_stream)
        slot["event"] = ev
        m = LabelMask.pending(slot["hm"], ev, owned=False)
        st = FrameStats.pending(slot["hs"], ev)
        slot["owners"] = (m, st)
        self._last_mask_dev = slot["mask"]
        return m, st

    def _stage(self, frame, out: np.ndarray) -> None:
        """Validate a host frame (cascade.py:263-269) and copy it into the
        pinned staging array."""
        if isinstance(frame, torch.Tensor):
            frame = frame.numpy()
        if isinstance(frame, Frame):
            if (frame.height, frame.width) != (self.height, self.width):
                raise DataError(
                    f"frame {frame.index} geometry {frame.height}x"
                    f"{frame.width} != model {self.height}x{self.width}")
            if frame.depth != self.depth:
                raise DataError(f"frame {frame.index} has {frame.depth} "
                                f"planes, model expects {self.depth}")
            _copy_rows([pl.data for pl in frame.planes], out)
            return
        arr = np.asarray(frame)
        if arr.ndim == 2:
            arr = arr[None]
        if arr.shape[1:] != (self.height, self.width):
            raise DataError(f"frame geometry {arr.shape[1]}x{arr.shape[2]} "
                            f"!= model {self.height}x{self.width}")
        if arr.shape[0] != self.depth:
            raise DataError(f"frame has {arr.shape[0]} planes, model "
                            f"expects {self.depth}")
        if arr.dtype != np.uint8:
            raise DataError("frames must be uint8")
        _copy_rows(list(arr), out)

    def process_frame_device(self, frame: torch.Tensor, mask: torch.Tensor,
                             stats: torch.Tensor) -> None:
        """Device-resident variant: frame (d,H,W) u8 CUDA tensor in, mask
        (H,W) u8 and stats (16,) i64 CUDA tensors out; no host traffic and
        no synchronisation."""
        if self._host is not None:
            self._flush()
        self._launch_step(frame, mask, stats)

    def reorder_levels(self) -> None:
        """Re-sort the middle levels by hits, ties by prior mass; the hit
        window restarts (cascade.py:393-417)."""
        self.materialize()
        self._reorder_pending = True
        self.materialize()

    def clone(self) -> "CascadeEngine":
        self._flush()
        twin = CascadeEngine.__new__(CascadeEngine)
        for k, v in vars(self).items():
            if isinstance(v, np.ndarray):
                setattr(twin, k, v.copy())
            elif k == "dev":
                twin.dev = v.clone()
            else:
                setattr(twin, k, v)
        twin._host = None
        twin._snap = None
        twin._ring = None
        return twin

    # ------------------------------------------------------- inspection

    @property
    def last_kinds(self) -> np.ndarray:
        return self.dev.kind[0].cpu().numpy()

    @property
    def last_confidence(self) -> np.ndarray:
        return self.dev.conf[0].to(torch.float64).cpu().numpy()

    @property
    def sampling_clock(self) -> np.ndarray:
        return self.clock

    def level_order(self, y: int, x: int, channel: int = 0) -> list[int]:
        p = y * self.width + x
        mids = [int(j) for j in self.mid_order[channel, p] if j >= 0]
        return [LEVEL_CHP] + mids + [LEVEL_GMM]

    @property
    def dynamics(self) -> np.ndarray:
        return self.dev.cls[0].cpu().numpy()

    def _weights_col(self, j: int) -> np.ndarray:
        return self._wtab[self.dynamics, j].astype(np.float64)

    wa = property(lambda self: self._weights_col(0))
    wb = property(lambda self: self._weights_col(1))
    wc = property(lambda self: self._weights_col(2))

    @property
    def tables(self) -> np.ndarray:
        return self.dev.table_to_ref(0).cpu().numpy()

    @property
    def group_id(self) -> np.ndarray:
        g = self.dev.gid[0].cpu().numpy().astype(np.int64) & 0xFFFF
        return np.where(g == 0xFFFF, -1, g)

    def state_dict(self) -> dict:
        """All per-pixel state in the reference's dtypes and layouts."""
        return {k: v.copy() for k, v in self._cached().items()}


def _state_property(name):
    def get(self):
        return self._cached()[name]

    def set_(self, value):
        cache = self._cached()
        cache[name][...] = np.asarray(value)
    return property(get, set_)


for _name in _STATE_FIELDS + _GROUP_FIELDS:
    setattr(CascadeEngine, _name, _state_property(_name))


def export_state(dev: DeviceState, s: int, k: int, lib, stream) -> dict:
    """Stream s of ``dev`` in the reference's dtypes and layouts
    (cascade.py:143-158) via ``cog_export_state``; group modes (d, G)."""
    d, P = dev.depth, dev.P
    dv = dev.device
    shapes = {
        "mu": ((d, P, k), torch.float64), "var": ((d, P, k), torch.float64),
        "w": ((d, P, k), torch.float64), "count": ((d, P), torch.int64),
        "mid_order": ((d, P, 3), torch.int8),
        "mode_ref": ((d, P, 2), torch.int8),
        "chp_prev": ((d, P), torch.uint8), "last_label": ((d, P), torch.uint8),
        "last_active": ((d, P), torch.int8), "waking": ((d, P), torch.uint8),
        "streak": ((d, P), torch.int64), "clock": ((d, P), torch.int64),
        "hits": ((d, P, 5), torch.int64)}
    bufs = {n: torch.empty(sh, dtype=t, device=dv)
            for n, (sh, t) in shapes.items()}
    rs = _ref_struct(bufs)
    rc = lib.cog_export_state(_lib.ref(dev.single_geom()),
                              _lib.ref(dev.stream_view(s)), _lib.ref(rs),
                              stream)
    _lib.check(rc, "cog_export_state")
    out = {n: b.cpu().numpy() for n, b in bufs.items()}
    G = dev.n_groups
    out["group_mu"] = dev.g_mu[s, :, :G].cpu().numpy().copy()
    out["group_var"] = dev.g_var[s, :, :G].cpu().numpy().copy()
    return out


def frame_tensor(frame, depth: int, height: int, width: int,
                 device) -> torch.Tensor:
    """(d, H, W) uint8 CUDA tensor from a Frame, array or tensor, checked
    against the model geometry (cascade.py:263-269 -> DataError)."""
    if isinstance(frame, torch.Tensor):
        t = frame if frame.dim() == 3 else frame.unsqueeze(0)
    else:
        if isinstance(frame, Frame):
            arr = frame.stacked()
        else:
            arr = np.asarray(frame)
        if arr.ndim == 2:
            arr = arr[None]
        t = torch.from_numpy(np.ascontiguousarray(arr))
    if tuple(t.shape) != (depth, height, width):
        raise DataError(f"frame shape {tuple(t.shape)} != model "
                        f"{(depth, height, width)}")
    if t.dtype != torch.uint8:
        raise DataError("frames must be uint8")
    return t.to(device, non_blocking=True).contiguous()


def _ref_struct(bufs: dict) -> "_lib.RefState":
    rs = _lib.RefState()
    rs.mu = bufs["mu"].data_ptr()
    rs.var = bufs["var"].data_ptr()
    rs.w = bufs["w"].data_ptr()
    rs.count = bufs["count"].data_ptr()
    rs.mid = bufs["mid_order"].data_ptr()
    rs.ref = bufs["mode_ref"].data_ptr()
    rs.chp = bufs["chp_prev"].data_ptr()
    rs.label = bufs["last_label"].data_ptr()
    rs.active = bufs["last_active"].data_ptr()
    rs.waking = bufs["waking"].data_ptr()
    rs.streak = bufs["streak"].data_ptr()
    rs.clock = bufs["clock"].data_ptr()
    rs.hits = bufs["hits"].data_ptr()
    return rs


def run_sequence(engine: CascadeEngine, frames):
    """Process frames in order, collecting masks and stats
    (cascade.py:433-444).  Masks / stats resolve lazily, so the loop only
    enqueues work."""
    masks, stats = [], []
    for frame in frames:
        mask, row = engine.process_frame(frame)
        if engine.config.majority_filter:
            mask = LabelMask(majority_filter(mask.labels))
        masks.append(mask)
        stats.append(row)
    return masks, stats


def majority_filter(labels: np.ndarray) -> np.ndarray:
    """Optional 3x3 majority vote (cascade.py:447-453; off the hot path)."""
    from scipy.ndimage import uniform_filter
    fg = (labels > 0).astype(np.float64)
    return (uniform_filter(fg, size=3, mode="nearest") > 0.5).astype(
        np.uint8) * 255
