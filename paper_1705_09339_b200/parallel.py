"""Multi-stream and row-band execution of the CoG path.

Two ways the per-pixel work shards, both with all state resident in HBM:

* **Independent streams** (BASELINE C5: 64 streams of 1280x720): a
  ``BatchEngine`` keeps S streams of one geometry in one set of buffers
  (``cog_geom.streams = S``); one ``cog_step`` launch steps all of them and
  every per-stream global (group update, illumination test, statistics)
  stays on the device.  Across GPUs each rank owns ``streams_for_rank`` --
  no collectives.

* **One stream in row bands** (BASELINE C4: one 3840x2160 stream): each
  shard is a ``CascadeEngine`` over rows [r0, r1) of the frame
  (``cog_geom.row0 = r0``, ``total_pixels`` = the whole frame).  Band starts
  are multiples of the sampling stride, so every copy pixel's anchor
  ``(y - y % stride, x - x % stride)`` (kernels_numba.py:363-373) lies in
  the same band and no halo is exchanged.  The two per-frame couplings of
  the reference -- the group update (cascade.py:320-344) and the
  illumination monitor (cascade.py:310-313) -- are whole-frame reductions:
  each shard's step leaves its exact partial sums (integer counts, integer
  intensity sums, 2^-52 fixed-point confidence sums) in ``accum``, a
  reducer sums them across shards (one ~0.5 KB all-reduce), and
  ``cog_finalize`` applies the identical update on every shard.  Because the
  partials are exact integers, the sharded run equals the single-engine run
  bit for bit.

Training shards the same way, except the k-means grouping, which is global:
each shard computes its band's behaviour features on the GPU, the features
are gathered, every shard runs the (deterministic) host clustering on the
whole frame and installs its band's slice of the group map.
"""

from __future__ import annotations

from typing import Callable, Sequence

import numpy as np
import torch

from . import _lib
from .cascade import (CascadeEngine, DeviceState, FrameStats, export_state,
                      frame_tensor, params_from_config, weight_table)
from .config import EngineConfig
from .errors import DataError, TrainingError
from .frame_io import LabelMask
from .grouping import GroupMap, build_groups
from .scene_prior import silverman_bandwidth, stack_training
from .training import install_groups, train_device

Gather = Callable[[np.ndarray, np.ndarray], tuple[np.ndarray, np.ndarray]]


# ----------------------------------------------------------------- bands


def band_rows(height: int, parts: int, stride: int) -> list[tuple[int, int]]:
    """Split ``height`` rows into ``parts`` contiguous bands whose starts are
    multiples of ``stride`` (as equal as the stride blocks allow)."""
    if parts < 1 or stride < 1 or height < 1:
        raise DataError("band_rows: height, parts and stride must be >= 1")
    blocks = -(-height // stride)
    if parts > blocks:
        raise DataError(f"{height} rows (stride {stride}) cannot form "
                        f"{parts} non-empty stride-aligned bands")
    per, extra = divmod(blocks, parts)
    out, b = [], 0
    for i in range(parts):
        nb = per + (1 if i < extra else 0)
        r0, r1 = b * stride, min(height, (b + nb) * stride)
        out.append((r0, r1))
        b += nb
    return out


def streams_for_rank(n_streams: int, rank: int, world: int) -> list[int]:
    """Contiguous block of stream indices owned by ``rank``."""
    per, extra = divmod(n_streams, world)
    start = rank * per + min(rank, extra)
    return list(range(start, start + per + (1 if rank < extra else 0)))


# -------------------------------------------------------------- reducers


class DistReducer:
    """Sums a shard's ``accum`` partials over a torch.distributed group
    (NCCL on the GPU box, gloo in the CPU tests).  The words are u64 bit
    patterns of non-negative sums stored in int64, so a two's-complement
    integer all-reduce is exact."""

    def __init__(self, group=None):
        self.group = group

    def __call__(self, accum: torch.Tensor) -> None:
        import torch.distributed as dist
        if accum.is_cuda and dist.get_backend(self.group) == "gloo":
            # gloo reduces host tensors: stage through the host
            host = accum.cpu()
            dist.all_reduce(host, op=dist.ReduceOp.SUM, group=self.group)
            accum.copy_(host)
            return
        dist.all_reduce(accum, op=dist.ReduceOp.SUM, group=self.group)


class PeerMailbox:
    """One row-band shard's side of the fused cross-shard sum
    (``cog_step_p2p``, include/cog_b200.h ``cog_peers``): every rank's
    mailbox mapped into this process, this rank's index and the step
    sequence number.  With it set as ``engine.peers`` a frame is two kernels
    on every rank -- hot pass, deep pass -- and the deep pass's last CTA
    stores the frame's partials into every peer's mailbox over NVLink, waits
    for theirs and runs the frame tail: no NCCL call, no host
    synchronisation, no extra launch per frame.

    The sequence number is shared by every engine holding this object (an
    engine and its clones), so ranks that issue the same sequence of steps
    -- SPMD -- stay in step."""

    def __init__(self, depth: int, n_groups: int, n_ranks: int, rank: int,
                 ptrs: Sequence[int], keep=None, fused: bool = True,
                 barrier: Callable[[], None] | None = None):
        if not 2 <= n_ranks <= _lib.MAX_RANKS or len(ptrs) != n_ranks:
            raise DataError(f"peer mailbox over {n_ranks} ranks")
        self.n_ranks, self.rank = n_ranks, rank
        self.ptrs = [int(x) for x in ptrs]
        self.keep = keep          # the allocations behind the pointers
        self.fused = fused
        # unfused across processes (ranks sharing a GPU): called between a
        # step's push and its cog_finalize_p2p, after which every rank's
        # push has landed -- so no kernel waits for one that cannot run
        self.barrier = barrier
        self.seq = 0
        self.words = int(_lib.load().cog_mailbox_words(depth, n_groups,
                                                       n_ranks))
        self._c = _lib.Peers()
        self._c.n_ranks, self._c.rank = n_ranks, rank
        for r, ptr in enumerate(self.ptrs):
            self._c.mailbox[r] = ptr

    def next(self) -> "_lib.Peers":
        """The peers struct of the next step."""
        self.seq += 1
        self._c.seq = self.seq
        return self._c

    def current(self) -> "_lib.Peers":
        return self._c

    @staticmethod
    def size(depth: int, n_groups: int, n_ranks: int) -> int:
        n = int(_lib.load().cog_mailbox_words(depth, n_groups, n_ranks))
        if n < 0:
            raise DataError(f"peer mailbox over {n_ranks} ranks")
        return n

    @classmethod
    def local(cls, depth: int, n_groups: int, n_ranks: int,
              device=None) -> list["PeerMailbox"]:
        """All ranks' mailboxes in one process on one GPU (``BandSet``, the
        single-GPU parity tests): the unfused form -- every band's step
        pushes, then every band's ``cog_finalize_p2p`` finds its flags set
        -- so no kernel ever waits on a later one."""
        n = cls.size(depth, n_groups, n_ranks)
        boxes = [torch.zeros(n, dtype=torch.int64, device=device or "cuda")
                 for _ in range(n_ranks)]
        ptrs = [b.data_ptr() for b in boxes]
        return [cls(depth, n_groups, n_ranks, r, ptrs, keep=boxes,
                    fused=False) for r in range(n_ranks)]

    @classmethod
    def symmetric(cls, depth: int, n_groups: int,
                  group=None) -> "PeerMailbox":
        """One rank per GPU: the mailboxes are torch symmetric memory
        (peer-mapped over NVLink), exchanged through the process group."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        group = group if group is not None else dist.group.WORLD
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        n = cls.size(depth, n_groups, world)
        dev = torch.device("cuda", torch.cuda.current_device())
        box = symm.empty(n, dtype=torch.int64, device=dev)
        box.zero_()
        hdl = symm.rendezvous(box, group)
        torch.cuda.synchronize(dev)
        dist.barrier(group)     # every mailbox is zero before any push
        return cls(depth, n_groups, world, rank, list(hdl.buffer_ptrs),
                   keep=(box, hdl), fused=True)


    @classmethod
    def ipc(cls, depth: int, n_groups: int, group=None,
            fused: bool = True) -> "PeerMailbox":
        """The mailboxes as plain device allocations shared through CUDA IPC
        handles (torch's storage sharing), exchanged over the process group.
        ``fused=False`` is for ranks that share one GPU (the two-process
        test): push, host barrier, then ``cog_finalize_p2p``."""
        import torch.distributed as dist
        group = group if group is not None else dist.group.WORLD
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        n = cls.size(depth, n_groups, world)
        dev = torch.device("cuda", torch.cuda.current_device())
        box = torch.zeros(n, dtype=torch.int64, device=dev)
        torch.cuda.synchronize(dev)
        handles = [None] * world
        dist.all_gather_object(handles, box.untyped_storage()._share_cuda_(),
                               group=group)
        keep, ptrs = [box], []
        for r, h in enumerate(handles):
            if r == rank:
                ptrs.append(box.data_ptr())
                continue
            with torch.cuda.device(h[0]):
                st = torch.UntypedStorage._new_shared_cuda(*h)
            peer = torch.empty(0, dtype=torch.int64,
                               device=st.device).set_(st)
            if peer.device != dev:
                peer[:1].to(dev)    # enables peer access dev -> owner
            keep.append(peer)
            ptrs.append(peer.data_ptr())
        dist.barrier(group)

        def barrier():
            torch.cuda.current_stream(dev).synchronize()
            dist.barrier(group)
        return cls(depth, n_groups, world, rank, ptrs, keep=keep, fused=fused,
                   barrier=None if fused else barrier)


def dist_gather_rows(group=None) -> Gather:
    """Gather callable for ``train_band_engine``: all-gathers the per-band
    feature rows of every rank (in rank = band order)."""
    import torch.distributed as dist

    def gather(feats: np.ndarray, w_final: np.ndarray):
        world = dist.get_world_size(group)
        n = torch.tensor([feats.shape[0]], dtype=torch.int64)
        backend = dist.get_backend(group)
        dev = torch.device("cuda", torch.cuda.current_device()) \
            if backend == "nccl" else torch.device("cpu")
        n = n.to(dev)
        sizes = [torch.zeros_like(n) for _ in range(world)]
        dist.all_gather(sizes, n, group=group)
        sizes = [int(s.item()) for s in sizes]
        m = max(sizes)
        buf = torch.zeros((m, 3), dtype=torch.float64, device=dev)
        buf[:feats.shape[0], :2] = torch.from_numpy(feats).to(dev)
        buf[:feats.shape[0], 2] = torch.from_numpy(w_final).to(dev)
        parts = [torch.zeros_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
        full = torch.cat([q[:k] for q, k in zip(parts, sizes)]).cpu().numpy()
        return np.ascontiguousarray(full[:, :2]), np.ascontiguousarray(full[:, 2])
    return gather


def band_group_map(groups: GroupMap, r0: int, r1: int, width: int) -> GroupMap:
    """The band's slice of a whole-frame group map (group parameters are
    global and shared by every band)."""
    return GroupMap(groups.group_id[r0 * width:r1 * width].copy(), groups.mu,
                    groups.var, groups.weight, groups.member_count)


# ------------------------------------------------------ row-band training


def train_band_engine(frames, config: EngineConfig, rows: tuple[int, int],
                      gather: Gather | None = None, device=None,
                      kde_windows=None) -> CascadeEngine:
    """Train the shard of rows [r0, r1) of a stream.

    ``frames``: the whole training sequence (list of Frame or (N, d, H, W)
    uint8) -- only the band's rows go to the device; the whole frames stay
    on the host for the global clustering.  ``gather(feats, w_final)``
    returns the whole frame's features in row order (identity when None,
    i.e. a single band covering the frame)."""
    config.validate()
    arr = stack_training(frames)
    n, d, h, w = arr.shape
    r0, r1 = rows
    if not (0 <= r0 < r1 <= h) or r0 % config.stride:
        raise DataError(f"band rows {rows} must be stride-aligned inside "
                        f"0..{h}")
    bw = silverman_bandwidth(arr) if config.kde_auto_bandwidth \
        else float(config.kde_bandwidth)
    eng = CascadeEngine(config, r1 - r0, w, d, device=device, row0=r0,
                        total_pixels=h * w)
    band = np.ascontiguousarray(arr[:, :, r0:r1, :].reshape(n, d, -1))
    values = torch.from_numpy(band).to(eng.dev.device)
    eng.prior, feats, w_final = train_device(eng, values, config, bw,
                                             kde_windows)
    flat = np.ascontiguousarray(arr.reshape(n, d, h * w))
    if config.grouping:
        f_loc, w_loc = feats.cpu().numpy(), w_final.cpu().numpy()
        f_all, w_all = gather(f_loc, w_loc) if gather else (f_loc, w_loc)
        if f_all.shape[0] != h * w:
            raise TrainingError(f"gathered features cover {f_all.shape[0]} "
                                f"pixels, frame has {h * w}")
        groups = build_groups(f_all, w_all, flat, config)
    else:
        groups = GroupMap.empty(h * w, d)
    install_groups(eng, band_group_map(groups, r0, r1, w))
    lib = _lib.load()
    rc = lib.cog_set_levels(_lib.ref(eng.dev.geom), _lib.ref(eng.dev.cstate),
                            torch.cuda.current_stream(eng.dev.device).cuda_stream)
    _lib.check(rc, "cog_set_levels")
    eng.bandwidth = bw
    eng.sample_count = n
    return eng


class BandSet:
    """All row bands of one stream in one process -- the single-GPU form of
    the row-band decomposition (used by the parity tests and to run C4 on
    fewer GPUs than bands).  Per frame: every band's step with the frame
    tail deferred, one device-side sum of the partials, every band's
    ``cog_finalize``.  No shard waits on another inside a kernel."""

    def __init__(self, engines: Sequence[CascadeEngine]):
        self.engines = list(engines)
        if not self.engines:
            raise DataError("BandSet needs at least one band")
        # set by use_mailboxes(): the bands sum their partials through peer
        # mailboxes (the multi-GPU data path, unfused) instead of torch ops
        self.mailboxes = None
        e0 = self.engines[0]
        self.width, self.depth = e0.width, e0.depth
        self.height = sum(e.height for e in self.engines)
        self.rows = [(e.row0, e.row0 + e.height) for e in self.engines]

    @classmethod
    def train(cls, frames, config: EngineConfig, parts: int, device=None,
              kde_windows=None) -> "BandSet":
        arr = stack_training(frames)
        rows = band_rows(arr.shape[2], parts, config.stride)
        # features of every band are needed before any band can cluster:
        # train the device phase of all bands first, cluster once
        engines = []
        n, d, h, w = arr.shape
        bw = silverman_bandwidth(arr) if config.kde_auto_bandwidth \
            else float(config.kde_bandwidth)
        feats, wfin = [], []
        for r0, r1 in rows:
            eng = CascadeEngine(config, r1 - r0, w, d, device=device,
                                row0=r0, total_pixels=h * w)
            band = np.ascontiguousarray(arr[:, :, r0:r1, :].reshape(n, d, -1))
            values = torch.from_numpy(band).to(eng.dev.device)
            eng.prior, f, wf = train_device(eng, values, config, bw,
                                            kde_windows)
            if config.grouping:
                feats.append(f.cpu().numpy())
                wfin.append(wf.cpu().numpy())
            eng.bandwidth = bw
            eng.sample_count = n
            engines.append(eng)
        flat = np.ascontiguousarray(arr.reshape(n, d, h * w))
        groups = (build_groups(np.concatenate(feats), np.concatenate(wfin),
                               flat, config)
                  if config.grouping else GroupMap.empty(h * w, d))
        lib = _lib.load()
        for eng, (r0, r1) in zip(engines, rows):
            install_groups(eng, band_group_map(groups, r0, r1, w))
            rc = lib.cog_set_levels(
                _lib.ref(eng.dev.geom), _lib.ref(eng.dev.cstate),
                torch.cuda.current_stream(eng.dev.device).cuda_stream)
            _lib.check(rc, "cog_set_levels")
        return cls(engines)

    def use_mailboxes(self) -> None:
        """Sum the bands' partials the way ranks on several GPUs do
        (``PeerMailbox``): each band's step pushes into every band's
        mailbox, each band's ``cog_finalize_p2p`` sums its own."""
        if len(self.engines) < 2:
            raise DataError("mailboxes need at least two bands")
        e0 = self.engines[0]
        self.mailboxes = PeerMailbox.local(e0.depth, e0.dev.n_groups,
                                           len(self.engines), e0.dev.device)

    def _frame_p2p(self, frame, mask, stats) -> None:
        bands = []
        for eng, box, (r0, r1) in zip(self.engines, self.mailboxes, self.rows):
            eng._flush()
            st = torch.empty(16, dtype=torch.int64, device=stats.device)
            x = frame[:, r0:r1].contiguous()
            geom, prm, cst = (_lib.ref(eng.dev.geom), _lib.ref(eng._params()),
                              _lib.ref(eng.dev.cstate))
            rc = eng.lib.cog_step_p2p(
                geom, prm, cst, x.data_ptr(), mask[r0:r1].data_ptr(),
                eng.dev.conf.data_ptr(), eng.dev.kind.data_ptr(),
                st.data_ptr(), eng.frame_count, int(eng._reorder_pending), 0,
                _lib.ref(box.next()), eng.stream)
            _lib.check(rc, "cog_step_p2p")
            bands.append((eng, box, geom, prm, cst, x))
        for eng, box, geom, prm, cst, x in bands:
            rc = eng.lib.cog_finalize_p2p(geom, prm, cst, stats.data_ptr(),
                                          eng.frame_count,
                                          _lib.ref(box.current()), eng.stream)
            _lib.check(rc, "cog_finalize_p2p")
            eng._advance()

    def process_frame_device(self, frame: torch.Tensor, mask: torch.Tensor,
                             stats: torch.Tensor) -> None:
        """frame (d, H, W) u8, mask (H, W) u8, stats (16,) i64 -- CUDA."""
        if self.mailboxes is not None:
            return self._frame_p2p(frame, mask, stats)
        bands = []
        for eng, (r0, r1) in zip(self.engines, self.rows):
            eng._flush()
            st = torch.empty(16, dtype=torch.int64, device=stats.device)
            x = frame[:, r0:r1].contiguous()
            m = mask[r0:r1]
            geom, prm, cst = (_lib.ref(eng.dev.geom), _lib.ref(eng._params()),
                              _lib.ref(eng.dev.cstate))
            rc = eng.lib.cog_step(
                geom, prm, cst, x.data_ptr(), m.data_ptr(),
                eng.dev.conf.data_ptr(), eng.dev.kind.data_ptr(),
                st.data_ptr(), eng.frame_count, int(eng._reorder_pending), 0,
                eng.stream)
            _lib.check(rc, "cog_step")
            bands.append((eng, geom, prm, cst, x))
        total = torch.stack([e.dev.accum for e in self.engines]).sum(dim=0)
        for eng, geom, prm, cst, x in bands:
            eng.dev.accum.copy_(total)
            rc = eng.lib.cog_finalize(geom, prm, cst, stats.data_ptr(),
                                      eng.frame_count, eng.stream)
            _lib.check(rc, "cog_finalize")
            eng._reorder_pending = False
            cfg = eng.config
            eng.frame_count += 1
            if (not cfg.compat and cfg.reorder_interval > 0
                    and eng.frame_count % cfg.reorder_interval == 0):
                eng._reorder_pending = True

    def process_frame(self, frame) -> tuple[LabelMask, FrameStats]:
        dev = self.engines[0].dev.device
        x = frame_tensor(frame, self.depth, self.height, self.width, dev)
        mask = torch.empty((self.height, self.width), dtype=torch.uint8,
                           device=dev)
        stats = torch.empty(16, dtype=torch.int64, device=dev)
        self.process_frame_device(x, mask, stats)
        return LabelMask(mask.cpu().numpy()), FrameStats(*stats.cpu().tolist()[:10])

    def state(self, name: str) -> np.ndarray:
        """A whole-frame state array assembled from the bands (reference
        layout: pixel axis = rows of every band in order)."""
        parts = [getattr(e, name) for e in self.engines]
        if name in ("group_mu", "group_var"):
            return parts[0]
        return np.concatenate(parts, axis=1)


# --------------------------------------------------------- batch engine


class BatchResult:
    """Masks (S, H, W) u8 and statistics rows (S, 10) i64 of one batch
    step, downloaded asynchronously into a pinned slot of the engine's ring;
    ``masks`` / ``stats`` block on the download.  The first read copies the
    result out of the slot into arrays the result owns (the slot is reused
    three submissions later), so arrays a caller already holds are never
    overwritten by later frames."""

    def __init__(self, slot: dict) -> None:
        self._slot = slot
        self._own = None

    def _wait(self):
        if self._own is None:
            slot = self._slot
            slot["down"].synchronize()
            self._own = (slot["hm"].numpy().copy(),
                         slot["hs"].numpy()[:, :10].copy())
            if slot.get("owner") is self:
                slot["owner"] = None
            self._slot = None
        return self._own

    def detach(self) -> None:
        """Copy out of the slot (called before the slot is reused)."""
        self._wait()

    @property
    def masks(self) -> np.ndarray:
        return self._wait()[0]

    @property
    def stats(self) -> np.ndarray:
        return self._wait()[1]


class BatchEngine:
    """S independent streams of one geometry in one set of HBM buffers;
    one launch steps every stream (no collectives, per-stream globals on
    the device)."""

    def __init__(self, config: EngineConfig, height: int, width: int,
                 depth: int, streams: int, device=None):
        config.validate()
        self.config = config
        self.height, self.width, self.depth = height, width, depth
        self.streams = streams
        self.n_pix = height * width
        self.lib = _lib.load()
        self.dev = DeviceState(config, height, width, depth, streams=streams,
                               device=device)
        self._wtab = weight_table(config)
        self.frame_count = 0
        self._reorder_pending = False
        self.group_w: list[np.ndarray] = [np.zeros(0)] * streams

    @property
    def stream(self) -> int:
        return torch.cuda.current_stream(self.dev.device).cuda_stream

    def _params(self):
        q = params_from_config(self.config, self._wtab)
        q.variant = _lib.VARIANTS[getattr(self, "kernel_variant", "auto")]
        return q

    @classmethod
    def train(cls, frames_per_stream: Sequence, config: EngineConfig,
              device=None, kde_windows=None) -> "BatchEngine":
        """frames_per_stream[s]: training frames of stream s (list of Frame
        or (N, d, H, W) uint8)."""
        first = stack_training(frames_per_stream[0])
        n, d, h, w = first.shape
        S = len(frames_per_stream)
        eng = cls(config, h, w, d, S, device=device)
        proxy = CascadeEngine.__new__(CascadeEngine)  # param/geom carrier
        proxy.config, proxy.dev, proxy._wtab = config, eng.dev, eng._wtab
        proxy.exact_group_sums = False
        proxy.kernel_variant = "auto"
        maps = []
        for s in range(S):
            arr = first if s == 0 else stack_training(frames_per_stream[s])
            if arr.shape[1:] != (d, h, w):
                raise DataError(f"stream {s} geometry {arr.shape[1:]} != "
                                f"{(d, h, w)}")
            bw = silverman_bandwidth(arr) if config.kde_auto_bandwidth \
                else float(config.kde_bandwidth)
            flat = np.ascontiguousarray(arr.reshape(arr.shape[0], d, h * w))
            values = torch.from_numpy(flat).to(eng.dev.device)
            _, feats, wf = train_device(proxy, values, config, bw,
                                        kde_windows, stream=s)
            maps.append(build_groups(feats, wf, flat, config,
                                     values_dev=values)
                        if config.grouping else GroupMap.empty(h * w, d))
            del values
        g = max(m.group_count for m in maps)
        eng.dev.set_groups(g)
        for s, m in enumerate(maps):
            proxy.group_w = np.zeros(0)
            install_groups(proxy, m, stream=s, resize=False)
            eng.group_w[s] = m.weight.copy()
        rc = eng.lib.cog_set_levels(_lib.ref(eng.dev.geom),
                                    _lib.ref(eng.dev.cstate), eng.stream)
        _lib.check(rc, "cog_set_levels")
        return eng

    def process_frames_device(self, frames: torch.Tensor, masks: torch.Tensor,
                              stats: torch.Tensor) -> None:
        """frames (S, d, H, W) u8, masks (S, H, W) u8, stats (S, 16) i64."""
        if tuple(frames.shape) != (self.streams, self.depth, self.height,
                                   self.width) or frames.dtype != torch.uint8:
            raise DataError(f"frames must be ({self.streams}, {self.depth}, "
                            f"{self.height}, {self.width}) uint8")
        rc = self.lib.cog_step(
            _lib.ref(self.dev.geom), _lib.ref(self._params()),
            _lib.ref(self.dev.cstate), frames.data_ptr(), masks.data_ptr(),
            self.dev.conf.data_ptr(), self.dev.kind.data_ptr(),
            stats.data_ptr(), self.frame_count, int(self._reorder_pending), 1,
            self.stream)
        _lib.check(rc, "cog_step")
        self._reorder_pending = False
        self.frame_count += 1
        cfg = self.config
        if (not cfg.compat and cfg.reorder_interval > 0
                and self.frame_count % cfg.reorder_interval == 0):
            self._reorder_pending = True

    def process_frames(self, frames) -> tuple[np.ndarray, np.ndarray]:
        """frames (S, d, H, W) uint8 (host or CUDA) -> masks (S, H, W) u8,
        stats (S, 10) int64 rows (FrameStats layout)."""
        if isinstance(frames, torch.Tensor) and frames.is_cuda:
            x = frames.contiguous()
            masks = torch.empty((self.streams, self.height, self.width),
                                dtype=torch.uint8, device=self.dev.device)
            stats = torch.empty((self.streams, 16), dtype=torch.int64,
                                device=self.dev.device)
            self.process_frames_device(x, masks, stats)
            return masks.cpu().numpy(), stats[:, :10].cpu().numpy()
        res = self.submit_frames(frames)
        return res.masks.copy(), res.stats.copy()

    def submit_frames(self, frames) -> BatchResult:
        """Host frames (S, d, H, W) uint8 -- a pinned tensor is DMA'd as is,
        anything else is staged into the slot's pinned buffer -- through a
        ring of three slots: upload on a copy stream (overlapping the
        previous step), step on the engine's stream, download of masks and
        statistics on the copy stream.  Returns at once."""
        dev = self.dev.device
        if getattr(self, "_ring", None) is None:
            S, d, H, W = self.streams, self.depth, self.height, self.width
            self._copy = torch.cuda.Stream(device=dev)
            self._ring = [{
                "in": torch.empty((S, d, H, W), dtype=torch.uint8,
                                  pin_memory=True),
                "x": torch.empty((S, d, H, W), dtype=torch.uint8, device=dev),
                "m": torch.empty((S, H, W), dtype=torch.uint8, device=dev),
                "s": torch.empty((S, 16), dtype=torch.int64, device=dev),
                "hm": torch.empty((S, H, W), dtype=torch.uint8,
                                  pin_memory=True),
                "hs": torch.empty((S, 16), dtype=torch.int64,
                                  pin_memory=True),
                "up": torch.cuda.Event(), "step": torch.cuda.Event(),
                "down": torch.cuda.Event(), "owner": None, "used": False,
            } for _ in range(3)]
            self._next = 0
        slot = self._ring[self._next]
        self._next = (self._next + 1) % len(self._ring)
        if slot["owner"] is not None:
            slot["owner"].detach()     # keep the old result valid
            slot["owner"] = None
        if slot["used"]:
            slot["down"].synchronize()  # pinned in/out buffers free again
        shape = (self.streams, self.depth, self.height, self.width)
        if (isinstance(frames, torch.Tensor) and not frames.is_cuda
                and frames.is_pinned() and frames.dtype == torch.uint8
                and frames.is_contiguous() and tuple(frames.shape) == shape):
            src = frames
        else:
            arr = np.asarray(frames.numpy() if isinstance(frames, torch.Tensor)
                             else frames)
            if arr.shape != shape or arr.dtype != np.uint8:
                raise DataError(f"frames must be {shape} uint8")
            np.copyto(slot["in"].numpy(), arr)
            src = slot["in"]
        compute = torch.cuda.current_stream(dev)
        with torch.cuda.stream(self._copy):
            if slot["used"]:
                self._copy.wait_event(slot["step"])  # device input reusable
            slot["x"].copy_(src, non_blocking=True)
            slot["up"].record(self._copy)
        if src is frames:
            slot["up"].synchronize()   # caller-owned pinned input: reusable
        compute.wait_event(slot["up"])
        self.process_frames_device(slot["x"], slot["m"], slot["s"])
        slot["step"].record(compute)
        with torch.cuda.stream(self._copy):
            self._copy.wait_event(slot["step"])
            slot["hm"].copy_(slot["m"], non_blocking=True)
            slot["hs"].copy_(slot["s"], non_blocking=True)
            slot["down"].record(self._copy)
        slot["used"] = True
        slot["src"] = src              # the DMA source stays alive
        res = BatchResult(slot)
        slot["owner"] = res
        return res

    def export_stream(self, s: int) -> dict:
        """Reference-layout state of stream s (after materialising any
        pending reset / reorder of every stream)."""
        rc = self.lib.cog_apply_pending(
            _lib.ref(self.dev.geom), _lib.ref(self._params()),
            _lib.ref(self.dev.cstate), int(self._reorder_pending), self.stream)
        _lib.check(rc, "cog_apply_pending")
        self._reorder_pending = False
        return export_state(self.dev, s, self.config.k_max, self.lib,
                            self.stream)
