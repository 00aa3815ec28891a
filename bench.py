"""Benchmark of the CoG hot path (BASELINE.json metric: pixel-frames/s of
classify+update, and % of HBM roofline at 1/2/4/8 B200).

Workload (default, N=1): BASELINE config C4 -- one 3840x2160 RGB stream,
K=5, trained on the first 150 frames of the seeded synthetic scene
(paper_1705_09339_b200.synth), the largest configuration a single GPU
holds.  A step is one frame through the step kernels.  At N>1 the 4K frame
is split into N stride-aligned row bands, one per rank, with the frame's
exact partials summed over peer mailboxes inside the step's tail (or, when
those cannot be mapped, by one NCCL all-reduce) per frame (strong scaling:
the ranks share each frame).
Other workloads (--workload): c3 (1920x1080, one stream per rank), c2
(640x480, one stream per rank), c5 (64 independent 1280x720 streams split
over the ranks, processed in waves of --streams resident streams).

``--gpus N`` without a torchrun environment re-launches this script under
``torch.distributed.run`` with N ranks (one per GPU).

value    device-resident frames, CUDA events around each step's launches on
         the engine stream, L2 flushed (256 MiB write, untimed) between
         steps; MAX over ranks of the summed step time.
e2e      the public API ``process_frame`` (c5: ``submit_frames``) fed frames
         from pinned host memory: H2D, step, D2H of mask + stats inside the
         timed region, results read two frames behind the submission.
         extra.e2e_pageable: the same with pageable numpy frames, as a
         reference caller passes them (+ the staging copy).
roofline the fused frame step (fast_kernel + deep_kernel): SURVEY.md 8(d)
         algorithmic bytes of each timed frame (B_frame from that frame's
         own level populations) / step time; when the committed ncu
         capture of the same workload (profiles/traffic_<workload>.json)
         shows fewer DRAM bytes than B_frame, the fraction uses those.
cpu_baseline  the oracle (C restatement of the reference's serial numba
         kernels, 1 thread) on a bounded sample of the same stream, seeded
         with the GPU engine's trained state (c4: a 270-row band).

--impl reference: the reference's CPU path (the oracle port, all host
threads) on the same workload; rank 0 only (c4: a 270-row band, trained by
the oracle itself).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM = 6650.0
METRIC = "pixel-frames/sec (CoG classify+update)"
C5_STREAMS = 64
BAND_ROWS = 270       # c4 CPU samples: rows 0-269 (1/8 of the 4K frame)


def hbm_peak():
    try:
        v = json.loads(PEAKS.read_text())["hbm_gbs"]
        return float(v), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def byte_model(row, depth, k):
    """SURVEY.md 8(d) algorithmic HBM bytes of one frame from its level
    populations (FrameStats row: frame, chp, group, mean, meanvar, gmm,
    skipped, ...):
      B = sum_level n_level * (R(K) + W_level(K)) + n_skipped * 12 + 3 * P
      R(K) = 57 + 12K             full record read of an evaluated plane-pixel
      W_chp = W_group = 13        chp_prev, flags, streak, u16 hit, conf, kind
      W_mean = 17                 + one mu
      W_meanvar = W_gmm = 16 + 12K   full mixture + count + refs
      3 * P                       class + group id read, mask write"""
    _, n_chp, n_group, n_mean, n_meanvar, n_gmm, n_skip = (int(x) for x in row[:7])
    pixels = (n_chp + n_group + n_mean + n_meanvar + n_gmm + n_skip) // depth
    r = 57 + 12 * k
    return ((n_chp + n_group) * (r + 13) + n_mean * (r + 17)
            + (n_meanvar + n_gmm) * (r + 16 + 12 * k) + n_skip * 12
            + 3 * pixels)


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) during the timed region."""

    def __init__(self, index=0, period=0.02):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(
                self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass
        self.period = period
        self._stop = threading.Event()

    def _poll(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(
                nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(
                nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
        }
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(
                self.h, nv.NVML_CLOCK_SM))
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for k, bit in names.items():
                if r & bit:
                    self.reasons.add(k)
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._poll()
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.ok:
            self.t.join()
            self._poll()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(n: int) -> int:
    """Re-run this command under torch.distributed.run with n ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def oracle_from_engine(eng, cfg, threads, p0=0, p1=None):
    """An oracle engine holding pixels [p0, p1) of the GPU engine's state
    (whole rows), exactly as exported in the reference's layouts."""
    from oracle import oracle as orc
    p1 = eng.n_pix if p1 is None else p1
    rows = (p1 - p0) // eng.width
    oe = orc.OracleEngine(cfg, rows, eng.width, eng.depth)
    oe.threads = threads
    st = eng.state_dict()
    for k, v in st.items():
        if k in ("group_mu", "group_var"):
            setattr(oe, k, np.array(v))
        else:
            setattr(oe, k, np.ascontiguousarray(v[:, p0:p1]))
    oe.tables = np.ascontiguousarray(
        eng.dev.table[0][:, p0:p1].cpu().numpy())
    oe.finalize_tables()
    oe.dynamics = eng.dynamics[p0:p1]
    wt = np.array([cfg.weights_static, cfg.weights_oscillating,
                   cfg.weights_dynamic])[oe.dynamics]
    oe.wa, oe.wb, oe.wc = (np.ascontiguousarray(wt[:, i]) for i in range(3))
    oe.group_id = np.ascontiguousarray(eng.group_id[p0:p1])
    oe.group_w = eng.group_w.copy()
    oe.group_members = eng.group_members.copy()
    return oe


def oracle_from_batch(beng, s, cfg, threads):
    """An oracle engine holding stream s of a batch engine's state."""
    from oracle import oracle as orc
    oe = orc.OracleEngine(cfg, beng.height, beng.width, beng.depth)
    oe.threads = threads
    for k, v in beng.export_stream(s).items():
        setattr(oe, k, np.ascontiguousarray(v))
    dev = beng.dev
    oe.tables = np.ascontiguousarray(dev.table[s].cpu().numpy())
    oe.finalize_tables()
    oe.dynamics = dev.cls[s].cpu().numpy()
    wt = np.array([cfg.weights_static, cfg.weights_oscillating,
                   cfg.weights_dynamic])[oe.dynamics]
    oe.wa, oe.wb, oe.wc = (np.ascontiguousarray(wt[:, i]) for i in range(3))
    g = dev.gid[s].cpu().numpy().astype(np.int64) & 0xFFFF
    oe.group_id = np.where(g == 0xFFFF, -1, g)
    G = dev.n_groups
    gw = np.zeros(G)
    gw[:len(beng.group_w[s])] = beng.group_w[s]
    oe.group_w = gw
    oe.group_members = dev.g_members[s, :G].cpu().numpy().astype(np.int64)
    oe.frame_count = beng.frame_count
    return oe


def cpu_baseline(frames, eng, cfg, rows, seconds, min_frames, stream=None):
    """The oracle (1 thread: the reference's kernels are serial) seeded with
    the GPU engine's trained state, timed over a bounded sample of the same
    stream's post-training frames: at least `min_frames` frames and
    `seconds` of CPU work (cycled if the host set is shorter)."""
    os.environ["COG_ORACLE_THREADS"] = "1"
    r0, r1 = rows
    if stream is None:
        oe = oracle_from_engine(eng, cfg, 1, r0 * eng.width, r1 * eng.width)
        band = [np.ascontiguousarray(f[:, r0:r1]) for f in frames]
    else:   # one stream of a batch engine, frames (T, S, d, H, W)
        oe = oracle_from_batch(eng, stream, cfg, 1)
        band = [np.ascontiguousarray(f[stream]) for f in frames]
    oe.process(band[0])  # warm
    t0 = time.perf_counter()
    done, dt = 0, 0.0
    while done < min_frames or dt < seconds:
        oe.process(band[1 + done % (len(band) - 1)])
        done += 1
        dt = time.perf_counter() - t0
    return oe.n_pix * done / dt, dt, done


REF_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                       "oracle", "_ref")


def real_reference_available():
    """The unmodified reference package installed under oracle/_ref by
    __graft_entry__.build() (git-ignored; it travels with the snapshot),
    plus numba for its default backend."""
    if not os.path.isdir(os.path.join(REF_DIR, "cogbg")):
        return False
    try:
        import numba  # noqa: F401
    except ImportError:
        return False
    return True


_REF_BARRIER = None


def _ref_init(barrier):
    global _REF_BARRIER
    _REF_BARRIER = barrier


def _ref_worker(job):
    """One host process of the real-reference arm: the reference's own
    train_engine / process_frame (cogbg, numba backend) on one row band."""
    train, run, k_max, warmup = job
    barrier = _REF_BARRIER
    sys.path.insert(0, REF_DIR)
    from cogbg.config import EngineConfig as RefConfig
    from cogbg.frame_io import Frame, FramePlane
    from cogbg.training import train_engine as ref_train

    def frames_of(arr, base):
        return [Frame(index=base + i,
                      planes=[FramePlane(c, arr[i, c])
                              for c in range(arr.shape[1])])
                for i in range(arr.shape[0])]
    cfg = RefConfig(k_max=k_max, color=True, training_frames=train.shape[0])
    t0 = time.perf_counter()
    eng = ref_train(frames_of(train, 0), cfg)
    t_train = time.perf_counter() - t0
    fr = frames_of(run, train.shape[0])
    for f in fr[:warmup]:
        eng.process_frame(f)          # includes the numba compile
    barrier.wait()
    t0 = time.perf_counter()
    for f in fr[warmup:]:
        eng.process_frame(f)
    dt = time.perf_counter() - t0
    return dt, t_train, eng.n_pix


def run_real_reference(args, world):
    """--impl reference with the REAL reference (oracle/_ref/cogbg): its
    numba kernels are serial, so every host core runs its own engine on a
    disjoint band of rows of the same frames (as a user of the reference
    would spread a stream over processes); value = all bands' pixel-frames
    over the slowest band's time."""
    import multiprocessing as mp
    from paper_1705_09339_b200 import synth
    cid = {"c2": 2, "c3": 3, "c4": 4, "c5": 5}[args.workload]
    spec = synth.CONFIGS[cid].for_stream(0)
    cores = len(os.sched_getaffinity(0))
    n_train = spec.training
    gen = max(1, min(16, cores))
    scene = synth.Scene(spec)
    train = scene.frames(0, n_train, gen)
    run = scene.frames(n_train, n_train + args.warmup + args.steps, gen)
    # bounded sample: rows_per even rows per core (stride-aligned bands)
    rows_per = max(2, min(16, (spec.height // cores) & ~1))
    nb = min(cores, spec.height // rows_per)
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(nb)
    jobs = [(np.ascontiguousarray(train[:, :, b * rows_per:(b + 1) * rows_per]),
             np.ascontiguousarray(run[:, :, b * rows_per:(b + 1) * rows_per]),
             spec.k_max, args.warmup) for b in range(nb)]
    with ctx.Pool(nb, initializer=_ref_init, initargs=(barrier,)) as pool:
        res = pool.map(_ref_worker, jobs, chunksize=1)
    total = max(r[0] for r in res)
    pix = sum(r[2] for r in res)
    value = pix * args.steps / total
    band = (f" (rows 0-{nb * rows_per - 1} of the {spec.width}x{spec.height} "
            f"frame, {nb} bands of {rows_per} rows)")
    line = {
        "metric": METRIC, "value": value, "unit": "pixel-frames/s",
        "impl": "reference", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if cid == 4 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded BASELINE generator)",
        "config": {"workload": f"{args.workload.upper()} "
                               f"{spec.width}x{spec.height}x3 K={spec.k_max} "
                               f"N={n_train}{band}",
                   "frames": f"post-training frames {n_train}.."},
        "cpu_baseline": {"value": value, "unit": "pixel-frames/s",
                         "cores": nb, "kind": "reference",
                         "sample": f"{args.steps} frames after {args.warmup} "
                                   f"warm-up frames{band}; the unmodified "
                                   f"reference (cogbg, numba backend), one "
                                   f"process per core; its own training "
                                   f"{max(r[1] for r in res):.1f}s excluded"},
        "e2e": {"value": value, "unit": "pixel-frames/s",
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_reference(args):
    """--impl reference: the reference's CPU path on the same workload; rank
    0 only.  The real reference (oracle/_ref, see run_real_reference) when it
    is installed; else the oracle port of its numba kernels on all host
    threads.  c4 runs a band of the 4K frame: the full frame needs ~100 GB
    of host RAM in the reference's layout."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return 0
    if real_reference_available() and not args.port:
        return run_real_reference(args, world)
    from oracle import oracle as orc
    from paper_1705_09339_b200 import synth
    from paper_1705_09339_b200.config import EngineConfig
    cid = {"c2": 2, "c3": 3, "c4": 4, "c5": 5}[args.workload]
    spec = synth.CONFIGS[cid].for_stream(0)
    cores = len(os.sched_getaffinity(0))
    os.environ["COG_ORACLE_THREADS"] = str(cores)
    scene = synth.Scene(spec)
    n_train = spec.training
    workers = max(1, min(16, cores))
    train = scene.frames(0, n_train, workers)
    run = scene.frames(n_train, n_train + args.warmup + args.steps, workers)
    band = ""
    if cid == 4:
        train = np.ascontiguousarray(train[:, :, :BAND_ROWS])
        run = np.ascontiguousarray(run[:, :, :BAND_ROWS])
        band = f" (rows 0-{BAND_ROWS - 1} of the 4K frame)"
    cfg = EngineConfig(k_max=spec.k_max, color=True,
                       training_frames=n_train).validate()
    t0 = time.perf_counter()
    eng = orc.train(train, cfg)
    t_train = time.perf_counter() - t0
    eng.threads = cores
    for f in run[:args.warmup]:
        eng.process(f)
    times = []
    for f in run[args.warmup:]:
        t = time.perf_counter()
        eng.process(f)
        times.append(time.perf_counter() - t)
    total = sum(times)
    value = eng.n_pix * args.steps / total
    line = {
        "metric": METRIC, "value": value, "unit": "pixel-frames/s",
        "impl": "reference", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if cid == 4 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded BASELINE generator)",
        "config": {"workload": f"{args.workload.upper()} "
                               f"{spec.width}x{spec.height}x3 K={spec.k_max} "
                               f"N={n_train}{band}",
                   "frames": f"post-training frames {n_train}.."},
        "cpu_baseline": {"value": value, "unit": "pixel-frames/s",
                         "cores": cores, "kind": "port",
                         "sample": f"{args.steps} frames after {args.warmup} "
                                   f"warm-up frames{band}; oracle C kernels "
                                   f"(restatement of the reference's numba "
                                   f"kernels, pixels split over {cores} "
                                   f"threads); training {t_train:.1f}s "
                                   f"excluded"},
        "e2e": {"value": value, "unit": "pixel-frames/s",
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def attach_band_reduce(eng, mode):
    """How a C4 row-band rank sums the frame partials with its peers: the
    one-shot all-reduce over peer mailboxes fused into the step's tail
    (PeerMailbox over torch symmetric memory, else over CUDA IPC handles) --
    adopted only if every rank could map the mailboxes AND two trial frames
    on a clone give, on every rank, exactly the statistics the NCCL path
    gives -- else one NCCL all-reduce per frame.  Returns the description."""
    import torch
    import torch.distributed as dist
    from paper_1705_09339_b200.parallel import DistReducer, PeerMailbox
    dev = eng.dev.device
    nccl = "one NCCL all-reduce of the frame partials per frame"

    def agreed(ok):
        t = torch.tensor([int(ok)], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return bool(t.item())

    def trial(twin, frames):
        stats = torch.zeros((len(frames), 16), dtype=torch.int64, device=dev)
        mask = torch.empty((eng.height, eng.width), dtype=torch.uint8,
                           device=dev)
        for i, f in enumerate(frames):
            twin.process_frame_device(f, mask, stats[i])
        torch.cuda.synchronize(dev)
        return stats

    if mode != "nccl":
        g = torch.Generator(device="cpu").manual_seed(1234)
        frames = [torch.randint(0, 256, (eng.depth, eng.height, eng.width),
                                dtype=torch.uint8, generator=g).to(dev)
                  for _ in range(2)]
        ref = eng.clone()
        ref.reducer = DistReducer()
        want = trial(ref, frames)
        del ref
        for name, make in (("torch symmetric memory", PeerMailbox.symmetric),
                           ("CUDA IPC", PeerMailbox.ipc)):
            box = None
            try:
                box = make(eng.depth, eng.dev.n_groups)
            except Exception as exc:   # noqa: BLE001 - any failure = fallback
                print(f"[bench] peer mailboxes over {name} unavailable: "
                      f"{type(exc).__name__}: {exc}", file=sys.stderr)
            if not agreed(box is not None):
                continue
            twin = eng.clone()
            twin.peers = box
            got = trial(twin, frames)
            del twin
            if agreed(bool((got == want).all())):
                eng.peers = box
                return (f"one-shot all-reduce of the frame partials over "
                        f"peer mailboxes ({name}), fused into the step's "
                        f"last CTA: no collective call, no extra launch")
            print(f"[bench] peer mailboxes over {name}: trial frames differ "
                  f"from the NCCL path, not used", file=sys.stderr)
    eng.reducer = DistReducer()
    return nccl


class Workload:
    """One bench workload on this rank: a trained engine plus its frames.

    c4 (default): one 3840x2160x3 stream; at N>1 one stride-aligned row band
        per rank, partials all-reduced over NCCL each frame.
    c3 / c2: one stream per rank (seed offset by rank), no collectives.
    c5: independent 1280x720x3 streams (K=5); this rank's 64 / N streams in
        waves of `--streams` resident streams (one batch engine per wave).
    """

    def __init__(self, name, args, world, rank, streams=None):
        import torch
        from paper_1705_09339_b200 import synth
        from paper_1705_09339_b200.config import EngineConfig
        from paper_1705_09339_b200.training import train_engine
        self.name = name
        cid = {"c2": 2, "c3": 3, "c4": 4, "c5": 5}[name]
        base = synth.CONFIGS[cid]
        workers = max(1, min(16, len(os.sched_getaffinity(0))))
        total_steps = args.warmup + args.steps
        self.total_steps = total_steps
        n_host = total_steps + 1
        t0 = time.perf_counter()
        self.cfg = EngineConfig(k_max=base.k_max, color=True,
                                training_frames=base.training,
                                state_dtype=args.state).validate()
        if name in ("c2", "c3"):
            spec = base.for_stream(rank)
            sc = synth.Scene(spec)
            train = sc.frames(0, spec.training, workers)
            self.t_gen = time.perf_counter() - t0
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            self.eng = train_engine(train, self.cfg)
            torch.cuda.synchronize()
            self.t_train = time.perf_counter() - t0
            self.host = sc.frames(spec.training, spec.training + n_host,
                                  workers)
            self.streams, self.spec = 1, spec
            self.rows = (0, spec.height)
            self.pixels = spec.n_pix
            self.workload = (f"{name.upper()} {spec.width}x{spec.height}x3 "
                             f"K={spec.k_max} N={spec.training}")
        elif name == "c4":
            from paper_1705_09339_b200.parallel import (
                DistReducer, band_rows, dist_gather_rows, train_band_engine)
            spec = base
            sc = synth.Scene(spec)
            train = sc.frames(0, spec.training, workers)
            self.t_gen = time.perf_counter() - t0
            rows = band_rows(spec.height, world, self.cfg.stride)[rank]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if world > 1:
                self.eng = train_band_engine(train, self.cfg, rows,
                                             gather=dist_gather_rows())
                self.band_reduce = attach_band_reduce(self.eng,
                                                      args.band_reduce)
            else:
                self.eng = train_engine(train, self.cfg)
            torch.cuda.synchronize()
            self.t_train = time.perf_counter() - t0
            del train
            full = sc.frames(spec.training, spec.training + n_host, workers)
            self.host = np.ascontiguousarray(full[:, :, rows[0]:rows[1]])
            self.streams, self.spec = 1, spec
            self.rows = rows
            self.pixels = (rows[1] - rows[0]) * spec.width
            self.workload = ("C4 3840x2160x3 K=5 N=150" if world == 1 else
                             f"C4 3840x2160x3 K=5 N=150, rows {rows[0]}-"
                             f"{rows[1] - 1} on rank {rank}")
        else:
            from paper_1705_09339_b200.parallel import BatchEngine
            mine = streams
            specs = [base.for_stream(i) for i in mine]
            scenes = [synth.Scene(sp) for sp in specs]
            trains = [sc.frames(0, base.training, workers) for sc in scenes]
            self.t_gen = time.perf_counter() - t0
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            self.eng = BatchEngine.train(trains, self.cfg)
            torch.cuda.synchronize()
            self.t_train = time.perf_counter() - t0
            del trains
            per = [sc.frames(base.training, base.training + n_host, workers)
                   for sc in scenes]
            self.host = np.ascontiguousarray(np.stack(per, axis=1))  # (T,S,d,H,W)
            self.streams, self.spec = len(mine), base
            self.rows = (0, base.height)
            self.pixels = len(mine) * base.n_pix
            self.workload = (f"C5 {len(mine)} x 1280x720x3 K=5 N=100 "
                             f"(seeds {specs[0].seed}-{specs[-1].seed})")
        self.dev_frames = [torch.from_numpy(f).cuda() for f in self.host]
        dev = torch.device("cuda", torch.cuda.current_device())
        if self.streams == 1:
            h, w = self.dev_frames[0].shape[1:]
            self.mask = torch.empty((h, w), dtype=torch.uint8, device=dev)
            self.stats = torch.empty((total_steps, 16), dtype=torch.int64,
                                     device=dev)
        else:
            h, w = self.dev_frames[0].shape[2:]
            self.mask = torch.empty((self.streams, h, w), dtype=torch.uint8,
                                    device=dev)
            self.stats = torch.empty((total_steps, self.streams, 16),
                                     dtype=torch.int64, device=dev)

    def step(self, i, j):
        """Frame i of the device-resident set, stats slot j."""
        f = self.dev_frames[i % len(self.dev_frames)]
        if self.streams == 1:
            self.eng.process_frame_device(f, self.mask, self.stats[j])
        else:
            self.eng.process_frames_device(f, self.mask, self.stats[j])

    def rows_stats(self, lo):
        r = self.stats[lo:].cpu().numpy()
        return r.reshape(-1, 16)

    def e2e_submit(self, eng, i, pinned=True):
        """The public API with host frames: enqueue frame i from this
        rank's frames in pinned host memory (the contract's e2e: H2D, step,
        D2H of mask + stats) or, pinned=False, from pageable numpy arrays as
        a reference caller passes them (+ the staging copy); returns the
        pending result and the bytes moved each way."""
        if pinned:
            if getattr(self, "host_pinned", None) is None:
                import torch
                self.host_pinned = [torch.from_numpy(x).pin_memory()
                                    for x in self.host]
            f = self.host_pinned[i % len(self.host_pinned)]
            nb = f.numel()
        else:
            f = self.host[i % len(self.host)]
            nb = f.nbytes
        if self.streams == 1:
            m, st = eng.process_frame(f)
            return (m, st), nb, self.pixels + 16 * 8
        res = eng.submit_frames(f)
        return (res,), nb, self.pixels + self.streams * 16 * 8

    @staticmethod
    def e2e_read(res):
        """Read a submitted frame's result on the host (blocks until its
        copies land)."""
        if len(res) == 1:
            res[0].stats                  # batch: blocks on the download
        else:
            m, st = res
            m.labels
            st.n_foreground


def time_device_loop(wl, args, world, local):
    """W untimed warm-up steps, then K steps, each bracketed by CUDA events
    on the engine stream with an L2 flush (untimed) in between; returns the
    per-step durations (ms) and the clock record."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    for i in range(args.warmup):
        flush.zero_()
        wl.step(i, i)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            wl.step(args.warmup + i, args.warmup + i)
            ends[i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    del flush
    return [s.elapsed_time(e) for s, e in zip(starts, ends)], clk


def time_e2e(wl, args, world, pinned=True):
    """The public API end to end: frames from host memory, results read on
    the host two frames behind the submission (so copies and host work
    overlap later steps)."""
    import torch
    eng = wl.eng
    for i in range(args.warmup):
        r, _, _ = wl.e2e_submit(eng, i, pinned)
        wl.e2e_read(r)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    bi = bo = 0
    inflight = []
    for i in range(args.steps):
        cur, bi, bo = wl.e2e_submit(eng, args.warmup + i, pinned)
        inflight.append(cur)
        if len(inflight) > 2:
            wl.e2e_read(inflight.pop(0))
    for r in inflight:
        wl.e2e_read(r)
    return time.perf_counter() - t0, bi, bo


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64,
                     device=torch.device("cuda", torch.cuda.current_device()))
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="cog", choices=["cog", "reference"])
    ap.add_argument("--workload", default="c4",
                    choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--streams", type=int, default=32,
                    help="c5: resident streams per wave (per rank)")
    ap.add_argument("--state", default="float32",
                    choices=["float32", "float64"])
    ap.add_argument("--cpu-frames", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="minimum CPU time of the cpu_baseline sample")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--port", action="store_true",
                    help="--impl reference: time the oracle port even when "
                         "the real reference is installed (oracle/_ref)")
    ap.add_argument("--band-reduce", default="auto", choices=["auto", "nccl"],
                    help="c4 at N > 1: fused peer-mailbox all-reduce when it "
                         "validates (auto), or NCCL")
    ap.add_argument("--variant", default="auto",
                    help="step kernel (engine.kernel_variant; A/B tooling)")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus)

    import torch

    world, rank, local = dist_setup()
    if args.workload == "c5":
        from paper_1705_09339_b200.parallel import streams_for_rank
        mine = streams_for_rank(C5_STREAMS, rank, world)
        cap = max(1, args.streams)
        waves = [mine[i:i + cap] for i in range(0, len(mine), cap)]
    else:
        waves = [None]

    durs_all, e2e_s, e2e_pg_s, rows_all = [], 0.0, 0.0, []
    t_train = t_gen = 0.0
    bi = bo = 0
    clk = None
    wl = None
    for wave in waves:
        if wl is not None:
            # free the previous wave's engine (its streams are done)
            import gc
            wl.eng = eng = None
            del wl
            gc.collect()
            torch.cuda.empty_cache()
        wl = Workload(args.workload, args, world, rank, streams=wave)
        wl.eng.kernel_variant = args.variant
        t_train += wl.t_train
        t_gen += wl.t_gen
        eng, cfg = wl.eng, wl.cfg
        twins = ([eng.clone(), eng.clone()] if hasattr(eng, "clone")
                 else [None, None])
        durs, c = time_device_loop(wl, args, world, local)
        clk = c if clk is None else clk
        durs_all.extend(durs)
        rows_all.append(wl.rows_stats(args.warmup))
        # e2e from pinned host frames (the contract), then from pageable
        # numpy frames (what a reference caller passing arrays pays: + the
        # staging copy), each on a twin starting from the trained state
        for twin, pinned in zip(twins, (True, False)):
            if twin is not None:
                wl.eng = twin
            dt, bi_, bo_ = time_e2e(wl, args, world, pinned)
            if pinned:
                e2e_s += dt
                bi += bi_
                bo += bo_
            else:
                e2e_pg_s += dt
            wl.eng = eng
        del twins
    total_ms = max_over_ranks(float(np.sum(durs_all)), world)
    e2e_s = max_over_ranks(e2e_s, world)
    e2e_pg_s = max_over_ranks(e2e_pg_s, world)
    rows = np.concatenate(rows_all)
    k = wl.cfg.k_max
    spec = wl.spec
    if args.workload == "c4":
        units = spec.n_pix                # the ranks share each frame
    elif args.workload == "c5":
        units = C5_STREAMS * spec.n_pix   # every stream, over all waves
    else:
        units = world * spec.n_pix
    value = units * args.steps / (total_ms * 1e-3)
    e2e = units * args.steps / e2e_s
    e2e_pg = units * args.steps / e2e_pg_s
    step_ms = float(np.mean(durs_all))
    b_frame = float(np.mean([byte_model(r, 3, k) for r in rows]))
    b_step = b_frame * (rows.shape[0] / (args.steps * len(waves)))
    peak, peak_kind = hbm_peak()
    if args.workload == "c4":
        # every rank's stats row describes the whole frame, which the
        # world's ranks process together: compare with the world's HBM
        peak *= world

    line = None
    if rank == 0:
        cpu = None
        if not args.no_cpu and world == 1:
            r = (0, BAND_ROWS) if args.workload == "c4" else (0, spec.height)
            if args.workload == "c5":
                v, dt, nf = cpu_baseline(wl.host, wl.eng, wl.cfg, r,
                                         args.cpu_seconds, args.cpu_frames,
                                         stream=0)
                what = "stream 0 (of the last wave) of the"
            else:
                v, dt, nf = cpu_baseline(wl.host, wl.eng.clone(), wl.cfg, r,
                                         args.cpu_seconds, args.cpu_frames)
                what = (f"rows {r[0]}-{r[1] - 1} of the"
                        if args.workload == "c4" else "the whole")
            cpu = {"value": v, "unit": "pixel-frames/s", "cores": 1,
                   "kind": "port",
                   "sample": f"{nf} post-training frames of {what} "
                             f"{args.workload.upper()} frame, from the "
                             f"GPU engine's state; oracle C "
                             f"kernels (restatement of the serial numba "
                             f"kernels), 1 thread, {dt:.1f}s"}
        traffic = None
        tpath = ROOT / "profiles" / f"traffic_{args.workload}.json"
        if tpath.exists():
            traffic = json.loads(tpath.read_text()).get("bytes_per_step")
        # the contract's definition: algorithmic bytes (SURVEY 8(d) model
        # over this run's own level populations) / measured duration; the
        # ncu DRAM traffic of the same step is reported beside it
        achieved = b_step / (step_ms * 1e-3) / 1e9
        lvl = rows[:, 1:7].sum(axis=0) / max(1, rows[:, 1:7].sum())
        wave_txt = (f", {len(waves)} wave(s) of <= {args.streams} resident "
                    f"streams per rank" if args.workload == "c5" else "")
        line = {
            "metric": METRIC, "value": value, "unit": "pixel-frames/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / (args.steps * len(waves)),
            "higher_is_better": True,
            "scaling": "strong" if args.workload == "c4" else "weak",
            "vs_baseline": None,
            "dtype": "f32-state/f32-filtered+f64-exact-decisions"
                     if args.state == "float32" else "f64",
            "data": "synthetic (seeded BASELINE generator, "
                    "paper_1705_09339_b200.synth)",
            "config": {"workload": wl.workload if world == 1 and
                       args.workload != "c5" else
                       {"c4": "C4 3840x2160x3 K=5 N=150",
                        "c5": "C5 64 x 1280x720x3 K=5 N=100",
                        "c3": "C3 1920x1080x3 K=5 N=200",
                        "c2": "C2 640x480x3 K=3 N=200"}[args.workload],
                       "l2": "flushed between steps (256 MiB write, "
                             "untimed); the per-frame state is also far "
                             "larger than L2",
                       "parallelism": (f"{world} row band(s), "
                                       f"{wl.band_reduce}"
                                       if args.workload == "c4"
                                       and world > 1 else
                                       f"{world} rank(s), independent "
                                       f"streams{wave_txt}")},
            "roofline": {"bound": "hbm",
                         "kernel": "the frame step (hot_kernel + "
                                   "deep_kernel), CUDA events on the engine "
                                   "stream",
                         "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak,
                         "algorithmic_bytes_per_step": b_step,
                         "traffic": traffic,
                         "bytes_used": "algorithmic (SURVEY 8(d) model); "
                                       "traffic = ncu DRAM bytes of the "
                                       "same step"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "pixel-frames/s",
                    "h2d_bytes_per_step": int(bi // len(waves)),
                    "d2h_bytes_per_step": int(bo // len(waves))},
            "gpu_launches": 2 * args.steps * len(waves),
            "clocks": clk.summary() if clk else None,
            "extra": {"train_s": t_train, "scene_gen_s": t_gen,
                      "e2e_pageable": {
                          "value": e2e_pg, "unit": "pixel-frames/s",
                          "what": "process_frame / submit_frames fed "
                                  "pageable numpy frames (+ the staging "
                                  "copy into pinned memory; host-memory "
                                  "bound on this box)"},
                      "step_ms_min": float(np.min(durs_all)),
                      "step_ms_max": float(np.max(durs_all)),
                      "level_fractions": {k_: float(x) for k_, x in zip(
                          ("chp", "group", "mean", "meanvar", "gmm", "skip"),
                          lvl)}},
        }
        print(json.dumps(line), flush=True)
        if args.out:
            Path(args.out).write_text(json.dumps(line, indent=1))
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
