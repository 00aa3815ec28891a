"""Benchmark of the CoG hot path (BASELINE.json metric: pixel-frames/s of
classify+update, and % of HBM roofline).

Workload (N=1, default): BASELINE config C2 -- 640x480 RGB, K=3, trained
on the first 200 frames of the seeded synthetic scene
(paper_1705_09339_b200.synth); a step is one frame through the step kernels.
For N>1 every rank runs its own independent C2-shaped stream (seed 1+rank,
no collectives: weak scaling), timed on the device, MAX over ranks.
--workload c3 / c4 / c5 measure the other BASELINE configs (c4 at N>1: one
4K stream in row bands with a per-frame NCCL all-reduce, strong scaling;
c5: a batch engine of independent 720p streams).

value    device-resident frames, CUDA events around each step's launch on the
         engine stream, L2 flushed (256 MiB write) between steps (outside
         the events).
e2e      the public API: ``process_frame(Frame)`` from pinned host memory +
         reading ``mask.labels`` back every step.
roofline achieved = algorithmic bytes of the frame (from its own level
         populations, byte model in DESIGN.md) / step-kernel duration.
cpu_baseline  the oracle (C restatement of the reference kernels, 1 thread
         like the serial reference) on a bounded sample of the same stream.

--impl reference runs the reference's CPU path (the oracle port, all host
threads) on the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM = 6650.0


def hbm_peak():
    try:
        v = json.loads(PEAKS.read_text())["hbm_gbs"]
        return float(v), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def byte_model(row, depth, k, f64=False):
    """Algorithmic HBM bytes of one frame from its level populations.

    per plane-pixel: frame 1 + dyn 4r/4w + kind 1w + conf 4w         = 14
    evaluated: + meta 2 + streak 4r/4w + hits 4r/4w + table sector 32
               + peak 4 + top-level mode mu/var 2x4                   = +62
    MEAN: + mu write 4; MEANVAR / GMM: + mixture 12K read + 12K write
          + meta write 2 (mixture bytes double with float64 storage)
    per pixel: class 1 + group id 2 + mask 1                          = 4
    """
    _, n_chp, n_group, n_mean, n_meanvar, n_gmm, n_skip = row[:7]
    pixels = (n_chp + n_group + n_mean + n_meanvar + n_gmm + n_skip) // depth
    mb = 8 if f64 else 4
    ev = 14 + 62 + (2 * mb - 8)
    mix = 2 * 3 * mb * k + 2
    return (n_skip * 14 + (n_chp + n_group) * ev + n_mean * (ev + mb)
            + (n_meanvar + n_gmm) * (ev + mix) + pixels * 4)


class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) during the timed region."""

    def __init__(self, index=0, period=0.05):
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

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(
                nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(
                nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(
                    self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
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

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples),
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


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


def cpu_baseline(frames, eng, cfg, n_frames, threads, seconds=10.0):
    """Oracle engine seeded with the GPU engine's trained state, timed over
    a bounded run sample (same stream)."""
    from oracle import oracle as orc
    os.environ["COG_ORACLE_THREADS"] = str(threads)
    oe = orc.OracleEngine(cfg, eng.height, eng.width, eng.depth)
    oe.threads = threads
    st = eng.state_dict()
    for k, v in st.items():
        setattr(oe, k, np.array(v))
    oe.tables = eng.tables.copy()
    oe.finalize_tables()
    oe.dynamics = eng.dynamics
    wt = np.array([cfg.weights_static, cfg.weights_oscillating,
                   cfg.weights_dynamic])[oe.dynamics]
    oe.wa, oe.wb, oe.wc = (np.ascontiguousarray(wt[:, i]) for i in range(3))
    oe.group_id = eng.group_id
    oe.group_w = eng.group_w.copy()
    oe.group_members = eng.group_members.copy()
    oe.process(frames[0])  # warm
    # a bounded sample: the stream's next frames (cycled if the host set is
    # shorter), at least n_frames of them and at least `seconds` of CPU work
    t0 = time.perf_counter()
    done, dt = 0, 0.0
    while done < n_frames or dt < seconds:
        oe.process(frames[1 + done % (len(frames) - 1)])
        done += 1
        dt = time.perf_counter() - t0
    return eng.n_pix * done / dt, dt, done


def run_reference(args):
    """--impl reference: the reference's CPU path (the oracle port of its
    numba kernels, all host threads) on the same workload; rank 0 only.
    c4 runs a 270-row band (1/8) of the 4K frame: the full frame needs
    ~100 GB of host RAM in the reference's layout."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
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
        train = np.ascontiguousarray(train[:, :, :270])
        run = np.ascontiguousarray(run[:, :, :270])
        band = " (rows 0-269 of the 4K frame)"
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
        "metric": "pixel-frames/sec (CoG classify+update)",
        "value": value, "unit": "pixel-frames/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator)",
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
    print(json.dumps(line))
    return 0


def m_bytes(spec):
    return spec.width * spec.height


class Workload:
    """One bench workload: a trained engine plus its frame sources.

    c2 (default, BASELINE configs[1]): one 640x480x3 stream per rank.
    c3: one 1920x1080x3 stream per rank (K=5).
    c4: one 3840x2160x3 stream; at N>1 split into stride-aligned row bands,
        one per rank, partials all-reduced over NCCL each frame.
    c5: independent 1280x720x3 streams (K=5), `streams` resident per rank
        in one batch engine (64 / N in total, waves of <= 32 on one GPU).
    """

    def __init__(self, name, args, world, rank):
        import torch
        from paper_1705_09339_b200 import synth
        from paper_1705_09339_b200.config import EngineConfig
        from paper_1705_09339_b200.training import train_engine
        self.name = name
        self.pinned = None
        cid = {"c2": 2, "c3": 3, "c4": 4, "c5": 5}[name]
        base = synth.CONFIGS[cid]
        workers = max(1, min(16, len(os.sched_getaffinity(0))))
        total_steps = args.warmup + args.steps
        self.total_steps = total_steps
        self.extra_frames = 2 * total_steps
        t0 = time.perf_counter()
        if name in ("c2", "c3"):
            spec = base.for_stream(rank)
            sc = synth.Scene(spec)
            train = sc.frames(0, spec.training, workers)
            self.cfg = EngineConfig(k_max=spec.k_max, color=True,
                                    training_frames=spec.training,
                                    state_dtype=args.state).validate()
            self.t_gen = time.perf_counter() - t0
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            self.eng = train_engine(train, self.cfg)
            torch.cuda.synchronize()
            self.t_train = time.perf_counter() - t0
            self.host = sc.frames(spec.training,
                                  spec.training + self.extra_frames, workers)
            self.streams, self.spec = 1, spec
            self.pixels = spec.n_pix            # per rank per step
            self.workload = (f"{name.upper()} {spec.width}x{spec.height}x3 "
                             f"K={spec.k_max} N={spec.training}")
        elif name == "c4":
            from paper_1705_09339_b200.parallel import (
                DistReducer, band_rows, dist_gather_rows, train_band_engine)
            spec = base
            sc = synth.Scene(spec)
            train = sc.frames(0, spec.training, workers)
            self.cfg = EngineConfig(k_max=spec.k_max, color=True,
                                    training_frames=spec.training,
                                    state_dtype=args.state).validate()
            self.t_gen = time.perf_counter() - t0
            rows = band_rows(spec.height, world, self.cfg.stride)[rank]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            self.eng = train_band_engine(
                train, self.cfg, rows,
                gather=dist_gather_rows() if world > 1 else None)
            if world > 1:
                self.eng.reducer = DistReducer()
            torch.cuda.synchronize()
            self.t_train = time.perf_counter() - t0
            full = sc.frames(spec.training, spec.training + self.extra_frames,
                             workers)
            self.host = np.ascontiguousarray(full[:, :, rows[0]:rows[1]])
            self.streams, self.spec = 1, spec
            self.pixels = (rows[1] - rows[0]) * spec.width
            self.workload = (f"C4 3840x2160x3 K=5 N=150, rows {rows[0]}-"
                             f"{rows[1]} of 2160 on this rank")
        else:
            from paper_1705_09339_b200.parallel import BatchEngine, streams_for_rank
            mine = streams_for_rank(64, rank, world)[:args.streams]
            specs = [base.for_stream(i) for i in mine]
            scenes = [synth.Scene(sp) for sp in specs]
            trains = [sc.frames(0, base.training, workers) for sc in scenes]
            self.cfg = EngineConfig(k_max=base.k_max, color=True,
                                    training_frames=base.training,
                                    state_dtype=args.state).validate()
            self.t_gen = time.perf_counter() - t0
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            self.eng = BatchEngine.train(trains, self.cfg)
            torch.cuda.synchronize()
            self.t_train = time.perf_counter() - t0
            del trains
            per = [sc.frames(base.training, base.training + self.extra_frames,
                             workers) for sc in scenes]
            self.host = np.ascontiguousarray(np.stack(per, axis=1))  # (T,S,d,H,W)
            self.streams, self.spec = len(mine), base
            self.pixels = len(mine) * base.n_pix
            self.workload = (f"C5 {len(mine)} x 1280x720x3 K=5 N=100 streams "
                             f"resident on this rank (seeds {specs[0].seed}-"
                             f"{specs[-1].seed})")
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

    def rows(self, lo):
        r = self.stats[lo:].cpu().numpy()
        return r.reshape(-1, 16)

    def e2e_engine(self):
        return self.eng.clone() if hasattr(self.eng, "clone") else self.eng

    def e2e_submit(self, eng, i):
        """Public API from host memory: enqueue frame i (H2D from the
        engine's pinned staging, step, D2H of mask + stats); returns the
        pending result and the bytes moved each way."""
        if self.streams == 1:
            if self.pinned is None:
                import torch
                self.pinned = [torch.from_numpy(f).pin_memory()
                               for f in self.host]
            f = self.pinned[i % len(self.pinned)]
            m, st = eng.process_frame(f)   # pinned host tensor -> DMA
            return (m, st), f.numel(), m_bytes(self.spec) + 16 * 8
        if self.pinned is None:        # first (untimed warm-up) call
            import torch
            self.pinned = [torch.from_numpy(f).pin_memory()
                           for f in self.host[:self.total_steps]]
        f = self.pinned[i % len(self.pinned)]
        res = eng.submit_frames(f)     # pinned host tensor -> DMA
        return (res,), f.numel(), (self.streams * self.spec.n_pix
                                   + self.streams * 16 * 8)

    @staticmethod
    def e2e_read(res):
        """Read a submitted frame's result on the host (blocks until its
        copies land)."""
        if res is not None and len(res) == 1:
            res[0].stats                  # batch: blocks on the download
        elif res is not None:
            m, st = res
            m.labels
            st.n_foreground


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="cog", choices=["cog", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--streams", type=int, default=32,
                    help="c5: resident streams per rank (<= 64 / N)")
    ap.add_argument("--state", default="float32",
                    choices=["float32", "float64"])
    ap.add_argument("--cpu-frames", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="minimum CPU time of the cpu_baseline sample")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch

    world, rank, local = dist_setup()
    wl = Workload(args.workload, args, world, rank)
    eng, cfg = wl.eng, wl.cfg
    total_steps = args.warmup + args.steps
    dev = torch.device("cuda", torch.cuda.current_device())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    e2e_eng = wl.e2e_engine()
    launches_per_step = 2  # hot kernel + deep/finalize kernel

    # ---- device-resident loop
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
    durs = [s.elapsed_time(e) for s, e in zip(starts, ends)]  # ms
    step_ms = float(np.mean(durs))
    total_ms = float(np.sum(durs))
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    rows = wl.rows(args.warmup)
    k = cfg.k_max
    bytes_frames = [byte_model(r, 3, k, args.state == "float64") for r in rows]
    steps_bytes = float(np.sum(bytes_frames)) / args.steps
    achieved = steps_bytes / (step_ms * 1e-3) / 1e9
    peak, peak_kind = hbm_peak()
    if args.workload == "c4":
        # strong scaling: the ranks share one frame
        value = wl.spec.n_pix * args.steps / (total_ms * 1e-3)
    else:
        value = world * wl.pixels * args.steps / (total_ms * 1e-3)

    # ---- warm-L2 back-to-back (diagnostic)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(True), torch.cuda.Event(True)
    ev0.record(stream)
    for i in range(args.steps):
        wl.step(total_steps + i, i % total_steps)
    ev1.record(stream)
    torch.cuda.synchronize()
    warm_ms = ev0.elapsed_time(ev1) / args.steps

    # ---- end-to-end through the public API (host frames in, mask and
    # stats read back every step; results are read two frames behind the
    # submission, so the copies and the host work overlap later steps)
    for i in range(args.warmup):
        r, _, _ = wl.e2e_submit(e2e_eng, i)
        wl.e2e_read(r)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    bi = bo = 0
    inflight = []
    for i in range(args.steps):
        cur, bi, bo = wl.e2e_submit(e2e_eng, args.warmup + i)
        inflight.append(cur)
        if len(inflight) > 2:          # results read two frames behind
            wl.e2e_read(inflight.pop(0))
    for r in inflight:
        wl.e2e_read(r)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    if args.workload == "c4":
        e2e = wl.spec.n_pix * args.steps / e2e_s
    else:
        e2e = world * wl.pixels * args.steps / e2e_s

    line = None
    if rank == 0:
        cpu = None
        if not args.no_cpu and world == 1 and args.workload in ("c2", "c3"):
            v, dt, nf = cpu_baseline(wl.host, eng.clone(), cfg,
                                     args.cpu_frames, 1, args.cpu_seconds)
            cpu = {"value": v, "unit": "pixel-frames/s", "cores": 1,
                   "kind": "port",
                   "sample": f"{nf} {args.workload.upper()} frames (the "
                             f"stream's post-training frames, cycled over "
                             f"{len(wl.host) - 1}) from the GPU engine's "
                             f"trained state, oracle C kernels (restatement "
                             f"of the serial numba kernels), 1 thread, "
                             f"{dt:.1f}s"}
        lvl = rows[:, 1:7].sum(axis=0) / max(1, rows[:, 1:7].sum())
        traffic = None
        tpath = ROOT / "profiles" / f"traffic_{args.workload}.json"
        if tpath.exists():
            traffic = json.loads(tpath.read_text()).get("bytes_per_step")
        line = {
            "metric": "pixel-frames/sec (CoG classify+update)",
            "value": value, "unit": "pixel-frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.workload == "c4" else "weak",
            "vs_baseline": None,
            "dtype": "f32-state/f32-filtered+f64-exact-decisions"
                     if args.state == "float32" else "f64",
            "data": "synthetic (seeded BASELINE generator, "
                    "paper_1705_09339_b200.synth)",
            "config": {"workload": wl.workload,
                       "l2": "flushed between steps (256 MiB write, untimed)",
                       "parallelism": (f"{world} row bands" if
                                       args.workload == "c4" else
                                       f"{world} ranks x {wl.streams} "
                                       f"independent stream(s)")},
            "roofline": {"bound": "hbm",
                         "kernel": "the frame step: fast_kernel (hot pass) + "
                                   "deep_kernel (worklist + finalize), timed "
                                   "together with CUDA events on the engine "
                                   "stream; ncu share in profiles/",
                         "achieved": achieved,
                         "peak": peak * (world if args.workload == "c4" else 1),
                         "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / (peak * (world if args.workload
                                                     == "c4" else 1)),
                         "bytes_per_step": steps_bytes,
                         "traffic": traffic},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "pixel-frames/s",
                    "h2d_bytes_per_step": int(bi),
                    "d2h_bytes_per_step": int(bo)},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
            "extra": {"train_s": wl.t_train, "scene_gen_s": wl.t_gen,
                      "warm_l2_ms_per_step": warm_ms,
                      "step_ms_min": float(np.min(durs)),
                      "step_ms_max": float(np.max(durs)),
                      "level_fractions": {k_: float(x) for k_, x in zip(
                          ("chp", "group", "mean", "meanvar", "gmm", "skip"),
                          lvl)}},
        }
        print(json.dumps(line))
        if args.out:
            Path(args.out).write_text(json.dumps(line, indent=1))
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
