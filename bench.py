"""Benchmark of the CoG hot path (BASELINE.json metric: pixel-frames/s of
classify+update, and % of HBM roofline).

Workload (N=1): BASELINE config C2 -- 640x480 RGB, K=3, trained on the
first 200 frames of the seeded synthetic scene (paper_1705_09339_b200.synth);
a step is one frame through the fused step kernel.  For N>1 every rank runs
its own independent C2-shaped stream (seed 1+rank, no collectives: weak
scaling), timed on the device and reduced with MAX over ranks.

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


def cpu_baseline(frames, eng, cfg, n_frames, threads):
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
    t0 = time.perf_counter()
    for f in frames[1:1 + n_frames]:
        oe.process(f)
    dt = time.perf_counter() - t0
    return eng.n_pix * n_frames / dt, dt


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle port) on the
    same workload, all host threads, rank 0 only."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as orc
    from paper_1705_09339_b200 import synth
    from paper_1705_09339_b200.config import EngineConfig
    spec = synth.CONFIGS[2]
    cores = len(os.sched_getaffinity(0))
    os.environ["COG_ORACLE_THREADS"] = str(cores)
    scene = synth.Scene(spec)
    n_train = spec.training
    train = scene.frames(0, n_train)
    cfg = EngineConfig(k_max=spec.k_max, color=True,
                       training_frames=n_train).validate()
    t0 = time.perf_counter()
    eng = orc.train(train, cfg)
    t_train = time.perf_counter() - t0
    eng.threads = cores
    run = scene.frames(n_train, n_train + args.warmup + args.steps)
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
        "data": "synthetic (seeded C2 generator)",
        "config": {"workload": "C2 640x480x3 K=3 N=200 (BASELINE configs[1])",
                   "frames": "post-training frames 200.."},
        "cpu_baseline": {"value": value, "unit": "pixel-frames/s",
                         "cores": cores, "kind": "port",
                         "sample": f"{args.steps} C2 frames after "
                                   f"{args.warmup} warm-up frames; oracle "
                                   f"training {t_train:.1f}s excluded"},
        "e2e": {"value": value, "unit": "pixel-frames/s",
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="cog", choices=["cog", "reference"])
    ap.add_argument("--state", default="float32",
                    choices=["float32", "float64"])
    ap.add_argument("--cpu-frames", type=int, default=20)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    from paper_1705_09339_b200 import synth
    from paper_1705_09339_b200.config import EngineConfig
    from paper_1705_09339_b200.frame_io import Frame
    from paper_1705_09339_b200.training import train_engine

    world, rank, local = dist_setup()
    spec = synth.CONFIGS[2].for_stream(rank)
    scene = synth.Scene(spec)
    n_train = spec.training
    cfg = EngineConfig(k_max=spec.k_max, color=True, training_frames=n_train,
                       state_dtype=args.state).validate()
    t0 = time.perf_counter()
    train = scene.frames(0, n_train)
    t_gen = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng = train_engine(train, cfg)
    torch.cuda.synchronize()
    t_train = time.perf_counter() - t0
    total_steps = args.warmup + args.steps
    host_frames = scene.frames(n_train, n_train + 2 * total_steps)
    dev_frames = [torch.from_numpy(f).cuda() for f in host_frames]
    e2e_eng = eng.clone()
    dev = torch.device("cuda", torch.cuda.current_device())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    mask = torch.empty((spec.height, spec.width), dtype=torch.uint8, device=dev)
    stats = torch.empty((total_steps, 16), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream()

    # ---- device-resident loop
    for i in range(args.warmup):
        flush.zero_()
        eng.process_frame_device(dev_frames[i], mask, stats[i])
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            eng.process_frame_device(dev_frames[args.warmup + i], mask,
                                     stats[args.warmup + i])
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
    rows = stats.cpu().numpy()[args.warmup:]
    bytes_frames = [byte_model(r, spec.depth, spec.k_max,
                               args.state == "float64") for r in rows]
    achieved = float(np.mean(bytes_frames)) / (step_ms * 1e-3) / 1e9
    peak, peak_kind = hbm_peak()
    value = world * spec.n_pix * args.steps / (total_ms * 1e-3)

    # ---- warm-L2 back-to-back (diagnostic)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(True), torch.cuda.Event(True)
    ev0.record(stream)
    for i in range(args.steps):
        eng.process_frame_device(dev_frames[(total_steps + i) % len(dev_frames)],
                                 mask, stats[i % total_steps])
    ev1.record(stream)
    torch.cuda.synchronize()
    warm_ms = ev0.elapsed_time(ev1) / args.steps

    # ---- end-to-end through the public API (host frames in, mask out)
    frames_api = [Frame.from_array(f, i) for i, f in enumerate(host_frames)]
    for i in range(args.warmup):
        m, s = e2e_eng.process_frame(frames_api[i])
        m.labels
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        m, s = e2e_eng.process_frame(frames_api[args.warmup + i])
        m.labels
        s.n_foreground
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = world * spec.n_pix * args.steps / e2e_s

    line = None
    if rank == 0:
        cpu = None
        if not args.no_cpu and world == 1:
            v, dt = cpu_baseline(host_frames, eng.clone(), cfg,
                                 args.cpu_frames, 1)
            cpu = {"value": v, "unit": "pixel-frames/s", "cores": 1,
                   "kind": "port",
                   "sample": f"{args.cpu_frames} C2 frames (640x480x3) from "
                             f"the GPU engine's trained state, oracle "
                             f"C kernels, 1 thread, {dt:.1f}s"}
        lvl = rows[:, 1:7].sum(axis=0) / max(1, rows[:, 1:7].sum())
        line = {
            "metric": "pixel-frames/sec (CoG classify+update)",
            "value": value, "unit": "pixel-frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f64-arith/" + ("f32" if args.state == "float32"
                                     else "f64") + "-state",
            "data": "synthetic (seeded C2 generator, paper_1705_09339_b200.synth)",
            "config": {"workload": "C2 640x480x3 K=3 N=200 (BASELINE configs[1])",
                       "l2": "flushed between steps (256 MiB write, untimed)",
                       "parallelism": f"{world} independent streams"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak,
                         "bytes_per_frame": float(np.mean(bytes_frames)),
                         "traffic": None},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "pixel-frames/s",
                    "h2d_bytes_per_step": spec.depth * spec.n_pix,
                    "d2h_bytes_per_step": spec.n_pix + 16 * 8},
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
            "extra": {"train_s": t_train, "scene_gen_s": t_gen,
                      "warm_l2_ms_per_step": warm_ms,
                      "step_ms_min": float(np.min(durs)),
                      "step_ms_max": float(np.max(durs)),
                      "level_fractions": {k: float(x) for k, x in zip(
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
