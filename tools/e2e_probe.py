"""Where the end-to-end (host frames -> public API) time goes, per frame:
python tools/e2e_probe.py [c4|c2]"""
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1705_09339_b200 import synth
from paper_1705_09339_b200.config import EngineConfig
from paper_1705_09339_b200.training import train_engine

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cid = {"c2": 2, "c3": 3, "c4": 4}[name]
spec = synth.CONFIGS[cid]
sc = synth.Scene(spec)
cfg = EngineConfig(k_max=spec.k_max, color=True,
                   training_frames=spec.training).validate()
eng = train_engine(sc.frames(0, spec.training, 16), cfg)
host = sc.frames(spec.training, spec.training + 24, 16)
pinned = [torch.from_numpy(f).pin_memory() for f in host]
dev = [torch.from_numpy(f).cuda() for f in host]
n = 20


def loop(src, lag=2):
    pend = []
    t0 = time.perf_counter()
    for i in range(n):
        pend.append(eng.process_frame(src[i % len(src)]))
        if len(pend) > lag:
            m, st = pend.pop(0)
            m.labels
            st.n_foreground
    for m, st in pend:
        m.labels
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / n


for src, what in ((host, "numpy"), (pinned, "pinned"), (dev, "device")):
    loop(src)
    print(f"{name} {what:7s} ms/frame {loop(src):.3f}  (lag 2)  "
          f"{loop(src, 4):.3f} (lag 4)", flush=True)
ring_in = torch.empty_like(pinned[0])
t0 = time.perf_counter()
for i in range(n):
    eng._stage(host[i % len(host)], ring_in.numpy())
print(f"{name} staging copy ms/frame {1e3 * (time.perf_counter() - t0) / n:.3f}")
x = torch.empty_like(dev[0])
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(n):
    x.copy_(pinned[i % len(pinned)], non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / n
print(f"{name} H2D pinned ms/frame {1e3 * dt:.3f} ({pinned[0].numel() / dt / 1e9:.1f} GB/s)")
m = torch.empty((spec.height, spec.width), dtype=torch.uint8, device="cuda")
stt = torch.empty(16, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(n):
    eng.process_frame_device(dev[i % len(dev)], m, stt)
torch.cuda.synchronize()
print(f"{name} device step ms/frame {1e3 * (time.perf_counter() - t0) / n:.3f}")

# ---- host-side split of the numpy path: staging vs the rest of the call
acc = {"stage": 0.0, "call": 0.0}
orig = eng._stage


def timed_stage(frame, out):
    t = time.perf_counter()
    orig(frame, out)
    acc["stage"] += time.perf_counter() - t


eng._stage = timed_stage
pend = []
t_all = time.perf_counter()
for i in range(n):
    t = time.perf_counter()
    pend.append(eng.process_frame(host[i % len(host)]))
    acc["call"] += time.perf_counter() - t
    if len(pend) > 2:
        m_, st_ = pend.pop(0)
        m_.labels
        st_.n_foreground
for m_, st_ in pend:
    m_.labels
torch.cuda.synchronize()
t_all = time.perf_counter() - t_all
print(f"{name} numpy loop ms/frame {1e3 * t_all / n:.3f}: process_frame "
      f"{1e3 * acc['call'] / n:.3f} (staging {1e3 * acc['stage'] / n:.3f}), "
      f"result reads {1e3 * (t_all - acc['call']) / n:.3f}")
import os
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
