"""Host-side cost of one process_frame_device call vs its GPU time (C2)."""
import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import time
import torch
from paper_1705_09339_b200 import synth
from paper_1705_09339_b200.config import EngineConfig
from paper_1705_09339_b200.training import train_engine

spec = synth.CONFIGS[2]
sc = synth.Scene(spec)
cfg = EngineConfig(k_max=3, color=True, training_frames=200).validate()
eng = train_engine(sc.frames(0, 200), cfg)
frames = [torch.from_numpy(f).cuda() for f in sc.frames(200, 260)]
mask = torch.empty((480, 640), dtype=torch.uint8, device="cuda")
stats = torch.empty(16, dtype=torch.int64, device="cuda")
for f in frames[:10]:
    eng.process_frame_device(f, mask, stats)
torch.cuda.synchronize()
t0 = time.perf_counter()
for f in frames[10:60]:
    eng.process_frame_device(f, mask, stats)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e6*(t1-t0)/50:.1f} us/frame, wall incl. GPU {1e6*(t2-t0)/50:.1f} us/frame")
# GPU-only time per frame: a long queue behind a big memset
big = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
big.zero_()
e0.record()
for f in frames[10:60]:
    eng.process_frame_device(f, mask, stats)
e1.record()
torch.cuda.synchronize()
print(f"events around 50 queued frames: {1e3*e0.elapsed_time(e1)/50:.1f} us/frame")
