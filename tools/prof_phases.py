"""Phase cycle breakdown of the pipelined step kernel (COG_PROF build):
COG_LIB=build_variants_PROF.so python tools/prof_phases.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1705_09339_b200 import _lib, synth  # noqa: E402
from paper_1705_09339_b200.config import EngineConfig  # noqa: E402
from paper_1705_09339_b200.training import train_engine  # noqa: E402

lib = _lib.load()
lib.cog_debug_prof.argtypes = [ctypes.c_void_p, ctypes.c_int]
spec = synth.CONFIGS[2]
sc = synth.Scene(spec)
eng = train_engine(sc.frames(0, spec.training), EngineConfig(k_max=3, color=True))
frames = [torch.from_numpy(f).cuda() for f in sc.frames(200, 220)]
mask = torch.empty((spec.height, spec.width), dtype=torch.uint8, device="cuda")
st = torch.empty(16, dtype=torch.int64, device="cuda")
buf = np.zeros(16, dtype=np.uint64)
for f in frames[:5]:
    eng.process_frame_device(f, mask, st)
torch.cuda.synchronize()
lib.cog_debug_prof(buf.ctypes.data, 1)
for f in frames[5:]:
    eng.process_frame_device(f, mask, st)
torch.cuda.synchronize()
lib.cog_debug_prof(buf.ctypes.data, 0)
names = ["stage_a issue", "wait A", "stage_b issue", "wait B", "tile compute",
         "tiles", "tail flush/fold", "publish", "hot planes (in tile)"]
tiles = buf[5]
for i, n in enumerate(names):
    if i == 5:
        print(f"{n:24s} {int(buf[i])}")
    else:
        print(f"{n:24s} {buf[i] / max(tiles, 1):12.0f} cycles/tile")
