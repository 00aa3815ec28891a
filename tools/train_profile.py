"""Host-side profile of training a BASELINE workload engine:
python tools/train_profile.py [config_id]"""
import cProfile
import pathlib
import pstats
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1705_09339_b200 import synth  # noqa: E402
from paper_1705_09339_b200.config import EngineConfig  # noqa: E402
from paper_1705_09339_b200.training import train_engine  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
spec = synth.CONFIGS[cid]
train = synth.Scene(spec).frames(0, spec.training, 16)
cfg = EngineConfig(k_max=spec.k_max, color=True,
                   training_frames=spec.training).validate()
torch.cuda.synchronize()
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
eng = train_engine(train, cfg)
torch.cuda.synchronize()
pr.disable()
print("train_s", time.perf_counter() - t)
pstats.Stats(pr).sort_stats("cumtime").print_stats(30)
