"""Host-side profile of the public per-frame API (C2)."""
import cProfile, pstats, sys, pathlib, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1705_09339_b200 import synth
from paper_1705_09339_b200.config import EngineConfig
from paper_1705_09339_b200.frame_io import Frame
from paper_1705_09339_b200.training import train_engine
spec = synth.CONFIGS[2]
sc = synth.Scene(spec)
cfg = EngineConfig(k_max=3, color=True, training_frames=200).validate()
eng = train_engine(sc.frames(0, 200, 8), cfg)
host = [torch.from_numpy(f).pin_memory() for f in sc.frames(200, 320, 8)]
def loop(n):
    prev = None
    for i in range(n):
        m, st = eng.process_frame(host[i % len(host)])
        if prev:
            prev[0].labels; prev[1].n_foreground
        prev = (m, st)
    prev[0].labels
loop(20); torch.cuda.synchronize()
t = time.perf_counter(); loop(200); print("us/frame", 1e6 * (time.perf_counter() - t) / 200)
pr = cProfile.Profile(); pr.enable(); loop(200); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
