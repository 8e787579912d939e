"""K-NN refresh statistics / timings at a config: the unseeded refresh, a
seeded refresh of the same state, and a seeded refresh after 30 fit epochs
(points and means moved).  Built with -DGSVR_KNN_STATS the kernel prints
per-warp candidate / row / heap counts (KNNSTATS lines)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from bench import build_workload
from paper_2512_11624_b200.engine import DeviceBatch, FitEngine
from paper_2512_11624_b200.train import LossConfig, OptimConfig

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg, stacks, batch, field, states, psf = build_workload(name, 0, 50)
db = DeviceBatch(batch, K=50)
eng = FitEngine(db, field, states, psf, LossConfig(), OptimConfig())


def timed(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    print(f"{label:34s} {(time.perf_counter() - t0) * 1e3:8.2f} ms", flush=True)


timed("refresh unseeded (warm-up)", lambda: eng.refresh(50))
eng.b.refresh.__self__.K = 50
from paper_2512_11624_b200._native import lib
timed("refresh seeded, same state", lambda: eng.refresh(50))
for e in range(30):
    eng.epoch(1.0, e >= 10, True, 0, sync=False)
torch.cuda.synchronize()
timed("refresh seeded after 30 epochs", lambda: eng.refresh(50))
for e in range(30):
    eng.epoch(1.0, True, True, 0, sync=False)
torch.cuda.synchronize()
timed("refresh seeded after 30 more", lambda: eng.refresh(50))
