"""Stage timing of the refresh and drop-in paths (CUDA events)."""
import sys, time, ctypes
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from bench import build_workload
from paper_2512_11624_b200 import _dev
from paper_2512_11624_b200._native import lib, check
from paper_2512_11624_b200.engine import DeviceBatch, FitEngine
from paper_2512_11624_b200.knn import NeighborIndex, _build_handle, query_device
from paper_2512_11624_b200.train import LossConfig, OptimConfig

cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
K = 50
cfg, stacks, batch, field, states, psf = build_workload(cfgname, 0, K)
torch.cuda.synchronize()

def timed(name, fn, reps=1):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    print(f"{name:32s} {(time.perf_counter() - t0) / reps * 1e3:10.2f} ms", flush=True)

db = DeviceBatch(batch, K=K)
eng = FitEngine(db, field, states, psf, LossConfig(), OptimConfig())
mu = eng.mu
timed("knn build", lambda: _build_handle(mu))
index = NeighborIndex(np.empty((field.count, 3)), _build_handle(mu))
x = db.corrected_points(eng.Rc, eng.tv)
out = _dev.empty((db.P, K), np.int32)
timed("knn query (Morton API)", lambda: query_device(index, x, K, out_i64=False))
timed("refresh = knn + bin", lambda: db.refresh(index, K, eng.Rc, eng.tv))
nbr = db.neighbors()
timed("bin (from caller nbr int64)", lambda: db.bin(nbr, field.count))
timed("batch_create", lambda: DeviceBatch(batch, K=K))
timed("train pass", lambda: eng.train_pass(), reps=5)
timed("epoch", lambda: eng.epoch(1.0, True, False, 0), reps=5)
lib().gsvr_set_kernel_variant(1)
timed("train pass (general 3D kernel)", lambda: eng.train_pass(), reps=5)
lib().gsvr_set_kernel_variant(0)
print("planar batch:", lib().gsvr_batch_is_planar(db.raw), "max unique/tile:", "n/a")
