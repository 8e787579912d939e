"""K-NN refresh timing at a config: unseeded + seeded, A/B via env (GSVR_KNN_LANE / GSVR_KNN_SEEDS)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from bench import build_workload
from paper_2512_11624_b200.engine import DeviceBatch, FitEngine
from paper_2512_11624_b200.knn import NeighborIndex, _build_handle, query_device
from paper_2512_11624_b200 import _dev
from paper_2512_11624_b200.train import LossConfig, OptimConfig
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg, stacks, batch, field, states, psf = build_workload(name, 0, 50)
db = DeviceBatch(batch, K=50)
eng = FitEngine(db, field, states, psf, LossConfig(), OptimConfig())
index = NeighborIndex(np.empty((field.count, 3)), _build_handle(eng.mu))
x = db.corrected_points(eng.Rc, eng.tv)
out = _dev.empty((db.P, 50), np.int32)
def t(label, fn, reps=3):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); print(f"{label:28s} {(time.perf_counter() - t0) / reps * 1e3:8.2f} ms", flush=True)
t("query (Morton API, unseeded)", lambda: query_device(index, x, 50, out_i64=False))
t("refresh (seeded after 1st)", lambda: db.refresh(index, 50, eng.Rc, eng.tv))
