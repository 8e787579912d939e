"""GPU timeline of steady-state epochs (torch profiler / CUPTI): kernel durations and idle gaps."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from torch.profiler import profile, ProfilerActivity
from bench import build_workload
from paper_2512_11624_b200.engine import DeviceBatch, FitEngine
from paper_2512_11624_b200.train import LossConfig, OptimConfig
cfg, stacks, batch, field, states, psf = build_workload(sys.argv[1] if len(sys.argv) > 1 else "cfg2", 0, 50)
db = DeviceBatch(batch, K=50)
eng = FitEngine(db, field, states, psf, LossConfig(), OptimConfig())
eng.refresh(50)
for _ in range(5):
    eng.epoch(1.0, True, False, 0)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        eng.epoch(1.0, True, False, 0, sync=False)
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev_end = t0
for e in evs:
    gap = (e.time_range.start - prev_end) / 1e3
    print(f"{(e.time_range.start - t0) / 1e3:8.3f} ms  gap {gap:7.3f}  dur {e.time_range.elapsed_us() / 1e3:7.3f}  {e.name[:60]}")
    prev_end = max(prev_end, e.time_range.end)
