"""Stage timing of the drop-in kernels.train_step_backward (host buffers) at cfg2."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import bench
from paper_2512_11624_b200 import _dev, kernels
from paper_2512_11624_b200._native import check, lib
from paper_2512_11624_b200.engine import DeviceBatch, FitEngine
from paper_2512_11624_b200.train import LossConfig, OptimConfig

cfg, stacks, batch, field, states, psf = bench.build_workload("cfg2", 0, 50)
db = DeviceBatch(batch, K=50)
eng = FitEngine(db, field, states, psf, LossConfig(), OptimConfig())
eng.refresh(50)
P, S, N = batch.n_points, batch.n_slices, field.count
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
nbr_h = pin(_dev.to_host(db.neighbors()))
x0 = pin(batch.lifted)

def t(name, fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    print(f"{name:40s} {(time.perf_counter() - t0) / reps * 1e3:9.2f} ms", flush=True)

t("H2D nbr int64 (pinned)", lambda: nbr_h.to("cuda"))
t("H2D x0 (pinned)", lambda: x0.to("cuda"))
nbr_d = nbr_h.to("cuda")
t("DeviceBatch create", lambda: DeviceBatch(batch, K=50))
t("bin from device nbr", lambda: db.bin(nbr_d, N))
t("np.asarray(pinned tensor)", lambda: np.asarray(nbr_h))
import cProfile, pstats
ins = [pin(a) for a in (batch.lifted, batch.slice_ids.astype(np.int32), _dev.to_host(eng.Rc).reshape(S, 3, 3),
                        _dev.to_host(eng.tv), _dev.to_host(eng.p6), _dev.to_host(eng.sig), _dev.to_host(eng.w),
                        batch.intensities)]
fl = [pin(_dev.to_host(x)) for x in (eng.mu, eng.cov6, eng.c)]
outs = [torch.empty(P, dtype=torch.float64).pin_memory() for _ in range(2)]
grads = [torch.zeros(s, dtype=torch.float64).pin_memory()
         for s in [(1, N, 3), (1, N, 6), (1, N), (1, S, 3), (1, S, 3, 3), (1, S, 6), (1, S)]]
call = lambda: kernels.train_step_backward(*ins, nbr_h, *fl, 1e-8, 1, outs[0], outs[1], *grads)
t("full drop-in call", call)
pr = cProfile.Profile(); pr.enable(); call(); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    call(); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
tail_from = evs[-1].time_range.end - 6000  # last 6 ms: every launch
for e in evs:
    if e.time_range.elapsed_us() > 200 or e.time_range.start > tail_from:
        print(f"{(e.time_range.start - t0) / 1e3:8.2f} ms  +{e.time_range.elapsed_us() / 1e3:7.2f} ms  {e.name[:70]}")
