"""Breakdown of the fit's setup at a config: host (numpy) vs device (init.cu) batch + initial field,
then DeviceBatch and FitEngine construction."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
import paper_2512_11624_b200 as g
from paper_2512_11624_b200 import initialization as ini, synthetic
from paper_2512_11624_b200.device_setup import DeviceStacks, device_init_field, device_point_batch
from paper_2512_11624_b200.engine import DeviceBatch, FitEngine

cfg = synthetic.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
stacks, _ = synthetic.make_stacks(cfg, seed=0)
icfg = g.InitConfig(n_gaussians=cfg.n_gaussians, seed=0)
torch.zeros(1).cuda()


def clock(T, name, fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    T[name] = round(time.perf_counter() - t, 4)
    return out


for rep in range(3):
    T = {}
    clock(T, "host sample_init_positions", lambda: ini.sample_init_positions(stacks, icfg))
    clock(T, "host build_point_batch", lambda: g.build_point_batch(stacks))
    ds = clock(T, "device stacks upload", lambda: DeviceStacks(stacks))
    b = clock(T, "device batch", lambda: device_point_batch(ds))
    f = clock(T, "device init field", lambda: device_init_field(ds, icfg))
    db = clock(T, "DeviceBatch", lambda: DeviceBatch(b, K=50))
    psf = g.slice_psf_diags(b, stacks)
    eng = clock(T, "FitEngine", lambda: FitEngine(db, f, g.init_states(stacks), psf, g.LossConfig(), g.OptimConfig()))
    clock(T, "first refresh", lambda: eng.refresh(50))
    print(T, flush=True)
    del eng, db, ds
