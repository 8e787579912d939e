"""A/B of the cfg3 fit with the device setup (init.cu) vs the host numpy setup: wall, setup, loop."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2512_11624_b200 as g
from paper_2512_11624_b200 import device_setup as ds, initialization as ini, motion, synthetic

cfg = synthetic.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
stacks, _ = synthetic.make_stacks(cfg, seed=0)
dev = (ds.DeviceStacks, ds.device_point_batch, ds.device_init_field)
host = (lambda st: st, motion.build_point_batch,
        lambda st, c: ini.init_field(ini.sample_init_positions(st, c), st, c))
for mode in ["device", "host", "device", "host"]:
    ds.DeviceStacks, ds.device_point_batch, ds.device_init_field = dev if mode == "device" else host
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, _, hist = g.fit(stacks, g.InitConfig(n_gaussians=cfg.n_gaussians, seed=0), None, g.OptimConfig(epochs=500))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    loop = hist[-1]["seconds"]
    print(f"{mode:6s} wall {wall:.2f} s setup {wall - loop:.2f} s loop {loop:.2f} s final loss {hist[-1]['loss']:.6e}",
          flush=True)
