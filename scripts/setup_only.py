"""The fit's device setup at a config for ncu launch lists: one warm-up pass
outside the profiler range, then DeviceStacks + device_point_batch +
device_init_field inside it."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2512_11624_b200 as g
from paper_2512_11624_b200 import synthetic
from paper_2512_11624_b200.device_setup import DeviceStacks, device_init_field, device_point_batch

cfg = synthetic.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
stacks, _ = synthetic.make_stacks(cfg, seed=0)
icfg = g.InitConfig(n_gaussians=cfg.n_gaussians, seed=0)
for prof in (False, True):
    torch.cuda.synchronize()
    if prof:
        torch.cuda.cudart().cudaProfilerStart()
    ds = DeviceStacks(stacks)
    b = device_point_batch(ds)
    f = device_init_field(ds, icfg)
    torch.cuda.synchronize()
    if prof:
        torch.cuda.cudart().cudaProfilerStop()
    del ds, b, f
