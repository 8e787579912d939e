"""Wall-clock of the cfg3 fit (6 stacks 320x320x40, 500k Gaussians, 500 epochs) with the
number and total time of neighbour refreshes (the engine's refresh is wrapped and timed)."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2512_11624_b200 as g
from paper_2512_11624_b200 import engine, synthetic

cfg = synthetic.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 500
stacks, truth = synthetic.make_stacks(cfg, seed=0)
stats = {"n": 0, "s": 0.0}
orig = engine.FitEngine.refresh


def timed_refresh(self, K):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    orig(self, K)
    torch.cuda.synchronize()
    stats["n"] += 1
    stats["s"] += time.perf_counter() - t0


engine.FitEngine.refresh = timed_refresh
for rep in range(2):
    stats.update(n=0, s=0.0)
    t0 = time.perf_counter()
    _, _, hist = g.fit(stacks, g.InitConfig(n_gaussians=cfg.n_gaussians, seed=0), None, g.OptimConfig(epochs=epochs))
    wall = time.perf_counter() - t0
    print(f"{cfg.name} fit {epochs} epochs: {wall:.2f} s (loop {hist[-1]['seconds']:.2f} s); "
          f"{stats['n']} refreshes {stats['s']:.2f} s (timed with syncs)", flush=True)
