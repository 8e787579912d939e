"""Robustness/scale check: the full fit at BASELINE configs[3] size on one GPU
(12 stacks 320x320x40, 49 M slice pixels, 2M Gaussians).  argv: epochs
(default 100, reseed every 50); with 500 epochs the default reseed policy."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2512_11624_b200 as g
from paper_2512_11624_b200 import synthetic
cfg = synthetic.CONFIGS["cfg4"]
t0 = time.perf_counter()
stacks, truth = synthetic.make_stacks(cfg, seed=0)
t_gen = time.perf_counter() - t0
epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 100
t0 = time.perf_counter()
field, states, hist = g.fit(stacks, g.InitConfig(n_gaussians=cfg.n_gaussians, seed=0), None,
                            g.OptimConfig(epochs=epochs, reseed_every=50) if epochs < 500
                            else g.OptimConfig(epochs=epochs))
wall = time.perf_counter() - t0
print(json.dumps({"config": "cfg4", "epochs": epochs, "wall_s": wall, "generate_s": t_gen,
                  "loss_first": hist[0]["loss"], "loss_last": hist[-1]["loss"],
                  "pixels": int(sum(np.prod(s.data.shape) for s in stacks)), "gaussians": cfg.n_gaussians}))
