"""cProfile of the whole fit() at a config (host-side view of where wall time goes)."""
import sys, cProfile, pstats
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_2512_11624_b200 as g
from paper_2512_11624_b200 import synthetic
cfg = synthetic.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
stacks, truth = synthetic.make_stacks(cfg, seed=0)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
g.fit(stacks, g.InitConfig(n_gaussians=cfg.n_gaussians, seed=0), None, g.OptimConfig(epochs=500))
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
