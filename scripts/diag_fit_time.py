"""Where does fit() time go at cfg2?  Counts refreshes/reseeds and times them."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_2512_11624_b200 as g
from paper_2512_11624_b200 import synthetic, engine
cfg = synthetic.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
stacks, truth = synthetic.make_stacks(cfg, seed=0)
stats = {"refresh": [0, 0.0], "reseed": [0, 0.0], "epoch": [0, 0.0], "b.refresh": [0, 0.0], "b.bin": [0, 0.0]}
log = []
def wrap(cls, name, key):
    orig = getattr(cls, name)
    def f(self, *a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = orig(self, *a, **k)
        torch.cuda.synchronize(); stats[key][0] += 1; stats[key][1] += time.perf_counter() - t0
        if key == "b.refresh":
            log.append(time.perf_counter() - t0)
        if key == "refresh" and time.perf_counter() - t0 > 0.3:
            mu = self.mu.cpu().numpy()
            q = np.percentile(mu, [0, 0.1, 1, 50, 99, 99.9, 100], axis=0)
            print("slow refresh", time.perf_counter() - t0, "N", len(mu), "\n", q.T)
        return r
    setattr(cls, name, f)
wrap(engine.FitEngine, "refresh", "refresh")
wrap(engine.FitEngine, "reseed", "reseed")
wrap(engine.FitEngine, "epoch", "epoch")
wrap(engine.DeviceBatch, "refresh", "b.refresh")
wrap(engine.DeviceBatch, "bin", "b.bin")
t0 = time.perf_counter()
g.fit(stacks, g.InitConfig(n_gaussians=cfg.n_gaussians, seed=0), None, g.OptimConfig(epochs=500))
print("total", time.perf_counter() - t0)
for k, (n, s) in stats.items():
    print(f"{k:8s} n={n:4d} total {s:.3f}s  mean {s / max(n, 1) * 1e3:.2f} ms")
print("per-refresh ms:", " ".join(f"{1e3 * v:.0f}" for v in log))
