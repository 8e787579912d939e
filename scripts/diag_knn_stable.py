"""Fraction of rows whose K-neighbour SET is unchanged by each refresh of a
cfg3 (or cfg2) fit -- the rows a count-only seeded pass could settle."""
import sys, json
from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2512_11624_b200 import engine
import bench
stats = []
orig = engine.DeviceBatch.refresh
def refresh(self, index, K, Rc, tvec):
    prev = self.neighbors().sort(dim=1).values if self.K else None
    orig(self, index, K, Rc, tvec)
    if prev is not None:
        cur = self.neighbors().sort(dim=1).values
        stats.append(round(float((prev == cur).all(dim=1).float().mean()), 4))
engine.DeviceBatch.refresh = refresh
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
out = bench.fit_cfg3() if cfg == "cfg3" else bench.fit_cfg2()
print(json.dumps({"cfg": cfg, "refreshes": len(stats), "unchanged_frac": stats}))
