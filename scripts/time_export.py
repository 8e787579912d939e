"""cfg5 HR export timing on a synthetic field (cfg3-sized: 500k Gaussians in a ~200 mm box)."""
import sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2512_11624_b200 as g
import bench
rng = np.random.default_rng(0)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 500_000
mu = rng.uniform(-100, 100, size=(N, 3))
f = g.GaussianField(mu, np.log(rng.uniform(0.8, 2.0, size=(N, 3))), rng.normal(size=(N, 4)),
                    rng.uniform(0.1, 0.9, size=N))
print(json.dumps(bench.export_cfg5(f)))
