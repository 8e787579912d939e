"""Where does fit_cfg3's wall time go, run to run?  Wraps FitEngine.refresh /
reseed / epoch with host wall timers (epoch() already blocks on its loss read)
and samples the SM clock with NVML while the fit runs."""
import sys, json, time, threading
from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import bench
from paper_2512_11624_b200 import engine

acc = {}
def wrap(name):
    f = getattr(engine.FitEngine, name)
    def g(self, *a, **k):
        t = time.perf_counter()
        r = f(self, *a, **k)
        if name != "epoch":
            import torch; torch.cuda.synchronize()
        acc.setdefault(name, []).append(time.perf_counter() - t)
        return r
    setattr(engine.FitEngine, name, g)
for n in ("refresh", "reseed", "epoch"):
    wrap(n)

import pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
clk = []; stop = False
def sample():
    while not stop:
        clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)); time.sleep(0.05)
th = threading.Thread(target=sample, daemon=True); th.start()
runs = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for r in range(runs):
    acc.clear(); clk.clear()
    out = bench.fit_cfg3()
    s = {k: (len(v), round(sum(v), 3), round(float(np.median(v)) * 1e3, 2), round(max(v) * 1e3, 1)) for k, v in acc.items()}
    ep = np.array(acc["epoch"]) * 1e3
    print(json.dumps({"run": r, "wall": round(out["wall_s"], 3), "loop": round(out["loop_s"], 3),
                      "calls(n,sum_s,med_ms,max_ms)": s,
                      "epoch_pct": [round(float(x), 2) for x in np.percentile(ep, [10, 50, 90, 99])],
                      "sm_mhz": [int(np.min(clk)), int(np.median(clk)), int(np.max(clk))]}), flush=True)
stop = True
