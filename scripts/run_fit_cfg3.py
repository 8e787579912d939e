import sys, json, time
from pathlib import Path; sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench
print(json.dumps(bench.fit_cfg3()), flush=True)
