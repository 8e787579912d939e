import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
from conftest import load_golden
import paper_2512_11624_b200 as g
from paper_2512_11624_b200.engine import DeviceBatch
d = load_golden("train_medium_s0")
b = g.PointBatch(d["lifted"], d["slice_ids"].astype(np.int32), d["slice_ids"] * 0, d["intensities_obs"],
                 d["slice_to_stack"], d["stack_rotations"])
db = DeviceBatch(b, K=50)
print("planar", db.planar)
ts, tn, tsl, uoff, gid, perm = (None,) * 6
o, bas, ab = db.tile_geometry()
import paper_2512_11624_b200._native as nat
T = db.n_tiles
from paper_2512_11624_b200 import _dev
ts_ = _dev.empty((T,), np.int64); tn_ = _dev.empty((T,), np.int32)
pm = _dev.empty((db.P,), np.int32)
nat.check(nat.lib().gsvr_batch_tile_info(db.raw, _dev.ptr(ts_), _dev.ptr(tn_), 0, 0, 0, _dev.ptr(pm), _dev.stream_ptr()))
ts_, tn_, pm = map(_dev.to_host, (ts_, tn_, pm))
for t in range(T):
    rows = pm[ts_[t]:ts_[t] + tn_[t]]
    x = b.lifted[rows] - o[t]
    b1, b2 = bas[t, :3], bas[t, 3:]
    n = np.cross(b1, b2)
    res = np.abs(x @ n).max()
    if res > 1e-8 or t < 3:
        print(t, tn_[t], "res", res, "|b1|", np.linalg.norm(b1), "|b2|", np.linalg.norm(b2), "b1.b2", b1 @ b2)
print("--- compare")
for t in range(3):
    rows = pm[ts_[t]:ts_[t] + tn_[t]]
    p = b.lifted[rows]
    oc = 0.5 * (p.min(0) + p.max(0))
    dd = p - oc
    w, V = np.linalg.eigh(dd.T @ dd)
    print(t, "origin dev", o[t], "host", oc)
    print("   normal host", V[:, 0], "b1 dev", bas[t, :3], "b2 dev", bas[t, 3:])
    print("   sid of rows", np.unique(b.slice_ids[rows]), "ab dev first", ab[ts_[t]:ts_[t]+2])
print("--- reconstruct")
ab_int = ab  # internal order
for t in range(4):
    rows = pm[ts_[t]:ts_[t] + tn_[t]]
    p = b.lifted[rows]
    rec = o[t] + ab_int[ts_[t]:ts_[t]+tn_[t], 0:1] * bas[t, :3] + ab_int[ts_[t]:ts_[t]+tn_[t], 1:2] * bas[t, 3:]
    n = np.cross(bas[t, :3], bas[t, 3:])
    print(t, "recon err", np.abs(rec - p).max(), "res", np.abs((p - o[t]) @ n).max())
import os
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/dbg_planar.npz", o=o, bas=bas, ab=ab, ts=ts_, tn=tn_, pm=pm, lifted=b.lifted)
