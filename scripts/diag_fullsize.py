"""Worst render pixels of the full-size device backward vs the oracle (diagnostic)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from bench import build_workload
from oracle import host as oracle
from paper_2512_11624_b200 import _dev, kernels
from paper_2512_11624_b200.engine import DeviceBatch, FitEngine
from paper_2512_11624_b200.train import LossConfig, OptimConfig
K = 50
cfg, stacks, batch, field, states, psf = build_workload("cfg2", 0, K)
P, S, N = batch.n_points, batch.n_slices, field.count
db = DeviceBatch(batch, K=K)
eng = FitEngine(db, field, states, psf, LossConfig(), OptimConfig())
eng.refresh(K)
nbr = _dev.to_host(db.neighbors())
Rc, _, psf6s, sig = oracle.slice_inputs(states.quaternions, batch.stack_rotations, batch.slice_to_stack,
                                        states.log_sigma, psf)
sid = batch.slice_ids
cov6 = oracle.covariances6(field.log_scales, field.quaternions)
w = np.exp(-states.eta)
I_ref, _, gref = oracle.train_step_backward(batch.lifted, sid, Rc, states.translations, psf6s, sig, w,
                                            batch.intensities, nbr, field.means, cov6, field.intensities)
I_hat, absres = np.empty(P), np.empty(P)
bufs = [np.zeros((1, N, 3)), np.zeros((1, N, 6)), np.zeros((1, N)), np.zeros((1, S, 3)),
        np.zeros((1, S, 3, 3)), np.zeros((1, S, 6)), np.zeros((1, S))]
kernels.train_step_backward(batch.lifted, sid, Rc, states.translations, psf6s, sig, w, batch.intensities,
                            nbr, field.means, cov6, field.intensities, 1e-8, 1, I_hat, absres, *bufs)
err = np.abs(I_hat - I_ref) - (1e-5 * np.abs(I_ref) + 1e-9)
bad = np.argsort(-err)[:8]
print("violations:", int((err > 0).sum()), "of", P)
for p in bad:
    print(f"p={p} I_ref={I_ref[p]:.6e} I_hat={I_hat[p]:.6e} diff={I_hat[p]-I_ref[p]:.3e} sid={sid[p]}")
p = bad[0]
x0 = batch.lifted[p]; s = sid[p]
X = Rc[s] @ x0 + states.translations[s]
us = []
for j in nbr[p]:
    A = oracle.unpack_sym6(cov6[j]) + oracle.unpack_sym6(psf6s[s])
    v = X - field.means[j]
    u = -0.5 * v @ np.linalg.solve(A, v)
    us.append(u)
us = np.array(us)
print("u range", us.min(), us.max(), "num e>1e-30:", int((us > -69).sum()))
e = np.where(us < -80, 0.0, np.exp(np.maximum(us, -80)))
print("sum e", e.sum(), "sum c e", (field.intensities[nbr[p]] * e).sum(), "sigma", sig[s])
