"""Debug: the self-consistency fixture (tests/test_train.py:196-214) through the
device backward / fit with the float64 L1 sign refinement."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
import paper_2512_11624_b200 as g
from test_gpu_fit import _self_consistency_fixture, _frozen

truth, stack = _self_consistency_fixture(g)
batch = g.build_point_batch([stack])
psf = g.slice_psf_diags(batch, [stack])
nbr = np.zeros((batch.n_points, 1), dtype=np.int64)
st = g.init_states([stack])
terms, grads, I_hat = g.backward(batch, truth.astype(np.float64), st, psf, g.LossConfig(lambda_reg=0.0), nbr)
r = I_hat - batch.intensities
print("terms", terms)
print("max|r|", np.abs(r).max(), "max|I|", np.abs(batch.intensities).max())
i = np.argsort(-np.abs(r))[:8]
print(np.c_[i, I_hat[i], batch.intensities[i], r[i]])
print({k: float(np.abs(v).max()) for k, v in grads.items()})
_, _, hist = g.fit([stack], loss_cfg=g.LossConfig(lambda_reg=0.0), optim_cfg=_frozen(g, 5),
                   field=truth.astype(np.float64))
print([h["data_term"] for h in hist])
