make -s -C paper_2512_11624_b200/csrc EXTRA=-DGSVR_L1_DEBUG >/dev/null 2>&1
python - <<'PY' 2>&1 | head -40
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, paper_2512_11624_b200 as g
from test_gpu_fit import _self_consistency_fixture
truth, stack = _self_consistency_fixture(g)
batch = g.build_point_batch([stack]); psf = g.slice_psf_diags(batch, [stack])
nbr = np.zeros((batch.n_points, 1), dtype=np.int64)
terms, grads, I_hat = g.backward(batch, truth, g.init_states([stack]), psf, g.LossConfig(lambda_reg=0.0), nbr)
import torch; torch.cuda.synchronize()
print(batch.lifted[[8,164]], batch.intensities[[8,164]], I_hat[[8,164]])
PY
