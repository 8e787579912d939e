"""Host-side batch construction and initial-field placement vs the reference
(tests/golden/host_cases.json, made by oracle/gen_host_golden.py from the
reference's own build_point_batch / sample_init_positions / init_field on its
cfg1 acquisitions): SHA-256 of the output bytes must match, i.e. the batch and
the starting field are bit-identical, numpy RNG stream included."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden"
CASES = json.loads((GOLDEN / "host_cases.json").read_text())


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def load_stacks(g, name):
    z = dict(np.load(GOLDEN / name))
    return [g.SliceStack(z[f"s{i}_data"].astype(np.float64), z[f"s{i}_affine"], z[f"s{i}_spacing"],
                         float(z[f"s{i}_thickness"]), z[f"s{i}_mask"]) for i in range(3)]


@pytest.fixture(scope="module")
def g():
    import paper_2512_11624_b200 as pkg
    return pkg


@pytest.mark.parametrize("name", sorted(CASES["batches"]))
def test_build_point_batch_bit_identical(g, name):
    ref = CASES["batches"][name]
    b = g.build_point_batch(load_stacks(g, name))
    assert b.lifted.shape[0] == ref["n_points"]
    assert digest(b.lifted) == ref["lifted"]
    assert digest(b.slice_ids) == ref["slice_ids"]
    assert digest(b.intensities) == ref["intensities"]


@pytest.mark.parametrize("case", CASES["inits"], ids=lambda c: f"{c['data']}-n{c['n_gaussians']}-s{c['seed']}")
def test_init_field_bit_identical(g, case):
    stacks = load_stacks(g, case["data"])
    cfg = g.InitConfig(n_gaussians=case["n_gaussians"], lambda_init=case["lambda_init"], seed=case["seed"],
                       initial_scale=case["initial_scale"], intensity_policy=case["intensity_policy"])
    pos = g.sample_init_positions(stacks, cfg)
    assert digest(pos) == case["positions"]
    f = g.init_field(pos, stacks, cfg)
    assert digest(f.intensities) == case["intensities"]
    assert digest(f.log_scales) == case["log_scales"]
