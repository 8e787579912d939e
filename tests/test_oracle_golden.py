"""The CPU oracle (oracle/) against golden vectors produced by the reference.

Pins the restatement before any CUDA result is judged against it.  Goldens come
from oracle/gen_golden.py, which runs /root/reference's gsvr package; the frozen
constants below are the reference tests' own (cited file:line).
"""
import numpy as np
import pytest

from conftest import TRAIN_CASES, load_golden, loss_kwargs, output_prefix

# /root/reference/pkg/tests/test_train.py:28-31
IHAT_ORACLE = (0.48293569946096643, 0.67596320104737873)
DATA_ORACLE = 0.39302750158641236
REG_ORACLE = 0.005100000000000001
TOTAL_ORACLE = 0.39812750158641236
# /root/reference/pkg/tests/test_optim.py:12
ADAMW_TRAJ = (0.899000002, 0.8789511989397751, 0.8433294795899422)


def test_frozen_constants(oracle):
    d = load_golden("train_frozen")
    assert np.allclose(oracle.render_batch(d), IHAT_ORACLE, rtol=1e-12, atol=0)
    terms, grads, I_hat = oracle.backward(d, **loss_kwargs(d))
    assert np.allclose(I_hat, IHAT_ORACLE, rtol=1e-12)
    assert np.isclose(terms["data_term"], DATA_ORACLE, rtol=1e-12)
    assert np.isclose(terms["reg_term"], REG_ORACLE, rtol=1e-12)
    assert np.isclose(terms["loss"], TOTAL_ORACLE, rtol=1e-12)
    # outlier form: tests/test_train.py:91-102
    terms, grads, _ = oracle.backward(d, **loss_kwargs(d, "outlier_"))
    assert np.isclose(terms["data_term"], np.exp(-0.3) * DATA_ORACLE, rtol=1e-12)
    assert np.isclose(terms["outlier_term"], 0.6, rtol=1e-12)
    assert np.isclose(grads["eta"][0], -np.exp(-0.3) * DATA_ORACLE + 2, rtol=1e-11)


@pytest.mark.parametrize("name", TRAIN_CASES)
def test_raw_kernel_matches_reference(oracle, name):
    d = load_golden(name)
    I_hat, absres, g = oracle.train_step_backward(
        d["lifted"], d["slice_ids"], d["raw_Rc"], d["slice_translations"], d["raw_psf6s"],
        d["raw_sigma_s"], d["raw_wdata_s"], d["intensities_obs"], d["nbr"], d["means"],
        d["raw_cov6"], d["intensities"])
    np.testing.assert_allclose(I_hat, d["raw_I_hat"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(absres, d["raw_absres"], rtol=1e-10, atol=1e-14)
    for k in ("dmu", "dcov6", "dc", "dt", "dRc", "dpsf6", "dsigraw"):
        ref = d["raw_" + k]
        np.testing.assert_allclose(g[k], ref, rtol=1e-9, atol=1e-12 * max(1.0, np.abs(ref).max()))


@pytest.mark.parametrize("name", TRAIN_CASES)
def test_backward_chain_matches_reference(oracle, name):
    d = load_golden(name)
    pre = output_prefix(name)
    terms, grads, I_hat = oracle.backward(d, **loss_kwargs(d, pre))
    np.testing.assert_allclose(I_hat, d[pre + "I_hat"], rtol=1e-12, atol=1e-15)
    for k in ("loss", "data_term", "reg_term", "outlier_term"):
        assert np.isclose(terms[k], d[pre + "term_" + k], rtol=1e-11, atol=1e-14), k
    for k, v in grads.items():
        ref = d[pre + "grad_" + k]
        np.testing.assert_allclose(v, ref, rtol=1e-8, atol=1e-11 * max(1.0, np.abs(ref).max()),
                                   err_msg=k)
    np.testing.assert_allclose(oracle.render_batch(d), d[pre + "render"], rtol=1e-12, atol=1e-15)


def test_knn_matches_reference(oracle):
    d = load_golden("knn_cases")
    for key in sorted(d):
        if "_K" not in key:
            continue
        case, K = key.split("_K")
        got = oracle.knn_query(d[case + "_means"], d[case + "_points"], int(K))
        np.testing.assert_array_equal(got, d[key], err_msg=key)


def test_adamw_matches_reference(oracle):
    d = load_golden("misc_cases")
    p = {"p": np.array([1.0])}
    m = {"p": np.zeros(1)}
    v = {"p": np.zeros(1)}
    t = 0
    for g, want, ref in zip((0.5, -0.3, 0.2), ADAMW_TRAJ, d["adamw_traj"]):
        t = oracle.adamw_step(p, {"p": np.array([g])}, m, v, t, {"p": 0.1}, 1.0,
                              weight_decay=0.01)
        assert abs(p["p"][0] - want) < 1e-12 and abs(p["p"][0] - ref) < 1e-15
    params = {"a": d["adamw_a0"].copy(), "b": d["adamw_b0"].copy()}
    m = {k: np.zeros_like(x) for k, x in params.items()}
    v = {k: np.zeros_like(x) for k, x in params.items()}
    t = 0
    for i in range(6):
        t = oracle.adamw_step(params, {"a": d["adamw_ga"][i], "b": d["adamw_gb"][i]}, m, v, t,
                              {"a": 0.05, "b": 0.002}, float(d["adamw_scales"][i]))
    np.testing.assert_allclose(params["a"], d["adamw_a"], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(params["b"], d["adamw_b"], rtol=1e-13, atol=1e-15)


def test_evaluate_field_matches_reference(oracle):
    d = load_golden("misc_cases")
    got = oracle.evaluate_field(d["ev_points"], d["ev_means"], d["ev_log_scales"],
                                d["ev_quats"], d["ev_cvals"], d["ev_nbr"])
    np.testing.assert_allclose(got, d["ev_out"], rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("case", ["a", "b", "c"])
def test_rasterize_matches_reference(oracle, case):
    d = load_golden("export_cases")
    p = case + "_"
    tr = (d[p + "R"], d[p + "t"]) if (p + "R") in d else None
    got = oracle.rasterize(d[p + "means"], d[p + "log_scales"], d[p + "quats"], d[p + "cvals"],
                           d[p + "out"].shape, d[p + "affine"], int(d[p + "K"]), d.get(p + "mask"), tr)
    np.testing.assert_allclose(got, d[p + "out"], rtol=1e-12, atol=1e-15)
