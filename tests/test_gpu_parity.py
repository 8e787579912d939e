"""CUDA path vs the reference (golden vectors) and the oracle, through the
reference-shaped public API and the drop-in kernels module.

Tolerances (north_star):
  * rendered intensities (fp32 tile kernel):  |I - I_ref| <= 1e-5 |I_ref| + 1e-9
  * gradients, per parameter array:           ||g - g_ref||_inf <= 1e-3 ||g_ref||_inf
  * float64 forward (render_batch / compute_loss / evaluate_field): rtol 1e-10
  * neighbour ids and (slice, tile) binning: exact
"""
import numpy as np
import pytest

from conftest import TRAIN_CASES, load_golden, loss_kwargs, output_prefix

pytestmark = pytest.mark.gpu

RENDER_RTOL, RENDER_ATOL, GRAD_TOL = 1e-5, 1e-9, 1e-3


@pytest.fixture(scope="module")
def g():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    import paper_2512_11624_b200 as pkg
    from paper_2512_11624_b200 import _native
    _native.lib()
    return pkg


def objects(g, d):
    batch = g.PointBatch(d["lifted"], d["slice_ids"].astype(np.int32), d["slice_ids"] * 0,
                         d["intensities_obs"].copy(), d["slice_to_stack"], d["stack_rotations"])
    field = g.GaussianField(d["means"], d["log_scales"], d["quaternions"], d["intensities"])
    states = g.SliceStates(d["slice_quaternions"], d["slice_translations"], d["log_sigma"], d["eta"])
    return batch, field, states


def assert_render(got, ref):
    err = np.abs(got - ref) - (RENDER_RTOL * np.abs(ref) + RENDER_ATOL)
    assert err.max() <= 0, f"render off by {np.max(np.abs(got - ref) / (np.abs(ref) + 1e-12)):.3e} rel"


def assert_grads(got, ref):
    for k, v in ref.items():
        scale = max(np.max(np.abs(v)), 1e-300)
        e = np.max(np.abs(np.asarray(got[k]) - v)) / scale
        assert e <= GRAD_TOL, f"gradient {k}: rel inf-norm error {e:.3e}"


@pytest.mark.parametrize("name", TRAIN_CASES)
def test_backward_matches_reference(g, name):
    d = load_golden(name)
    pre = output_prefix(name)
    batch, field, states = objects(g, d)
    cfg = g.LossConfig(**loss_kwargs(d, pre))
    terms, grads, I_hat = g.backward(batch, field, states, d["psf_diags"], cfg, d["nbr"])
    assert_render(I_hat, d[pre + "I_hat"])
    assert_grads(grads, {k[len(pre) + 5:]: d[k] for k in d if k.startswith(pre + "grad_")})
    for k in ("loss", "data_term", "reg_term", "outlier_term"):
        ref = float(d[pre + "term_" + k])
        assert abs(terms[k] - ref) <= 1e-5 * abs(ref) + 1e-9, k


@pytest.mark.parametrize("name", TRAIN_CASES)
def test_render_and_loss_float64(g, name):
    d = load_golden(name)
    pre = output_prefix(name)
    batch, field, states = objects(g, d)
    got = g.render_batch(batch, field, states, d["psf_diags"], d["nbr"])
    np.testing.assert_allclose(got, d[pre + "render"], rtol=1e-10, atol=1e-14)
    loss, _ = g.compute_loss(batch, field, states, d["psf_diags"], g.LossConfig(**loss_kwargs(d, pre)),
                             d["nbr"])
    assert abs(loss - float(d[pre + "loss_fwd"])) <= 1e-10 * abs(float(d[pre + "loss_fwd"]))


def test_frozen_oracle_constants(g):
    """/root/reference/pkg/tests/test_train.py:28-31 IHAT/DATA/TOTAL_ORACLE."""
    d = load_golden("train_frozen")
    batch, field, states = objects(g, d)
    I = g.render_batch(batch, field, states, d["psf_diags"], d["nbr"])
    np.testing.assert_allclose(I, (0.48293569946096643, 0.67596320104737873), rtol=1e-12)
    terms, _, I2 = g.backward(batch, field, states, d["psf_diags"], g.LossConfig(), d["nbr"])
    np.testing.assert_allclose(I2, (0.48293569946096643, 0.67596320104737873), rtol=1e-5)
    assert abs(terms["loss"] - 0.39812750158641236) < 1e-5 * 0.4


@pytest.mark.parametrize("name", ["train_grad_acc_s1", "train_medium_s0"])
def test_dropin_kernels_module(g, name):
    """kernels.train_step_backward / render_forward with the reference's own
    positional arguments and (B, ...) block buffers."""
    from paper_2512_11624_b200 import kernels
    d = load_golden(name)
    P, S, N = d["lifted"].shape[0], d["raw_Rc"].shape[0], d["means"].shape[0]
    B = kernels.default_block_count(P)
    I_hat, absres = np.empty(P), np.empty(P)
    bufs = [np.zeros((B, N, 3)), np.zeros((B, N, 6)), np.zeros((B, N)), np.zeros((B, S, 3)),
            np.zeros((B, S, 3, 3)), np.zeros((B, S, 6)), np.zeros((B, S))]
    kernels.train_step_backward(d["lifted"], d["slice_ids"].astype(np.int32), d["raw_Rc"],
                                d["slice_translations"], d["raw_psf6s"], d["raw_sigma_s"],
                                d["raw_wdata_s"], d["intensities_obs"], d["nbr"], d["means"],
                                d["raw_cov6"], d["intensities"], 1e-8, B, I_hat, absres, *bufs)
    assert_render(I_hat, d["raw_I_hat"])
    names = ["dmu", "dcov6", "dc", "dt", "dRc", "dpsf6", "dsigraw"]
    assert_grads({n: b.sum(axis=0) for n, b in zip(names, bufs)}, {n: d["raw_" + n] for n in names})
    # render_forward: per-point PSF and sigma, clamp semantics, float64
    sid = d["slice_ids"]
    Rc = d["raw_Rc"]
    X = np.einsum("pij,pj->pi", Rc[sid], d["lifted"]) + d["slice_translations"][sid]
    out = np.empty(P)
    kernels.render_forward(X, d["raw_psf6s"][sid], d["raw_sigma_s"][sid], d["nbr"], d["means"],
                           d["raw_cov6"], d["intensities"], 1e-8, out)
    pre = output_prefix(name)
    np.testing.assert_allclose(out, d[pre + "render"], rtol=1e-10, atol=1e-14)
    out32 = np.empty(P, dtype=np.float32)
    kernels.render_forward(X.astype(np.float32), d["raw_psf6s"][sid].astype(np.float32),
                           d["raw_sigma_s"][sid].astype(np.float32), d["nbr"], d["means"].astype(np.float32),
                           d["raw_cov6"].astype(np.float32), d["intensities"].astype(np.float32),
                           np.float32(1e-8), out32)
    np.testing.assert_allclose(out32, d[pre + "render"], rtol=1e-3, atol=1e-6)


def test_knn_exact(g):
    d = load_golden("knn_cases")
    for key in sorted(d):
        if "_K" not in key:
            continue
        case, K = key.split("_K")
        got = g.query(g.build_index(d[case + "_means"]), d[case + "_points"], int(K))
        np.testing.assert_array_equal(got, d[key], err_msg=key)


def test_knn_large_vs_oracle(g, oracle):
    rng = np.random.default_rng(7)
    # duplicated means + clustered density + queries outside the cloud
    base = rng.normal(scale=12.0, size=(6000, 3))
    means = np.concatenate([base, base[:2500], rng.uniform(-60, 60, (1500, 3))])
    pts = np.concatenate([rng.normal(scale=14.0, size=(20000, 3)), rng.uniform(-90, 90, (3000, 3)),
                          means[:2000]])
    got = g.query(g.build_index(means), pts, 50)
    np.testing.assert_array_equal(got, oracle.knn_query(means, pts, 50))


def test_knn_validation(g):
    idx = g.build_index(np.random.default_rng(0).normal(size=(10, 3)))
    with pytest.raises(g.InvalidParameterError):
        g.query(idx, np.zeros((1, 3)), 0)
    with pytest.raises(g.InvalidParameterError):
        g.query(idx, np.zeros((1, 3)), 11)
    assert g.query(idx, np.zeros((1, 3)), 10).shape == (1, 10)
    with pytest.raises(g.InvalidParameterError):
        g.build_index(np.array([[np.nan, 0, 0]]))


def test_evaluate_field(g):
    d = load_golden("misc_cases")
    f = g.GaussianField(d["ev_means"], d["ev_log_scales"], d["ev_quats"], d["ev_cvals"])
    got = g.evaluate_field(d["ev_points"], f, d["ev_nbr"])
    np.testing.assert_allclose(got, d["ev_out"], rtol=1e-10, atol=1e-15)


def test_binning_counts_exact(g):
    """(slice, tile) unique-Gaussian lists equal those derived on the host from
    the neighbour lists (ids ascending, counts bit-exact)."""
    from paper_2512_11624_b200.engine import DeviceBatch
    d = load_golden("train_medium_s1")
    batch, field, _ = objects(g, d)
    db = DeviceBatch(batch, K=50, tile_points=64)
    db.bin(d["nbr"], field.count)
    ts, tn, tsl, uoff, gid, perm = db.tile_info()
    assert sorted(perm.tolist()) == list(range(batch.n_points))
    assert np.all(np.diff(batch.slice_ids[perm]) >= 0)
    for t in range(len(ts)):
        rows = perm[ts[t]:ts[t] + tn[t]]
        assert np.all(batch.slice_ids[rows] == tsl[t])
        want = np.unique(d["nbr"][rows])
        np.testing.assert_array_equal(gid[uoff[t]:uoff[t + 1]], want)


def test_gradcheck_finite_differences(g):
    """tests/test_train.py:159-179 style: analytic (fp32 tile kernel) vs central
    differences of the float64 device loss."""
    d = load_golden("train_grad_unit_s0")
    batch, field, states = objects(g, d)
    cfg = g.LossConfig(**loss_kwargs(d))
    _, grads, _ = g.backward(batch, field, states, d["psf_diags"], cfg, d["nbr"])
    params = {"means": field.means, "log_scales": field.log_scales, "quaternions": field.quaternions,
              "intensities": field.intensities, "slice_quaternions": states.quaternions,
              "slice_translations": states.translations, "log_sigma": states.log_sigma,
              "eta": states.eta}
    worst = 0.0
    for name, arr in params.items():
        flat = arr.reshape(-1)
        for i in range(flat.size):
            h = 1e-6 * max(1.0, abs(flat[i]))
            keep = flat[i]
            flat[i] = keep + h
            up, _ = g.compute_loss(batch, field, states, d["psf_diags"], cfg, d["nbr"])
            flat[i] = keep - h
            down, _ = g.compute_loss(batch, field, states, d["psf_diags"], cfg, d["nbr"])
            flat[i] = keep
            fd = (up - down) / (2 * h)
            a = grads[name].reshape(-1)[i]
            worst = max(worst, abs(a - fd) / max(abs(a), abs(fd), 1e-6))
    assert worst < 1e-3, worst


def test_unused_primitive_zero_gradient(g):
    """tests/test_train.py:182-193."""
    d = load_golden("train_grad_unit_s1")
    batch, field, states = objects(g, d)
    nbr = np.where(d["nbr"] == 4, 3, d["nbr"])
    _, grads, _ = g.backward(batch, field, states, d["psf_diags"], g.LossConfig(lambda_reg=0.0), nbr)
    assert not grads["means"][4].any()
    assert not grads["log_scales"][4].any()
    assert not grads["quaternions"][4].any()
    assert grads["intensities"][4] == 0.0
    assert grads["means"][:4].any()


def test_error_contract(g):
    """train.py:155-169 messages and classes."""
    d = load_golden("train_frozen")
    batch, field, states = objects(g, d)
    bad = g.GaussianField(field.means, np.log(np.full((2, 3), 1e-4)), field.quaternions,
                          field.intensities)
    with pytest.raises(g.NumericalDegeneracyError, match="floor"):
        g.backward(batch, bad, states, d["psf_diags"], g.LossConfig(), d["nbr"])
    nanf = g.GaussianField(field.means, field.log_scales, field.quaternions, np.array([np.nan, 0.3]))
    with pytest.raises(g.TrainingDivergedError, match="slice 0"):
        g.render_batch(batch, nanf, states, d["psf_diags"], d["nbr"])
    with pytest.raises(g.TrainingDivergedError, match="slice 0"):
        g.backward(batch, nanf, states, d["psf_diags"], g.LossConfig(), d["nbr"])
    with pytest.raises(g.InvalidParameterError):
        g.backward(batch, field, states, d["psf_diags"], g.LossConfig(), np.array([[0, 5], [0, 1]]))


@pytest.mark.parametrize("name", ["train_medium_s0", "train_medium_s1", "train_grad_acc_s3"])
def test_planar_and_general_kernels_agree(g, name):
    """The slice-plane kernel (2D conditional form) and the general 3D tile kernel
    give the same render and gradients (both vs the reference)."""
    from paper_2512_11624_b200._native import lib
    from paper_2512_11624_b200.engine import DeviceBatch
    d = load_golden(name)
    batch, field, states = objects(g, d)
    db = DeviceBatch(batch, K=d["nbr"].shape[1])
    assert lib().gsvr_batch_is_planar(db.raw) == 1
    cfg = g.LossConfig(**loss_kwargs(d))
    out = []
    for general in (0, 1):
        lib().gsvr_set_kernel_variant(general)
        try:
            out.append(g.backward(batch, field, states, d["psf_diags"], cfg, d["nbr"]))
        finally:
            lib().gsvr_set_kernel_variant(0)
    for terms, grads, I_hat in out:
        assert_render(I_hat, d["I_hat"])
        assert_grads(grads, {k[5:]: d[k] for k in d if k.startswith("grad_")})


def test_nonplanar_points_use_general_kernel(g, oracle):
    """Arbitrary (non-coplanar) points through the drop-in kernel API."""
    from paper_2512_11624_b200 import kernels
    from paper_2512_11624_b200._native import lib
    from paper_2512_11624_b200.engine import DeviceBatch
    rng = np.random.default_rng(3)
    P, S, N, K = 3000, 4, 300, 20
    x0 = rng.uniform(-6, 6, size=(P, 3))
    sid = np.sort(rng.integers(0, S, size=P)).astype(np.int32)
    mu = rng.uniform(-6, 6, size=(N, 3))
    ls = np.log(rng.uniform(0.6, 1.6, size=(N, 3)))
    q = rng.normal(size=(N, 4))
    c = rng.uniform(0.1, 0.9, size=N)
    cov6 = oracle.covariances6(ls, q)
    qs = rng.normal(scale=0.02, size=(S, 4)) + [1, 0, 0, 0]
    Rc = oracle.quat_to_rotation(qs)
    tv = rng.normal(scale=0.3, size=(S, 3))
    psf6s = oracle.pack_sym6(np.einsum("sik,k,sjk->sij", Rc, [0.1, 0.1, 0.8], Rc))
    sig = np.exp(rng.normal(scale=0.05, size=S))
    w = np.exp(-rng.normal(scale=0.2, size=S))
    X = np.einsum("pij,pj->pi", Rc[sid], x0) + tv[sid]
    nbr = oracle.knn_query(mu, X, K)
    I_ref0 = oracle.render_forward(X, psf6s[sid], sig[sid], nbr, mu, cov6, c)
    I_obs = I_ref0 + np.where(rng.random(P) < 0.5, -1, 1) * rng.uniform(0.02, 0.2, P)
    b = g.PointBatch(x0, sid, sid * 0, I_obs, np.zeros(S, np.int32), np.eye(3)[None])
    db = DeviceBatch(b, K=K)
    assert lib().gsvr_batch_is_planar(db.raw) == 0
    I_ref, _, gr = oracle.train_step_backward(x0, sid, Rc, tv, psf6s, sig, w, I_obs, nbr, mu, cov6, c)
    I_hat, absres = np.empty(P), np.empty(P)
    bufs = [np.zeros((1, N, 3)), np.zeros((1, N, 6)), np.zeros((1, N)), np.zeros((1, S, 3)),
            np.zeros((1, S, 3, 3)), np.zeros((1, S, 6)), np.zeros((1, S))]
    kernels.train_step_backward(x0, sid, Rc, tv, psf6s, sig, w, I_obs, nbr, mu, cov6, c, 1e-8, 1,
                                I_hat, absres, *bufs)
    assert_render(I_hat, I_ref)
    names = ["dmu", "dcov6", "dc", "dt", "dRc", "dpsf6", "dsigraw"]
    assert_grads({n: b_[0] for n, b_ in zip(names, bufs)}, {n: gr[n] for n in names})


def test_refresh_seeded_matches_oracle(g, oracle):
    """Device refresh (K-NN of the motion-corrected points + binning) against the
    oracle's exact K-NN, over a sequence of refreshes: the 2nd.. refreshes prune
    with the previous lists (seeds); means move, collapse onto a lattice (ties)
    and duplicate between refreshes, slices move, and N changes (seeds dropped)."""
    import torch
    from paper_2512_11624_b200._native import lib
    from paper_2512_11624_b200.engine import DeviceBatch
    from paper_2512_11624_b200.knn import NeighborIndex, _build_handle
    rng = np.random.default_rng(11)
    S, n, K = 3, 24, 12
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    x0 = np.concatenate([np.stack([ii.ravel() * 0.8 - 9, jj.ravel() * 0.8 - 9, np.full(n * n, 3.0 * s - 3)], 1)
                         for s in range(S)])
    sid = np.repeat(np.arange(S), n * n).astype(np.int32)
    b = g.PointBatch(x0, sid, sid * 0, rng.random(len(x0)), np.zeros(S, np.int32), np.eye(3)[None])
    db = DeviceBatch(b, K=K)
    N = 400
    mu = rng.uniform(-10, 10, size=(N, 3))
    for step in range(6):
        if step == 2:   # lattice means: many exact distance ties
            mu = np.round(mu / 2.0) * 2.0
        if step == 3:   # duplicated means
            mu[: N // 4] = mu[N // 4: N // 2]
        if step == 5:   # different N: seeds must be dropped
            mu = np.concatenate([mu, rng.uniform(-10, 10, size=(37, 3))])
        qs = rng.normal(scale=0.03, size=(S, 4)) + [1, 0, 0, 0]
        Rc = oracle.quat_to_rotation(qs)
        tv = rng.normal(scale=0.4, size=(S, 3))
        mud = torch.from_numpy(mu).cuda()
        index = NeighborIndex(np.empty((len(mu), 3)), _build_handle(mud))
        db.refresh(index, K, torch.from_numpy(Rc).cuda().contiguous(), torch.from_numpy(tv).cuda())
        R = Rc[sid]  # train.py:305-309 order: ((R0 a0 + R1 a1) + R2 a2) + t
        X = ((R[:, :, 0] * x0[:, :1] + R[:, :, 1] * x0[:, 1:2]) + R[:, :, 2] * x0[:, 2:]) + tv[sid]
        got = db.neighbors().cpu().numpy()
        np.testing.assert_array_equal(got, oracle.knn_query(mu, X, K), err_msg=f"refresh {step}")
        fb = int(lib().gsvr_batch_knn_fallback_rows(db.raw))
        print(f"refresh {step}: selection-kernel fallback rows {fb} of {len(x0)}")
        if step in (1, 4):  # seeded, same N: the heap-free selection kernel ran
            assert 0 <= fb < len(x0)
        mu = mu + rng.normal(scale=0.3, size=mu.shape)


@pytest.mark.parametrize("case", ["a", "b", "c"])
def test_rasterize_matches_reference(g, case):
    """HR export: field.py:138-175 on rotated grids, masked /
    unmasked, with a rigid transform, K < N and K > N (clipped), vs the
    reference's own rasterize output (tests/golden/export_cases.npz)."""
    d = load_golden("export_cases")
    p = case + "_"
    f = g.GaussianField(d[p + "means"], d[p + "log_scales"], d[p + "quats"], d[p + "cvals"])
    ref = d[p + "out"]
    grid = g.VolumeGrid(np.zeros(ref.shape), d[p + "affine"], d.get(p + "mask"))
    tr = (d[p + "R"], d[p + "t"]) if (p + "R") in d else None
    got = g.rasterize(f, grid, int(d[p + "K"]), transform=tr)
    np.testing.assert_allclose(got.data, ref, rtol=1e-10, atol=1e-15)


@pytest.mark.parametrize("pinned,raw_every", [(False, "3"), (True, "3"), (True, "0"), (True, "1")])
def test_dropin_host_path_matches_device_path(g, pinned, raw_every, monkeypatch):
    """kernels.train_step_backward with host buffers (gsvr_train_step_backward_host:
    int64 ids narrowed on host threads and/or on the device, chunked upload
    overlapped with planning and per-tile binning) gives the same bits as the
    CUDA-tensor path, and accumulates into the caller's block-0 buffers."""
    import torch
    from paper_2512_11624_b200 import kernels
    from paper_2512_11624_b200.knn import build_index, query
    monkeypatch.setenv("GSVR_UPLOAD_CHUNK_MB", "4")  # many chunks at test size
    monkeypatch.setenv("GSVR_RAW_EVERY", raw_every)  # 0: all host-narrowed, 1: all device-narrowed
    rng = np.random.default_rng(21)
    S, n, K, N = 6, 96, 20, 3000
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    x0 = np.concatenate([np.stack([ii.ravel() * 0.7 - 33, jj.ravel() * 0.7 - 33, np.full(n * n, 2.5 * s - 6)], 1)
                         for s in range(S)])
    sid = np.repeat(np.arange(S), n * n).astype(np.int32)
    P = len(sid)
    mu = rng.uniform(-35, 35, size=(N, 3)) * [1, 1, 0.3]
    cov6 = np.tile([2.0, 0.1, 0.0, 1.5, 0.05, 1.2], (N, 1)) * rng.uniform(0.5, 1.5, size=(N, 1))
    c = rng.uniform(0.1, 0.9, size=N)
    Rc = np.tile(np.eye(3), (S, 1, 1))
    tv = rng.normal(scale=0.2, size=(S, 3))
    psf6s = np.tile([0.3, 0, 0, 0.3, 0, 1.1], (S, 1))
    sig, w = np.ones(S), np.ones(S)
    I_obs = rng.uniform(0, 1, size=P)
    nbr = query(build_index(mu), x0 + tv[sid], K)
    shapes = [(1, N, 3), (1, N, 6), (1, N), (1, S, 3), (1, S, 3, 3), (1, S, 6), (1, S)]
    pre = [rng.normal(size=s) for s in shapes]  # accumulate semantics

    def run(conv):
        I_hat, absres = conv(np.zeros(P)), conv(np.zeros(P))
        bufs = [conv(p.copy()) for p in pre]
        kernels.train_step_backward(*[conv(a) for a in (x0, sid, Rc, tv, psf6s, sig, w, I_obs, nbr, mu, cov6, c)],
                                    1e-8, 1, I_hat, absres, *bufs)
        tonp = lambda a: a.cpu().numpy() if hasattr(a, "cpu") else a
        return tonp(I_hat), [tonp(b) for b in bufs]

    host = (lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()) if pinned else (lambda a: a)
    I_h, g_h = run(host)
    I_d, g_d = run(lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda())
    np.testing.assert_array_equal(I_h, I_d)
    for a, b_ in zip(g_h, g_d):
        np.testing.assert_array_equal(a, b_)
    assert np.abs(g_h[0] - pre[0]).max() > 0  # gradients were added to the prefilled block


@pytest.mark.parametrize("raw_every", ["0", "1"])
@pytest.mark.parametrize("bad_id", ["N", "2**32+1", "-1"])
def test_dropin_host_path_rejects_bad_ids(g, bad_id, raw_every, monkeypatch):
    """int64 neighbour ids are narrowed to int32 on host threads before the
    upload; an id outside [0, N) -- including one that only differs in the high
    word -- must still raise InvalidParameterError (status 1)."""
    from paper_2512_11624_b200 import kernels
    monkeypatch.setenv("GSVR_UPLOAD_CHUNK_MB", "1")
    monkeypatch.setenv("GSVR_RAW_EVERY", raw_every)
    rng = np.random.default_rng(5)
    S, n, K, N = 2, 32, 8, 200
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    x0 = np.concatenate([np.stack([ii.ravel() * 0.7 - 11, jj.ravel() * 0.7 - 11, np.full(n * n, 2.5 * s)], 1)
                         for s in range(S)])
    sid = np.repeat(np.arange(S), n * n).astype(np.int32)
    P = len(sid)
    mu = rng.uniform(-12, 12, size=(N, 3))
    cov6 = np.tile([2.0, 0.1, 0.0, 1.5, 0.05, 1.2], (N, 1))
    nbr = np.stack([rng.choice(N, K, replace=False) for _ in range(P)]).astype(np.int64)
    nbr[P // 2, 3] = {"N": N, "2**32+1": 2 ** 32 + 1, "-1": -1}[bad_id]
    args = (x0, sid, np.tile(np.eye(3), (S, 1, 1)), np.zeros((S, 3)), np.tile([0.3, 0, 0, 0.3, 0, 1.1], (S, 1)),
            np.ones(S), np.ones(S), rng.uniform(size=P), nbr, mu, cov6, rng.uniform(0.1, 0.9, size=N))
    bufs = [np.zeros(s) for s in [(1, N, 3), (1, N, 6), (1, N), (1, S, 3), (1, S, 3, 3), (1, S, 6), (1, S)]]
    with pytest.raises(g.InvalidParameterError):
        kernels.train_step_backward(*args, 1e-8, 1, np.zeros(P), np.zeros(P), *bufs)
    nbr[P // 2, 3] = (nbr[P // 2, 3] + 1) % N if bad_id == "-1" else 0  # repaired: runs
    nbr[P // 2] = rng.choice(N, K, replace=False)
    kernels.train_step_backward(*args, 1e-8, 1, np.zeros(P), np.zeros(P), *bufs)


def test_staleness_displacement_exact(g, oracle):
    """gsvr_batch_displacement (train.py:457-461: max_p |x_a - x_b|^2, x = Rc x0 + t)
    scans only tiles whose bound reaches the best exact value; it must equal
    the full scan bit for bit."""
    import torch
    from paper_2512_11624_b200 import _dev
    from paper_2512_11624_b200._native import check, lib
    from paper_2512_11624_b200.engine import DeviceBatch
    rng = np.random.default_rng(8)
    S, n = 5, 40
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    x0 = np.concatenate([np.stack([ii.ravel() * 0.9 - 18, jj.ravel() * 0.9 - 18, np.full(n * n, 3.0 * s - 6)], 1)
                         for s in range(S)])
    x0 = x0 + rng.normal(scale=0.05, size=x0.shape) * (np.arange(len(x0)) % 7 == 0)[:, None]  # off-plane too
    sid = np.repeat(np.arange(S), n * n).astype(np.int32)
    b = g.PointBatch(x0, sid, sid * 0, rng.random(len(x0)), np.zeros(S, np.int32), np.eye(3)[None])
    db = DeviceBatch(b, K=8)
    for scale in (0.0, 1e-4, 0.02, 0.3):
        Ra = oracle.quat_to_rotation(rng.normal(scale=scale, size=(S, 4)) + [1, 0, 0, 0])
        Rb = oracle.quat_to_rotation(rng.normal(scale=scale, size=(S, 4)) + [1, 0, 0, 0])
        ta, tb = rng.normal(scale=scale, size=(S, 3)), rng.normal(scale=scale, size=(S, 3))
        if scale == 0.0:
            Rb, tb = Ra.copy(), ta.copy()

        def X(R, t):
            A = R[sid]
            return ((A[:, :, 0] * x0[:, :1] + A[:, :, 1] * x0[:, 1:2]) + A[:, :, 2] * x0[:, 2:]) + t[sid]
        d = X(Ra, ta) - X(Rb, tb)
        want = np.max((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])
        out = torch.zeros(1, dtype=torch.float64, device="cuda")
        dv = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (Ra, ta, Rb, tb)]
        check(lib().gsvr_batch_displacement(db.raw, *map(_dev.ptr, dv), _dev.ptr(out), _dev.stream_ptr()))
        assert out.item() == want, (scale, out.item(), want)


def test_hash_binning_equals_sort_binning():
    """The hash + pixel-mask binning kernel produces the sorting kernel's
    unique lists, CSR, pair lists and pixel-major local ids bit for bit (tiles
    with a repeated id in a row go to the sort): identical tile lists and
    identical tile-kernel outputs under GSVR_BIN_SORT=0 (hash) and =1 (sort)."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path
    code = r"""
import hashlib, json, os, sys, numpy as np, torch
sys.path.insert(0, %r)
sys.path.insert(0, os.path.dirname(sys.path[0]))
import paper_2512_11624_b200 as g
from conftest import load_golden
from paper_2512_11624_b200 import kernels
from paper_2512_11624_b200.engine import DeviceBatch
d = load_golden("train_medium_s1")
nbr = d["nbr"].copy()
nbr[5, 3] = nbr[5, 4]  # a repeated id in one row
b = g.PointBatch(d["lifted"], d["slice_ids"].astype(np.int32), d["slice_ids"] * 0, d["intensities_obs"],
                 d["slice_to_stack"], d["stack_rotations"])
out = {}
for name, rows in (("clean", d["nbr"]), ("dup", nbr)):
    db = DeviceBatch(b, K=50, tile_points=64)
    db.bin(rows, d["means"].shape[0])
    ts, tn, tsl, uoff, gid, perm = db.tile_info()
    P, S, N = d["lifted"].shape[0], d["raw_Rc"].shape[0], d["means"].shape[0]
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    I_hat, absres = cu(np.zeros(P)), cu(np.zeros(P))
    bufs = [cu(np.zeros(s)) for s in [(1, N, 3), (1, N, 6), (1, N), (1, S, 3), (1, S, 3, 3), (1, S, 6), (1, S)]]
    kernels.train_step_backward(*[cu(a) for a in (d["lifted"], d["slice_ids"].astype(np.int32), d["raw_Rc"],
                                d["slice_translations"], d["raw_psf6s"], d["raw_sigma_s"], d["raw_wdata_s"],
                                d["intensities_obs"], rows, d["means"], d["raw_cov6"], d["intensities"])],
                                1e-8, 1, I_hat, absres, *bufs)
    h = hashlib.sha256()
    for t in [I_hat] + bufs:
        h.update(t.cpu().numpy().tobytes())
    out[name] = [uoff.tolist(), gid.tolist(), h.hexdigest()]
print(json.dumps(out))
"""
    root = str(Path(__file__).resolve().parent)
    env = dict(os.environ)
    res = []
    for mode in ("0", "1"):
        env["GSVR_BIN_SORT"] = mode
        r = subprocess.run([sys.executable, "-c", code % root], capture_output=True, text=True, env=env,
                           cwd=root, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert res[0] == res[1]


@pytest.mark.parametrize("K", [1, 2, 7, 96])
def test_dropin_unusual_K_vs_oracle(g, oracle, K):
    """kernels.train_step_backward at K = 1, 2, an odd K and K = 96 (pairs per
    tile above the shared-memory sort's 12,800 -> the segmented-sort binning
    path) against the oracle.  At K = 1 the model is degenerate: the render is
    sigma c e / (e + delta) and every position gradient is proportional to
    delta / e, far below fp32 resolution of the (c - ratio) factor, so only the
    render is compared there."""
    from paper_2512_11624_b200 import kernels
    rng = np.random.default_rng(30 + K)
    S, n, N = 3, 40, 500
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    x0 = np.concatenate([np.stack([ii.ravel() * 0.8 - 16, jj.ravel() * 0.8 - 16, np.full(n * n, 3.0 * s - 3)], 1)
                         for s in range(S)])
    sid = np.repeat(np.arange(S), n * n).astype(np.int32)
    P = len(sid)
    mu = rng.uniform(-17, 17, size=(N, 3)) * [1, 1, 0.4]
    ls = np.log(rng.uniform(0.6, 1.8, size=(N, 3)))
    q = rng.normal(size=(N, 4))
    c = rng.uniform(-0.3, 0.9, size=N)
    cov6 = oracle.covariances6(ls, q)
    qs = rng.normal(scale=0.02, size=(S, 4)) + [1, 0, 0, 0]
    Rc = oracle.quat_to_rotation(qs)
    tv = rng.normal(scale=0.3, size=(S, 3))
    psf6s = oracle.pack_sym6(np.einsum("sik,k,sjk->sij", Rc, [0.1, 0.1, 0.8], Rc))
    sig = np.exp(rng.normal(scale=0.05, size=S))
    w = np.exp(-rng.normal(scale=0.2, size=S))
    R = Rc[sid]
    X = ((R[:, :, 0] * x0[:, :1] + R[:, :, 1] * x0[:, 1:2]) + R[:, :, 2] * x0[:, 2:]) + tv[sid]
    nbr = oracle.knn_query(mu, X, K)
    I0 = oracle.render_forward(X, psf6s[sid], sig[sid], nbr, mu, cov6, c)
    I_obs = I0 + np.where(rng.random(P) < 0.5, -1, 1) * rng.uniform(0.02, 0.2, P)
    I_ref, _, gr = oracle.train_step_backward(x0, sid, Rc, tv, psf6s, sig, w, I_obs, nbr, mu, cov6, c)
    I_abs, _, _ = oracle.train_step_backward(x0, sid, Rc, tv, psf6s, sig, w, I_obs, nbr, mu, cov6, np.abs(c))
    I_hat, absres = np.empty(P), np.empty(P)
    bufs = [np.zeros((1, N, 3)), np.zeros((1, N, 6)), np.zeros((1, N)), np.zeros((1, S, 3)),
            np.zeros((1, S, 3, 3)), np.zeros((1, S, 6)), np.zeros((1, S))]
    kernels.train_step_backward(x0, sid, Rc, tv, psf6s, sig, w, I_obs, nbr, mu, cov6, c, 1e-8, 1,
                                I_hat, absres, *bufs)
    assert (np.abs(I_hat - I_ref) <= RENDER_RTOL * np.abs(I_abs) + RENDER_ATOL).all()
    if K > 1:
        names = ["dmu", "dcov6", "dc", "dt", "dRc", "dpsf6", "dsigraw"]
        assert_grads({n: b_[0] for n, b_ in zip(names, bufs)}, {n: gr[n] for n in names})


def test_dropin_ragged_slices_vs_oracle(g, oracle):
    """Ragged batch through kernels.train_step_backward: a 1-pixel slice, an
    empty slice (no points at all), a slice one pixel over a tile (257) and a
    large one, points in shuffled caller order (kernels.py takes any order);
    render and gradients vs the oracle, and the empty slice's gradients exactly 0."""
    from paper_2512_11624_b200 import kernels
    rng = np.random.default_rng(77)
    S, N, K = 4, 300, 12
    counts = [1, 0, 257, 700]
    pts, sids = [], []
    for s, cnt in enumerate(counts):
        if cnt == 0:
            continue
        side = int(np.ceil(np.sqrt(cnt)))
        ii, jj = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
        xy = np.stack([ii.ravel(), jj.ravel()], 1)[:cnt] * 0.7 - 0.35 * side
        pts.append(np.concatenate([xy, np.full((cnt, 1), 2.5 * s - 4.0)], 1))
        sids.append(np.full(cnt, s))
    x0 = np.concatenate(pts)
    sid = np.concatenate(sids).astype(np.int32)
    order = rng.permutation(len(sid))
    x0, sid = np.ascontiguousarray(x0[order]), np.ascontiguousarray(sid[order])
    P = len(sid)
    mu = rng.uniform(-10, 10, size=(N, 3)) * [1, 1, 0.6]
    ls = np.log(rng.uniform(0.6, 1.8, size=(N, 3)))
    c = rng.uniform(0.1, 0.9, size=N)
    cov6 = oracle.covariances6(ls, rng.normal(size=(N, 4)))
    qs = rng.normal(scale=0.02, size=(S, 4)) + [1, 0, 0, 0]
    Rc = oracle.quat_to_rotation(qs)
    tv = rng.normal(scale=0.3, size=(S, 3))
    psf6s = oracle.pack_sym6(np.einsum("sik,k,sjk->sij", Rc, [0.1, 0.1, 0.8], Rc))
    sig, w = np.exp(rng.normal(scale=0.05, size=S)), np.exp(-rng.normal(scale=0.2, size=S))
    R = Rc[sid]
    X = ((R[:, :, 0] * x0[:, :1] + R[:, :, 1] * x0[:, 1:2]) + R[:, :, 2] * x0[:, 2:]) + tv[sid]
    nbr = oracle.knn_query(mu, X, K)
    I0 = oracle.render_forward(X, psf6s[sid], sig[sid], nbr, mu, cov6, c)
    I_obs = I0 + np.where(rng.random(P) < 0.5, -1, 1) * rng.uniform(0.02, 0.2, P)
    I_ref, _, gr = oracle.train_step_backward(x0, sid, Rc, tv, psf6s, sig, w, I_obs, nbr, mu, cov6, c)
    I_hat, absres = np.empty(P), np.empty(P)
    bufs = [np.zeros((1, N, 3)), np.zeros((1, N, 6)), np.zeros((1, N)), np.zeros((1, S, 3)),
            np.zeros((1, S, 3, 3)), np.zeros((1, S, 6)), np.zeros((1, S))]
    kernels.train_step_backward(x0, sid, Rc, tv, psf6s, sig, w, I_obs, nbr, mu, cov6, c, 1e-8, 1,
                                I_hat, absres, *bufs)
    assert (np.abs(I_hat - I_ref) <= RENDER_RTOL * np.abs(I_ref) + RENDER_ATOL).all()
    names = ["dmu", "dcov6", "dc", "dt", "dRc", "dpsf6", "dsigraw"]
    assert_grads({n: b_[0] for n, b_ in zip(names, bufs)}, {n: gr[n] for n in names})
    for b_ in bufs[3:]:
        assert not np.any(b_[0][1])  # the empty slice


def test_dropin_multipage_tile_vs_oracle(g, oracle):
    """A tile whose unique-Gaussian list exceeds one shared-memory record page
    (> 1,536 Gaussians: 256 pixels 6 mm apart, K = 96 out of 30,000): the hash
    binning overflows to the sort, the tile kernel stages its records through
    the global pages and accumulates the partials with atomics.  vs the oracle."""
    from paper_2512_11624_b200 import kernels
    rng = np.random.default_rng(91)
    S, N, K, n = 1, 30000, 96, 16
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    x0 = np.stack([ii.ravel() * 6.0 - 45, jj.ravel() * 6.0 - 45, np.zeros(n * n)], 1)
    sid = np.zeros(n * n, np.int32)
    P = len(sid)
    mu = rng.uniform(-50, 50, size=(N, 3)) * [1, 1, 0.05]
    ls = np.log(rng.uniform(0.6, 1.5, size=(N, 3)))
    c = rng.uniform(0.1, 0.9, size=N)
    cov6 = oracle.covariances6(ls, rng.normal(size=(N, 4)))
    Rc, tv = np.eye(3)[None].copy(), np.zeros((1, 3))
    psf6s = oracle.pack_sym6(np.diag([0.1, 0.1, 0.8])[None])
    sig, w = np.ones(1), np.ones(1)
    nbr = oracle.knn_query(mu, x0, K)
    assert len(np.unique(nbr)) > 1536
    I0 = oracle.render_forward(x0, psf6s[sid], sig[sid], nbr, mu, cov6, c)
    I_obs = I0 + np.where(rng.random(P) < 0.5, -1, 1) * rng.uniform(0.02, 0.2, P)
    I_ref, _, gr = oracle.train_step_backward(x0, sid, Rc, tv, psf6s, sig, w, I_obs, nbr, mu, cov6, c)
    I_hat, absres = np.empty(P), np.empty(P)
    bufs = [np.zeros((1, N, 3)), np.zeros((1, N, 6)), np.zeros((1, N)), np.zeros((1, S, 3)),
            np.zeros((1, S, 3, 3)), np.zeros((1, S, 6)), np.zeros((1, S))]
    kernels.train_step_backward(x0, sid, Rc, tv, psf6s, sig, w, I_obs, nbr, mu, cov6, c, 1e-8, 1,
                                I_hat, absres, *bufs)
    assert (np.abs(I_hat - I_ref) <= RENDER_RTOL * np.abs(I_ref) + RENDER_ATOL).all()
    names = ["dmu", "dcov6", "dc", "dt", "dRc", "dpsf6", "dsigraw"]
    assert_grads({n_: b_[0] for n_, b_ in zip(names, bufs)}, {n_: gr[n_] for n_ in names})


@pytest.mark.parametrize("name", ["train_medium_s0", "train_medium_s1"])
def test_backward_records_in_global_memory(g, name):
    """The large-tile configuration of the planar kernel (backward record halves
    in global memory, chosen when shared memory would cut residency, e.g. cfg4)
    forced on the reference goldens: same parity bounds."""
    from paper_2512_11624_b200._native import lib
    d = load_golden(name)
    batch, field, states = objects(g, d)
    cfg = g.LossConfig(**loss_kwargs(d, ""))
    lib().gsvr_set_kernel_variant(2)
    try:
        terms, grads, I_hat = g.backward(batch, field, states, d["psf_diags"], cfg, d["nbr"])
    finally:
        lib().gsvr_set_kernel_variant(0)
    assert_render(I_hat, d["I_hat"])
    assert_grads(grads, {k[5:]: d[k] for k in d if k.startswith("grad_")})


def test_dropin_concurrent_calls_from_threads(g, oracle):
    """kernels.train_step_backward with host buffers called from two Python
    threads at once (ctypes releases the GIL): the per-device lock serialises
    the calls, so each gets exactly the result of a lone call."""
    import threading
    from paper_2512_11624_b200 import kernels
    names = ["train_medium_s0", "train_medium_s1"]
    args, lone = [], []
    for name in names:
        d = load_golden(name)
        S = len(d["slice_to_stack"])
        Rc, _, psf6s, sig = oracle.slice_inputs(d["slice_quaternions"], d["stack_rotations"], d["slice_to_stack"],
                                                d["log_sigma"], d["psf_diags"])
        cov6 = oracle.covariances6(d["log_scales"], d["quaternions"])
        a = [d["lifted"], d["slice_ids"], Rc, d["slice_translations"], psf6s, sig, np.ones(S),
             d["intensities_obs"], d["nbr"], d["means"], cov6, d["intensities"]]
        args.append(a)

    def call(a):
        P, N, S = len(a[0]), len(a[9]), len(a[2])
        I_hat, absres = np.empty(P), np.empty(P)
        bufs = [np.zeros((1, N, 3)), np.zeros((1, N, 6)), np.zeros((1, N)), np.zeros((1, S, 3)),
                np.zeros((1, S, 3, 3)), np.zeros((1, S, 6)), np.zeros((1, S))]
        kernels.train_step_backward(*a, 1e-8, 1, I_hat, absres, *bufs)
        return I_hat, bufs

    lone = [call(a) for a in args]
    out = [None, None]

    def worker(i):
        for _ in range(5):
            out[i] = call(args[i])

    th = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for (I0, b0), (I1, b1) in zip(lone, out):
        assert np.array_equal(I0, I1)
        for x, y in zip(b0, b1):
            assert np.array_equal(x, y)
