"""Device-resident fit loop: one-epoch parity with the oracle (backward + AdamW)
and the reference's fit-loop behaviour tests (/root/reference/pkg/tests/
test_train.py:196-355), with fp32-appropriate floors where the reference
asserts float64 exactness."""
import numpy as np
import pytest

from conftest import load_golden, loss_kwargs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g():
    import torch
    assert torch.cuda.is_available()
    import paper_2512_11624_b200 as pkg
    return pkg


def _self_consistency_fixture(g):
    """tests/test_train.py:196-214: one primitive, a stack of its own rendering."""
    truth = g.GaussianField(means=[[0.1, -0.2, 0.3]], log_scales=np.log([[2.0, 1.7, 2.3]]),
                            quaternions=[[1.0, 0, 0, 0]], intensities=[0.7])
    affine = np.diag([1.0, 1.0, 2.0, 1.0])
    affine[:3, 3] = [-4.0, -4.0, -2.0]
    shell = g.SliceStack(data=np.zeros((9, 9, 3)), affine=affine, inplane_spacing=1.0, thickness=2.0)
    batch = g.build_point_batch([shell])
    psf = g.slice_psf_diags(batch, [shell])
    nbr = np.zeros((batch.n_points, 1), dtype=np.int64)
    vals = g.render_batch(batch, truth, g.init_states([shell]), psf, nbr)
    # The reference writes ``data[shell.mask] = vals``, which fills the raster in
    # C order (slice index fastest) while the batch is slice-major
    # (motion.py:210-237): its "own rendering" is a permutation of the render,
    # off by up to ~2e-6 relative.  Written back in batch order here, so the
    # data IS the rendering and the fixed point is exact.
    data = np.zeros((9, 9, 3))
    i = 0
    for k in range(3):
        uu, vv = np.nonzero(shell.mask[:, :, k])
        data[uu, vv, k] = vals[i:i + len(uu)]
        i += len(uu)
    return truth, g.SliceStack(data=data, affine=affine, inplane_spacing=1.0, thickness=2.0)


def _frozen(g, epochs, **kw):
    kw.setdefault("scheduler", g.SchedulerConfig(factor=0.5, every=20))
    return g.OptimConfig(epochs=epochs, k_neighbors=1, motion_warmup=10 ** 6,
                         rotation_warmup=10 ** 6, reseed_every=0, **kw)


def test_one_epoch_matches_oracle_step(g, oracle):
    """FitEngine epoch == reference backward (train.py:220-302) + AdamW step
    (optim.py:69-88) for field and slices, from the same start."""
    from paper_2512_11624_b200.engine import DeviceBatch, FitEngine
    d = load_golden("train_medium_s1")
    kw = loss_kwargs(d)
    batch = g.PointBatch(d["lifted"], d["slice_ids"].astype(np.int32), d["slice_ids"] * 0,
                         d["intensities_obs"], d["slice_to_stack"], d["stack_rotations"])
    field = g.GaussianField(d["means"].copy(), d["log_scales"].copy(), d["quaternions"].copy(),
                            d["intensities"].copy())
    states = g.SliceStates(d["slice_quaternions"], d["slice_translations"], d["log_sigma"], d["eta"])
    ocfg = g.OptimConfig(epochs=1, motion_warmup=0, rotation_warmup=0, reseed_every=0)
    db = DeviceBatch(batch, K=50)
    db.bin(d["nbr"], field.count)
    eng = FitEngine(db, field, states, d["psf_diags"], g.LossConfig(**kw), ocfg)
    terms = eng.epoch(1.0, True, False, None)
    ref_terms, grads, _ = oracle.backward(d, **kw)
    for k in ("loss", "data_term", "reg_term", "outlier_term"):
        assert abs(terms[k] - ref_terms[k]) <= 1e-5 * abs(ref_terms[k]) + 1e-9, k
    # reference AdamW step on float64 copies
    fp = {"means": d["means"].copy(), "log_scales": d["log_scales"].copy(),
          "quaternions": d["quaternions"].copy(), "intensities": d["intensities"].copy()}
    sp = {"slice_quaternions": d["slice_quaternions"].copy(),
          "slice_translations": d["slice_translations"].copy(),
          "log_sigma": d["log_sigma"].copy(), "eta": d["eta"].copy()}
    for params, lrs in ((fp, ocfg.field_lrs()), (sp, ocfg.slice_lrs())):
        m = {k: np.zeros_like(v) for k, v in params.items()}
        v = {k: np.zeros_like(x) for k, x in params.items()}
        oracle.adamw_step(params, {k: grads[k] for k in params}, m, v, 0, lrs)
    got_f, got_s = eng.field_host(), eng.states_host()
    got = {"means": got_f.means, "log_scales": got_f.log_scales, "quaternions": got_f.quaternions,
           "intensities": got_f.intensities, "slice_quaternions": got_s.quaternions,
           "slice_translations": got_s.translations, "log_sigma": got_s.log_sigma, "eta": got_s.eta}
    lrs = {**ocfg.field_lrs(), **ocfg.slice_lrs()}
    for name, ref in {**fp, **sp}.items():
        gr = np.asarray(grads[name])
        # first Adam step moves each entry by lr * g/(|g| + eps): exact where the
        # gradient is resolved; an entry whose |g| is at the fp32 noise floor may flip
        resolved = np.abs(gr) > 1e-4 * np.abs(gr).max()
        err = np.abs(got[name] - ref)
        assert np.all(err[resolved] <= 1e-3 * lrs[name] + 1e-12), name
        assert np.all(err <= 2 * lrs[name] + 1e-12), name


def test_own_rendering_is_a_training_fixed_point(g):
    """tests/test_train.py:223-230, with the reference's own bound (data term
    < 1e-9): residuals inside the fp32 render tolerance are re-rendered in
    float64 (batch.cuh pixel_l1), so the exact fit stays put."""
    truth, stack = _self_consistency_fixture(g)
    _, _, hist = g.fit([stack], loss_cfg=g.LossConfig(lambda_reg=0.0), optim_cfg=_frozen(g, 200),
                       field=truth.astype(np.float64))
    assert max(h["data_term"] for h in hist) < 1e-9


def test_fit_recovers_own_rendering_from_perturbed_start(g):
    """tests/test_train.py:233-249."""
    truth, stack = _self_consistency_fixture(g)
    start = g.GaussianField(means=[[0.35, -0.5, 0.05]], log_scales=np.log([[1.5, 2.1, 1.9]]),
                            quaternions=[[1.0, 0, 0, 0]], intensities=[0.5])
    _, _, hist = g.fit([stack], loss_cfg=g.LossConfig(lambda_reg=0.0), optim_cfg=_frozen(g, 200),
                       field=start.astype(np.float64))
    data = np.array([h["data_term"] for h in hist])
    n_pix = int(stack.mask.sum())
    assert data.min() / n_pix < 1e-5
    assert data[-1] < 1e-2 * data[0]


def test_loss_window_means_non_increasing(g):
    """tests/test_train.py:252-263 (the reference fails this one through its
    N=K=1 knn shape bug; the device K-NN has no such bug)."""
    truth, stack = _self_consistency_fixture(g)
    start = g.GaussianField(means=[[0.35, -0.5, 0.05]], log_scales=np.log([[1.5, 2.1, 1.9]]),
                            quaternions=[[1.0, 0, 0, 0]], intensities=[0.5])
    _, _, hist = g.fit([stack], loss_cfg=g.LossConfig(lambda_reg=0.0), optim_cfg=_frozen(g, 200),
                       field=start.astype(np.float64))
    w = np.array([h["loss"] for h in hist]).reshape(4, 50).mean(axis=1)
    assert all(w[i + 1] <= w[i] for i in range(3))


def test_scale_regularizer_pulls_toward_target(g):
    """tests/test_train.py:266-278."""
    truth, stack = _self_consistency_fixture(g)
    cfg = _frozen(g, 60)
    f0, _, _ = g.fit([stack], loss_cfg=g.LossConfig(lambda_reg=0.0), optim_cfg=cfg,
                     field=truth.astype(np.float64))
    np.testing.assert_allclose(f0.scales(), truth.scales(), rtol=1e-4)
    f1, _, _ = g.fit([stack], loss_cfg=g.LossConfig(lambda_reg=2.5e-3), optim_cfg=cfg,
                     field=truth.astype(np.float64))
    assert f1.scales().mean() < truth.scales().mean()
    assert f1.scales().mean() > 1.0


def test_motion_warmup_freezes_slice_states(g):
    """tests/test_train.py:290-301."""
    truth, stack = _self_consistency_fixture(g)
    cfg = g.OptimConfig(epochs=5, k_neighbors=1, motion_warmup=10, rotation_warmup=0, reseed_every=0)
    _, states, _ = g.fit([stack], optim_cfg=cfg, field=truth.astype(np.float64))
    ident = np.zeros_like(states.quaternions)
    ident[:, 0] = 1.0
    assert np.array_equal(states.quaternions, ident)
    assert not states.translations.any()
    assert not states.log_sigma.any()


def test_rotation_warmup_freezes_rotations_only(g):
    """tests/test_train.py:304-315."""
    truth, stack = _self_consistency_fixture(g)
    start = truth.astype(np.float64)
    start.intensities = start.intensities * 0.5
    cfg = g.OptimConfig(epochs=6, k_neighbors=1, motion_warmup=0, rotation_warmup=100, reseed_every=0,
                        anchor_slice=None)
    _, states, _ = g.fit([stack], optim_cfg=cfg, field=start)
    ident = np.zeros_like(states.quaternions)
    ident[:, 0] = 1.0
    assert np.array_equal(states.quaternions, ident)
    assert states.translations.any()


def test_anchor_slice_state_never_moves(g):
    """tests/test_train.py:318-327."""
    truth, stack = _self_consistency_fixture(g)
    start = truth.astype(np.float64)
    start.intensities = start.intensities * 0.5
    cfg = g.OptimConfig(epochs=6, k_neighbors=1, motion_warmup=0, rotation_warmup=0, reseed_every=0,
                        anchor_slice=1)
    _, states, _ = g.fit([stack], optim_cfg=cfg, field=start)
    assert np.array_equal(states.quaternions[1], [1.0, 0, 0, 0])
    assert not states.translations[1].any()
    assert states.translations[[0, 2]].any()


def test_reseed_schedule_and_history_flags(g):
    """tests/test_train.py:330-344."""
    truth, stack = _self_consistency_fixture(g)
    cfg = g.OptimConfig(epochs=10, k_neighbors=1, motion_warmup=0, rotation_warmup=0, reseed_every=2)
    _, _, hist = g.fit([stack], optim_cfg=cfg, field=truth.astype(np.float64))
    assert [h["epoch"] for h in hist if h["reseeded"]] == [2, 4, 6]
    cfg = g.OptimConfig(epochs=10, k_neighbors=1, motion_warmup=0, rotation_warmup=0, reseed_every=0)
    _, _, hist = g.fit([stack], optim_cfg=cfg, field=truth.astype(np.float64))
    assert not any(h["reseeded"] for h in hist)


def test_history_record_layout(g):
    """tests/test_train.py:347-358."""
    truth, stack = _self_consistency_fixture(g)
    cfg = g.OptimConfig(epochs=4, k_neighbors=1, motion_warmup=0, rotation_warmup=0, reseed_every=0)
    _, _, hist = g.fit([stack], optim_cfg=cfg, field=truth.astype(np.float64))
    assert [h["epoch"] for h in hist] == [0, 1, 2, 3]
    sec = [h["seconds"] for h in hist]
    assert all(b >= a for a, b in zip(sec, sec[1:]))
    for h in hist:
        assert {"loss", "data_term", "reg_term", "outlier_term", "lr_scale", "reseeded", "psnr",
                "ssim"} <= set(h)
        assert h["psnr"] is None and h["ssim"] is None


def test_reseed_field_modes(g):
    """tests/test_train.py:364-420 (reseed_field unit behaviour)."""
    truth, stack = _self_consistency_fixture(g)
    batch = g.build_point_batch([stack])
    states = g.init_states([stack])
    states.translations[:] = [[0.2, -0.1, 0.3]] * len(states)
    src = g.GaussianField(
        means=np.random.default_rng(0).normal(scale=2.0, size=(6, 3)),
        log_scales=np.log(np.random.default_rng(1).uniform(0.8, 1.6, (6, 3))),
        quaternions=np.random.default_rng(2).normal(size=(6, 4)) + [4, 0, 0, 0],
        intensities=np.linspace(0.1, 0.9, 6))
    f = g.reseed_field(batch, states, 20, initial_scale=1.4, seed=0, mode="observed")
    assert f.count == 20 and np.allclose(f.log_scales, np.log(1.4))
    corrected = g.corrected_points(batch, states)
    assert all(np.isclose(corrected, m, atol=1e-12).all(axis=1).any() for m in f.means)
    f = g.reseed_field(batch, states, 15, initial_scale=1.4, seed=2, source_field=src, k_neighbors=6,
                       mode="resample")
    for ls, q, m in zip(f.log_scales, f.quaternions, f.means):
        j = int(np.argmin(np.sum((src.means - m) ** 2, axis=1)))
        assert np.array_equal(ls, src.log_scales[j]) and np.array_equal(q, src.quaternions[j])
    a = g.reseed_field(batch, states, 10, 1.4, 7, source_field=src, mode="resample")
    b = g.reseed_field(batch, states, 10, 1.4, 7, source_field=src, mode="resample")
    assert np.array_equal(a.means, b.means)
    with pytest.raises(g.InvalidParameterError, match="mode"):
        g.reseed_field(batch, states, 5, 1.4, 0, mode="sideways")


def test_cfg1_fit_quality_and_wallclock(g):
    """BASELINE configs[0] (reference simulator data, tests/golden/cfg1_data.npz):
    200 epochs, 10k Gaussians, K=50 through the device fit; PSNR/SSIM vs the GT
    phantom at least as good as the reference's own fit (tests/golden/cfg1_ref_fit.json)."""
    import json
    import time
    from conftest import GOLDEN
    z = dict(np.load(GOLDEN / "cfg1_data.npz"))
    stacks = [g.SliceStack(z[f"s{i}_data"].astype(np.float64), z[f"s{i}_affine"], z[f"s{i}_spacing"],
                           float(z[f"s{i}_thickness"]), z[f"s{i}_mask"]) for i in range(3)]
    ref = g.VolumeGrid(z["gt_data"].astype(np.float64), z["gt_affine"], z["gt_mask"])
    t0 = time.perf_counter()
    field, states, hist = g.fit(stacks, g.InitConfig(n_gaussians=10_000, seed=0), None,
                                g.OptimConfig(epochs=200), reference=ref, eval_every=50)
    wall = time.perf_counter() - t0
    last = hist[-1]
    refj = json.loads((GOLDEN / "cfg1_ref_fit.json").read_text())
    rlast = refj["history"][-1]
    print(f"cfg1 fit: {wall:.2f} s, psnr {last['psnr']:.2f} (ref {rlast['psnr']:.2f}), "
          f"ssim {last['ssim']:.4f} (ref {rlast['ssim']:.4f}), ref wall {refj['wall_s']:.1f} s")
    assert last["psnr"] >= rlast["psnr"] - 0.5
    assert last["ssim"] >= rlast["ssim"] - 0.01


def test_cfg1_noisy_fit_tracks_reference_trajectory(g):
    """Reference simulator data with noise 0.02 (tests/golden/cfg1_noisy_data.npz): the
    reference's own fit peaks early and then over-fits the noise (PSNR 28.3 -> 25.1 dB
    over 300 epochs, tests/golden/cfg1_noisy_ref_fit.json).  The device fit follows the
    same trajectory."""
    import json
    from conftest import GOLDEN
    z = dict(np.load(GOLDEN / "cfg1_noisy_data.npz"))
    stacks = [g.SliceStack(z[f"s{i}_data"].astype(np.float64), z[f"s{i}_affine"], z[f"s{i}_spacing"],
                           float(z[f"s{i}_thickness"]), z[f"s{i}_mask"]) for i in range(3)]
    ref = g.VolumeGrid(z["gt_data"].astype(np.float64), z["gt_affine"], z["gt_mask"])
    _, _, hist = g.fit(stacks, g.InitConfig(n_gaussians=10_000, seed=0), None, g.OptimConfig(epochs=300),
                       reference=ref, eval_every=25)
    got = {h["epoch"]: h for h in hist if h["psnr"] is not None}
    want = json.loads((GOLDEN / "cfg1_noisy_ref_fit.json").read_text())["evals"]
    for w in want:
        h = got[w["epoch"]]
        print(f"epoch {w['epoch']}: psnr {h['psnr']:.2f} (ref {w['psnr']:.2f}) "
              f"ssim {h['ssim']:.4f} (ref {w['ssim']:.4f})")
        assert abs(h["psnr"] - w["psnr"]) < 1.0
        assert abs(h["ssim"] - w["ssim"]) < 0.03


def test_fit_is_bitwise_deterministic(g):
    """No atomics in any reduction of the epoch (per-(tile, Gaussian) partials
    gathered in tile order, per-tile slice partials summed per slice in order),
    so repeated fits are bit-identical -- the reference's fixed block partition
    gives it the same property (kernels.py:7-9)."""
    from conftest import GOLDEN
    z = dict(np.load(GOLDEN / "cfg1_data.npz"))
    stacks = [g.SliceStack(z[f"s{i}_data"].astype(np.float64), z[f"s{i}_affine"], z[f"s{i}_spacing"],
                           float(z[f"s{i}_thickness"]), z[f"s{i}_mask"]) for i in range(3)]
    runs = []
    for _ in range(2):
        f, st, hist = g.fit(stacks, g.InitConfig(n_gaussians=4000, seed=0), None,
                            g.OptimConfig(epochs=40, motion_warmup=5, rotation_warmup=10, reseed_every=20))
        runs.append((f, st, [h["loss"] for h in hist]))
    (f1, s1, l1), (f2, s2, l2) = runs
    assert l1 == l2
    assert np.array_equal(f1.means, f2.means) and np.array_equal(f1.quaternions, f2.quaternions)
    assert np.array_equal(s1.translations, s2.translations)


def _desk_case(g, tag="desk_motion"):
    from conftest import GOLDEN
    z = dict(np.load(GOLDEN / f"{tag}_data.npz"))
    stacks = [g.SliceStack(z[f"s{i}_data"], z[f"s{i}_affine"], z[f"s{i}_spacing"],
                           float(z[f"s{i}_thickness"]), z[f"s{i}_mask"]) for i in range(3)]
    ref = g.VolumeGrid(z["gt_data"], z["gt_affine"], z["gt_mask"])
    truth = g.SliceStates(z["truth_q"], z["truth_t"], z["truth_logsig"], z["truth_eta"])
    return stacks, ref, truth


def run_desk_fit(g, tag="desk_motion"):
    """The reference's acceptance desk run (tests/test_acceptance.py:60-100) on the
    device: 64^3 phantom @ 0.5 mm, 3 stacks with 6 deg / 4 mm slice motion,
    N=5000, K=50, lambda 2.5e-3, 500 epochs, gauge-removed evaluation every 25."""
    from paper_2512_11624_b200.metrics import motion_error, motion_gauge, psnr, ssim
    stacks, ref, truth = _desk_case(g, tag)
    field, states, hist = g.fit(stacks, g.InitConfig(n_gaussians=5000, seed=0),
                                g.LossConfig(lambda_reg=2.5e-3),
                                g.OptimConfig(epochs=500, k_neighbors=50),
                                reference=ref, truth_states=truth, eval_every=25)
    aligned = g.rasterize(field, ref, K=50, transform=motion_gauge(states, truth))
    rot, trans = motion_error(states, truth)
    return {"evals": {h["epoch"]: h for h in hist if h["psnr"] is not None},
            "final_psnr": psnr(aligned.data, ref.data, mask=ref.mask),
            "final_ssim": ssim(aligned.data, ref.data, mask=ref.mask),
            "rot": rot, "trans": trans, "seconds": hist[-1]["seconds"]}


@pytest.mark.parametrize("tag", ["desk_motion", "desk_motion_clean"])
def test_desk_motion_fit_tracks_reference(g, tag):
    """Slice-pose descent ("S" of SVR, train.py:473-479) at trajectory level: the
    device fit of the reference's own motion-corrupted desk acquisition tracks the
    reference's fit of it (tests/golden/<tag>_ref_fit.json, oracle/gen_desk_motion.py):
    PSNR within 1 dB and SSIM within 0.03 at every evaluation, final aligned
    PSNR/SSIM likewise, median per-slice motion error within 0.5 deg / 0.3 mm."""
    import json
    from conftest import GOLDEN
    want = json.loads((GOLDEN / f"{tag}_ref_fit.json").read_text())
    got = run_desk_fit(g, tag)
    worst_p = worst_s = 0.0
    for w in want["evals"]:
        h = got["evals"][w["epoch"]]
        print(f"{tag} epoch {w['epoch']}: psnr {h['psnr']:.2f} (ref {w['psnr']:.2f}) "
              f"ssim {h['ssim']:.4f} (ref {w['ssim']:.4f})")
        worst_p = max(worst_p, abs(h["psnr"] - w["psnr"]))
        worst_s = max(worst_s, abs(h["ssim"] - w["ssim"]))
    mr, mt = float(np.median(got["rot"])), float(np.median(got["trans"]))
    print(f"{tag} final psnr {got['final_psnr']:.2f} (ref {want['final_psnr']:.2f}) ssim "
          f"{got['final_ssim']:.4f} (ref {want['final_ssim']:.4f}); motion median {mr:.2f} deg "
          f"{mt:.3f} mm (ref {want['motion_rot_median']:.2f} / {want['motion_trans_median']:.3f}); "
          f"worst |dPSNR| {worst_p:.2f} |dSSIM| {worst_s:.4f}; fit {got['seconds']:.2f} s "
          f"(ref {want['wall_s']:.0f} s)")
    assert worst_p < 1.0 and worst_s < 0.03
    assert abs(got["final_psnr"] - want["final_psnr"]) < 1.0
    assert abs(got["final_ssim"] - want["final_ssim"]) < 0.03
    assert abs(mr - want["motion_rot_median"]) < 0.5
    assert abs(mt - want["motion_trans_median"]) < 0.3


def run_cfg2mini_fit(g, tag="cfg2mini"):
    """The synthetic cfg2 generator at a CPU-feasible size (oracle/gen_cfg2mini.py):
    cfg2 spacing / noise / motion, 96x96x22 FOV, 20.6k Gaussians, 500 epochs with
    the reference defaults, evaluated every 25 epochs on a 64^3 1.2 mm grid."""
    from conftest import GOLDEN
    from paper_2512_11624_b200.metrics import motion_error
    z = dict(np.load(GOLDEN / f"{tag}_data.npz"))
    stacks = [g.SliceStack(z[f"s{i}_data"].astype(np.float64), z[f"s{i}_affine"], z[f"s{i}_spacing"],
                           float(z[f"s{i}_thickness"])) for i in range(3)]
    ref = g.VolumeGrid(z["gt_data"], z["gt_affine"], mask=z["gt_data"] > 0)
    S = len(z["truth_q"])
    truth = g.SliceStates(z["truth_q"], z["truth_t"], np.zeros(S), np.zeros(S))
    _, states, hist = g.fit(stacks, g.InitConfig(n_gaussians=int(z["n_gaussians"]), seed=0), None,
                            g.OptimConfig(epochs=500), reference=ref, truth_states=truth, eval_every=25)
    r, t = motion_error(states, truth)
    return {h["epoch"]: h for h in hist if h["psnr"] is not None}, float(np.median(r)), float(np.median(t))


@pytest.mark.parametrize("tag", ["cfg2mini", "cfg2mini_clean"])
def test_cfg2mini_fit_tracks_reference(g, tag):
    """The late-epoch quality drop of the fetal-scale synthetic fits is the
    reference's own behaviour: on the same generator at a CPU-feasible size the
    reference's fit peaks (26.0 dB at epoch 324) and ends at 20.9 dB / SSIM 0.52
    (tests/golden/cfg2mini_ref_fit.json); without noise (cfg2mini_clean) the
    reference ends at 26.2 dB / SSIM 0.947.  The device fit follows both
    trajectories: PSNR within 1 dB and SSIM within 0.04 at every evaluation."""
    import json
    from conftest import GOLDEN
    want = json.loads((GOLDEN / f"{tag}_ref_fit.json").read_text())
    got, mr, mt = run_cfg2mini_fit(g, tag)
    wp = ws = 0.0
    for w in want["evals"]:
        h = got[w["epoch"]]
        print(f"{tag} epoch {w['epoch']}: psnr {h['psnr']:.2f} (ref {w['psnr']:.2f}) "
              f"ssim {h['ssim']:.4f} (ref {w['ssim']:.4f})")
        wp, ws = max(wp, abs(h["psnr"] - w["psnr"])), max(ws, abs(h["ssim"] - w["ssim"]))
    print(f"{tag}: worst |dPSNR| {wp:.2f} |dSSIM| {ws:.4f}; motion median {mr:.2f} deg {mt:.3f} mm "
          f"(ref {want['motion_rot_median']:.2f} / {want['motion_trans_median']:.3f})")
    assert wp < 1.0 and ws < 0.04
