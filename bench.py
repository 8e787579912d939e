"""Benchmark: slice-pixel fwd+bwd evaluations per second of the GSVR hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

One step = one training epoch of the hot path over the whole synthetic batch:
fused tile forward + L1 + backward (gsvr_train_tiles), slice chain + AdamW,
field chain + AdamW, staleness measure, and the per-epoch loss read-back --
i.e. what ``fit`` runs every epoch between neighbour refreshes (refresh time is
reported separately).  Workload (N=1): BASELINE.json configs[1] ("cfg2",
fetal-brain scale: 3 stacks 256x256x30 @ 0.8x0.8x3.5 mm, 200k Gaussians, K=50,
per-slice motion), synthetic data (paper_2512_11624_b200/synthetic.py).

N>1 (torchrun, NCCL): weak scaling -- every rank holds its own cfg2-sized set
of stacks, the field is replicated and its gradient all-reduced every epoch.

``--impl reference`` times the reference algorithm's CPU path (the oracle's
C/OpenMP restatement of kernels.train_step_backward, all host threads) on a
bounded sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FLOP_PER_PAIR = 101      # 62 forward + 39 backward per (pixel, neighbour)
FLOP_PER_PIXEL = 50      # per-pixel transform / residual / slice terms
BYTES_PER_PIXEL_K = lambda K: 12 + 4 + 4 + 4 * K + 8  # x0, sid, I_obs, nbr int32, I_hat + |r|


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--k", type=int, default=50)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-fit", action="store_true", help="skip the wall-clock-to-convergence runs")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# workload

_WORKLOAD_CACHE = {}


def workload_name(cfg, K):
    """The `config.workload` string, identical on both arms."""
    return (f"{cfg.name}: {cfg.n_stacks} stacks {cfg.nx}x{cfg.ny}x{cfg.n_slices} "
            f"@ {cfg.inplane}x{cfg.inplane}x{cfg.thickness} mm, {cfg.n_gaussians} Gaussians, K={K}, motion")


def build_workload(cfg_name, rank, K):
    from paper_2512_11624_b200 import synthetic
    from paper_2512_11624_b200.initialization import InitConfig, init_field, sample_init_positions
    from paper_2512_11624_b200.motion import build_point_batch, init_states
    from paper_2512_11624_b200.train import slice_psf_diags

    cfg = synthetic.CONFIGS[cfg_name]
    stacks, truth = synthetic.make_stacks(cfg, seed=rank)
    _WORKLOAD_CACHE[(cfg_name, rank)] = (stacks, truth)
    batch = build_point_batch(stacks)
    icfg = InitConfig(n_gaussians=cfg.n_gaussians, seed=0)
    field = init_field(sample_init_positions(stacks, icfg), stacks, icfg)
    states = init_states(stacks)
    psf = slice_psf_diags(batch, stacks)
    return cfg, stacks, batch, field, states, psf


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.proc = None
        self.index = index
        self.path = ROOT / "gpurun_out" / f"clocks_bench_{index}.csv"

    def __enter__(self):
        self.path.parent.mkdir(exist_ok=True)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        rows = []
        try:
            for line in self.path.read_text().splitlines():
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 8 and f[0].replace(".", "").isdigit():
                    rows.append(f)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[4:8]) if v.lower() == "active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle restatement of kernels.train_step_backward

def cpu_reference_rate(batch, field, states, psf, nbr_host, seconds, seed=0):
    """slice-px/s of the reference algorithm (float64, per-pair inverse, 16-block
    private buffers) on a contiguous sample of the batch sized to ~`seconds`."""
    from oracle import host as oracle
    from paper_2512_11624_b200.geometry import pack_sym6
    oracle.set_threads(oracle.all_host_threads())

    P = batch.n_points
    S = batch.n_slices
    sid = batch.slice_ids
    Rc, R_eff, psf6s, sig = oracle.slice_inputs(states.quaternions, batch.stack_rotations,
                                                batch.slice_to_stack, states.log_sigma, psf)
    cov6 = oracle.covariances6(field.log_scales, field.quaternions)
    w = np.ones(S)

    B = oracle.default_block_count(P)
    N = field.count

    def run(lo, n):
        hi = lo + n
        # the reference zero-fills 16 private (N, 10) buffers per call
        # (train.py:247-253); done outside the timed region here so a bounded
        # sample is not dominated by that fixed cost
        bufs = {"dmu": np.zeros((B, N, 3)), "dcov6": np.zeros((B, N, 6)), "dc": np.zeros((B, N)),
                "dt": np.zeros((B, S, 3)), "dRc": np.zeros((B, S, 3, 3)), "dpsf6": np.zeros((B, S, 6)),
                "dsigraw": np.zeros((B, S))}
        t0 = time.perf_counter()
        oracle.train_step_backward(batch.lifted[lo:hi], sid[lo:hi], Rc, states.translations, psf6s,
                                   sig, w, batch.intensities[lo:hi], nbr_host[lo:hi], field.means,
                                   cov6, field.intensities, n_blocks=B, reduce=False, bufs=bufs)
        return time.perf_counter() - t0

    rng = np.random.default_rng(seed)
    n = 16384
    lo = int(rng.integers(0, max(1, P - n)))
    run(lo, n)                               # warm (page-in)
    t = run(lo, n)
    while t < 0.2 * seconds and n < P:       # grow the sample to ~seconds of CPU work
        n = int(min(P, n * max(2.0, 0.8 * seconds / max(t, 1e-3))))
        lo = int(rng.integers(0, max(1, P - n + 1)))
        t = run(lo, n)
    total_n, total_t = n, t
    while n == P and total_t < 0.8 * seconds:  # whole batch is < seconds: repeat passes
        total_t += run(0, P)
        total_n += P
    return total_n / total_t, total_n, total_t


# ---------------------------------------------------------------------------

def _log(msg):
    if os.environ.get("GSVR_BENCH_VERBOSE"):
        print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return main_reference(args, world, rank)

    import ctypes

    import torch
    import torch.distributed as dist
    from paper_2512_11624_b200._native import lib

    torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    comm = None
    if world > 1:
        backend = os.environ.get("GSVR_DIST_BACKEND", "nccl")  # gloo: multi-rank smoke on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        from paper_2512_11624_b200.parallel import Comm
        comm = Comm()
    from paper_2512_11624_b200 import _native, _dev
    from paper_2512_11624_b200.engine import DeviceBatch, FitEngine
    from paper_2512_11624_b200.train import LossConfig, OptimConfig

    K = args.k
    t0 = time.perf_counter()
    cfg, stacks, batch, field, states, psf = build_workload(args.config, rank, K)
    t_gen = time.perf_counter() - t0
    if comm is not None:  # replicate rank 0's field
        for name in ("means", "log_scales", "quaternions", "intensities"):
            t = torch.from_numpy(np.ascontiguousarray(getattr(field, name))).cuda()
            comm.broadcast(t)
            setattr(field, name, t.cpu().numpy())
    loss_cfg, optim_cfg = LossConfig(), OptimConfig(k_neighbors=K)

    _log("device batch")
    t0 = time.perf_counter()
    db = DeviceBatch(batch, K=K)
    eng = FitEngine(db, field, states, psf, loss_cfg, optim_cfg, comm=comm)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    eng.refresh(K)  # first refresh sizes the binning buffers; report the steady state
    torch.cuda.synchronize()
    ev0.record()
    eng.refresh(K)
    ev1.record()
    torch.cuda.synchronize()
    refresh_ms = ev0.elapsed_time(ev1)
    n_tiles, tile_g = db.n_tiles, db.tile_gaussians

    _log("warmup")
    for _ in range(args.warmup):
        eng.epoch(1.0, True, False, 0)
    torch.cuda.synchronize()

    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    orig_train = eng.train_pass
    it = {"i": 0}

    def timed_train(*a, **k):
        e = kev[it["i"]]
        e[0].record()
        orig_train(*a, **k)
        e[1].record()
        it["i"] += 1

    eng.train_pass = timed_train
    lib().gsvr_set_kernel_timing(1)  # events around the tile-kernel launch itself
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if comm is not None:
        comm.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        start.record()
        # steps are issued back to back; the loss terms (a host sync) are read
        # after the last one -- every step's kernels run inside the timed region
        for i in range(args.steps):
            terms = eng.epoch(1.0, True, False, 0, sync=(i == args.steps - 1))
        end.record()
        torch.cuda.synchronize()
    if comm is not None:
        comm.barrier()
    eng.train_pass = orig_train
    elapsed_ms = start.elapsed_time(end)
    pass_ms = float(np.mean([a.elapsed_time(b) for a, b in kev]))  # kernel + gradient gathers
    nl = ctypes.c_int64(0)
    kern_total = lib().gsvr_kernel_time_ms(ctypes.byref(nl))
    lib().gsvr_set_kernel_timing(0)
    kern_ms = kern_total / max(nl.value, 1)
    kern_name = "k_train_planar" if lib().gsvr_batch_is_planar(db.raw) else "k_train_tiles"
    if comm is not None:
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device="cuda")
        comm.allreduce_max(t)
        elapsed_ms = float(t.item())
    P_local = batch.n_points
    P_total = P_local * world
    value = P_total * args.steps / (elapsed_ms * 1e-3)

    out = None
    if rank == 0:
        peak = _probe_fp32()
        flop_launch = P_local * (FLOP_PER_PAIR * K + FLOP_PER_PIXEL)
        achieved = flop_launch / (kern_ms * 1e-3) / 1e12
        bytes_launch = P_local * BYTES_PER_PIXEL_K(K)
        hbm_gbs = bytes_launch / (kern_ms * 1e-3) / 1e9
        measured = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
            if (ROOT / "MEASURED_PEAKS.json").exists() else {}
        traffic = _ncu_traffic(P_local)
        out = {
            "metric": "slice-pixel fwd+bwd evals/sec",
            "value": value, "unit": "slice-px/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (analytic phantom, seeded per-slice motion, reference init policy)",
            "config": {"workload": workload_name(cfg, K),
                       "points_per_gpu": P_local, "gaussians": field.count, "K": K,
                       "tiles": n_tiles, "tile_gaussians": tile_g,
                       "l2": "inputs larger than L2 (per-epoch tile streams "
                             f"{P_local * K * 4 / 1e9:.2f} GB > 126 MB)",
                       "parallelism": f"slice-sharded dp{world}, field replicated, "
                                      f"{os.environ.get('GSVR_DIST_BACKEND', 'nccl').upper()} grad all-reduce"},
            "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak if peak else None, "traffic": traffic,
                         "kernel": kern_name, "kernel_ms": kern_ms, "launches_timed": nl.value,
                         "train_pass_ms": pass_ms,
                         "flop_per_launch": flop_launch,
                         "flop_per_pixel": FLOP_PER_PAIR * K + FLOP_PER_PIXEL,
                         "peak_source": "measured live: FFMA probe (gsvr_probe_fp32_peak)",
                         "hbm_achieved_gbs": hbm_gbs,
                         "hbm_peak_gbs": measured.get("hbm_gbs"),
                         "hbm_frac": hbm_gbs / measured["hbm_gbs"] if measured.get("hbm_gbs") else None},
            # per epoch: k_pack_grec, k_train_planar, k_gather_grads, k_slice_reduce, k_slice_step,
            # k_field_step, k_disp_bounds, k_disp_points (profiles/launches_r01.csv)
            "gpu_launches": (8 if eng.Rc_ref is not None else 6) * args.steps,
            "clocks": clk.summary(),
            "refresh_ms": refresh_ms,
            "setup_s": {"generate": t_gen, "device_batch": t_setup},
            "loss_last": terms["loss"],
        }
    _log("e2e")
    # e2e through the reference-facing drop-in (kernels.train_step_backward) with pinned host buffers
    e2e = _e2e(eng, db, batch, field, states, psf, K, args.e2e_steps, comm)
    if rank == 0:
        out["e2e"] = e2e
        _log("cpu baseline")
        if world == 1 and not args.no_cpu_baseline:
            nbr_host = _dev.to_host(db.neighbors())
            rate, n, secs = cpu_reference_rate(batch, field, states, psf, nbr_host, args.cpu_seconds)
            from oracle import host as oracle_host
            out["cpu_baseline"] = {"value": rate, "unit": "slice-px/s", "cores": oracle_host.threads_used(),
                                   "kind": "port",
                                   "sample": f"{n} batch pixels x K={K} of the same workload "
                                             f"({n / batch.n_points:.1f} passes when >= 1; full "
                                             f"{field.count}-Gaussian field), {secs:.1f} s of "
                                             "oracle/gsvr_oracle.c (kernels.py:78-198 restated, OpenMP, "
                                             "float64, 16 private block buffers zeroed outside the timer)"}
        _log("fits")
        if world == 1 and not args.no_fit:
            fits = (("fit_cfg1", fit_cfg1),
                    ("fit_cfg2", lambda: fit_cfg2(stacks_truth=_WORKLOAD_CACHE.get(("cfg2", 0)))),
                    ("fit_cfg3", fit_cfg3))
            for name, fn in fits:
                _log(name)
                try:
                    out[name] = fn()
                except Exception as exc:  # reported, never fatal for the bench line
                    out[name] = {"error": f"{type(exc).__name__}: {exc}"}
        print(json.dumps(out), flush=True)
    if comm is not None:
        dist.destroy_process_group()


def _probe_fp32():
    import ctypes
    from paper_2512_11624_b200 import _dev
    from paper_2512_11624_b200._native import check, lib
    v = ctypes.c_double()
    check(lib().gsvr_probe_fp32_peak(ctypes.byref(v), _dev.stream_ptr()))
    return float(v.value)


def _ncu_traffic(points):
    """DRAM bytes per launch of the tile kernel from the committed ncu capture
    (profiles/ncu_train_tiles_*.json), when it was taken on this workload size."""
    best = None
    for p in sorted((ROOT / "profiles").glob("ncu_train_tiles_*.json")):
        try:
            d = json.loads(p.read_text())
        except (OSError, ValueError):
            continue
        if d.get("points", 5898240) == points:
            best = d.get("dram_bytes_per_launch")
    return best


def _e2e(eng, db, batch, field, states, psf, K, steps, comm):
    """kernels.train_step_backward (the reference's operator boundary) with host
    buffers: H2D of every input and D2H of every output inside the timed region."""
    import torch
    from paper_2512_11624_b200 import _dev, kernels
    from paper_2512_11624_b200.geometry import pack_sym6

    P, S, N = batch.n_points, batch.n_slices, field.count
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    Rc = _dev.to_host(eng.Rc).reshape(S, 3, 3)
    ins = dict(x0pts=pin(batch.lifted), sid=pin(batch.slice_ids.astype(np.int32)), Rc=pin(Rc),
               tvec=pin(_dev.to_host(eng.tv)), psf6s=pin(_dev.to_host(eng.p6)),
               sigma_s=pin(_dev.to_host(eng.sig)), wdata_s=pin(_dev.to_host(eng.w)),
               I_obs=pin(batch.intensities), nbr=pin(_dev.to_host(db.neighbors())),
               mu=pin(_dev.to_host(eng.mu)), cov6=pin(_dev.to_host(eng.cov6)), cvals=pin(_dev.to_host(eng.c)))
    outs = [torch.empty(P, dtype=torch.float64).pin_memory() for _ in range(2)]
    grads = [torch.zeros(s, dtype=torch.float64).pin_memory()
             for s in [(1, N, 3), (1, N, 6), (1, N), (1, S, 3), (1, S, 3, 3), (1, S, 6), (1, S)]]
    h2d = sum(t.numel() * t.element_size() for t in ins.values())
    d2h = sum(t.numel() * t.element_size() for t in outs + grads)

    def call():
        for gbuf in grads:
            gbuf.zero_()
        kernels.train_step_backward(ins["x0pts"], ins["sid"], ins["Rc"], ins["tvec"], ins["psf6s"],
                                    ins["sigma_s"], ins["wdata_s"], ins["I_obs"], ins["nbr"], ins["mu"],
                                    ins["cov6"], ins["cvals"], 1e-8, 1, outs[0], outs[1], *grads)

    call()
    torch.cuda.synchronize()
    if comm is not None:
        comm.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        call()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    if comm is not None:
        t = torch.tensor([dt], dtype=torch.float64, device="cuda")
        comm.allreduce_max(t)
        dt = float(t.item())
    world = comm.world if comm is not None else 1
    del pack_sym6
    return {"value": P * world / dt, "unit": "slice-px/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": dt * 1e3,
            # caller bytes consumed per call; inside the (timed) call two of every
            # three id chunks are narrowed to int32 by host threads before the
            # bus, the third crosses as int64 and is narrowed on the device
            "h2d_note": "int64 neighbour ids: 2/3 of the chunks narrowed to int32 on host threads, "
                        "1/3 narrowed on the device (balances host memory bandwidth against PCIe)",
            "api": "paper_2512_11624_b200.kernels.train_step_backward (numpy-compatible drop-in, "
                   "pinned host tensors)"}


def fit_cfg1():
    """Wall-clock of the full device fit on BASELINE configs[0] (the reference
    simulator's own cfg1 stacks, tests/golden/cfg1_data.npz): 10k Gaussians, K=50,
    200 epochs, PSNR/SSIM vs the GT phantom; the reference's fit of the same data
    (measured in the build container, tests/golden/cfg1_ref_fit.json) beside it."""
    import paper_2512_11624_b200 as g
    z = dict(np.load(ROOT / "tests" / "golden" / "cfg1_data.npz"))
    stacks = [g.SliceStack(z[f"s{i}_data"].astype(np.float64), z[f"s{i}_affine"], z[f"s{i}_spacing"],
                           float(z[f"s{i}_thickness"]), z[f"s{i}_mask"]) for i in range(3)]
    ref = g.VolumeGrid(z["gt_data"].astype(np.float64), z["gt_affine"], z["gt_mask"])
    out = {}
    for eval_every in (0, 50):
        t0 = time.perf_counter()
        _, _, hist = g.fit(stacks, g.InitConfig(n_gaussians=10_000, seed=0), None, g.OptimConfig(epochs=200),
                           reference=ref if eval_every else None, eval_every=eval_every)
        wall = time.perf_counter() - t0
        if eval_every:
            out["psnr"], out["ssim"] = hist[-1]["psnr"], hist[-1]["ssim"]
        else:
            out["wall_s"] = wall
    refj = json.loads((ROOT / "tests" / "golden" / "cfg1_ref_fit.json").read_text())
    out.update(epochs=200, gaussians=10_000, K=50,
               reference={"wall_s": refj["wall_s"], "psnr": refj["history"][-1]["psnr"],
                          "ssim": refj["history"][-1]["ssim"],
                          "where": "gsvr.fit in the build container, numba 8 threads"})
    return out


def fit_cfg2(epochs=500, stacks_truth=None):
    """Wall-clock to convergence at fetal scale (cfg2, synthetic phantom with
    per-slice motion, paper protocol: 500 epochs, refresh/reseed policy of the
    reference): total fit time, and time to first SSIM >= 0.8 / to within 0.1 dB
    of the final PSNR from a second run evaluated every 25 epochs (gauge removed
    with the true slice states)."""
    import paper_2512_11624_b200 as g
    from paper_2512_11624_b200 import synthetic
    cfg = synthetic.CONFIGS["cfg2"]
    stacks, truth = stacks_truth or synthetic.make_stacks(cfg, seed=0)
    n = 128
    aff = np.diag([1.0, 1.0, 1.0, 1.0])
    aff[:3, 3] = -0.5 * (n - 1)
    grid = g.VolumeGrid(np.zeros((n, n, n)), aff)
    gt = synthetic.phantom(grid.voxel_centers()).reshape(n, n, n)
    ref = g.VolumeGrid(gt, aff, mask=gt > 0)
    icfg = g.InitConfig(n_gaussians=cfg.n_gaussians, seed=0)
    t0 = time.perf_counter()
    g.fit(stacks, icfg, None, g.OptimConfig(epochs=epochs))
    wall = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, _, hist = g.fit(stacks, icfg, None, g.OptimConfig(epochs=epochs), reference=ref,
                       truth_states=truth, eval_every=25)
    evals = [h for h in hist if h["psnr"] is not None]
    final = evals[-1]["psnr"]
    best = max(evals, key=lambda h: h["psnr"])
    first_ssim = next((h for h in evals if h["ssim"] >= 0.8), None)
    frac = lambda h: None if h is None else wall * (h["epoch"] + 1) / epochs
    return {"wall_s": wall, "epochs": epochs, "final_psnr": final, "final_ssim": evals[-1]["ssim"],
            "best_psnr": best["psnr"], "best_ssim": best["ssim"], "best_epoch": best["epoch"],
            "s_to_best": frac(best), "s_to_ssim_0.8": frac(first_ssim),
            "note": "milestone times = epoch fraction of the un-instrumented run; like the reference "
                    "(tests/golden/cfg1_noisy_ref_fit.json) the 500-epoch protocol peaks early and then "
                    "over-fits the 2% noise"}


def fit_cfg3(epochs=500):
    """Wall-clock of the full fit at BASELINE configs[2] scale on ONE B200 (6
    stacks 320x320x40 @ 0.7x0.7x3 mm, 500k Gaussians, per-slice motion): the
    north-star "fetal-brain-scale SVR (~6 stacks, ~500k Gaussians) converges in
    well under ~30 s" claim.  Quality of the final field is evaluated after the
    timed fit (motion gauge removed with the true slice states)."""
    import paper_2512_11624_b200 as g
    from paper_2512_11624_b200 import synthetic
    from paper_2512_11624_b200.train import _evaluate
    cfg = synthetic.CONFIGS["cfg3"]
    t0 = time.perf_counter()
    stacks, truth = synthetic.make_stacks(cfg, seed=0)
    t_gen = time.perf_counter() - t0
    icfg = g.InitConfig(n_gaussians=cfg.n_gaussians, seed=0)
    t0 = time.perf_counter()
    field, states, hist = g.fit(stacks, icfg, None, g.OptimConfig(epochs=epochs))
    wall = time.perf_counter() - t0
    n = 128
    aff = np.diag([1.0, 1.0, 1.0, 1.0])
    aff[:3, 3] = -0.5 * (n - 1)
    grid = g.VolumeGrid(np.zeros((n, n, n)), aff)
    gt = synthetic.phantom(grid.voxel_centers()).reshape(n, n, n)
    ref = g.VolumeGrid(gt, aff, mask=gt > 0)
    psnr, ssim = _evaluate(field, ref, 50, states, truth)
    pts = sum(int(np.prod(s.data.shape)) for s in stacks)
    loop = hist[-1]["seconds"]
    out = {"wall_s": wall, "setup_s": wall - loop, "loop_s": loop,
           "epochs": epochs, "stacks": cfg.n_stacks, "slice_pixels": pts,
           "gaussians": cfg.n_gaussians, "K": 50, "final_psnr": psnr, "final_ssim": ssim,
           "generate_s": t_gen, "target": "north star: well under ~30 s on one B200"}
    try:
        out["export_cfg5"] = export_cfg5(field)
    except Exception as exc:  # reported, never fatal
        out["export_cfg5"] = {"error": f"{type(exc).__name__}: {exc}"}
    return out


def export_cfg5(field, n=410, spacing=0.5, K=50):
    """BASELINE configs[4]: the trained field evaluated on a 0.5 mm isotropic grid
    over a ~205 mm box (410^3 = 68.9 M voxels): device voxel centres, exact K-NN
    of every voxel, PSF-free blend (field.py:138-175); the host array is filled."""
    import torch
    import paper_2512_11624_b200 as g
    aff = np.diag([spacing, spacing, spacing, 1.0])
    aff[:3, 3] = -0.5 * spacing * (n - 1)
    grid = g.VolumeGrid(np.zeros((n, n, n)), aff)
    g.rasterize(field, g.VolumeGrid(np.zeros((8, 8, 8)), aff), K)  # warm-up (module load, pools)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    vol = g.rasterize(field, grid, K)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    return {"voxels": n ** 3, "spacing_mm": spacing, "K": K, "gaussians": field.count, "wall_s": wall,
            "voxels_per_s": n ** 3 / wall, "finite": bool(np.isfinite(vol.data).all()),
            "note": "wall includes device centres, K-NN, evaluation and the 551 MB device->host copy"}


def main_reference(args, world, rank):
    """Reference arm: the reference's CPU algorithm for this path (the oracle's C
    restatement of kernels.py:78-198, float64, 16 private block buffers, all host
    threads) on a bounded contiguous sample of the same cfg2 workload: 2^20 pixels
    per step, neighbour lists of the sample from scipy's cKDTree (the reference's
    own K-NN dependency, knn.py:33-75) outside the timer, block buffers zero-filled
    outside the timer (the reference pays that once per full-batch call)."""
    if rank != 0:
        return
    K = args.k
    cfg, stacks, batch, field, states, psf = build_workload(args.config, 0, K)
    from scipy.spatial import cKDTree
    from oracle import host as oracle
    oracle.set_threads(oracle.all_host_threads())  # torchrun exports OMP_NUM_THREADS=1
    t0 = time.perf_counter()
    P, S, N = batch.n_points, batch.n_slices, field.count
    n_sample = min(P, 1 << 20)
    lo = int(np.random.default_rng(1).integers(0, P - n_sample + 1))
    hi = lo + n_sample
    Rc, _, psf6s, sig = oracle.slice_inputs(states.quaternions, batch.stack_rotations,
                                            batch.slice_to_stack, states.log_sigma, psf)
    X = np.einsum("pij,pj->pi", Rc[batch.slice_ids[lo:hi]], batch.lifted[lo:hi]) + \
        states.translations[batch.slice_ids[lo:hi]]
    nbr = cKDTree(field.means).query(X, k=K, workers=-1)[1].astype(np.int64)
    cov6 = oracle.covariances6(field.log_scales, field.quaternions)
    B = oracle.default_block_count(P)
    rates = []
    for step in range(args.warmup + args.steps):
        bufs = {"dmu": np.zeros((B, N, 3)), "dcov6": np.zeros((B, N, 6)), "dc": np.zeros((B, N)),
                "dt": np.zeros((B, S, 3)), "dRc": np.zeros((B, S, 3, 3)), "dpsf6": np.zeros((B, S, 6)),
                "dsigraw": np.zeros((B, S))}
        ts = time.perf_counter()
        oracle.train_step_backward(batch.lifted[lo:hi], batch.slice_ids[lo:hi], Rc, states.translations,
                                   psf6s, sig, np.ones(S), batch.intensities[lo:hi], nbr, field.means, cov6,
                                   field.intensities, n_blocks=B, reduce=False, bufs=bufs)
        dt = time.perf_counter() - ts
        if step >= args.warmup:
            rates.append(n_sample / dt)
    value = float(np.median(rates))
    wall = time.perf_counter() - t0
    sample = (f"{n_sample} contiguous batch pixels x K={K} per step (full {N}-Gaussian field), "
              "oracle/gsvr_oracle.c restating kernels.py:78-198, float64, OpenMP, 16 block buffers "
              "zeroed outside the timer")
    out = {"metric": "slice-pixel fwd+bwd evals/sec", "value": value, "unit": "slice-px/s",
           "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": n_sample / value * 1e3, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": workload_name(cfg, K), "points_per_gpu": batch.n_points, "gaussians": N,
                      "K": K, "sample_pixels_per_step": n_sample},
           "cpu_baseline": {"value": value, "unit": "slice-px/s", "cores": oracle.threads_used(),
                            "kind": "port", "sample": sample},
           "e2e": {"value": value, "unit": "slice-px/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "wall_s": wall}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
