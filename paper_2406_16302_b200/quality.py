"""Equal-budget quality harness (the paper's comparison protocol).

Estimators of the residual Delta = I(new) - I(old):
  * "pt_difference"    -- path tracing from scratch in each state with independent seeds;
  * "correlated_pt"    -- camera paths only (T7), random-number replay in both states (mask {7}, one-way;
                          P:L510-511);
  * "residual"         -- the paper's method: all seven techniques, path mapping, two-way;
ablations of the method:
  * "residual_no_pm"   -- "incremental w/o PM" (Table num_of_dynamics): both states sampled by the
                          dynamic techniques separately, no path mapping (RR_NO_PATH_MAPPING);
  * "residual_replay"  -- two-way, no reconnection: diverged paths are replayed only (RR_RECONNECT off);
  * "residual_one_way" -- one side per technique, replay only (flags 0; SPEC's "mapping off" run knob);
  * "residual_vndf"    -- the paper's mode with GGX visible-normal sampling (RR_VNDF);
  * "residual_t6_light", "residual_tobj", "residual_recon_bidir", "residual_variants" -- the paper's mode with
                          RR_T6_TOWARD_LIGHT, RR_TOBJ_MIDPATH, RR_RECONNECT_BIDIR, and all three (row 4).

The reference is NOT any of these estimators: it is the GPU primal renderer (unidirectional NEE/BSDF-MIS path
tracing, rr_primal.cu, checked against the CPU reference's primal renderer by the tests) run in both states with the SAME random numbers
(RR_PRIMAL_SHARED_STREAMS) at high spp -- a correlated, unbiased estimate of I(new) - I(old) that shares no code
with the residual estimator.  Its own variance is estimated from its chunks and subtracted from every MSE
(mse = mean |x - ref|^2 - var(ref)), so a reference noisier than intended cannot flatter or hurt an estimator.
Every estimator is timed with CUDA events on the device; efficiency = 1 / (mse * seconds), and the
MSE "at equal time" of estimator e against the paper's residual = mse_e * t_e / t_residual (the paper's tables).
Scenes are the synthetic stand-ins of rr_inputs (no measured data).
"""
from __future__ import annotations

import dataclasses
from typing import Dict

import numpy as np

PAPER_FLAGS = 7
NO_PATH_MAPPING = 256


def _timed(fn):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    img = fn()
    e1.record()
    torch.cuda.synchronize()
    return img[..., :3].double().cpu().numpy(), e0.elapsed_time(e1) / 1e3


def reference(r, args, spp: int = 65536, chunk: int = 4096, seed: int = 1 << 20):
    """(mean, variance of the mean per pixel) of the correlated primal difference primal(N) - primal(O) at `spp`
    samples per pixel, in chunks of `chunk` spp with distinct seeds."""
    imgs = []
    for k in range(max(1, spp // chunk)):
        img, _ = _timed(lambda: r.render_primal(0, chunk, seed + k, args.max_depth, shared_streams=True).clone()
                        - r.render_primal(1, chunk, seed + k, args.max_depth, shared_streams=True))
        imgs.append(img)
    a = np.stack(imgs)
    return a.mean(0), (a.var(0) / len(a) if len(a) > 1 else np.zeros_like(a[0]))


def reference_primal(r, state: int, max_depth: int, spp: int = 16384, chunk: int = 4096, seed: int = 3 << 20):
    """(mean, variance of the mean) of primal(state) at `spp` spp: the reference of PT from scratch"""
    imgs = [_timed(lambda: r.render_primal(state, chunk, seed + k, max_depth).clone())[0]
            for k in range(max(1, spp // chunk))]
    a = np.stack(imgs)
    return a.mean(0), (a.var(0) / len(a) if len(a) > 1 else np.zeros_like(a[0]))


def estimators(r, args, spp: int, seed: int = 0, ablations: bool = False) -> Dict[str, tuple]:
    """{name: (image, seconds)} at `spp` samples per pixel per technique (PT: spp per state)."""
    out = {}
    out["pt_difference"] = _timed(lambda: r.render_primal(0, spp, seed + 11, args.max_depth).clone()
                                  - r.render_primal(1, spp, seed + 12, args.max_depth))
    corr = dataclasses.replace(args, spp=spp, seed=seed + 13, technique_mask=0x40, flags=0)
    out["correlated_pt"] = _timed(lambda: r.render_residual(corr).clone())
    full = dataclasses.replace(args, spp=spp + (spp & 1), seed=seed + 14, flags=PAPER_FLAGS)
    out["residual"] = _timed(lambda: r.render_residual(full).clone())
    nopm = dataclasses.replace(full, seed=seed + 18, flags=1 | NO_PATH_MAPPING)
    out["residual_no_pm"] = _timed(lambda: r.render_residual(nopm).clone())
    if ablations:
        rep = dataclasses.replace(full, seed=seed + 15, flags=PAPER_FLAGS & ~2)
        out["residual_replay"] = _timed(lambda: r.render_residual(rep).clone())
        one = dataclasses.replace(args, spp=spp, seed=seed + 16, flags=0)
        out["residual_one_way"] = _timed(lambda: r.render_residual(one).clone())
        vn = dataclasses.replace(full, seed=seed + 17, flags=PAPER_FLAGS | 32)
        out["residual_vndf"] = _timed(lambda: r.render_residual(vn).clone())
        # the other SURVEY 8(f) row 4 variants (each alone and all three together)
        for name, f in (("residual_t6_light", 512), ("residual_tobj", 1024), ("residual_recon_bidir", 2048),
                        ("residual_variants", 512 | 1024 | 2048)):
            va = dataclasses.replace(full, seed=seed + 19, flags=PAPER_FLAGS | f)
            out[name] = _timed(lambda: r.render_residual(va).clone())
    return out


def mse(img: np.ndarray, ref, ref_var=None) -> float:
    """mean squared error against the reference, minus the reference's own variance (unbiased for the error
    of `img` when the reference's noise is independent of it)"""
    m = float(((img - ref) ** 2).mean())
    return m - float(ref_var.mean()) if ref_var is not None else m


def _box(a: np.ndarray, k: int) -> np.ndarray:
    """mean over every k x k window (valid positions only), via a summed-area table"""
    c = np.pad(a, ((1, 0), (1, 0))).cumsum(0).cumsum(1)
    return (c[k:, k:] - c[:-k, k:] - c[k:, :-k] + c[:-k, :-k]) / (k * k)


def ssim(img: np.ndarray, ref: np.ndarray, k: int = 7) -> float:
    """Mean structural similarity (Wang et al. 2004) of the channel-mean images, k x k uniform windows,
    C1 = (0.01 L)^2, C2 = (0.03 L)^2 with L the reference's value range (residuals are signed)."""
    x, y = img.mean(axis=-1), ref.mean(axis=-1)
    L = float(y.max() - y.min()) or 1.0
    c1, c2 = (0.01 * L) ** 2, (0.03 * L) ** 2
    mx, my = _box(x, k), _box(y, k)
    vx, vy, cxy = _box(x * x, k) - mx * mx, _box(y * y, k) - my * my, _box(x * y, k) - mx * my
    s = ((2 * mx * my + c1) * (2 * cxy + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2))
    return float(s.mean())


def compare(r, args, spp: int, ref, seed: int = 0, ablations: bool = False) -> Dict[str, dict]:
    """ref = (mean, variance of the mean) from reference()"""
    ref_mean, ref_var = ref
    res = {}
    estimators(r, args, spp, seed + 1000, ablations)  # warm-up: first launches of each kernel are not timed
    for name, (img, sec) in estimators(r, args, spp, seed, ablations).items():
        m = mse(img, ref_mean, ref_var)
        res[name] = {"mse": m, "ssim": ssim(img, ref_mean), "seconds": sec,
                     "efficiency": 1.0 / (m * sec) if m > 0 and sec > 0 else float("inf")}
    t0 = res["residual"]["seconds"]
    for v in res.values():
        v["mse_at_residual_time"] = v["mse"] * v["seconds"] / t0
    res["_reference"] = {"variance_of_mean": float(ref_var.mean()), "max_abs": float(np.abs(ref_mean).max())}
    return res


def technique_variance(r, args, spp: int, n_seeds: int = 16, seed: int = 500) -> Dict[int, dict]:
    """Per technique l: the variance its MIS-weighted layer adds to the residual (mean over pixels of the
    per-pixel variance over n_seeds renders; the layers of different techniques are independent), and its
    device time per render.  Shows which technique's samples the estimator's noise and cost come from."""
    import torch
    layers = {}
    times = {}
    a0 = dataclasses.replace(args, spp=spp + (spp & 1), flags=PAPER_FLAGS)
    for k in range(n_seeds):
        a = dataclasses.replace(a0, seed=seed + k)
        for l in range(1, 8):
            if not (int(a.technique_mask) >> (l - 1)) & 1:
                continue
            img, sec = _timed(lambda: r.render_residual(dataclasses.replace(a, layer_mask=1 << (l - 1))).clone())
            layers.setdefault(l, []).append(img)
            times.setdefault(l, []).append(sec)
    torch.cuda.synchronize()
    out = {}
    tot_var = sum(float(np.stack(v).var(0).mean()) for v in layers.values())
    tot_t = sum(float(np.median(t)) for t in times.values())
    for l, v in layers.items():
        var = float(np.stack(v).var(0).mean())
        t = float(np.median(times[l]))
        out[l] = {"variance": var, "variance_share": var / tot_var if tot_var > 0 else 0.0, "seconds": t,
                  "time_share": t / tot_t if tot_t > 0 else 0.0,
                  "mean_abs": float(np.abs(np.stack(v).mean(0)).mean())}
    return out


def sweep_row(r, w, spp: int, ref_spp: int = 65536, pt_ref_spp: int = 16384) -> dict:
    """One row of the paper's Table num_of_dynamics / Table material_editing: MSE at equal time (the paper's
    residual's time) and SSIM of PT from scratch (of the NEW image against its own high-spp reference),
    correlated PT, incremental w/o PM and incremental w/ PM (residuals: I_new = I_old + Delta with a converged
    I_old, so the error of I_new is the error of Delta)."""
    args = w.args
    ref = reference(r, args, ref_spp)
    res = compare(r, args, spp, ref)
    new_mean, new_var = reference_primal(r, 0, args.max_depth, pt_ref_spp)
    _timed(lambda: r.render_primal(0, spp, 77, args.max_depth))  # warm-up
    img, sec = _timed(lambda: r.render_primal(0, spp, 78, args.max_depth).clone())
    m = mse(img, new_mean, new_var)
    res["pt_from_scratch"] = {"mse": m, "ssim": ssim(img, new_mean), "seconds": sec,
                              "efficiency": 1.0 / (m * sec) if m > 0 else float("inf"),
                              "mse_at_residual_time": m * sec / res["residual"]["seconds"]}
    return res
