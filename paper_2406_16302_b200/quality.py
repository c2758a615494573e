"""Equal-budget quality harness (the paper's comparison protocol).

Estimators of the residual Delta = I(new) - I(old) compared against a high-sample reference:
  * "pt_difference"   -- path tracing from scratch in each state with independent seeds;
  * "correlated_pt"   -- camera paths only (T7), random-number replay in both states (mask {7}, one-way;
                         P:L510-511);
  * "residual"        -- the paper's method: all seven techniques, path mapping, two-way;
ablations of the method (the mapping components of P:L387-436, one at a time):
  * "residual_replay" -- two-way, no reconnection: diverged paths are replayed only (RR_RECONNECT off);
  * "residual_one_way"-- one side per technique, replay only (flags 0; SPEC's "mapping off" run knob);
and the paper's mode with GGX visible-normal sampling ("residual_vndf", RR_VNDF).
Each is timed with CUDA events on the device; mse() and ssim() are taken against the reference and
efficiency = 1 / (mse * seconds).  Scenes are the synthetic stand-ins of rr_inputs (no
measured data).
"""
from __future__ import annotations

import dataclasses
from typing import Dict

import numpy as np

PAPER_FLAGS = 7


def _timed(fn):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    img = fn()
    e1.record()
    torch.cuda.synchronize()
    return img[..., :3].double().cpu().numpy(), e0.elapsed_time(e1) / 1e3


def reference(r, args, spp: int = 1024, seed: int = 1 << 20) -> np.ndarray:
    """High-sample residual (all techniques, two-way) on seeds disjoint from every estimator below.  Unbiased
    (record-level parity with the CPU reference implementation, whose residual converges to I(new) - I(old) in
    its tests), and its variance is far below a path-traced difference of the same spp, which would dominate
    every MSE."""
    a = dataclasses.replace(args, spp=spp + (spp & 1), seed=seed, flags=PAPER_FLAGS)
    img, _ = _timed(lambda: r.render_residual(a).clone())
    return img


def estimators(r, args, spp: int, seed: int = 0, ablations: bool = False) -> Dict[str, tuple]:
    """{name: (image, seconds)} at `spp` samples per pixel per technique (PT: spp per state)."""
    out = {}
    out["pt_difference"] = _timed(lambda: r.render_primal(0, spp, seed + 11, args.max_depth).clone()
                                  - r.render_primal(1, spp, seed + 12, args.max_depth))
    corr = dataclasses.replace(args, spp=spp, seed=seed + 13, technique_mask=0x40, flags=0)
    out["correlated_pt"] = _timed(lambda: r.render_residual(corr).clone())
    full = dataclasses.replace(args, spp=spp + (spp & 1), seed=seed + 14, flags=PAPER_FLAGS)
    out["residual"] = _timed(lambda: r.render_residual(full).clone())
    if ablations:
        rep = dataclasses.replace(full, seed=seed + 15, flags=PAPER_FLAGS & ~2)
        out["residual_replay"] = _timed(lambda: r.render_residual(rep).clone())
        one = dataclasses.replace(args, spp=spp, seed=seed + 16, flags=0)
        out["residual_one_way"] = _timed(lambda: r.render_residual(one).clone())
        vn = dataclasses.replace(full, seed=seed + 17, flags=PAPER_FLAGS | 32)
        out["residual_vndf"] = _timed(lambda: r.render_residual(vn).clone())
    return out


def mse(img: np.ndarray, ref: np.ndarray) -> float:
    return float(((img - ref) ** 2).mean())


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


def compare(r, args, spp: int, ref: np.ndarray, seed: int = 0, ablations: bool = False) -> Dict[str, dict]:
    res = {}
    estimators(r, args, spp, seed + 1000, ablations)  # warm-up: first launches of each kernel are not timed
    for name, (img, sec) in estimators(r, args, spp, seed, ablations).items():
        m = mse(img, ref)
        res[name] = {"mse": m, "ssim": ssim(img, ref), "seconds": sec,
                     "efficiency": 1.0 / (m * sec) if m > 0 and sec > 0 else float("inf")}
    return res
