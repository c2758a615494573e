"""Equal-budget quality harness (the paper's comparison protocol).

Estimators of the residual Delta = I(new) - I(old) compared against a high-sample reference:
  * "pt_difference"   -- path tracing from scratch in each state with independent seeds;
  * "correlated_pt"   -- camera paths only (T7), random-number replay in both states (mask {7}, one-way;
                         P:L510-511);
  * "residual"        -- the paper's method: all seven techniques, path mapping, two-way.
Each is timed with CUDA events on the device; mse() is taken against the reference and efficiency =
1 / (mse * seconds).  Scenes are the synthetic stand-ins of rr_inputs (no measured data).
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


def estimators(r, args, spp: int, seed: int = 0) -> Dict[str, tuple]:
    """{name: (image, seconds)} at `spp` samples per pixel per technique (PT: spp per state)."""
    out = {}
    out["pt_difference"] = _timed(lambda: r.render_primal(0, spp, seed + 11, args.max_depth).clone()
                                  - r.render_primal(1, spp, seed + 12, args.max_depth))
    corr = dataclasses.replace(args, spp=spp, seed=seed + 13, technique_mask=0x40, flags=0)
    out["correlated_pt"] = _timed(lambda: r.render_residual(corr).clone())
    full = dataclasses.replace(args, spp=spp + (spp & 1), seed=seed + 14, flags=PAPER_FLAGS)
    out["residual"] = _timed(lambda: r.render_residual(full).clone())
    return out


def mse(img: np.ndarray, ref: np.ndarray) -> float:
    return float(((img - ref) ** 2).mean())


def compare(r, args, spp: int, ref: np.ndarray, seed: int = 0) -> Dict[str, dict]:
    res = {}
    for name, (img, sec) in estimators(r, args, spp, seed).items():
        m = mse(img, ref)
        res[name] = {"mse": m, "seconds": sec, "efficiency": 1.0 / (m * sec) if m > 0 and sec > 0 else float("inf")}
    return res
