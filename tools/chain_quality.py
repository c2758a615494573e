"""Config-5 chain quality (Eq.3): error growth over 16 chained residuals.

  python tools/chain_quality.py [W H SPP REF_SPP]      (default 320 180 8 1024)

I_0 = a REF_SPP primal of the first state; frame f applies the edit S_f -> S_f+1 and adds its residual
(SPP per technique, seed 5000 + f).  After every frame the chained image I_0 + sum Delta is compared with an
independent REF_SPP primal of S_f+1 (disjoint seeds), and with a fresh SPP-matched primal of S_f+1 at the
same device time as the residual (path tracing the new frame from scratch instead of chaining).  MSE over RGB;
the reference's own noise is reported as 2 x its variance estimate from two half-spp renders."""
import dataclasses
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from rr_inputs import scenes as S  # noqa: E402
from paper_2406_16302_b200 import Renderer  # noqa: E402


def main():
    import torch
    W, H, spp, ref_spp = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (320, 180, 8, 1024)))
    w = S.config5(W, H, spp=spp)
    D = w.args.max_depth
    r = Renderer(0)
    r.upload(w.scene)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def timed(fn):
        torch.cuda.synchronize()
        ev[0].record()
        out = fn()
        ev[1].record()
        torch.cuda.synchronize()
        return out, ev[0].elapsed_time(ev[1]) / 1e3

    r.set_edit(w.frames[0])
    chain = r.render_primal(1, ref_spp, 777, D).clone()  # I_0 (old state of frame 0)
    rows = []
    for f, edits in enumerate(w.frames):
        r.set_edit(edits)
        a = dataclasses.replace(w.args, seed=int(w.args.seed) + f)
        r.render_residual(a)  # warm (first launch of the frame's kernels is not timed)
        delta, t_res = timed(lambda: r.render_residual(a).clone())
        chain += delta
        ref = r.render_primal(0, ref_spp, 100000 + f, D).clone()
        half = [r.render_primal(0, ref_spp // 2, 200000 + 2 * f + k, D).clone() for k in (0, 1)]
        ref_noise = float(((half[0] - half[1])[..., :3] ** 2).mean().item()) / 4.0  # var of the REF_SPP mean
        # a fresh primal of S_f+1 at the residual's device time: spp scaled by measured primal throughput
        _, t_p = timed(lambda: r.render_primal(0, 8, 300000 + f, D))
        pt_spp = max(1, int(round(8 * t_res / t_p)))
        fresh, t_fresh = timed(lambda: r.render_primal(0, pt_spp, 400000 + f, D).clone())
        mse = lambda x: float(((x - ref)[..., :3] ** 2).mean().item())  # noqa: E731
        rows.append({"frame": f, "mse_chain": mse(chain), "mse_fresh_pt": mse(fresh), "fresh_pt_spp": pt_spp,
                     "ref_noise_mse": ref_noise, "residual_s": t_res, "fresh_pt_s": t_fresh})
        print(json.dumps(rows[-1]), flush=True)
    print(json.dumps({"config": 5, "resolution": [W, H], "spp": spp, "reference_spp": ref_spp, "frames": rows}))


if __name__ == "__main__":
    main()
