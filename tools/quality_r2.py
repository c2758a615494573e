"""Round-2 quality study: every estimator against the correlated
primal-difference reference on configs 1-3 at 256^2, the per-technique variance / time split, and the sweeps of
the paper's Table num_of_dynamics (dynamic count 1/2/4/8, displacement ladder) and Table material_editing.
  python tools/quality_r2.py [out.json]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from rr_inputs import scenes as S  # noqa: E402
from paper_2406_16302_b200 import Renderer, quality as Q  # noqa: E402

out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/quality_r2.json"
W, SPP = 256, 16
out = {"resolution": W, "spp": SPP, "configs": {}, "technique_variance": {}, "sweeps": {}}


def renderer(w):
    r = Renderer(0)
    r.upload(w.scene)
    r.set_edit(w.edits)
    return r


def short(res):
    return {k: (f"{v['mse']:.2e}", f"eq-time {v['mse_at_residual_time']:.2e}", round(v["ssim"], 3),
                round(1e3 * v["seconds"], 1)) for k, v in res.items() if not k.startswith("_")}


t0 = time.time()
for c in (1, 2, 3):
    w = S.load_config(c, width=W, height=W)
    r = renderer(w)
    ref = Q.reference(r, w.args, 65536 if c < 3 else 16384)
    res = Q.compare(r, w.args, SPP, ref, ablations=True)
    out["configs"][f"config{c}"] = res
    print(f"config {c}:", short(res), flush=True)
    if c in (1, 3):
        tv = Q.technique_variance(r, w.args, SPP, n_seeds=8)
        out["technique_variance"][f"config{c}"] = tv
        print("   per technique (variance share, time share):",
              {l: (round(v["variance_share"], 3), round(v["time_share"], 3)) for l, v in tv.items()}, flush=True)
    # reconnection threshold on the material edit: alpha_min just above the edited roughness 0.1
    if c == 2:
        import dataclasses
        a2 = dataclasses.replace(w.args, alpha_min=0.15)
        res2 = Q.compare(r, a2, SPP, ref)
        out["configs"]["config2_alpha_min_0.15"] = res2
        print("config 2, alpha_min 0.15:", short(res2), flush=True)
    del r
rows = [(f"dynamics{n}", S.cornell_dynamics(n, width=W, height=W)) for n in (1, 2, 4, 8)]
rows += [(f"displacement{d}", S.cornell_displacement(d, width=W, height=W)) for d in S.DISPLACEMENT_LADDER]
rows += [(f"material_{k}", S.cornell_material_edit(k, width=W, height=W)) for k in S.MATERIAL_EDITS]
for name, w in rows:
    r = renderer(w)
    res = Q.sweep_row(r, w, SPP)
    out["sweeps"][name] = res
    print(name, short(res), flush=True)
    del r
out["wall_s"] = time.time() - t0
json.dump(out, open(out_path, "w"), indent=1)
