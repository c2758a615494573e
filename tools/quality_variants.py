"""SURVEY 8(f) row 4 variants against the paper's mode, at 256^2 / 16 spp on configs 1-3 (MSE against the
correlated primal-difference reference, device time), as in tools/quality_r2.py.
  python tools/quality_variants.py [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from rr_inputs import scenes as S  # noqa: E402
from paper_2406_16302_b200 import Renderer, quality as Q  # noqa: E402

out = {}
for c in (1, 2, 3):
    w = S.load_config(c, width=256, height=256)
    r = Renderer(0)
    r.upload(w.scene)
    r.set_edit(w.edits)
    ref = Q.reference(r, w.args, 65536 if c < 3 else 16384)
    res = Q.compare(r, w.args, 16, ref, ablations=True)
    keep = ("residual", "residual_vndf", "residual_t6_light", "residual_tobj", "residual_recon_bidir",
            "residual_variants", "residual_replay", "correlated_pt")
    out[f"config{c}"] = {k: res[k] for k in keep if k in res}
    print(c, {k: (f"{v['mse']:.3e}", f"{v['mse_at_residual_time']:.3e}", round(1e3 * v["seconds"], 1))
              for k, v in out[f"config{c}"].items()}, flush=True)
    del r
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/quality_variants.json", "w"), indent=1)
