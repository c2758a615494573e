"""Render one residual image of a (reduced) config for ncu captures: python tools/profile_run.py CFG W MASK [SPP]"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from rr_inputs import scenes as S  # noqa: E402
from paper_2406_16302_b200 import Renderer  # noqa: E402

cfg, W, mask = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3], 0)
spp = int(sys.argv[4]) if len(sys.argv) > 4 else None
w = S.load_config(cfg)
w = S.subsample(w, W, W)
args = dataclasses.replace(w.args, technique_mask=mask, **({"spp": spp} if spp else {}))
r = Renderer(0)
r.upload(w.scene)
r.set_edit(w.edits)
for _ in range(2):
    img = r.render_residual(args)
torch.cuda.synchronize()
st = r.get_stats()
print("samples", st["samples"], "rays", st["closest_rays"] + st["shadow_rays"], "timings", r.last_timings(4)[:3])
