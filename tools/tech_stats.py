import os, sys
sys.path.insert(0, os.getcwd())
import torch
from rr_inputs import scenes as S
from paper_2406_16302_b200 import Renderer
import dataclasses
w = S.load_config(4)
r = Renderer(0); r.upload(w.scene); r.set_edit(w.edits)
for l in range(1, 8):
    a = dataclasses.replace(w.args, layer_mask=1 << (l - 1))
    r.render_residual(a); torch.cuda.synchronize()
    st = r.get_stats()
    print(l, {k: st[k] for k in ("samples", "connections", "splats", "offscreen", "zero_pairs", "closest_rays", "shadow_rays", "instance_queries")})
