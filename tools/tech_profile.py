"""Per-technique cost breakdown of one config (diagnostics): for each technique l, a render of exactly its
launches (layer_mask = T_l, full technique mask so MIS and pairing are the production ones), timed, then
counted (RR_COUNT_TRAVERSAL): samples, ns per sample, queries / node visits per sample, share of node visits
in dynamic-instance and ghost-crossing jobs, warp-round statistics.   python tools/tech_profile.py CFG [W]"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from rr_inputs import scenes as S  # noqa: E402
from paper_2406_16302_b200 import Renderer  # noqa: E402

cfg = int(sys.argv[1])
w = S.load_config(cfg)
if len(sys.argv) > 2:
    w = S.subsample(w, int(sys.argv[2]), int(sys.argv[2]))
r = Renderer(0)
r.upload(w.scene)
r.set_edit(w.edits)
img = r.render_residual(w.args)
torch.cuda.synchronize()
tot_ms = 0.0
for l in range(1, 8):
    a = dataclasses.replace(w.args, layer_mask=1 << (l - 1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r.render_residual(a, image=img)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    tot_ms += ms
    r.render_residual(a, image=img, count_traversal=True)
    torch.cuda.synchronize()
    st = r.get_stats()
    n = max(st["samples"], 1)
    sc = st["sched"]
    q = st["closest_rays"] + st["shadow_rays"]
    print(f"T{l}: {ms:8.1f} ms  samples {st['samples']:>10}  {1e6 * ms / n:6.1f} ns/sample  "
          f"closest {st['closest_rays'] / n:5.2f} shadow {st['shadow_rays'] / n:5.2f} inst {st['instance_queries'] / n:5.2f} /sample  "
          f"nodes {st['nodes_visited'] / n:7.1f} /sample ({st['nodes_visited'] / max(q, 1):5.1f} /static query; "
          f"inst jobs {sc[6] / max(st['nodes_visited'], 1):.2f}, ghost jobs {sc[7] / max(st['nodes_visited'], 1):.2f})  "
          f"tris {st['tris_tested'] / n:6.1f}  queries/round {sc[3] / max(sc[0], 1):5.1f} lanes {sc[4] / max(sc[0], 1):4.1f}",
          flush=True)
print(f"total {tot_ms:.1f} ms")
