"""Quick GPU timing of one residual render per config (diagnostics, not the bench)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from rr_inputs import scenes as S  # noqa: E402
from paper_2406_16302_b200 import Renderer  # noqa: E402

cfgs = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2", "3", "4"])]
for k in cfgs:
    w = S.load_config(k)
    r = Renderer(0)
    t0 = time.time()
    r.upload(w.scene)
    r.set_edit(w.edits)
    torch.cuda.synchronize()
    t_up = time.time() - t0
    img = r.render_residual(w.args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    img = r.render_residual(w.args, image=img)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    tm = r.last_timings(16)
    r.render_residual(w.args, image=img, count_traversal=True)  # node / triangle counts (untimed)
    st = r.get_stats()
    n = st["samples"]
    print(f"config {k}: upload+lbvh {t_up:.2f}s  render {ms:.1f} ms  samples {n} ({n / ms / 1e3:.1f} M/s)  "
          f"closest {st['closest_rays']} shadow {st['shadow_rays']} inst {st['instance_queries']} "
          f"Mrays/s {(st['closest_rays'] + st['shadow_rays']) / ms / 1e3:.1f}  nodes {st['nodes_visited']} tris {st['tris_tested']} "
          f"GB/s(alg) {(64 * st['nodes_visited'] + 48 * st['tris_tested']) / ms / 1e6:.1f}", flush=True)
    sc = st["sched"]
    if sc[0]:
        print(f"   sched: queries/round {sc[3] / sc[0]:.1f}, lanes holding {sc[4] / sc[0]:.1f}/32, bvh depth {sc[5]}",
              flush=True)
    print("   per launch ms:", [round(x, 2) for x in tm[1:15]], " img sum", img[..., :3].sum().item(), flush=True)
    del r
