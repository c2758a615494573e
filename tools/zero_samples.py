"""How many two-ended (T3 / T6) samples contribute nothing?  (diagnostics, GPU box)
Per technique: queries per sample (layer renders), and from dumped records of 2^16 strided indices per side the
fraction of samples whose every connection term (base and partner) is exactly zero."""
import collections
import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from rr_inputs import scenes as S  # noqa: E402
from paper_2406_16302_b200 import Renderer  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = S.load_config(cfg)
r = Renderer(0)
r.upload(w.scene)
r.set_edit(w.edits)
for l in range(1, 8):
    a = dataclasses.replace(w.args, layer_mask=1 << (l - 1))
    r.render_residual(a)
    torch.cuda.synchronize()
    st = r.get_stats()
    n = max(1, st["samples"])
    print(f"T{l}: samples {n} closest/sample {st['closest_rays'] / n:.2f} shadow/sample {st['shadow_rays'] / n:.2f} "
          f"inst/sample {st['instance_queries'] / n:.2f} conns/sample {st['connections'] / n:.2f} splats/sample {st['splats'] / n:.3f}",
          flush=True)
n_all = w.scene.camera.width * w.scene.camera.height * w.args.spp // 2
for l in (3, 6, 7, 2, 5):
    recs = []
    for i0 in np.linspace(0, n_all - 4096, 16).astype(int):
        recs += r.dump_paths(w.args, l, 0, int(i0), int(i0) + 4096)
    by = collections.defaultdict(lambda: [0, 0])
    for rec in recs:
        nz = any(abs(x) > 0 for x in rec.term_p) or any(abs(x) > 0 for x in rec.term_q)
        by[int(rec.i)][0] += 1
        by[int(rec.i)][1] += nz
    tot = 16 * 4096
    withrec = len(by)
    nz = sum(1 for v in by.values() if v[1] > 0)
    print(f"T{l}: {tot} samples, {withrec} with records, {nz} with a nonzero term ({nz / tot:.3f}); records/sample "
          f"{len(recs) / tot:.2f}", flush=True)
