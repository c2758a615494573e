"""CUDA-graph capture of one residual render (VERDICT r1 missing #5): rr_render_residual only enqueues work on the
given stream (memsets, the ordering pre-pass with its CUB sorts, one launch per (technique, side), event records),
so after one warm-up render (which grows the scratch buffers) the whole render can be captured and replayed.
Times direct calls against graph replays per config (diagnostics, not the bench)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from rr_inputs import scenes as S  # noqa: E402
from paper_2406_16302_b200 import Renderer  # noqa: E402

cfgs = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2", "3", "4"])]
for k in cfgs:
    w = S.load_config(k)
    r = Renderer(0)
    r.upload(w.scene)
    r.set_edit(w.edits)
    reps = {1: 200, 2: 50, 3: 5}.get(k, 2)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        img = r.render_residual(w.args)
        img = r.render_residual(w.args, image=img)
        s.synchronize()
        ref = img.clone()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            r.render_residual(w.args, image=img)
        e1.record()
        s.synchronize()
        direct = e0.elapsed_time(e1) / reps
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        r.render_residual(w.args, image=img)
    with torch.cuda.stream(s):
        g.replay()
        s.synchronize()
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        s.synchronize()
        graph = e0.elapsed_time(e1) / reps
    d = (img[..., :3] - ref[..., :3]).abs().max().item()
    sc = ref[..., :3].abs().max().item()
    print(f"config {k}: direct {direct:.3f} ms  graph replay {graph:.3f} ms  ({100 * (graph / direct - 1):+.2f}%)  "
          f"max |graph - direct| {d:.3e} of {sc:.3e} (atomic splat order)", flush=True)
    del g, r
