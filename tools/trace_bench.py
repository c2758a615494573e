"""Traversal-only microbenchmark: rr_trace (closest hit, one query per thread) on random camera-like
rays of a config's scene.  python tools/trace_bench.py CFG [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from rr_inputs import scenes as S  # noqa: E402
from paper_2406_16302_b200 import Renderer  # noqa: E402

cfg = int(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else (1 << 22)
w = S.load_config(cfg)
r = Renderer(0)
r.upload(w.scene)
r.set_edit(w.edits)
g = torch.Generator(device="cuda").manual_seed(1)
cam = w.scene.camera
o = torch.tensor(cam.pos, dtype=torch.float32, device="cuda")
look = torch.tensor(cam.look_at, dtype=torch.float32, device="cuda")
fwd = (look - o) / torch.linalg.norm(look - o)
coherent = os.environ.get("COHERENT", "0") == "1"
if coherent:  # pixel-ordered pinhole rays over a square image (adjacent lanes: adjacent pixels)
    side = int(n ** 0.5)
    n = side * side
    up = torch.tensor(cam.up, dtype=torch.float32, device="cuda")
    right = torch.linalg.cross(fwd, up)
    right = right / torch.linalg.norm(right)
    up2 = torch.linalg.cross(right, fwd)
    ys, xs = torch.meshgrid(torch.linspace(-0.5, 0.5, side, device="cuda"), torch.linspace(-0.5, 0.5, side, device="cuda"), indexing="ij")
    d = fwd + xs.reshape(-1, 1) * right + ys.reshape(-1, 1) * up2
else:
    d = torch.randn((n, 3), generator=g, device="cuda") * 0.35 + fwd
d = d / torch.linalg.norm(d, dim=1, keepdim=True)
rays = torch.zeros((n, 8), dtype=torch.float32, device="cuda")
rays[:, 0:3] = o
rays[:, 3:6] = d
rays[:, 6] = torch.tensor([-1], dtype=torch.int32).view(torch.float32).item()
for _ in range(2):
    h = r.trace(0, rays)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 5
for _ in range(reps):
    h = r.trace(0, rays)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
hit = (h[:, 0] >= 0).float().mean().item()
print(f"config {cfg}: {n} {'coherent' if coherent else 'random'} camera rays, {ms:.2f} ms, {n / ms / 1e3:.1f} Mrays/s, hit fraction {hit:.3f}")
