"""Traversal throughput of a stand-alone trace kernel on the residual estimator's kind of rays (diagnostics):
camera rays, then cosine-weighted secondary rays from the hit points (incoherent), then segments from the hit
points to random emitter points.  One query per thread, full warps (what a wavefront trace kernel would see).
  python tools/wave_probe.py CFG [N]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
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
up = torch.tensor(cam.up, dtype=torch.float32, device="cuda")
right = torch.linalg.cross(fwd, up); right /= torch.linalg.norm(right)
up2 = torch.linalg.cross(right, fwd)
th = np.tan(np.radians(cam.vfov_deg) / 2)
u = torch.rand((n, 2), generator=g, device="cuda") * 2 - 1
d = fwd + u[:, :1] * th * right + u[:, 1:] * th * up2
d = d / torch.linalg.norm(d, dim=1, keepdim=True)
nofl = torch.tensor([-1], dtype=torch.int32).view(torch.float32).item()


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record(); torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) / reps


rays = torch.zeros((n, 8), dtype=torch.float32, device="cuda")
rays[:, 0:3] = o; rays[:, 3:6] = d; rays[:, 6] = nofl
h, ms = timed(lambda: r.trace(0, rays))
print(f"config {cfg}: camera rays {n}: {ms:.2f} ms, {n / ms / 1e3:.1f} Mrays/s, hit {float((h[:, 0] >= 0).float().mean()):.3f}")
m = h[:, 0] >= 0
p, nrm, tri = h[m, 2:5], h[m, 5:8], h[m, 1]
dd = d[m]
flip = ((nrm * dd).sum(1, keepdim=True) > 0).float() * -2 + 1
nrm = nrm * flip                                           # facing the incoming ray
a = torch.rand((p.shape[0], 2), generator=g, device="cuda")
rr_, ph = a[:, :1].sqrt(), a[:, 1:] * 2 * np.pi
t1 = torch.where(nrm[:, :1].abs() < 0.9, torch.tensor([[1.0, 0, 0]], device="cuda"), torch.tensor([[0, 1.0, 0]], device="cuda"))
b1 = torch.linalg.cross(nrm, t1); b1 /= torch.linalg.norm(b1, dim=1, keepdim=True)
b2 = torch.linalg.cross(nrm, b1)
wd = b1 * rr_ * torch.cos(ph) + b2 * rr_ * torch.sin(ph) + nrm * (1 - a[:, :1]).sqrt()
sec = torch.zeros((p.shape[0], 8), dtype=torch.float32, device="cuda")
sec[:, 0:3] = p; sec[:, 3:6] = wd; sec[:, 6] = tri
h2, ms = timed(lambda: r.trace(0, sec))
k = sec.shape[0]
print(f"   secondary (cosine) rays {k}: {ms:.2f} ms, {k / ms / 1e3:.1f} Mrays/s, hit {float((h2[:, 0] >= 0).float().mean()):.3f}")
# segments from the hit points toward random points of the lights' bounding box (emissive objects)
em = np.nonzero(np.abs(np.asarray(w.scene.obj_emission)).sum(1) > 0)[0]
tris = np.nonzero(np.isin(np.asarray(w.scene.tri_object), em[:3] if len(em) > 3 else em))[0]
verts = np.asarray(w.scene.positions)[np.asarray(w.scene.indices)[tris]].reshape(-1, 3)
if cfg == 3:
    verts = verts[verts[:, 1] > 2.0]
lo, hi = verts.min(0), verts.max(0)
tgt = torch.tensor(lo, device="cuda") + torch.rand((k, 3), generator=g, device="cuda") * torch.tensor(hi - lo + 1e-3, device="cuda")
segs = torch.cat([p + nrm * 1e-3, tgt.float()], 1).contiguous()
s_out, ms = timed(lambda: r.segment(segs))
print(f"   segments to lights {k}: {ms:.2f} ms, {k / ms / 1e3:.1f} Msegs/s (both states), visible {float((s_out[:, 0] > 0.5).float().mean()):.3f}")
