"""Where does a GPU-vs-oracle image difference come from?  (diagnostics, GPU box)

  python tools/pixel_diff.py CFG W H SPP
Renders the residual per technique on the GPU and in the oracle (spawn pool over the host cores), reports the
worst pixel and each technique's share of its difference, then joins the per-connection records of the worst
technique that splat into that pixel and prints the mismatching ones."""
import dataclasses
import multiprocessing as mp
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from rr_inputs import scenes as S  # noqa: E402


def workload(cfg, W, H, spp):
    return S.load_config(cfg, width=W, height=H, spp=spp)


def oracle_part(a):
    (cfg, W, H, spp), l, side, i0, i1, pix = a
    from oracle import binding as OB
    w = workload(cfg, W, H, spp)
    o = OB.Oracle(w.scene, w.edits)
    img = np.zeros((o.H, o.W, 3))
    _, recs, _ = o.residual(w.args, l, side, i0, i1, records=pix is not None, image=img)
    keep = []
    if pix is not None:
        for r in recs:
            if r.pix_p == pix or r.pix_q == pix:
                keep.append((int(r.tech), int(r.side), int(r.i), int(r.key_kind), int(r.key_a), int(r.key_b),
                             int(r.status), int(r.reason), int(r.pix_p), list(r.term_p), int(r.pix_q), list(r.term_q),
                             float(r.R)))
    return img, keep


def main():
    cfg, W, H, spp = (int(x) for x in sys.argv[1:5])
    key = (cfg, W, H, spp)
    import torch
    from paper_2406_16302_b200 import Renderer
    from oracle import binding as OB
    w = workload(*key)
    r = Renderer(0)
    r.upload(w.scene)
    r.set_edit(w.edits)
    layers = {l: x[..., :3].double().cpu().numpy() for l, x in r.render_layers(w.args).items()}
    torch.cuda.synchronize()
    o = OB.Oracle(w.scene, w.edits)
    n = o.sample_range(w.args)
    mask = o.effective_mask(w.args.technique_mask)
    nt = os.cpu_count() or 8
    ctx = mp.get_context("spawn")
    olay = {}
    with ctx.Pool(nt) as p:
        for l in range(1, 8):
            if not (mask >> (l - 1)) & 1:
                continue
            jobs = [(key, l, s, n * k // nt, n * (k + 1) // nt, None) for s in o.sides(w.args) for k in range(nt)]
            olay[l] = sum(img for img, _ in p.map(oracle_part, jobs))
    g = sum(layers[l] for l in olay)
    ref = sum(olay.values())
    err = np.abs(g - ref).max(axis=2)
    P = np.unravel_index(np.argmax(err), err.shape)
    pix = int(P[0]) * W + int(P[1])
    print(f"config {cfg} {W}x{H} {spp} spp: max|ref| {np.abs(ref).max():.4g}, rmse {np.sqrt(((g - ref) ** 2).mean()):.4g}, "
          f"worst pixel {P} err {err.max():.4g} (gpu {g[P].tolist()} oracle {ref[P].tolist()})")
    per = {l: float(np.abs(layers[l][P] - olay[l][P]).max()) for l in olay}
    print("   per-technique |diff| at the worst pixel:", {l: round(v, 6) for l, v in per.items()})
    L = max(per, key=per.get)
    # records of technique L that splat into the pixel
    grec = {}
    chunk = 1 << 16
    for s in o.sides(w.args):
        for i0 in range(0, n, chunk):
            for rec in r.dump_paths(w.args, L, s, i0, min(n, i0 + chunk)):
                if rec.pix_p == pix or rec.pix_q == pix:
                    grec[(L, s, int(rec.i), int(rec.key_kind), int(rec.key_a), int(rec.key_b))] = (
                        int(rec.status), int(rec.reason), int(rec.pix_p), list(rec.term_p), int(rec.pix_q),
                        list(rec.term_q), float(rec.R))
    orec = {}
    with ctx.Pool(nt) as p:
        jobs = [(key, L, s, n * k // nt, n * (k + 1) // nt, pix) for s in o.sides(w.args) for k in range(nt)]
        for _, keep in p.map(oracle_part, jobs):
            for t in keep:
                orec[t[:6]] = t[6:]
    print(f"   technique {L}: {len(grec)} gpu / {len(orec)} oracle records touch the pixel")
    rows = []
    for k in set(grec) | set(orec):
        a, b = grec.get(k), orec.get(k)
        ga = np.zeros(3) if a is None else (np.array(a[3]) if a[2] == pix else 0) + (np.array(a[5]) if a[4] == pix else 0)
        ob = np.zeros(3) if b is None else (np.array(b[3]) if b[2] == pix else 0) + (np.array(b[5]) if b[4] == pix else 0)
        d = float(np.abs(np.asarray(ga) - np.asarray(ob)).max())
        rows.append((d, k, a, b))
    rows.sort(key=lambda x: -x[0])
    for d, k, a, b in rows[:8]:
        print(f"   diff {d:.4g} key {k}\n      gpu    {a}\n      oracle {b}")


if __name__ == "__main__":
    main()
