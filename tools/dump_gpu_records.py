"""Dump GPU per-connection records (and traced hits) to gpurun_out/*.npz for offline comparison."""
import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from rr_inputs import scenes as S  # noqa: E402
from paper_2406_16302_b200 import Renderer  # noqa: E402

OUT = os.environ.get("RR_REC_DIR", "gpurun_out")


def recs_to_np(recs):
    a = np.zeros((len(recs), 17), np.float64)
    for k, r in enumerate(recs):
        a[k] = [r.tech, r.side, r.i, r.key_kind, r.key_a, r.key_b, r.status, r.reason, r.pix_p, *r.term_p,
                r.pix_q, *r.term_q, r.R]
    return a


def dump(name, w, args, n_per):
    r = Renderer(0)
    r.upload(w.scene)
    r.set_edit(w.edits)
    out = []
    for l in range(1, 8):
        for s in ((0, 1) if args.flags & 1 else (0,)):
            out.append(recs_to_np(r.dump_paths(args, l, s, 0, n_per)))
    np.save(os.path.join(OUT, f"rec_{name}.npy"), np.concatenate(out))


def main():
    os.makedirs(OUT, exist_ok=True)
    if len(sys.argv) > 1 and sys.argv[1] == "c2full":
        w = S.config2()
        dump("c2full", w, w.args, 40000)
        return
    w = S.config1()
    dump("c1_f7", w, w.args, 3000)
    dump("c1_f1", w, dataclasses.replace(w.args, flags=1), 3000)
    w = S.config1(32, 32, spp=4, max_depth=8)
    dump("c1d8", w, w.args, 1000)
    w = S.config2()
    dump("c2", w, w.args, 2000)
    w = S.config3()
    dump("c3", w, w.args, 400)
    # traced hits, config 1
    import torch
    w = S.config1(16, 16)
    r = Renderer(0)
    r.upload(w.scene)
    r.set_edit(w.edits)
    rng = np.random.default_rng(1)
    n = 3000
    rays = np.zeros((n, 8), np.float32)
    rays[:, 0:3] = rng.uniform(0.02, 0.98, size=(n, 3))
    d = rng.normal(size=(n, 3))
    rays[:, 3:6] = d / np.linalg.norm(d, axis=1, keepdims=True)
    rays[:, 6] = np.array([-1] * n, np.int32).view(np.float32)
    h0 = r.trace(0, torch.from_numpy(rays).cuda()).cpu().numpy()
    h1 = r.trace(1, torch.from_numpy(rays).cuda()).cpu().numpy()
    np.savez(os.path.join(OUT, "trace_c1.npz"), rays=rays, h0=h0, h1=h1)


if __name__ == "__main__":
    main()
