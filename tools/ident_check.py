import os, sys, dataclasses
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from rr_inputs import scenes as S
from paper_2406_16302_b200 import Renderer
w = S.cornell_identity(64, 64, spp=8, max_depth=6)
r = Renderer(0); r.upload(w.scene); r.set_edit(w.edits)
bad = 0
for l in range(1, 8):
    for s in (0, 1):
        try:
            recs = r.dump_paths(w.args, l, s, 0, 64 * 64 * 4)
        except Exception as e:
            print(l, s, e); continue
        for rec in recs:
            tp, tq = np.array(rec.term_p), np.array(rec.term_q)
            if rec.pix_p == rec.pix_q and np.any(tp + tq != 0):
                bad += 1
                if bad <= 12:
                    print(l, s, rec.i, rec.key_kind, rec.key_a, rec.key_b, rec.status, rec.reason, tp, tq)
            elif rec.pix_p != rec.pix_q:
                bad += 1
                if bad <= 12: print("pix", l, s, rec.i, rec.key_kind, rec.key_a, rec.key_b, rec.status, rec.pix_p, rec.pix_q, tp, tq)
print("bad", bad)
for flags in (S.PAPER_FLAGS, S.TWO_WAY, 0):
    a = dataclasses.replace(w.args, flags=flags)
    for rep in range(3):
        img = r.render_residual(a)
        torch.cuda.synchronize()
        print("render flags", flags, "nonzero", int(torch.count_nonzero(img)), "sum", float(img.abs().sum()))
    bad = 0
    for l in range(1, 8):
        for s in ((0, 1) if flags & S.TWO_WAY else (0,)):
            recs = r.dump_paths(a, l, s, 0, 64 * 64 * (4 if flags & S.TWO_WAY else 8))
            for rec in recs:
                tp, tq = np.array(rec.term_p), np.array(rec.term_q)
                if np.any(tp + tq != 0) or rec.pix_p != rec.pix_q:
                    bad += 1
                    if bad <= 5: print(l, s, rec.i, rec.key_kind, rec.key_a, rec.key_b, rec.status, rec.pix_p, rec.pix_q, tp, tq)
    print("flags", flags, "bad records", bad)
