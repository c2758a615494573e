"""Offline comparison of dumped GPU records with the oracle (diagnostics)."""
import collections
import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import binding as OB  # noqa: E402
from rr_inputs import scenes as S  # noqa: E402


def load(name):
    return np.load(os.path.join(os.environ.get("RR_REC_DIR", "gpurun_out"), f"rec_{name}.npy"))


def close(g, o, rel=1e-4):
    g = np.where(np.abs(g) < 1e-30, 0, g)
    o = np.where(np.abs(o) < 1e-30, 0, o)
    return np.all(np.abs(g - o) <= rel * np.maximum(np.abs(g), np.abs(o)))


def compare(name, w, args, n_per, techs=range(1, 8), verbose=5):
    G = load(name)
    o = OB.Oracle(w.scene, w.edits)
    gmap = {tuple(int(x) for x in r[:6]): r for r in G}
    orecs = []
    mask = o.effective_mask(args.technique_mask)
    for l in techs:
        if not (mask >> (l - 1)) & 1:
            continue
        for s in ((0, 1) if args.flags & 1 else (0,)):
            _, rr, _ = o.residual(args, l, s, 0, n_per, records=True)
            orecs += rr
    omap = {(r.tech, r.side, r.i, r.key_kind, r.key_a, r.key_b): r for r in orecs}
    keys = set(k for k in gmap if k[0] in techs) | set(omap)
    bad = collections.Counter()
    ex = collections.defaultdict(list)
    ok = 0
    for k in keys:
        g, r = gmap.get(k), omap.get(k)
        if g is None or r is None:
            why = "missing_gpu" if g is None else "missing_oracle"
            bad[(k[0], why)] += 1
            ex[(k[0], why)].append((k, None if r is None else (r.status, r.pix_p, list(r.term_p))))
            continue
        st_ok = int(g[6]) == r.status
        nz = lambda a: bool(np.any(np.abs(np.asarray(a)) > 1e-30))
        pix_ok = ((int(g[8]) == r.pix_p or not (nz(g[9:12]) or nz(r.term_p))) and
                  (int(g[12]) == r.pix_q or not (nz(g[13:16]) or nz(r.term_q))))
        off_p = int(g[8]) < 0 and r.pix_p < 0  # dropped splats (reading 4)
        off_q = int(g[12]) < 0 and r.pix_q < 0
        tp_ok = off_p or close(g[9:12], np.array(r.term_p))
        tq_ok = off_q or close(g[13:16], np.array(r.term_q))
        if st_ok and pix_ok and tp_ok and tq_ok:
            ok += 1
            continue
        why = "status" if not st_ok else ("pix" if not pix_ok else ("term_p" if not tp_ok else "term_q"))
        bad[(k[0], why)] += 1
        ex[(k[0], why)].append((k, (int(g[6]), r.status, int(g[7]), r.reason), (int(g[8]), r.pix_p, int(g[12]), r.pix_q),
                                (g[9:12].tolist(), list(r.term_p)), (g[13:16].tolist(), list(r.term_q)), (g[16], r.R)))
    print(f"== {name}: {ok}/{len(keys)} = {ok / max(1, len(keys)):.5f}")
    for k, v in sorted(bad.items()):
        print("  ", k, v)
        for e in ex[k][:verbose]:
            print("      ", e)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1_f7"]
    for nm in which:
        if nm == "c1_f7":
            w = S.config1(); compare(nm, w, w.args, 3000)
        elif nm == "c1_f1":
            w = S.config1(); compare(nm, w, dataclasses.replace(w.args, flags=1), 3000)
        elif nm == "c1d8":
            w = S.config1(32, 32, spp=4, max_depth=8); compare(nm, w, w.args, 1000)
        elif nm == "c2full":
            w = S.config2(); compare(nm, w, w.args, 40000, verbose=40)
        elif nm == "c2":
            w = S.config2(); compare(nm, w, w.args, 2000)
        elif nm == "c3":
            w = S.config3(); compare(nm, w, w.args, 400)
