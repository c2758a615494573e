"""Dump GPU records of config 1 (32x32, D = 6) with RR_RECONNECT_BIDIR for T3 / T6 (diagnostics)."""
import dataclasses, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from rr_inputs import scenes as S  # noqa: E402
from paper_2406_16302_b200 import Renderer  # noqa: E402
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
from dump_gpu_records import recs_to_np  # noqa: E402
w = S.config1(32, 32, spp=4, max_depth=6)
a = dataclasses.replace(w.args, flags=S.PAPER_FLAGS | S.RECONNECT_BIDIR)
r = Renderer(0); r.upload(w.scene); r.set_edit(w.edits)
out = []
for l in (3, 6):
    for s in (0, 1):
        out.append(recs_to_np(r.dump_paths(a, l, s, 0, 2048)))
np.save("gpurun_out/rec_rb.npy", np.concatenate(out))
