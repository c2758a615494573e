"""Dump GPU records of config 3 with RR_RECONNECT_BIDIR for T3 side 0 over a few chunks (diagnostics)."""
import dataclasses, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
from rr_inputs import scenes as S  # noqa: E402
from paper_2406_16302_b200 import Renderer  # noqa: E402
from dump_gpu_records import recs_to_np  # noqa: E402
w = S.load_config(3)
a = dataclasses.replace(w.args, flags=S.PAPER_FLAGS | S.RECONNECT_BIDIR)
r = Renderer(0); r.upload(w.scene); r.set_edit(w.edits)
out = [recs_to_np(r.dump_paths(a, 3, 0, i0, i0 + 256)) for i0 in (69120, 3566848)]
np.save("gpurun_out/rec_rb3.npy", np.concatenate(out))
