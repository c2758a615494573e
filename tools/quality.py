"""Equal-budget comparison of residual estimators (paper_2406_16302_b200.quality) on a config.
  python tools/quality.py CFG W SPP [REF_SPP]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from rr_inputs import scenes as S  # noqa: E402
from paper_2406_16302_b200 import Renderer, quality as Q  # noqa: E402

cfg, W, spp = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
ref_spp = int(sys.argv[4]) if len(sys.argv) > 4 else 1024
w = S.load_config(cfg, width=W, height=W)
r = Renderer(0)
r.upload(w.scene)
r.set_edit(w.edits)
ref = Q.reference(r, w.args, ref_spp)
print(json.dumps({"config": cfg, "resolution": W, "spp": spp, "reference_spp": ref_spp,
                  "results": Q.compare(r, w.args, spp, ref, ablations=True)}, indent=1))
