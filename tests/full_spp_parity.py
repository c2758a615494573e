"""North-star image parity at the full 1024 spp (BASELINE.json north star), run as a script on the
GPU box (not collected by pytest: the fp64 oracle needs minutes to an hour per configuration on the host cores):

    python tests/full_spp_parity.py 2:128x128 3:64x64 ...   ->  gpurun_out/full_spp_parity.json

Same comparison as tests/test_gpu_parity.py image_parity (same seeds, sample for sample): RMSE(gpu - oracle) over
max |oracle| must be <= 1e-3.  Results are committed under profiles/."""
import json
import math
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from test_gpu_parity import _image_workload, _oracle_image, _renderer  # noqa: E402


def main():
    import torch
    spp = int(os.environ.get("RR_SPP", "1024"))
    out = []
    path = os.path.join(ROOT, "gpurun_out", "full_spp_parity.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    for spec in sys.argv[1:]:
        cfg, res = spec.split(":")
        W, H = (int(x) for x in res.split("x"))
        key = (int(cfg), W, H, spp)
        w = _image_workload(*key)
        r = _renderer(w)
        img = r.render_residual(w.args)
        torch.cuda.synchronize()
        g = img[..., :3].double().cpu().numpy()
        st = r.get_stats()
        del r
        nc = os.cpu_count() or 8
        nt = 8 * nc  # finer slices than cores: sample cost varies strongly over the index range
        t0 = time.time()
        with mp.get_context("spawn").Pool(nc) as p:
            parts = p.map(_oracle_image, [(key, k, nt) for k in range(nt)], chunksize=1)
        dt = time.time() - t0
        ref = sum(parts)
        scale = float(np.abs(ref).max())
        rmse = math.sqrt(float(((g - ref) ** 2).mean()))
        rec = {"config": int(cfg), "width": W, "height": H, "spp": spp, "samples": int(st["samples"]),
               "rmse": rmse, "max_abs_oracle": scale, "rmse_over_max": rmse / scale, "tolerance": 1e-3,
               "ok": bool(rmse <= 1e-3 * scale), "max_abs_diff": float(np.abs(g - ref).max()),
               "oracle_seconds": dt, "oracle_cores": nc}
        print(json.dumps(rec), flush=True)
        out.append(rec)
        with open(path, "w") as f:
            json.dump(out, f, indent=1)
    return 0 if all(x["ok"] for x in out) else 1


if __name__ == "__main__":
    sys.exit(main())
