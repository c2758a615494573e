#!/bin/bash
# equal-budget quality of configs 1-3 at 256^2, 16 spp (1024-spp reference) -> gpurun_out/quality_256px.json
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python - <<'PY'
import json, subprocess, sys
out = {}
for c in (1, 2, 3):
    r = subprocess.run([sys.executable, "tools/quality.py", str(c), "256", "16"], capture_output=True, text=True)
    if r.returncode:
        print(r.stderr[-2000:]); sys.exit(1)
    out[f"config{c}"] = json.loads(r.stdout)
json.dump(out, open("gpurun_out/quality_256px.json", "w"), indent=1)
for k, v in out.items():
    print(k, {n: (f"{x['mse']:.2e}", round(x['ssim'], 3), round(1e3 * x['seconds'], 1)) for n, x in v["results"].items()})
PY
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k equal_budget 2>&1 | tail -2
