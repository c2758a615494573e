"""Build tuning variants of the C-ABI library with extra -D flags into build/variants/<name>.so.

  python tools/variants.py name1:-DA=1,-DB=2 name2:-DA=3 ...
Select one at run time with RR_LIB_VARIANT=build/variants/<name>.so (diagnostics only)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_16302_b200 import build as B  # noqa: E402


def one(spec):
    name, flags = spec.split(":", 1) if ":" in spec else (spec, "")
    out = os.path.join(ROOT, "build", "variants", name + ".so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = ["nvcc", *[f for f in B.FLAGS if f not in ("-Xptxas", "-v")], *[f for f in flags.split(",") if f], "-o", out,
           *B.SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return name, r.returncode, r.stderr[-2000:]


if __name__ == "__main__":
    with ThreadPoolExecutor(4) as ex:
        for name, rc, err in ex.map(one, sys.argv[1:]):
            print(name, "ok" if rc == 0 else "FAILED\n" + err)
