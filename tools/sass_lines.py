"""Attribute an ncu --set full capture's per-SASS-instruction metrics to CUDA source lines.

  python tools/sass_lines.py REPORT.ncu-rep KERNEL_MANGLED [LIB.so] [--top N]

Uses `nvdisasm -g` on the kernel's cubin (compiled with -lineinfo) to map instruction offsets to
file:line, then sums warp-stall samples, warp instructions and thread instructions per line.
"""
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict


def line_map(lib, kernel):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
        sec = f".text.{kernel}:"
        if sec not in out:
            continue
        body = out.split(sec, 1)[1].split("//---------------------", 1)[0]
        cur = ("?", 0)
        m = {}
        for ln in body.splitlines():
            g = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if g:
                cur = (os.path.basename(g.group(1)), int(g.group(2)))
                continue
            g = re.match(r"\s*/\*([0-9a-f]+)\*/", ln)
            if g:
                m[int(g.group(1), 16)] = cur
        return m
    raise SystemExit("kernel not found in " + lib)


def main():
    rep, kernel = sys.argv[1], sys.argv[2]
    lib = sys.argv[3] if len(sys.argv) > 3 and not sys.argv[3].startswith("--") else \
        os.path.join(os.path.dirname(__file__), "..", "paper_2406_16302_b200", "librr_b200.so")
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    lm = line_map(lib, kernel)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, ist, iw, it = (hdr.index(k) for k in ("Address", "Warp Stall Sampling (All Samples)", "Instructions Executed",
                                             "Thread Instructions Executed"))
    base = None
    agg = defaultdict(lambda: [0, 0, 0])
    for r in rows[2:]:
        if len(r) <= it:
            continue
        a = int(r[ia], 16)
        base = a if base is None else base
        key = lm.get(a - base, ("?", 0))
        agg[key][0] += int(r[ist] or 0)
        agg[key][1] += int(r[iw] or 0)
        agg[key][2] += int(r[it] or 0)
    tot = [sum(v[i] for v in agg.values()) for i in range(3)]
    print(f"total stall samples {tot[0]}, warp insts {tot[1]:.4g}, thread insts {tot[2]:.4g}, "
          f"avg threads {tot[2] / max(1, tot[1]):.2f}")
    by_file = defaultdict(lambda: [0, 0, 0])
    for (f, _), v in agg.items():
        for i in range(3):
            by_file[f][i] += v[i]
    for f, v in sorted(by_file.items(), key=lambda x: -x[1][0]):
        print(f"  {f:24s} stall {100 * v[0] / tot[0]:5.1f}%  insts {100 * v[1] / tot[1]:5.1f}%  thr/inst {v[2] / max(1, v[1]):5.2f}")
    print(f"\n{'file:line':32s} {'stall%':>7s} {'inst%':>7s} {'thr/inst':>8s}")
    for (f, l), v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{f + ':' + str(l):32s} {100 * v[0] / tot[0]:7.2f} {100 * v[1] / tot[1]:7.2f} {v[2] / max(1, v[1]):8.2f}")


if __name__ == "__main__":
    main()
