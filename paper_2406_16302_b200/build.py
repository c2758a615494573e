"""Build the sm_100a C-ABI library librr_b200.so in-tree with nvcc (no JIT cache; the .so travels
with the repository snapshot to the GPU box)."""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "librr_b200.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("rr_capi.cu", "rr_lbvh.cu", "rr_residual.cu", "rr_residual_vndf.cu", "rr_residual_var.cu", "rr_primal.cu")]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false", "-prec-div=false", "-prec-sqrt=false", "-std=c++17", "--extended-lambda",
         "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


STAMP = LIB + ".flags"


def _stale() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(STAMP) or open(STAMP).read() != " ".join(FLAGS):
        return True
    t = os.path.getmtime(LIB)
    deps = SOURCES + glob.glob(os.path.join(HERE, "csrc", "*.h*")) + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(HERE, "..", "include", "rr.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or _stale():
        tmp = LIB + ".tmp"
        objdir = os.path.join(HERE, "build_obj")
        os.makedirs(objdir, exist_ok=True)
        cflags = [f for f in FLAGS if f != "-shared"]

        def compile_one(src):  # translation units compile in parallel, then one link
            obj = os.path.join(objdir, os.path.basename(src) + ".o")
            return obj, subprocess.run(["nvcc", *cflags, "-c", "-o", obj, src], capture_output=True, text=True)

        with ThreadPoolExecutor(len(SOURCES)) as ex:
            done = list(ex.map(compile_one, SOURCES))
        log = ""
        for obj, r in done:
            if r.returncode != 0:
                raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
            log += r.stderr
        r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp,
                            *[obj for obj, _ in done]], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc link failed:\n" + r.stdout + r.stderr)
        if verbose:
            print(log)
        with open(os.path.join(HERE, "csrc", "ptxas_info.txt"), "w") as f:
            f.write(log)
        os.replace(tmp, LIB)
        with open(STAMP, "w") as f:
            f.write(" ".join(FLAGS))
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
