"""Image I/O: Portable Float Map (PFM), the float format of the SPEC's image outputs.

write_pfm / read_pfm handle (H, W, 3) or (H, W) float arrays; rows are stored bottom-to-top and the scale
sign gives the byte order (negative: little-endian), per the PFM definition.  Composite of an edit:
I_new = I_old + residual (an (H, W, 3) add; Renderer.render_primal + Renderer.render_residual).
"""
from __future__ import annotations

import numpy as np


def write_pfm(path: str, img) -> None:
    a = np.asarray(img, dtype=np.float32)
    if a.ndim == 3 and a.shape[2] == 4:
        a = a[..., :3]
    if a.ndim not in (2, 3) or (a.ndim == 3 and a.shape[2] != 3):
        raise ValueError("expected (H, W) or (H, W, 3)")
    color = a.ndim == 3
    h, w = a.shape[:2]
    with open(path, "wb") as f:
        f.write(b"PF\n" if color else b"Pf\n")
        f.write(f"{w} {h}\n".encode())
        f.write(b"-1.0\n")
        f.write(np.ascontiguousarray(a[::-1]).astype("<f4").tobytes())


def read_pfm(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        kind = f.readline().strip()
        if kind not in (b"PF", b"Pf"):
            raise ValueError("not a PFM file")
        w, h = (int(x) for x in f.readline().split())
        scale = float(f.readline())
        dt = "<f4" if scale < 0 else ">f4"
        ch = 3 if kind == b"PF" else 1
        a = np.frombuffer(f.read(w * h * ch * 4), dtype=dt).astype(np.float32)
    a = a.reshape((h, w, ch) if ch == 3 else (h, w))
    return a[::-1].copy()
