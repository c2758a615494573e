"""Thin Python binding over the C ABI (include/rr.h): argument marshalling only.

Every step of the residual estimator runs in librr_b200.so's sm_100a kernels; PyTorch is used only
for device memory and streams.  Names mirror the ABI: upload / set_edit / render_residual / get_stats
/ dump_paths / trace / segment / philox.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import native as N


class RRError(RuntimeError):
    pass


def _mat(m) -> N.rr_material:
    r = N.rr_material()
    r.type = int(m.type)
    r.albedo[:] = [float(a) for a in m.albedo]
    r.roughness = float(m.roughness)
    return r


class Renderer:
    """One library context on one CUDA device."""

    def __init__(self, device: int = 0):
        self._L = N.lib()
        h = C.c_void_p()
        st = self._L.rr_create(int(device), C.byref(h))
        if st != N.RR_OK:
            raise RRError(f"rr_create failed ({st}) on device {device}")
        self.h = h
        self.device = device
        self.width = self.height = 0
        self._keep = []

    def close(self):
        if getattr(self, "h", None):
            self._L.rr_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int, what: str):
        if st != N.RR_OK:
            msg = self._L.rr_last_error(self.h)
            raise RRError(f"{what}: status {st}: {msg.decode() if msg else ''}")

    # ---------------------------------------------------------------- scene / edit
    def upload(self, scene) -> None:
        pos = np.ascontiguousarray(scene.positions, dtype=np.float32)
        idx = np.ascontiguousarray(scene.indices, dtype=np.uint32)
        tob = np.ascontiguousarray(scene.tri_object, dtype=np.uint32)
        no, nm = int(scene.obj_material.shape[0]), int(scene.mat_type.shape[0])
        objs = (N.rr_object * no)()
        for o in range(no):
            objs[o].material = int(scene.obj_material[o])
            objs[o].emission[:] = [float(x) for x in scene.obj_emission[o]]
            objs[o].flags = int(scene.obj_flags[o])
        mats = (N.rr_material * nm)()
        for m in range(nm):
            mats[m].type = int(scene.mat_type[m])
            mats[m].albedo[:] = [float(x) for x in scene.mat_albedo[m]]
            mats[m].roughness = float(scene.mat_roughness[m])
        d = N.rr_scene_desc()
        d.n_vertices = pos.shape[0]
        d.positions = pos.ctypes.data
        d.n_triangles = idx.shape[0]
        d.indices = idx.ctypes.data
        d.tri_object = tob.ctypes.data
        d.n_objects = no
        d.objects = objs
        d.n_materials = nm
        d.materials = mats
        cam = scene.camera
        d.camera.pos[:] = [float(x) for x in cam.pos]
        d.camera.look_at[:] = [float(x) for x in cam.look_at]
        d.camera.up[:] = [float(x) for x in cam.up]
        d.camera.vfov_deg = float(cam.vfov_deg)
        d.camera.width, d.camera.height = int(cam.width), int(cam.height)
        d.eps_rel = float(scene.eps_rel)
        self._check(self._L.rr_scene_upload(self.h, C.byref(d)), "rr_scene_upload")
        self.width, self.height = int(cam.width), int(cam.height)

    def set_edit(self, edits: Sequence) -> None:
        n = len(edits)
        arr = (N.rr_edit * max(n, 1))()
        for k, e in enumerate(edits):
            arr[k].object = int(e.object)
            arr[k].old_xform[:] = [float(x) for x in np.asarray(e.old_xform, np.float32)]
            arr[k].new_xform[:] = [float(x) for x in np.asarray(e.new_xform, np.float32)]
            arr[k].has_material = 1 if e.has_material else 0
            if e.has_material:
                arr[k].old_material = _mat(e.old_material)
                arr[k].new_material = _mat(e.new_material)
        self._check(self._L.rr_set_edit(self.h, n, arr), "rr_set_edit")

    # ---------------------------------------------------------------- rendering
    @staticmethod
    def make_args(a, shard_index: int = 0, shard_count: int = 1) -> N.rr_render_args:
        r = N.rr_render_args()
        r.spp, r.seed, r.max_depth = int(a.spp), int(a.seed), int(a.max_depth)
        r.technique_mask, r.flags = int(a.technique_mask), int(a.flags)
        r.jacobian_max, r.alpha_min, r.dmin_rel = float(a.jacobian_max), float(a.alpha_min), float(a.dmin_rel)
        r.shard_index, r.shard_count = int(shard_index), int(shard_count)
        r.layer_mask = int(getattr(a, "layer_mask", 0))
        return r

    def render_residual(self, args, image=None, stream: Optional[int] = None, shard_index: int = 0,
                        shard_count: int = 1, accumulate: bool = False, count_traversal: bool = False):
        """Render into a torch float32 (H, W, 4) CUDA tensor (allocated if None); asynchronous.
        count_traversal: also count BVH node fetches / triangle tests into get_stats() (diagnostic)."""
        import torch
        if image is None:
            image = torch.empty((self.height, self.width, 4), dtype=torch.float32, device=f"cuda:{self.device}")
        assert image.is_cuda and image.dtype == torch.float32 and image.is_contiguous()
        assert tuple(image.shape) == (self.height, self.width, 4)
        a = self.make_args(args, shard_index, shard_count)
        if accumulate:
            a.flags |= N.RR_ACCUMULATE
        if count_traversal:
            a.flags |= N.RR_COUNT_TRAVERSAL
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        self._check(self._L.rr_render_residual(self.h, C.byref(a), image.data_ptr(), int(stream)),
                    "rr_render_residual")
        return image

    def render_primal(self, state: int, spp: int, seed: int, max_depth: int, image=None, stream: Optional[int] = None,
                      count_traversal: bool = False, shared_streams: bool = False):
        """Primal image I^D(state) (state 0 = new, 1 = old) into a torch float32 (H, W, 4) CUDA tensor.
        shared_streams: the same random numbers in both states (correlated primal difference)."""
        import torch
        if image is None:
            image = torch.empty((self.height, self.width, 4), dtype=torch.float32, device=f"cuda:{self.device}")
        assert image.is_cuda and image.dtype == torch.float32 and image.is_contiguous()
        assert tuple(image.shape) == (self.height, self.width, 4)
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        flags = (N.RR_COUNT_TRAVERSAL if count_traversal else 0) | (N.RR_PRIMAL_SHARED_STREAMS if shared_streams else 0)
        self._check(self._L.rr_render_primal(self.h, int(state), int(spp), int(seed), int(max_depth), flags,
                                             image.data_ptr(), int(stream)), "rr_render_primal")
        return image

    def render_layers(self, args) -> dict:
        """Per-technique residual layers {l: (H, W, 4) CUDA tensor}: the samples of technique l only, MIS-weighted
        against every technique of args.technique_mask; the layers add up to render_residual(args).  A technique
        the library auto-disables (T4-T6 without a moved object) gives a zero layer."""
        import dataclasses
        out = {}
        for l in range(1, 8):
            if (int(args.technique_mask) >> (l - 1)) & 1:
                out[l] = self.render_residual(dataclasses.replace(args, layer_mask=1 << (l - 1))).clone()
        return out

    def render_sequence(self, frames, args, image=None, shard_index: int = 0, shard_count: int = 1,
                        checkpoint_dir: Optional[str] = None, start_frame: int = 0):
        """Chained residuals of an animation (config 5): frame f applies the edit S_f -> S_f+1
        (`frames[f]`, a list of edits), renders its residual with seed args.seed + f and adds it to `image`,
        so that after the last frame image = I_0 + sum_f Delta_f (I_0 = the given image, else 0).
        checkpoint_dir: after every frame the accumulated image is written there as `chain_fNNN.pfm` (float32,
        exact) with `chain_state.json` naming the last finished frame; `resume_sequence` continues from it.
        start_frame: the first frame to render (the frames before it are already in `image`)."""
        import dataclasses
        import json
        import os
        for f in range(start_frame, len(frames)):
            self.set_edit(frames[f])
            a = dataclasses.replace(args, seed=int(args.seed) + f)
            acc = image is not None
            image = self.render_residual(a, image=image, shard_index=shard_index, shard_count=shard_count,
                                         accumulate=acc)
            if checkpoint_dir is not None:
                from .io import write_pfm
                os.makedirs(checkpoint_dir, exist_ok=True)
                path = os.path.join(checkpoint_dir, f"chain_f{f:03d}.pfm")
                write_pfm(path, image.cpu().numpy())
                with open(os.path.join(checkpoint_dir, "chain_state.json"), "w") as fh:
                    json.dump({"frame": f, "image": os.path.basename(path), "frames": len(frames),
                               "seed": int(args.seed), "shard": [shard_index, shard_count]}, fh)
        return image

    def resume_sequence(self, frames, args, checkpoint_dir: str, shard_index: int = 0, shard_count: int = 1):
        """Continue an interrupted render_sequence from its last checkpoint (frame-level resume; the image is
        restored exactly from the float32 PFM, so the result equals an uninterrupted chain)."""
        import json
        import os
        import torch
        from .io import read_pfm
        with open(os.path.join(checkpoint_dir, "chain_state.json")) as fh:
            st = json.load(fh)
        rgb = read_pfm(os.path.join(checkpoint_dir, st["image"]))
        img = torch.zeros((self.height, self.width, 4), dtype=torch.float32, device=f"cuda:{self.device}")
        img[..., :3] = torch.from_numpy(rgb).to(img.device)
        return self.render_sequence(frames, args, image=img, shard_index=shard_index, shard_count=shard_count,
                                    checkpoint_dir=checkpoint_dir, start_frame=int(st["frame"]) + 1)

    def render_residual_host(self, args, out: Optional[np.ndarray] = None, shard_index: int = 0,
                             shard_count: int = 1) -> np.ndarray:
        """Render into HOST memory (the library copies the image back; blocking)."""
        if out is None:
            out = np.zeros((self.height, self.width, 4), np.float32)
        assert out.dtype == np.float32 and out.flags.c_contiguous
        a = self.make_args(args, shard_index, shard_count)
        self._check(self._L.rr_render_residual_host(self.h, C.byref(a), out.ctypes.data), "rr_render_residual_host")
        return out

    def get_stats(self) -> dict:
        s = N.rr_stats()
        self._check(self._L.rr_get_stats(self.h, C.byref(s)), "rr_get_stats")
        return s.as_dict()

    def last_timings(self, n: int = 16) -> list:
        buf = (C.c_float * n)()
        self._check(self._L.rr_last_timings(self.h, buf, n), "rr_last_timings")
        return list(buf)

    def dump_paths(self, args, technique: int, side: int, i_begin: int, i_end: int, capacity: Optional[int] = None):
        cap = capacity if capacity is not None else max(64, 64 * (i_end - i_begin))
        buf = (N.rr_path_record * cap)()
        n = C.c_uint64(0)
        a = self.make_args(args)
        self._check(self._L.rr_dump_paths(self.h, C.byref(a), technique, side, i_begin, i_end, buf, cap, C.byref(n)),
                    "rr_dump_paths")
        return [buf[k] for k in range(n.value)]

    # ---------------------------------------------------------------- test-only exports
    def trace(self, state: int, rays):
        """rays: torch CUDA float32 [n, 8]; returns hits [n, 8]."""
        import torch
        n = rays.shape[0]
        hits = torch.empty((n, 8), dtype=torch.float32, device=rays.device)
        self._check(self._L.rr_trace(self.h, state, n, rays.data_ptr(), hits.data_ptr(),
                                     torch.cuda.current_stream(self.device).cuda_stream), "rr_trace")
        return hits

    def segment(self, segs):
        import torch
        n = segs.shape[0]
        out = torch.empty((n, 10), dtype=torch.float32, device=segs.device)
        self._check(self._L.rr_segment(self.h, n, segs.data_ptr(), out.data_ptr(),
                                       torch.cuda.current_stream(self.device).cuda_stream), "rr_segment")
        return out

    def philox(self, ctr, key_lo: int, key_hi: int):
        import torch
        n = ctr.shape[0]
        out = torch.empty_like(ctr)
        self._check(self._L.rr_philox(self.h, n, ctr.data_ptr(), key_lo, key_hi, out.data_ptr(),
                                      torch.cuda.current_stream(self.device).cuda_stream), "rr_philox")
        return out

