"""ctypes loader for the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module.  The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "rr_oracle.cpp")
LIB = os.path.join(HERE, "librr_oracle.so")


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", LIB, SRC])
    return LIB


class Record(C.Structure):
    _fields_ = [("tech", C.c_int32), ("side", C.c_int32), ("i", C.c_uint64),
                ("key_kind", C.c_int32), ("key_a", C.c_int32), ("key_b", C.c_int32),
                ("status", C.c_int32), ("reason", C.c_int32),
                ("pix_p", C.c_int32), ("term_p", C.c_double * 3),
                ("pix_q", C.c_int32), ("term_q", C.c_double * 3),
                ("R", C.c_double), ("v_p", C.c_double * 3), ("v_q", C.c_double * 3),
                ("n_cand_p", C.c_int32), ("n_cand_q", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("samples", "connections", "accepted", "rejected", "unpaired",
                                          "mapped_only", "reconnected", "closest_rays", "shadow_rays",
                                          "splats", "offscreen")] + [("rejected_by", C.c_uint64 * 8)]

    def as_dict(self):
        d = {n: int(getattr(self, n)) for n, _ in self._fields_ if n != "rejected_by"}
        d["rejected_by"] = [int(x) for x in self.rejected_by]
        return d


class Input(C.Structure):
    _fields_ = [("n_vertices", C.c_int32), ("positions", C.c_void_p),
                ("n_triangles", C.c_int32), ("indices", C.c_void_p), ("tri_object", C.c_void_p),
                ("n_objects", C.c_int32), ("obj_material", C.c_void_p), ("obj_emission", C.c_void_p),
                ("obj_flags", C.c_void_p),
                ("n_materials", C.c_int32), ("mat_type", C.c_void_p), ("mat_albedo", C.c_void_p),
                ("mat_roughness", C.c_void_p),
                ("cam_pos", C.c_float * 3), ("cam_look", C.c_float * 3), ("cam_up", C.c_float * 3),
                ("vfov_deg", C.c_float), ("width", C.c_int32), ("height", C.c_int32), ("eps_rel", C.c_float),
                ("n_edits", C.c_int32), ("edit_object", C.c_void_p), ("edit_old_xform", C.c_void_p),
                ("edit_new_xform", C.c_void_p), ("edit_has_material", C.c_void_p),
                ("edit_mat_type", C.c_void_p), ("edit_mat_albedo", C.c_void_p),
                ("edit_mat_roughness", C.c_void_p)]


class Args(C.Structure):
    _fields_ = [("spp", C.c_uint32), ("seed", C.c_uint64), ("max_depth", C.c_uint32),
                ("technique_mask", C.c_uint32), ("flags", C.c_uint32),
                ("jacobian_max", C.c_double), ("alpha_min", C.c_double), ("dmin_rel", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        P, D = C.c_void_p, C.POINTER(C.c_double)
        L.orc_create.restype = P
        L.orc_create.argtypes = [C.POINTER(Input), C.c_char_p, C.c_int]
        L.orc_destroy.argtypes = [P]
        L.orc_effective_mask.argtypes = [P, C.c_uint32]
        L.orc_paired_tech.argtypes = [P, C.c_uint32, C.c_int]
        L.orc_scene_eps.restype = C.c_double
        L.orc_scene_eps.argtypes = [P]
        L.orc_scene_diag.restype = C.c_double
        L.orc_scene_diag.argtypes = [P]
        L.orc_residual.argtypes = [P, C.POINTER(Args), C.c_int, C.c_int, C.c_uint64, C.c_uint64, D,
                                   C.POINTER(Record), C.c_int64, C.POINTER(C.c_int64), C.POINTER(Stats)]
        L.orc_primal.argtypes = [P, C.c_int, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, D, C.POINTER(Stats)]
        L.orc_primal_streams.argtypes = [P, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, D,
                                         C.POINTER(Stats)]
        L.orc_philox.argtypes = [C.POINTER(C.c_uint32)] * 3
        L.orc_u01.restype = C.c_double
        L.orc_u01.argtypes = [C.c_uint32]
        L.orc_stream_dims.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, D]
        L.orc_closest.argtypes = [P, C.c_int, D, D, C.c_int, D]
        L.orc_closest_brute.argtypes = [P, C.c_int, D, D, C.c_int, D]
        L.orc_visible.argtypes = [P, C.c_int, D, D, C.c_int, C.c_int]
        L.orc_crossings.argtypes = [P, C.c_int, D, D, D, C.c_int]
        L.orc_crossings_brute.argtypes = [P, C.c_int, D, D]
        L.orc_bsdf.restype = C.c_double
        L.orc_bsdf.argtypes = [D, D, D, D, D]
        L.orc_bsdf_sample.argtypes = [D, D, D, C.c_double, C.c_double, D]
        for name in ("orc_geometric_term",):
            getattr(L, name).restype = C.c_double
            getattr(L, name).argtypes = [D, D, D, D]
        L.orc_vertex1pdf.restype = C.c_double
        L.orc_vertex1pdf.argtypes = [C.c_double, D, D, D, D, D]
        L.orc_g_term.restype = C.c_double
        L.orc_g_term.argtypes = [C.c_double, D, D, D, D, D]
        L.orc_reconnect_jacobian.restype = C.c_double
        L.orc_reconnect_jacobian.argtypes = [D, D, D, D]
        L.orc_candidates.argtypes = [C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int,
                                     C.POINTER(C.c_int32), C.c_int]
        L.orc_sample_set.argtypes = [P, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, D]
        L.orc_set_area.restype = C.c_double
        L.orc_set_area.argtypes = [P, C.c_int]
        L.orc_project.argtypes = [P, D]
        L.orc_debug_sample.argtypes = [P, C.POINTER(Args), C.c_int, C.c_int, C.c_uint64]
        L.orc_t3_light_dir.argtypes = [D, C.c_double, C.c_double, D]
        L.orc_reconnections.restype = C.c_int64
        L.orc_reconnections.argtypes = [P, C.POINTER(Args), C.c_int, C.c_int, C.c_uint64, C.c_uint64, D, C.c_int64]
        L.orc_pdf_check.restype = C.c_int64
        L.orc_pdf_check.argtypes = [P, C.POINTER(Args), C.c_int, C.c_int, C.c_uint64, C.c_uint64, D, C.c_int64]
    return _lib


def dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def vec(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _mat_tuple(m):
    return (int(m.type), [float(a) for a in m.albedo], float(m.roughness))


class Oracle:
    """One oracle scene (scene arrays + edit list)."""

    def __init__(self, scene, edits):
        L = lib()
        self._keep = []

        def arr(a, dt):
            a = np.ascontiguousarray(np.asarray(a, dtype=dt))
            self._keep.append(a)
            return a.ctypes.data

        inp = Input()
        inp.n_vertices = scene.positions.shape[0]
        inp.positions = arr(scene.positions, np.float32)
        inp.n_triangles = scene.indices.shape[0]
        inp.indices = arr(scene.indices, np.uint32)
        inp.tri_object = arr(scene.tri_object, np.uint32)
        inp.n_objects = scene.obj_material.shape[0]
        inp.obj_material = arr(scene.obj_material, np.uint32)
        inp.obj_emission = arr(scene.obj_emission, np.float32)
        inp.obj_flags = arr(scene.obj_flags, np.uint32)
        inp.n_materials = scene.mat_type.shape[0]
        inp.mat_type = arr(scene.mat_type, np.uint32)
        inp.mat_albedo = arr(scene.mat_albedo, np.float32)
        inp.mat_roughness = arr(scene.mat_roughness, np.float32)
        cam = scene.camera
        inp.cam_pos[:] = [float(v) for v in cam.pos]
        inp.cam_look[:] = [float(v) for v in cam.look_at]
        inp.cam_up[:] = [float(v) for v in cam.up]
        inp.vfov_deg = cam.vfov_deg
        inp.width, inp.height = cam.width, cam.height
        inp.eps_rel = scene.eps_rel
        n = len(edits)
        inp.n_edits = n
        inp.edit_object = arr([e.object for e in edits] or [0], np.uint32)
        inp.edit_old_xform = arr(np.concatenate([e.old_xform for e in edits]) if n else np.zeros(12), np.float32)
        inp.edit_new_xform = arr(np.concatenate([e.new_xform for e in edits]) if n else np.zeros(12), np.float32)
        inp.edit_has_material = arr([1 if e.has_material else 0 for e in edits] or [0], np.uint32)
        mt, ma, mr = [], [], []
        for e in edits:
            if e.has_material:
                for m in (e.old_material, e.new_material):
                    t, a, r = _mat_tuple(m)
                    mt.append(t); ma.extend(a); mr.append(r)
            else:
                mt.extend([0, 0]); ma.extend([0.0] * 6); mr.extend([1.0, 1.0])
        inp.edit_mat_type = arr(mt or [0, 0], np.uint32)
        inp.edit_mat_albedo = arr(ma or [0.0] * 6, np.float32)
        inp.edit_mat_roughness = arr(mr or [1.0, 1.0], np.float32)
        err = C.create_string_buffer(256)
        self.h = L.orc_create(C.byref(inp), err, 256)
        if not self.h:
            raise ValueError("oracle: " + err.value.decode())
        self.W, self.H = cam.width, cam.height
        self.npix = self.W * self.H

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    @property
    def eps(self) -> float:
        return lib().orc_scene_eps(self.h)

    @property
    def diag(self) -> float:
        return lib().orc_scene_diag(self.h)

    def effective_mask(self, mask: int) -> int:
        return lib().orc_effective_mask(self.h, mask)

    def paired_tech(self, mask: int, l: int) -> int:
        return lib().orc_paired_tech(self.h, mask, l)

    @staticmethod
    def make_args(a) -> Args:
        r = Args()
        r.spp, r.seed, r.max_depth = a.spp, a.seed, a.max_depth
        r.technique_mask, r.flags = a.technique_mask, a.flags
        r.jacobian_max, r.alpha_min, r.dmin_rel = a.jacobian_max, a.alpha_min, a.dmin_rel
        return r

    def residual(self, args, tech: int, side: int, i0: int, i1: int, records: bool = False,
                 image: Optional[np.ndarray] = None, cap: Optional[int] = None):
        img = np.zeros((self.H, self.W, 3), np.float64) if image is None else image
        st = Stats()
        a = self.make_args(args)
        recs_p, cap_ = None, 0
        buf = None
        if records:
            cap_ = cap if cap is not None else max(64, 64 * (i1 - i0))
            buf = (Record * cap_)()
            recs_p = buf
        n = C.c_int64(0)
        rc = lib().orc_residual(self.h, C.byref(a), tech, side, i0, i1, dptr(img), recs_p, cap_, C.byref(n),
                                C.byref(st))
        if rc != 0:
            raise ValueError("oracle residual: invalid arguments (mask must contain T7)")
        recs = [buf[k] for k in range(n.value)] if records else None
        return img, recs, st.as_dict()

    def sample_range(self, args) -> int:
        """Samples per (technique, side): N_pix spp / 2 two-way, N_pix spp one-way."""
        return self.npix * args.spp // 2 if (args.flags & 1) else self.npix * args.spp

    @staticmethod
    def sides(args):
        """Sides that run: both two-way; side N only one-way (the paired technique's replayed paths in O are
        counted from it) and in the diagnostic one-way ablation."""
        return (0, 1) if (args.flags & 1) else (0,)

    def render_residual(self, args, records: bool = False, techniques=None, limit: Optional[int] = None):
        """Full residual image (H,W,3) over every enabled technique and side."""
        mask = self.effective_mask(args.technique_mask)
        img = np.zeros((self.H, self.W, 3), np.float64)
        recs, stats = [], []
        n = self.sample_range(args)
        if limit is not None:
            n = min(n, limit)
        sides = self.sides(args)
        for l in range(1, 8):
            if not (mask >> (l - 1)) & 1:
                continue
            if techniques is not None and l not in techniques:
                continue
            for s in sides:
                _, r, st = self.residual(args, l, s, 0, n, records=records, image=img)
                stats.append(st)
                if records:
                    recs.extend(r)
        return img, recs, stats

    def primal(self, F: int, seed: int, spp: int, max_depth: int, i0: int = 0, i1: Optional[int] = None):
        img = np.zeros((self.H, self.W, 3), np.float64)
        st = Stats()
        i1 = self.npix * spp if i1 is None else i1
        lib().orc_primal(self.h, F, seed, max_depth, i0, i1, dptr(img), C.byref(st))
        return img / spp, st.as_dict()

    def pdf_check(self, args, tech: int, side: int, i0: int, i1: int) -> np.ndarray:
        """[n, 3]: per connection (generator-recorded density, eval_path pdf of the producing candidate or -1,
        number of candidates) -- the C5 self-consistency pin."""
        a = self.make_args(args)
        cap = 64 * (i1 - i0) + 64
        out = np.zeros(3 * cap)
        n = lib().orc_pdf_check(self.h, C.byref(a), tech, side, i0, i1, dptr(out), cap)
        return out[:3 * min(n, cap)].reshape(-1, 3)

    def reconnections(self, args, tech: int, side: int, i0: int, i1: int) -> np.ndarray:
        """[n, 39]: accepted reconnections {j - w, R, R of the inverse map, (p, n) of v_{w-1}, v_w, v'_{w-1},
        v'_w, v_{w+1}, v_{w+2}} (the R pins of SURVEY 8(c) C11)."""
        a = self.make_args(args)
        cap = 16 * (i1 - i0) + 16
        out = np.zeros(39 * cap)
        n = lib().orc_reconnections(self.h, C.byref(a), tech, side, i0, i1, dptr(out), cap)
        return out[:39 * min(n, cap)].reshape(-1, 39)

    def primal_difference(self, seed: int, spp: int, max_depth: int) -> np.ndarray:
        """I^D(N) - I^D(O) from the primal renderer with the SAME random numbers in both states (correlated,
        unbiased; independent of the residual estimator's code)."""
        out = []
        for F in (0, 1):
            img = np.zeros((self.H, self.W, 3), np.float64)
            lib().orc_primal_streams(self.h, F, 0, seed, max_depth, 0, self.npix * spp, dptr(img), None)
            out.append(img / spp)
        return out[0] - out[1]

    def debug_sample(self, args, tech, side, i):
        a = self.make_args(args)
        lib().orc_debug_sample(self.h, C.byref(a), tech, side, i)

    # ---- unit-test helpers
    def closest(self, F, o, d, excl=-1):
        out = np.zeros(9)
        lib().orc_closest(self.h, F, dptr(vec(o)), dptr(vec(d)), excl, dptr(out))
        return out

    def closest_brute(self, F, o, d, excl=-1):
        out = np.zeros(2)
        lib().orc_closest_brute(self.h, F, dptr(vec(o)), dptr(vec(d)), excl, dptr(out))
        return out

    def visible(self, F, a, b, ea=-1, eb=-1) -> bool:
        return bool(lib().orc_visible(self.h, F, dptr(vec(a)), dptr(vec(b)), ea, eb))

    def crossings(self, F, a, b):
        out = np.zeros(7 * 64)
        n = lib().orc_crossings(self.h, F, dptr(vec(a)), dptr(vec(b)), dptr(out), 64)
        return out[:7 * min(n, 64)].reshape(-1, 7)

    def crossings_brute(self, F, a, b) -> int:
        return lib().orc_crossings_brute(self.h, F, dptr(vec(a)), dptr(vec(b)))

    def sample_set(self, which, F, u0, u1, u2):
        out = np.zeros(7)
        rc = lib().orc_sample_set(self.h, which, F, u0, u1, u2, dptr(out))
        if rc != 0:
            raise ValueError("empty set")
        return out

    def set_area(self, which) -> float:
        return lib().orc_set_area(self.h, which)

    def project(self, x) -> int:
        return lib().orc_project(self.h, dptr(vec(x)))


# ---- stateless helpers
def philox(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    lib().orc_philox(c, k, o)
    return list(o)


def stream_dims(seed, i, l, side, slot):
    out = np.zeros(8)
    lib().orc_stream_dims(seed, i, l, side, slot, dptr(out))
    return out


def bsdf(mat, n, wi, wo):
    ev = np.zeros(3)
    pdf = lib().orc_bsdf(dptr(vec(mat)), dptr(vec(n)), dptr(vec(wi)), dptr(vec(wo)), dptr(ev))
    return ev, pdf


def bsdf_sample(mat, n, wi, u1, u2):
    wo = np.zeros(3)
    ok = lib().orc_bsdf_sample(dptr(vec(mat)), dptr(vec(n)), dptr(vec(wi)), u1, u2, dptr(wo))
    return bool(ok), wo


def t3_light_dir(n, u3, u4):
    """T3's cosine-weighted emitter-side start direction at a dynamic point with normal n; (w, pdf)."""
    out = np.zeros(4)
    lib().orc_t3_light_dir(dptr(vec(n)), u3, u4, dptr(out))
    return out[:3], out[3]


def geometric_term(x, nx, y, ny):
    return lib().orc_geometric_term(dptr(vec(x)), dptr(vec(nx)), dptr(vec(y)), dptr(vec(ny)))


def vertex1pdf(pG, a, xg, ng, x1, n1):
    return lib().orc_vertex1pdf(pG, dptr(vec(a)), dptr(vec(xg)), dptr(vec(ng)), dptr(vec(x1)), dptr(vec(n1)))


def g_term(pdir, ng, x1, n1, x2, n2):
    return lib().orc_g_term(pdir, dptr(vec(ng)), dptr(vec(x1)), dptr(vec(n1)), dptr(vec(x2)), dptr(vec(n2)))


def reconnect_jacobian(xprev, tprev, xi, ni):
    return lib().orc_reconnect_jacobian(dptr(vec(xprev)), dptr(vec(tprev)), dptr(vec(xi)), dptr(vec(ni)))


def candidates(k, dyn, ncross, mask=0x7F):
    d = (C.c_int32 * k)(*dyn)
    n = (C.c_int32 * (k - 1))(*ncross)
    out = (C.c_int32 * 256)()
    m = lib().orc_candidates(k, d, n, mask, out, 128)
    return [(out[2 * a], out[2 * a + 1]) for a in range(m)]
