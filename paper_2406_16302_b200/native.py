"""ctypes declarations of include/rr.h (argument marshalling only).

The library is REQUIRED: importing this module raises if librr_b200.so is missing, and every call
returns the library's status -- there is no CPU or PyTorch fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librr_b200.so")

RR_OK, RR_E_INVALID, RR_E_STATE, RR_E_CUDA, RR_E_OOM = 0, -1, -2, -3, -4
RR_TWO_WAY, RR_RECONNECT, RR_REJECT_MULTI, RR_ACCUMULATE, RR_COUNT_TRAVERSAL = 1, 2, 4, 8, 16
RR_VNDF = 32
RR_DIAG_ONE_WAY_ABLATION = 64  # diagnostic, deliberately biased (include/rr.h)
RR_PRIMAL_SHARED_STREAMS = 128  # rr_render_primal: one stream for both states
RR_NO_PATH_MAPPING = 256  # "incremental w/o PM" ablation (include/rr.h)
RR_T6_TOWARD_LIGHT = 512  # T6 directions toward the light (include/rr.h)
RR_TOBJ_MIDPATH = 1024  # object transform of the first mid-path moved-object hit (include/rr.h)
RR_RECONNECT_BIDIR = 2048  # reconnection inside the T3 / T6 emitter-side sub-walk (include/rr.h)


class rr_material(C.Structure):
    _fields_ = [("type", C.c_uint32), ("albedo", C.c_float * 3), ("roughness", C.c_float)]


class rr_object(C.Structure):
    _fields_ = [("material", C.c_uint32), ("emission", C.c_float * 3), ("flags", C.c_uint32)]


class rr_camera(C.Structure):
    _fields_ = [("pos", C.c_float * 3), ("look_at", C.c_float * 3), ("up", C.c_float * 3),
                ("vfov_deg", C.c_float), ("width", C.c_uint32), ("height", C.c_uint32)]


class rr_scene_desc(C.Structure):
    _fields_ = [("n_vertices", C.c_uint32), ("positions", C.c_void_p),
                ("n_triangles", C.c_uint32), ("indices", C.c_void_p), ("tri_object", C.c_void_p),
                ("n_objects", C.c_uint32), ("objects", C.POINTER(rr_object)),
                ("n_materials", C.c_uint32), ("materials", C.POINTER(rr_material)),
                ("camera", rr_camera), ("eps_rel", C.c_float)]


class rr_edit(C.Structure):
    _fields_ = [("object", C.c_uint32), ("old_xform", C.c_float * 12), ("new_xform", C.c_float * 12),
                ("has_material", C.c_uint32), ("old_material", rr_material), ("new_material", rr_material)]


class rr_render_args(C.Structure):
    _fields_ = [("spp", C.c_uint32), ("seed", C.c_uint64), ("max_depth", C.c_uint32),
                ("technique_mask", C.c_uint32), ("flags", C.c_uint32), ("jacobian_max", C.c_float),
                ("alpha_min", C.c_float), ("dmin_rel", C.c_float), ("shard_index", C.c_uint32),
                ("shard_count", C.c_uint32), ("layer_mask", C.c_uint32)]


class rr_stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("samples", "connections", "accepted", "rejected", "unpaired",
                                          "mapped_only", "reconnected", "closest_rays", "shadow_rays",
                                          "instance_queries", "splats", "offscreen", "zero_pairs",
                                          "nodes_visited", "tris_tested")] + \
               [("rejected_by", C.c_uint64 * 8), ("effective_mask", C.c_uint32), ("n_moved", C.c_uint32),
                ("sched", C.c_uint64 * 8), ("r_hist", C.c_uint64 * 16)]

    def as_dict(self):
        d = {n: int(getattr(self, n)) for n, _ in self._fields_ if n not in ("rejected_by", "sched", "r_hist")}
        d["rejected_by"] = [int(x) for x in self.rejected_by]
        d["sched"] = [int(x) for x in self.sched]
        d["r_hist"] = [int(x) for x in self.r_hist]
        return d


class rr_path_record(C.Structure):
    _fields_ = [("tech", C.c_int32), ("side", C.c_int32), ("i", C.c_uint64),
                ("key_kind", C.c_int32), ("key_a", C.c_int32), ("key_b", C.c_int32),
                ("status", C.c_int32), ("reason", C.c_int32), ("pix_p", C.c_int32),
                ("term_p", C.c_float * 3), ("pix_q", C.c_int32), ("term_q", C.c_float * 3), ("R", C.c_float)]


EXPORTS = ["rr_create", "rr_destroy", "rr_last_error", "rr_scene_upload", "rr_set_edit", "rr_render_residual",
           "rr_render_primal",
           "rr_render_residual_host", "rr_get_stats", "rr_trace", "rr_segment", "rr_philox", "rr_dump_paths",
           "rr_last_timings"]

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("RR_LIB_VARIANT") or LIB_PATH  # tuning experiments (tools/variants.py) only
    if not os.path.exists(path):
        raise RuntimeError(f"CUDA extension missing: {path} (run __graft_entry__.build())")
    L = C.CDLL(path)
    P, U32, U64 = C.c_void_p, C.c_uint32, C.c_uint64
    L.rr_create.argtypes = [C.c_int, C.POINTER(P)]
    L.rr_destroy.argtypes = [P]
    L.rr_destroy.restype = None
    L.rr_last_error.argtypes = [P]
    L.rr_last_error.restype = C.c_char_p
    L.rr_scene_upload.argtypes = [P, C.POINTER(rr_scene_desc)]
    L.rr_set_edit.argtypes = [P, U32, C.POINTER(rr_edit)]
    L.rr_render_residual.argtypes = [P, C.POINTER(rr_render_args), P, U64]
    L.rr_render_residual_host.argtypes = [P, C.POINTER(rr_render_args), P]
    L.rr_get_stats.argtypes = [P, C.POINTER(rr_stats)]
    L.rr_trace.argtypes = [P, U32, U32, P, P, U64]
    L.rr_segment.argtypes = [P, U32, P, P, U64]
    L.rr_philox.argtypes = [P, U32, P, U32, U32, P, U64]
    L.rr_dump_paths.argtypes = [P, C.POINTER(rr_render_args), U32, U32, U64, U64, C.POINTER(rr_path_record), U64,
                                C.POINTER(U64)]
    L.rr_last_timings.argtypes = [P, C.POINTER(C.c_float), U32]
    L.rr_render_primal.argtypes = [P, U32, U32, U64, U32, U32, P, U64]
    for name in EXPORTS:
        if name not in ("rr_destroy", "rr_last_error"):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L
