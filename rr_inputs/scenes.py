"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module only builds *inputs*: triangle meshes, materials, cameras, rigid edit
transforms and render arguments.  It contains none of the residual estimator's
arithmetic (no sampling, no pdfs, no intersection, no CDF tables) -- each side
derives everything it needs from these arrays on its own.

The paper measures on Bitterli's scenes ("Scenes courtesy of Benedikt
Bitterli"; Cornell Box, Glossy Cornell, Living room, Ninja Sponza, Staircase, Dining room:
L443, L454, L465).  None of them is available here; the five configurations of
BASELINE.json stand in for them, with the unstated parameters fixed as in SURVEY.md
section 8(d).  Scene randomness uses numpy's Philox bit generator keyed by
0x5EED0000 + config.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence

import numpy as np

LAMBERT = 0
GGX = 1

OBJ_DYNAMIC = 1  # object may carry an edit (rigid transform and/or material change)
OBJ_ENV = 2      # environment stand-in (excluded from the scene diagonal)

# technique bits (bit l-1 for technique l, PAPER.md Fig. importance_sample row A)
T1, T2, T3, T4, T5, T6, T7 = (1 << k for k in range(7))
ALL_TECHNIQUES = 0x7F

# render flags
TWO_WAY = 1
RECONNECT = 2
REJECT_MULTI = 4
ACCUMULATE = 8
PAPER_FLAGS = TWO_WAY | RECONNECT | REJECT_MULTI
VNDF = 32  # GGX directions from the visible normals (Heitz 2018), both implementations
DIAG_ONE_WAY = 64  # RR_DIAG_ONE_WAY_ABLATION: one-way with the two-way pairing rules (biased test mode)
NO_PATH_MAPPING = 256  # RR_NO_PATH_MAPPING: "incremental w/o PM", with TWO_WAY
T6_TOWARD_LIGHT = 512  # RR_T6_TOWARD_LIGHT: T6 directions "uniformly toward the light"
TOBJ_MIDPATH = 1024  # RR_TOBJ_MIDPATH: object transform of a mid-path hit on a moved object
RECONNECT_BIDIR = 2048  # RR_RECONNECT_BIDIR: reconnection inside the T3 / T6 emitter-side sub-walk


@dataclasses.dataclass
class Material:
    type: int
    albedo: Sequence[float]
    roughness: float = 1.0

    def as_tuple(self):
        return (int(self.type), tuple(float(a) for a in self.albedo), float(self.roughness))


@dataclasses.dataclass
class Camera:
    pos: Sequence[float]
    look_at: Sequence[float]
    up: Sequence[float]
    vfov_deg: float
    width: int
    height: int


@dataclasses.dataclass
class Scene:
    positions: np.ndarray   # float32 [V,3]; dynamic objects in OBJECT space
    indices: np.ndarray     # uint32 [T,3]
    tri_object: np.ndarray  # uint32 [T]
    obj_material: np.ndarray  # uint32 [O]
    obj_emission: np.ndarray  # float32 [O,3]
    obj_flags: np.ndarray     # uint32 [O]
    mat_type: np.ndarray      # uint32 [M]
    mat_albedo: np.ndarray    # float32 [M,3]
    mat_roughness: np.ndarray  # float32 [M]
    camera: Camera
    eps_rel: float = 1e-4
    name: str = ""

    @property
    def n_triangles(self) -> int:
        return int(self.indices.shape[0])

    @property
    def n_objects(self) -> int:
        return int(self.obj_material.shape[0])

    def with_camera(self, width: int, height: int) -> "Scene":
        c = dataclasses.replace(self.camera, width=int(width), height=int(height))
        return dataclasses.replace(self, camera=c)


@dataclasses.dataclass
class Edit:
    object: int
    old_xform: np.ndarray  # float32 [12], row-major 3x4 [R|t], x' = R x + t
    new_xform: np.ndarray
    old_material: Optional[Material] = None
    new_material: Optional[Material] = None

    @property
    def has_material(self) -> bool:
        return self.old_material is not None


@dataclasses.dataclass
class RenderArgs:
    spp: int = 4
    seed: int = 0
    max_depth: int = 4
    technique_mask: int = ALL_TECHNIQUES
    flags: int = PAPER_FLAGS
    jacobian_max: float = 10.0
    alpha_min: float = 0.1
    dmin_rel: float = 0.01       # SPEC.md L416 (x scene diagonal)
    layer_mask: int = 0          # GPU only: render the samples of these techniques (0 = all); see rr.h


@dataclasses.dataclass
class Workload:
    scene: Scene
    edits: List[Edit]
    args: RenderArgs
    frames: Optional[List[List[Edit]]] = None  # config 5: per-frame edit lists
    name: str = ""


# ----------------------------------------------------------------------------------------
# mesh construction helpers (pure geometry; winding fixes the wound normal direction)
# ----------------------------------------------------------------------------------------

class _Builder:
    def __init__(self):
        self.pos: List[np.ndarray] = []
        self.idx: List[np.ndarray] = []
        self.tobj: List[np.ndarray] = []
        self.nv = 0
        self.obj_material: List[int] = []
        self.obj_emission: List[Sequence[float]] = []
        self.obj_flags: List[int] = []
        self.materials: List[Material] = []

    def material(self, m: Material) -> int:
        self.materials.append(m)
        return len(self.materials) - 1

    def add(self, verts: np.ndarray, tris: np.ndarray, material: int,
            emission=(0.0, 0.0, 0.0), flags: int = 0) -> int:
        oid = len(self.obj_material)
        verts = np.asarray(verts, dtype=np.float64).reshape(-1, 3)
        tris = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
        self.pos.append(verts.astype(np.float32))
        self.idx.append((tris + self.nv).astype(np.uint32))
        self.tobj.append(np.full(tris.shape[0], oid, dtype=np.uint32))
        self.nv += verts.shape[0]
        self.obj_material.append(material)
        self.obj_emission.append(tuple(float(e) for e in emission))
        self.obj_flags.append(flags)
        return oid

    def add_many(self, meshes, materials, flags=0):
        """Bulk-add many objects of identical topology: meshes = [n_obj, nv, 3] verts, tris [nt,3]."""
        verts, tris = meshes
        n_obj, nv = verts.shape[0], verts.shape[1]
        nt = tris.shape[0]
        base = self.nv + np.arange(n_obj, dtype=np.int64)[:, None, None] * nv
        oid0 = len(self.obj_material)
        self.pos.append(verts.reshape(-1, 3).astype(np.float32))
        self.idx.append((tris[None, :, :] + base).reshape(-1, 3).astype(np.uint32))
        self.tobj.append(np.repeat(np.arange(oid0, oid0 + n_obj, dtype=np.uint32), nt))
        self.nv += n_obj * nv
        for k in range(n_obj):
            self.obj_material.append(int(materials[k]))
            self.obj_emission.append((0.0, 0.0, 0.0))
            self.obj_flags.append(flags)
        return list(range(oid0, oid0 + n_obj))

    def build(self, camera: Camera, eps_rel: float, name: str) -> Scene:
        mats = self.materials
        return Scene(
            positions=np.concatenate(self.pos).astype(np.float32),
            indices=np.concatenate(self.idx).astype(np.uint32),
            tri_object=np.concatenate(self.tobj).astype(np.uint32),
            obj_material=np.asarray(self.obj_material, dtype=np.uint32),
            obj_emission=np.asarray(self.obj_emission, dtype=np.float32).reshape(-1, 3),
            obj_flags=np.asarray(self.obj_flags, dtype=np.uint32),
            mat_type=np.asarray([m.type for m in mats], dtype=np.uint32),
            mat_albedo=np.asarray([m.albedo for m in mats], dtype=np.float32).reshape(-1, 3),
            mat_roughness=np.asarray([m.roughness for m in mats], dtype=np.float32),
            camera=camera, eps_rel=float(eps_rel), name=name)


def quad(corner, a, b, n: int = 1):
    """Grid quad corner + u a + v b, u,v in [0,1]; wound normal along a x b; 2 n^2 tris."""
    corner, a, b = (np.asarray(x, dtype=np.float64) for x in (corner, a, b))
    g = np.linspace(0.0, 1.0, n + 1)
    uu, vv = np.meshgrid(g, g, indexing="ij")
    verts = corner + uu[..., None] * a + vv[..., None] * b
    verts = verts.reshape(-1, 3)
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    v00 = (i * (n + 1) + j).ravel()
    v10 = ((i + 1) * (n + 1) + j).ravel()
    v11 = ((i + 1) * (n + 1) + j + 1).ravel()
    v01 = (i * (n + 1) + j + 1).ravel()
    tris = np.concatenate([np.stack([v00, v10, v11], 1), np.stack([v00, v11, v01], 1)])
    return verts, tris


def _merge(parts):
    vs, ts, off = [], [], 0
    for v, t in parts:
        vs.append(v)
        ts.append(t + off)
        off += v.shape[0]
    return np.concatenate(vs), np.concatenate(ts)


def box(lo, hi, n: int = 1, inward: bool = False, faces: Sequence[str] = ("-x", "+x", "-y", "+y", "-z", "+z")):
    """Axis-aligned box; wound normals outward (or inward)."""
    x0, y0, z0 = lo
    x1, y1, z1 = hi
    sx, sy, sz = x1 - x0, y1 - y0, z1 - z0
    ex, ey, ez = np.array([sx, 0, 0.0]), np.array([0, sy, 0.0]), np.array([0, 0, sz])
    spec = {
        "-x": ((x0, y0, z0), ez, ey), "+x": ((x1, y0, z0), ey, ez),
        "-y": ((x0, y0, z0), ex, ez), "+y": ((x0, y1, z0), ez, ex),
        "-z": ((x0, y0, z0), ey, ex), "+z": ((x0, y0, z1), ex, ey),
    }
    parts = []
    for f in faces:
        c, a, b = spec[f]
        if inward:
            a, b = b, a
        parts.append(quad(c, a, b, n))
    return _merge(parts)


def _orient_outward(verts, tris, ref_fn):
    """Flip triangles whose wound normal points toward ref_fn(centroid) (inside)."""
    v0, v1, v2 = verts[tris[:, 0]], verts[tris[:, 1]], verts[tris[:, 2]]
    nrm = np.cross(v1 - v0, v2 - v0)
    cen = (v0 + v1 + v2) / 3.0
    out = cen - ref_fn(cen)
    bad = np.einsum("ij,ij->i", nrm, out) < 0
    tris = tris.copy()
    tris[bad] = tris[bad][:, [0, 2, 1]]
    return tris


def uv_ellipsoid(radii, slices: int, stacks: int):
    """UV ellipsoid about the origin (poles on +-y); 2*slices + 2*slices*(stacks-2) tris."""
    rx, ry, rz = radii
    verts = [np.array([0.0, ry, 0.0])]
    for k in range(1, stacks):
        th = math.pi * k / stacks
        for s in range(slices):
            ph = 2.0 * math.pi * s / slices
            verts.append(np.array([rx * math.sin(th) * math.cos(ph), ry * math.cos(th),
                                   rz * math.sin(th) * math.sin(ph)]))
    verts.append(np.array([0.0, -ry, 0.0]))
    verts = np.stack(verts)
    tris = []
    bottom = verts.shape[0] - 1
    for s in range(slices):
        s1 = (s + 1) % slices
        tris.append((0, 1 + s1, 1 + s))
    for k in range(stacks - 2):
        r0, r1 = 1 + k * slices, 1 + (k + 1) * slices
        for s in range(slices):
            s1 = (s + 1) % slices
            tris.append((r0 + s, r0 + s1, r1 + s1))
            tris.append((r0 + s, r1 + s1, r1 + s))
    rl = 1 + (stacks - 2) * slices
    for s in range(slices):
        s1 = (s + 1) % slices
        tris.append((bottom, rl + s, rl + s1))
    tris = np.asarray(tris, dtype=np.int64)
    tris = _orient_outward(verts, tris, lambda c: np.zeros_like(c))
    return verts, tris


def torus_x(R: float, r: float, n_major: int, n_minor: int):
    """Torus with symmetry axis along x, centred at the origin; 2*n_major*n_minor tris."""
    verts = []
    for i in range(n_major):
        a = 2.0 * math.pi * i / n_major
        cy, cz = math.cos(a), math.sin(a)
        for j in range(n_minor):
            b = 2.0 * math.pi * j / n_minor
            rr = R + r * math.cos(b)
            verts.append((r * math.sin(b), rr * cy, rr * cz))
    verts = np.asarray(verts, dtype=np.float64)
    tris = []
    for i in range(n_major):
        i1 = (i + 1) % n_major
        for j in range(n_minor):
            j1 = (j + 1) % n_minor
            a, b_, c, d = i * n_minor + j, i1 * n_minor + j, i1 * n_minor + j1, i * n_minor + j1
            tris.append((a, b_, c))
            tris.append((a, c, d))
    tris = np.asarray(tris, dtype=np.int64)

    def ring(cen):
        yz = cen[:, 1:3]
        nrm = np.linalg.norm(yz, axis=1, keepdims=True)
        on = R * yz / np.maximum(nrm, 1e-12)
        return np.concatenate([np.zeros((cen.shape[0], 1)), on], axis=1)
    tris = _orient_outward(verts, tris, ring)
    return verts, tris


def translate_xform(t) -> np.ndarray:
    x = np.zeros(12, dtype=np.float32)
    x[0] = x[5] = x[10] = 1.0
    x[3], x[7], x[11] = t
    return x


def rot_y_xform(deg: float, t) -> np.ndarray:
    """x' = Ry(deg) x + t."""
    c, s = math.cos(math.radians(deg)), math.sin(math.radians(deg))
    R = np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]], dtype=np.float64)
    x = np.zeros((3, 4), dtype=np.float64)
    x[:, :3] = R
    x[:, 3] = t
    return x.reshape(12).astype(np.float32)


def _rng(config: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=0x5EED0000 + config))


# ----------------------------------------------------------------------------------------
# Config 1 / 2: Cornell box stand-ins ("move the small box slightly to the right")
# ----------------------------------------------------------------------------------------

_GRAY, _RED, _GREEN = (0.75, 0.75, 0.75), (0.75, 0.15, 0.15), (0.15, 0.75, 0.15)
CORNELL_CAMERA = dict(pos=(0.5, 0.5, -1.2), look_at=(0.5, 0.5, 0.5), up=(0.0, 1.0, 0.0), vfov_deg=45.0)


def _cornell_room(b: _Builder):
    gray = b.material(Material(LAMBERT, _GRAY))
    red = b.material(Material(LAMBERT, _RED))
    green = b.material(Material(LAMBERT, _GREEN))
    black = b.material(Material(LAMBERT, (0.0, 0.0, 0.0)))
    # inward-facing walls of [0,1]^3 with the front (z=0) open
    b.add(*box((0, 0, 0), (1, 1, 1), inward=True, faces=("-y", "+y", "+z")), gray)
    b.add(*box((0, 0, 0), (1, 1, 1), inward=True, faces=("-x",)), red)
    b.add(*box((0, 0, 0), (1, 1, 1), inward=True, faces=("+x",)), green)
    # area light 0.25 x 0.25 at y = 0.999 facing down
    lv, lt = quad((0.375, 0.999, 0.375), (0.25, 0.0, 0.0), (0.0, 0.0, 0.25))  # x cross z = -y
    b.add(lv, lt, black, emission=(15.0, 15.0, 15.0))
    # static block [0.55,0.85]x[0,0.6]x[0.7,1]: the four faces not touching floor/back wall
    b.add(*box((0.55, 0.0, 0.7), (0.85, 0.6, 1.0), faces=("-x", "+x", "+y", "-z")), gray)
    return gray


# the dynamic cube rests 1 mm above the floor: its bottom face is never coplanar with the floor, so
# ray/triangle ties cannot depend on floating-point rounding (readings)
CUBE_CENTER = np.array([0.3, 0.151, 0.4])
CUBE_MOVE = np.array([0.1, 0.0, 0.05])


def config1(width: int = 64, height: int = 64, spp: int = 4, max_depth: int = 4, seed: int = 0) -> Workload:
    """cornell-move: 32 triangles, dynamic 12-tri cube moved (0.1,0,0.05)."""
    b = _Builder()
    gray = _cornell_room(b)
    cube = b.add(*box((-0.15, -0.15, -0.15), (0.15, 0.15, 0.15)), gray, flags=OBJ_DYNAMIC)
    scene = b.build(Camera(width=width, height=height, **CORNELL_CAMERA), 1e-4, "cornell-move")
    ed = Edit(cube, translate_xform(CUBE_CENTER), translate_xform(CUBE_CENTER + CUBE_MOVE))
    return Workload(scene, [ed], RenderArgs(spp=spp, seed=seed, max_depth=max_depth), name="config1")


def config2(width: int = 256, height: int = 256, spp: int = 16, max_depth: int = 6, seed: int = 2) -> Workload:
    """cornell-material: sphere Lambert 0.8 -> 0.3, cube GGX alpha 0.5 -> 0.1."""
    b = _Builder()
    _cornell_room(b)
    sph_m = b.material(Material(LAMBERT, (0.8, 0.8, 0.8)))
    cube_m = b.material(Material(GGX, (0.8, 0.8, 0.8), 0.5))
    cube = b.add(*box((-0.15, -0.15, -0.15), (0.15, 0.15, 0.15)), cube_m, flags=OBJ_DYNAMIC)
    sv, st = uv_ellipsoid((0.18, 0.18, 0.18), 32, 32)
    sph = b.add(sv, st, sph_m, flags=OBJ_DYNAMIC)
    scene = b.build(Camera(width=width, height=height, **CORNELL_CAMERA), 1e-4, "cornell-material")
    eye = translate_xform(CUBE_CENTER)
    sph_x = translate_xform((0.7, 0.18, 0.35))
    edits = [
        Edit(cube, eye, eye.copy(), Material(GGX, (0.8, 0.8, 0.8), 0.5), Material(GGX, (0.8, 0.8, 0.8), 0.1)),
        Edit(sph, sph_x, sph_x.copy(), Material(LAMBERT, (0.8, 0.8, 0.8)), Material(LAMBERT, (0.3, 0.3, 0.3))),
    ]
    return Workload(scene, edits, RenderArgs(spp=spp, seed=seed, max_depth=max_depth), name="config2")


# ----------------------------------------------------------------------------------------
# Config 3: procedural room (~200k tris), torus rotated 15 deg and translated
# ----------------------------------------------------------------------------------------

TORUS_CENTER = np.array([5.0, 0.65, 4.0])


def config3(width: int = 512, height: int = 512, spp: int = 32, max_depth: int = 8, seed: int = 3) -> Workload:
    rng = _rng(3)
    b = _Builder()
    wall = b.material(Material(LAMBERT, (0.6, 0.6, 0.6)))
    black = b.material(Material(LAMBERT, (0.0, 0.0, 0.0)))
    b.add(*box((0, 0, 0), (10, 3, 10), n=40, inward=True, faces=("-y", "-x", "+x", "-z", "+z")), wall)
    # 400 boxes: 6 faces each a 6x6 grid (432 tris), resting on the floor
    centers = []
    while len(centers) < 400:
        x, z = rng.uniform(0.5, 9.5, size=2)
        if math.hypot(x - TORUS_CENTER[0], z - TORUS_CENTER[2]) < 1.0:
            continue
        if 4.0 <= x <= 6.0 and 0.0 <= z <= 5.0:
            continue
        centers.append((x, z))
    sizes = rng.uniform(0.05, 0.5, size=(400, 3))
    albedos = rng.uniform(0.1, 0.9, size=(400, 3))
    for (x, z), sz, al in zip(centers, sizes, albedos):
        m = b.material(Material(LAMBERT, tuple(al)))
        lo = (x - sz[0] / 2, 0.0, z - sz[2] / 2)
        hi = (x + sz[0] / 2, sz[1], z + sz[2] / 2)
        b.add(*box(lo, hi, n=6), m)
    lv, lt = quad((4.5, 2.95, 4.5), (1.0, 0.0, 0.0), (0.0, 0.0, 1.0))
    b.add(lv, lt, black, emission=(15.0, 15.0, 15.0))
    rc = np.array([5.0, 1.5, 5.0])
    b.add(*box(rc - 50.0, rc + 50.0, inward=True), black, emission=(0.2, 0.2, 0.2), flags=OBJ_ENV)
    tor_m = b.material(Material(LAMBERT, (0.7, 0.7, 0.7)))
    tv, tt = torus_x(0.5, 0.15, 100, 50)
    tor = b.add(tv, tt, tor_m, flags=OBJ_DYNAMIC)
    cam = Camera((5.0, 1.7, 0.3), (5.0, 0.8, 6.0), (0.0, 1.0, 0.0), 65.0, width, height)
    scene = b.build(cam, 1e-4, "room-200k")
    ed = Edit(tor, translate_xform(TORUS_CENTER), rot_y_xform(15.0, TORUS_CENTER + np.array([0.2, 0.0, 0.1])))
    return Workload(scene, [ed], RenderArgs(spp=spp, seed=seed, max_depth=max_depth), name="config3")


# ----------------------------------------------------------------------------------------
# Config 4 / 5: large instanced scene (~2M tris)
# ----------------------------------------------------------------------------------------

CHAR_CENTER = np.array([0.0, 0.9, -22.0])


def _yaw_boxes(rng, n):
    unit_v, unit_t = box((-0.5, -0.5, -0.5), (0.5, 0.5, 0.5))
    edges = rng.uniform(0.1, 0.6, size=(n, 3))
    yaw = rng.uniform(0.0, 2.0 * math.pi, size=n)
    c, s = np.cos(yaw), np.sin(yaw)
    v = unit_v[None, :, :] * edges[:, None, :]
    x = c[:, None] * v[..., 0] + s[:, None] * v[..., 2]
    z = -s[:, None] * v[..., 0] + c[:, None] * v[..., 2]
    return np.stack([x, v[..., 1], z], axis=-1), unit_t


def _large_scene(config: int, extra_dynamic: bool):
    rng = _rng(4)  # configs 4 and 5 share the static scene
    b = _Builder()
    ground = b.material(Material(LAMBERT, (0.5, 0.5, 0.5)))
    black = b.material(Material(LAMBERT, (0.0, 0.0, 0.0)))
    b.add(*quad((-30.0, 0.0, -30.0), (0.0, 0.0, 60.0), (60.0, 0.0, 0.0)), ground)

    def centers(n):
        out = np.empty((0, 3))
        while out.shape[0] < n:
            c = rng.uniform((-30, 0, -30), (30, 12, 30), size=(2 * n, 3))
            keep = ~((np.abs(c[:, 0]) <= 4.0) & (c[:, 2] >= -30.0) & (c[:, 2] <= -19.0))
            out = np.concatenate([out, c[keep]])
        return out[:n]

    def materials(n):
        ids = []
        is_ggx = rng.uniform(size=n) < 0.3
        f0 = rng.uniform(0.1, 0.9, size=(n, 3))
        alpha = rng.uniform(0.05, 0.8, size=n)
        alb = rng.uniform(0.1, 0.9, size=(n, 3))
        for k in range(n):
            if is_ggx[k]:
                ids.append(b.material(Material(GGX, tuple(f0[k]), float(alpha[k]))))
            else:
                ids.append(b.material(Material(LAMBERT, tuple(alb[k]))))
        return ids

    n_sph, n_box = 1500, 46000
    sv, st = uv_ellipsoid((1.0, 1.0, 1.0), 24, 21)
    sc = centers(n_sph)
    sr = rng.uniform(0.1, 0.5, size=n_sph)
    b.add_many((sv[None] * sr[:, None, None] + sc[:, None, :], st), materials(n_sph))
    bv, bt = _yaw_boxes(rng, n_box)
    bc = centers(n_box)
    b.add_many((bv + bc[:, None, :], bt), materials(n_box))
    for cx, cz in ((-15.0, -10.0), (10.0, 0.0), (0.0, 15.0)):
        lv, lt = quad((cx - 1.5, 16.0, cz - 1.5), (3.0, 0.0, 0.0), (0.0, 0.0, 3.0))
        b.add(lv, lt, black, emission=(30.0, 30.0, 30.0))
    char_m = b.material(Material(LAMBERT, (0.7, 0.7, 0.7)))
    cv, ct = uv_ellipsoid((0.35, 0.9, 0.25), 125, 201)
    dyn = [b.add(cv, ct, char_m, flags=OBJ_DYNAMIC)]
    centers_dyn = [CHAR_CENTER]
    if extra_dynamic:
        m1 = b.material(Material(GGX, (0.9, 0.9, 0.9), 0.2))
        v1, t1 = uv_ellipsoid((0.4, 0.4, 0.4), 24, 21)
        dyn.append(b.add(v1, t1, m1, flags=OBJ_DYNAMIC))
        centers_dyn.append(np.array([-2.0, 1.5, -20.0]))
        m2 = b.material(Material(LAMBERT, (0.8, 0.8, 0.8)))
        dyn.append(b.add(*box((-0.25, -0.25, -0.25), (0.25, 0.25, 0.25)), m2, flags=OBJ_DYNAMIC))
        centers_dyn.append(np.array([2.0, 0.251, -21.0]))  # 1 mm above the ground (no coplanar faces)
    return b, dyn, centers_dyn


def config4(width: int = 1024, height: int = 1024, spp: int = 64, max_depth: int = 8, seed: int = 4) -> Workload:
    b, dyn, cen = _large_scene(4, extra_dynamic=False)
    cam = Camera((0.0, 2.0, -30.0), (0.0, 1.5, 0.0), (0.0, 1.0, 0.0), 50.0, width, height)
    scene = b.build(cam, 1e-5, "large-2M")
    ed = Edit(dyn[0], translate_xform(cen[0]), translate_xform(cen[0] + np.array([0.2, 0.0, 0.0])))
    return Workload(scene, [ed], RenderArgs(spp=spp, seed=seed, max_depth=max_depth), name="config4")


def config5(width: int = 1920, height: int = 1080, spp: int = 128, max_depth: int = 8, seed: int = 5000,
            n_frames: int = 16) -> Workload:
    b, dyn, cen = _large_scene(5, extra_dynamic=True)
    cam = Camera((0.0, 2.0, -30.0), (0.0, 1.5, 0.0), (0.0, 1.0, 0.0), 50.0, width, height)
    scene = b.build(cam, 1e-5, "anim-16")
    rng = _rng(5)
    ang = rng.uniform(0.0, 2.0 * math.pi, size=len(dyn))
    speed = rng.uniform(0.05, 0.2, size=len(dyn))
    vel = np.stack([np.cos(ang) * speed, np.zeros_like(ang), np.sin(ang) * speed], 1)
    frames = []
    for f in range(n_frames):
        frames.append([Edit(o, translate_xform(c + f * v), translate_xform(c + (f + 1) * v))
                       for o, c, v in zip(dyn, cen, vel)])
    return Workload(scene, frames[0], RenderArgs(spp=spp, seed=seed, max_depth=max_depth),
                    frames=frames, name="config5")


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def load_config(k: int, **kw) -> Workload:
    return CONFIGS[k](**kw)


# ----------------------------------------------------------------------------------------
# Tiny validation fixtures (SURVEY 8(d) "Tiny validation scenes")
# ----------------------------------------------------------------------------------------

def furnace(albedo: float = 0.5, new_albedo: Optional[float] = None, le: float = 1.0, width: int = 8,
            height: int = 8, max_depth: int = 4, spp: int = 4, dynamic: bool = True) -> Workload:
    """White furnace: closed inward-facing cube, every face Lambert `albedo` and emitting `le`.

    The enclosure is the (material-edited) dynamic object when `new_albedo` is given.
    """
    b = _Builder()
    m = b.material(Material(LAMBERT, (albedo,) * 3))
    obj = b.add(*box((-1, -1, -1), (1, 1, 1), n=2, inward=True), m, emission=(le, le, le),
                flags=OBJ_DYNAMIC if dynamic else 0)
    cam = Camera((0.0, 0.0, -0.5), (0.0, 0.0, 1.0), (0.0, 1.0, 0.0), 60.0, width, height)
    scene = b.build(cam, 1e-4, "furnace")
    edits = []
    if dynamic:
        eye = translate_xform((0.0, 0.0, 0.0))
        na = albedo if new_albedo is None else new_albedo
        edits = [Edit(obj, eye, eye.copy(), Material(LAMBERT, (albedo,) * 3), Material(LAMBERT, (na,) * 3))]
    return Workload(scene, edits, RenderArgs(spp=spp, seed=1, max_depth=max_depth), name="furnace")


def cornell_albedo_scale(k: float = 0.5, width: int = 32, height: int = 32, spp: int = 4) -> Workload:
    """Direct-only (D=2) Cornell box, cube albedo a -> k a (material-only edit, no move)."""
    w = config1(width, height, spp, max_depth=2)
    cube = w.edits[0].object
    eye = translate_xform(CUBE_CENTER)
    a = np.asarray(_GRAY)
    w.edits = [Edit(cube, eye, eye.copy(), Material(LAMBERT, tuple(a)), Material(LAMBERT, tuple(k * a)))]
    w.name = "cornell-albedo-scale"
    return w


def cornell_identity(width: int = 32, height: int = 32, spp: int = 4, max_depth: int = 4) -> Workload:
    w = config1(width, height, spp, max_depth=max_depth)
    eye = translate_xform(CUBE_CENTER)
    w.edits = [Edit(w.edits[0].object, eye, eye.copy())]
    w.name = "cornell-identity"
    return w


def occluder_reveal(width: int = 32, height: int = 32, spp: int = 4, max_depth: int = 4) -> Workload:
    """An object moves out from behind a wall (SPEC.md L530 'occluder-reveal')."""
    b = _Builder()
    gray = _cornell_room(b)
    wall = b.material(Material(LAMBERT, (0.5, 0.5, 0.5)))
    b.add(*quad((0.05, 0.0, 0.3), (0.0, 0.7, 0.0), (0.45, 0.0, 0.0)), wall)  # faces -z toward the camera
    cube = b.add(*box((-0.1, -0.1, -0.1), (0.1, 0.1, 0.1)), gray, flags=OBJ_DYNAMIC)
    scene = b.build(Camera(width=width, height=height, **CORNELL_CAMERA), 1e-4, "occluder-reveal")
    c0 = np.array([0.25, 0.1, 0.5])
    ed = Edit(cube, translate_xform(c0), translate_xform(c0 + np.array([0.45, 0.0, 0.0])))
    return Workload(scene, [ed], RenderArgs(spp=spp, seed=7, max_depth=max_depth), name="occluder-reveal")


# ----------------------------------------------------------------------------------------
# Sweeps of the paper's Table num_of_dynamics and Table material_editing, on the
# Cornell stand-ins (the paper's own scenes are not available).  Displacements scale the paper's 40/100/160/220
# units on its ~550-unit Cornell box to the unit box: 0.073 / 0.18 / 0.29 / 0.40.
# ----------------------------------------------------------------------------------------
DISPLACEMENT_LADDER = (0.073, 0.18, 0.29, 0.40)


def cornell_dynamics(n_dyn: int, displacement: float = 0.1, width: int = 64, height: int = 64, spp: int = 4,
                     max_depth: int = 4, seed: int = 0) -> Workload:
    """n_dyn small cubes (side 0.12) scattered uniformly over the Cornell box (seeded, non-overlapping, clear of
    the static block and the light), each moved by `displacement` in a random horizontal direction ("we
    uniformly scatter eight moving objects across the scene")."""
    rng = np.random.Generator(np.random.Philox(key=0x5EED0100 + n_dyn))
    b = _Builder()
    gray = _cornell_room(b)
    h = 0.06
    placed, edits = [], []
    while len(placed) < n_dyn:
        c = rng.uniform([0.08, 0.07, 0.08], [0.92, 0.85, 0.92])
        c[1] = max(c[1], h + 0.001)
        d = rng.normal(size=2)
        d = d / np.linalg.norm(d) * displacement
        c2 = c + np.array([d[0], 0.0, d[1]])
        sep = 2 * h + 0.01  # boxes (old and new placements) never overlap another cube's
        ok = all(np.max(np.abs(a - q)) > sep for p, p2 in placed for a in (c, c2) for q in (p, p2))
        inside = np.all(c2 > h + 0.01) and np.all(c2 < 1 - h - 0.01) and c2[1] == c[1]
        block = lambda x: (0.55 - h < x[0] < 0.85 + h) and (x[1] < 0.6 + h) and (x[2] > 0.7 - h)  # noqa: E731
        if ok and inside and not block(c) and not block(c2):
            placed.append((c, c2))
            obj = b.add(*box((-h, -h, -h), (h, h, h)), gray, flags=OBJ_DYNAMIC)
            edits.append(Edit(obj, translate_xform(c), translate_xform(c2)))
    scene = b.build(Camera(width=width, height=height, **CORNELL_CAMERA), 1e-4, f"cornell-{n_dyn}dyn")
    return Workload(scene, edits, RenderArgs(spp=spp, seed=seed, max_depth=max_depth), name=f"dynamics{n_dyn}")


def cornell_displacement(d: float, width: int = 64, height: int = 64, spp: int = 4, max_depth: int = 4,
                         seed: int = 0) -> Workload:
    """config 1's cube moved by d along +x (Table num_of_dynamics (b), the displacement ladder)"""
    w = config1(width, height, spp, max_depth, seed)
    w.edits = [Edit(w.edits[0].object, translate_xform(CUBE_CENTER), translate_xform(CUBE_CENTER + np.array([d, 0, 0])))]
    w.name = f"displacement{d:g}"
    return w


MATERIAL_EDITS = ("white_to_blue", "ggx_0.1_to_0.5", "lambert_to_metallic")


def cornell_material_edit(kind: str, width: int = 64, height: int = 64, spp: int = 4, max_depth: int = 6,
                          seed: int = 2) -> Workload:
    """Table material_editing's three edits on config 2's scene (sphere + cube), one at a time:
    the sphere's Lambert white -> blue; the cube's GGX roughness 0.1 -> 0.5; the sphere Lambert -> metallic
    (GGX, F0 0.9, alpha 0.2)."""
    w = config2(width, height, spp, max_depth, seed)
    cube_e, sph_e = w.edits
    if kind == "white_to_blue":
        e = dataclasses.replace(sph_e, old_material=Material(LAMBERT, (0.8, 0.8, 0.8)),
                                new_material=Material(LAMBERT, (0.1, 0.1, 0.8)))
    elif kind == "ggx_0.1_to_0.5":
        e = dataclasses.replace(cube_e, old_material=Material(GGX, (0.8, 0.8, 0.8), 0.1),
                                new_material=Material(GGX, (0.8, 0.8, 0.8), 0.5))
    elif kind == "lambert_to_metallic":
        e = dataclasses.replace(sph_e, old_material=Material(LAMBERT, (0.8, 0.8, 0.8)),
                                new_material=Material(GGX, (0.9, 0.9, 0.9), 0.2))
    else:
        raise ValueError(kind)
    w.edits = [e]
    w.name = f"material-{kind}"
    return w


def subsample(w: Workload, width: int, height: int) -> Workload:
    """Same scene and camera, reduced resolution (SURVEY 8(c) C10 parity at 128x128)."""
    return dataclasses.replace(w, scene=w.scene.with_camera(width, height))
