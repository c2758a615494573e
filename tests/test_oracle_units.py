"""Pins of the oracle's building blocks against values and definitions fixed outside the oracle.

Each test names the paper / SPEC passage (P:Lnnn = PAPER.md, S:Lnnn = SPEC.md) whose value it checks.
"""
import json
import math
import os
import shutil
import subprocess

import numpy as np
import pytest

from oracle import binding as B
from rr_inputs import scenes as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")
VALS = json.load(open(os.path.join(GOLD, "paper_values.json")))


# ---------------------------------------------------------------- Philox
def test_philox_known_answer_vectors():
    n = 0
    for line in open(os.path.join(GOLD, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        assert B.philox(w[0:4], w[4:6]) == w[6:10]
        n += 1
    assert n == 3


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")
def test_philox_matches_curand_host_build(tmp_path):
    """Library routine: cuRAND's curand_Philox4x32_10 compiled for the host (no GPU needed)."""
    src = tmp_path / "c.cu"
    src.write_text(r'''
#include <cstdio>
#include <cuda_runtime.h>
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
int main(){ unsigned s=987654321u; for(int k=0;k<2000;k++){ uint4 c={s,s*7u+1u,s*13u+5u,s*17u+9u};
 uint2 key={s^0xdeadbeefu,s*3u}; uint4 o=curand_Philox4x32_10(c,key);
 printf("%u %u %u %u %u %u %u %u %u %u\n",c.x,c.y,c.z,c.w,key.x,key.y,o.x,o.y,o.z,o.w); s=s*1103515245u+12345u;} }
''')
    exe = tmp_path / "c"
    subprocess.check_call(["nvcc", "-Wno-deprecated-gpu-targets", "-o", str(exe), str(src)])
    out = subprocess.check_output([str(exe)]).decode().split("\n")
    rows = [list(map(int, l.split())) for l in out if l.strip()]
    assert len(rows) == 2000
    for r in rows:
        assert B.philox(r[0:4], r[4:6]) == r[6:10]


def test_u01_is_exact_24bit():
    assert B.lib().orc_u01(0) == 0.0
    assert B.lib().orc_u01(0x100) == 2.0 ** -24
    assert B.lib().orc_u01(0xFFFFFFFF) == (2 ** 24 - 1) / 2 ** 24
    d = B.stream_dims(7, 123, 3, 1, 5)
    assert np.all((d >= 0) & (d < 1))
    assert np.all(np.float32(d) == d)  # exact in fp32


# ---------------------------------------------------------------- closed forms
def test_geometric_term_values():
    v = VALS["geometric_term"]
    assert B.geometric_term([0, 0, 0], [0, 0, 1], [0, 0, 1], [0, 0, -1]) == pytest.approx(v["facing_distance_1"], rel=1e-14)
    assert B.geometric_term([0, 0, 0], [0, 0, 1], [0, 0, 2], [0, 0, -1]) == pytest.approx(v["facing_distance_2"], rel=1e-14)


def test_lambert_values():
    v = VALS["lambert"]
    ev, pdf = B.bsdf([0, 0.5, 0.5, 0.5, 1.0], [0, 0, 1], [0, 0, 1], [math.sin(math.pi / 3), 0, math.cos(math.pi / 3)])
    assert ev == pytest.approx([v["albedo_0.5_rho"]] * 3, rel=1e-14)
    assert pdf == pytest.approx(v["cos_pdf_at_60deg"], rel=1e-14)
    # two-sided: flipping the normal does not change anything; opposite sides give 0
    ev2, pdf2 = B.bsdf([0, 0.5, 0.5, 0.5, 1.0], [0, 0, -1], [0, 0, 1], [math.sin(math.pi / 3), 0, math.cos(math.pi / 3)])
    assert pdf2 == pdf and np.all(ev2 == ev)
    ev3, pdf3 = B.bsdf([0, 0.5, 0.5, 0.5, 1.0], [0, 0, 1], [0, 0, 1], [0, 0.6, -0.8])
    assert pdf3 == 0 and np.all(ev3 == 0)


def _rand_dirs(rng, n, hemi=True):
    v = rng.normal(size=(n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    if hemi:
        v[:, 2] = np.abs(v[:, 2])
    return v


@pytest.mark.parametrize("alpha", [0.05, 0.3, 0.8])
def test_ggx_reciprocity(alpha):
    rng = np.random.default_rng(1)
    mat = [1, 0.9, 0.5, 0.2, alpha]
    n = np.array([0.0, 0.0, 1.0])
    for wi, wo in zip(_rand_dirs(rng, 200), _rand_dirs(rng, 200)):
        a, _ = B.bsdf(mat, n, wi, wo)
        b, _ = B.bsdf(mat, n, wo, wi)
        assert a == pytest.approx(b, rel=1e-12, abs=1e-300)


@pytest.mark.parametrize("mat", [[0, 0.8, 0.8, 0.8, 1.0], [1, 1.0, 1.0, 1.0, 0.1], [1, 1.0, 1.0, 1.0, 0.6],
                                 [2, 1.0, 1.0, 1.0, 0.1], [2, 1.0, 1.0, 1.0, 0.6]])
def test_sampling_density_matches_pdf(mat):
    """E[1/pdf(wo)] over valid samples = 2 pi iff the sampler's density equals pdf on the hemisphere;
    E[rho cos / pdf] <= 1 (energy)."""
    rng = np.random.default_rng(2)
    n = np.array([0.0, 0.0, 1.0])
    N = 40000
    for wi in ([0, 0, 1.0], [math.sin(1.0), 0, math.cos(1.0)]):
        inv, en = [], []
        u = rng.random((N, 2))
        for u1, u2 in u:
            ok, wo = B.bsdf_sample(mat, n, wi, u1, u2)
            if not ok:
                inv.append(0.0); en.append(0.0)
                continue
            ev, pdf = B.bsdf(mat, n, wi, wo)
            inv.append(1.0 / pdf)
            en.append(ev[0] * wo[2] / pdf)
        inv, en = np.array(inv), np.array(en)
        m, s = inv.mean(), inv.std() / math.sqrt(N)
        assert abs(m - 2 * math.pi) < 4 * s + 1e-3, (m, s)
        assert en.mean() < 1.0 + 3 * en.std() / math.sqrt(N)


# ---------------------------------------------------------------- GGX visible-normal sampling
def _g1(a, c):
    """Smith G1 of GGX (Walter et al. 2007, Eq. 34 written with cos): 2 / (1 + sqrt(1 + a^2 tan^2))"""
    return 2.0 / (1.0 + math.sqrt(1.0 + a * a * (1.0 - c * c) / (c * c)))


@pytest.mark.parametrize("alpha", [0.1, 0.5, 1.0])
def test_vndf_equals_ndf_sampling_at_normal_incidence(alpha):
    """At wi = n the visible-normal distribution is D(h)(n.h) (G1(n) = 1), so Heitz's warp reduces to the
    classic inversion tan^2 = a^2 u1 / (1 - u1): same direction for the same (u1, u2), same pdf."""
    rng = np.random.default_rng(4)
    n, wi = np.array([0.0, 0.0, 1.0]), [0.0, 0.0, 1.0]
    for u1, u2 in rng.random((200, 2)):
        ok1, w1 = B.bsdf_sample([1, 1, 1, 1, alpha], n, wi, u1, u2)
        ok2, w2 = B.bsdf_sample([2, 1, 1, 1, alpha], n, wi, u1, u2)
        assert ok1 == ok2
        if ok1:
            assert np.allclose(w1, w2, atol=1e-9), (w1, w2)
            assert B.bsdf([2, 1, 1, 1, alpha], n, wi, w2)[1] == pytest.approx(B.bsdf([1, 1, 1, 1, alpha], n, wi, w1)[1],
                                                                              rel=1e-9)


@pytest.mark.parametrize("alpha", [0.1, 0.4, 0.9])
def test_vndf_sample_weight_is_g1_of_wo(alpha):
    """With F0 = 1 (Fresnel 1) every visible-normal sample has weight f cos_o / pdf = G1(wo) exactly
    (f = D G1(wi) G1(wo) / (4 cos_i cos_o), pdf = G1(wi) D / (4 cos_i)), at any incidence."""
    rng = np.random.default_rng(5)
    n = np.array([0.0, 0.0, 1.0])
    mat = [2, 1.0, 1.0, 1.0, alpha]
    for th in (0.2, 0.9, 1.4):
        wi = [math.sin(th), 0.0, math.cos(th)]
        for u1, u2 in rng.random((300, 2)):
            ok, wo = B.bsdf_sample(mat, n, wi, u1, u2)
            if not ok:
                continue
            ev, pdf = B.bsdf(mat, n, wi, wo)
            assert ev[0] * wo[2] / pdf == pytest.approx(_g1(alpha, wo[2]), rel=1e-9)


def test_vndf_pdf_is_not_symmetric_but_eval_is():
    """pdf(wo | wi) conditions on wi: G1(wi) / cos_i differs from G1(wo) / cos_o, unlike the classic
    half-vector pdf; f stays reciprocal."""
    n = np.array([0.0, 0.0, 1.0])
    wi, wo = [math.sin(1.2), 0.0, math.cos(1.2)], [-math.sin(0.3), 0.0, math.cos(0.3)]
    ea, pa = B.bsdf([2, 1, 1, 1, 0.5], n, wi, wo)
    eb, pb = B.bsdf([2, 1, 1, 1, 0.5], n, wo, wi)
    assert ea[0] == pytest.approx(eb[0], rel=1e-12)
    assert pa / pb == pytest.approx((_g1(0.5, wi[2]) / wi[2]) / (_g1(0.5, wo[2]) / wo[2]), rel=1e-9)
    _, qa = B.bsdf([1, 1, 1, 1, 0.5], n, wi, wo)
    _, qb = B.bsdf([1, 1, 1, 1, 0.5], n, wo, wi)
    assert qa == pytest.approx(qb, rel=1e-12)


def test_lambert_histogram_chi_square():
    """Cosine-hemisphere sampling: histogram of cos(theta)^2 is uniform."""
    rng = np.random.default_rng(3)
    n = np.array([0.0, 0.0, 1.0])
    N, K = 20000, 20
    c2 = []
    for u1, u2 in rng.random((N, 2)):
        ok, wo = B.bsdf_sample([0, 1, 1, 1, 1], n, [0, 0, 1.0], u1, u2)
        c2.append(wo[2] ** 2)
    h, _ = np.histogram(c2, bins=K, range=(0, 1))
    chi = ((h - N / K) ** 2 / (N / K)).sum()
    assert chi < 43.8  # p = 0.001 for 19 dof


def test_vertex1pdf_values():
    v = VALS["vertex1pdf"]
    pG = 0.7
    # coincident x_1 = x_G with equal normals -> p(x_G)
    assert B.vertex1pdf(pG, [0, 0, 0], [0, 0, 1], [0, 0, 1], [0, 0, 1], [0, 0, 1]) == pytest.approx(pG * v["coincident"], rel=1e-14)
    # x_G at distance 1, x_1 at distance 2, all cosines 1 -> p(x_G)/4
    assert B.vertex1pdf(pG, [0, 0, 0], [0, 0, 1], [0, 0, 1], [0, 0, 2], [0, 0, -1]) == pytest.approx(pG * v["distances_1_2"], rel=1e-14)


def test_vertex1pdf_finite_difference():
    """Eq. vertex1pdf against the numerically measured density of x_1: map an area element
    around x_G through the ray from x_L onto a tilted receiver plane and compare area ratios."""
    a = np.array([0.1, -0.2, 0.0])
    xg, ng = np.array([0.0, 0.0, 1.0]), np.array([0.2, 0.1, 1.0]) / np.linalg.norm([0.2, 0.1, 1.0])
    n1 = np.array([0.3, -0.2, -1.0]) / np.linalg.norm([0.3, -0.2, -1.0])
    p0 = np.array([0.0, 0.0, 2.5])

    def proj(x):  # ray a -> x intersected with the receiver plane (p0, n1)
        d = x - a
        t = np.dot(p0 - a, n1) / np.dot(d, n1)
        return a + t * d
    x1 = proj(xg)
    t1 = np.cross(ng, [1, 0, 0]); t1 /= np.linalg.norm(t1)
    t2 = np.cross(ng, t1)
    h = 1e-5
    e1 = proj(xg + h * t1) - x1
    e2 = proj(xg + h * t2) - x1
    ratio = h * h / np.linalg.norm(np.cross(e1, e2))  # dA(x_G) / dA(x_1)
    pG = 1.3
    assert B.vertex1pdf(pG, a, xg, ng, x1, n1) == pytest.approx(pG * ratio, rel=1e-4)


def test_g_term_values():
    v = VALS["g_term"]
    pdir = 1 / (4 * math.pi)
    assert B.g_term(pdir, [0, 0, 1], [0, 0, 0], [0, 0, 1], [0, 0, 1], [0, 0, -1]) == pytest.approx(v["unit"], rel=1e-14)
    assert B.g_term(pdir, [0, 0, 1], [0, 0, 0], [0, 0, 1], [0, 0, 2], [0, 0, -1]) == pytest.approx(v["distance_2"], rel=1e-14)


def test_reconnect_jacobian_values():
    v = VALS["reconnect_jacobian"]
    xi, ni = [0, 0, 0], [0, 0, 1]
    assert B.reconnect_jacobian([0.3, 0.1, 1.0], [0.3, 0.1, 1.0], xi, ni) == pytest.approx(v["identity"], rel=1e-14)
    assert B.reconnect_jacobian([0.3, 0.0, 1.0], [0.6, 0.0, 2.0], xi, ni) == pytest.approx(v["twice_as_far"], rel=1e-14)


def test_reconnect_jacobian_finite_difference():
    """Eq. P:L397-401 as the ratio of projected solid angles of a fixed small patch at x_i seen from
    x_{i-1} and t(x_{i-1})."""
    xi, ni = np.array([0.0, 0.0, 0.0]), np.array([0.0, 0.0, 1.0])
    xp, tp = np.array([0.4, 0.2, 1.0]), np.array([-0.7, 0.3, 1.8])

    def solid_angle(o, h=1e-4):
        c = [xi + np.array(v) for v in ([0, 0, 0], [h, 0, 0], [h, h, 0], [0, h, 0])]
        d = [(x - o) / np.linalg.norm(x - o) for x in c]
        # small quad -> solid angle ~ |(d1-d0) x (d3-d0)|
        return np.linalg.norm(np.cross(d[1] - d[0], d[3] - d[0]))
    ratio = solid_angle(tp) / solid_angle(xp)  # |t'| = dw(t)/dw(x) for the same patch
    assert B.reconnect_jacobian(xp, tp, xi, ni) == pytest.approx(ratio, rel=1e-3)


# ---------------------------------------------------------------- candidate enumeration
def test_fig_importance_sample_d_candidates():
    """E S- S D2 S D2 D S- S S- L: 1 dynamic vertex + 4 ghost crossings + PT = 6."""
    # vertices E,x1..x4,L ; x3 dynamic ; edges (1,2) and (2,3) each cross the ghost twice
    c = B.candidates(6, [0, 0, 0, 1, 0, 0], [0, 2, 2, 0, 0])
    assert len(c) == VALS["fig_importance_sample_d"]["candidates"]
    assert sorted(t for t, _ in c) == [3, 6, 6, 6, 6, 7]


def test_candidate_ownership_rules():
    # 3-vertex path with dynamic x_1: direct lighting belongs to T1, not T2
    assert sorted(B.candidates(3, [0, 1, 0], [0, 0])) == [(1, 1), (7, 0)]
    # 4-vertex: x_1 -> T2, x_2 (adjacent to L) -> T1
    assert sorted(t for t, _ in B.candidates(4, [0, 1, 1, 0], [0, 0, 0])) == [1, 2, 7]
    # crossings: first edge -> T5, last edge -> T4, interior -> T6
    assert sorted(t for t, _ in B.candidates(4, [0, 0, 0, 0], [1, 1, 1])) == [4, 5, 6, 7]
    # k = 2 has no candidate besides PT
    assert B.candidates(2, [0, 0], [3]) == [(7, 0)]
    # mask restricts
    assert B.candidates(4, [0, 1, 1, 0], [1, 0, 0], mask=0x40 | 0x2) == [(2, 1), (7, 0)]


# ---------------------------------------------------------------- geometry queries
def _single_triangle_scene():
    b = S._Builder()
    m = b.material(S.Material(S.LAMBERT, (0.5, 0.5, 0.5)))
    b.add(np.array([[-1, -1, 0], [2, -1, 0], [-1, 2, 0.0]]), np.array([[0, 1, 2]]), m)
    b.add(*S.quad((5, 5, 5), (1, 0, 0), (0, 0, 1)), m, emission=(1, 1, 1))
    return b.build(S.Camera((0, 0, -3), (0, 0, 0), (0, 1, 0), 40, 8, 8), 1e-4, "tri")


def test_ray_fixture_t_equals_one():
    o = B.Oracle(_single_triangle_scene(), [])
    r = o.closest(0, [0, 0, -1], [0, 0, 1])
    v = VALS["ray_fixture"]
    assert r[0] == pytest.approx(v["t"], rel=1e-15)
    assert r[3:6] == pytest.approx(v["hit"], abs=1e-15)


@pytest.mark.parametrize("cfg", [1, 2])
def test_bvh_matches_brute_force(cfg):
    w = S.load_config(cfg, width=16, height=16)
    o = B.Oracle(w.scene, w.edits)
    rng = np.random.default_rng(cfg)
    for F in (0, 1):
        for _ in range(1500):
            org = rng.uniform(0.02, 0.98, 3)
            d = rng.normal(size=3)
            a = o.closest(F, org, d)
            b = o.closest_brute(F, org, d)
            assert (a[0] < 0) == (b[0] < 0)
            if a[0] >= 0:
                assert int(a[1]) == int(b[1])
                assert a[0] == pytest.approx(b[0], rel=1e-12)


def test_crossings_match_brute_force():
    w = S.config1(16, 16)
    o = B.Oracle(w.scene, w.edits)
    rng = np.random.default_rng(5)
    hits = 0
    for F in (0, 1):
        for _ in range(1000):
            c = S.CUBE_CENTER + S.CUBE_MOVE * rng.uniform(0, 1)
            a = c + rng.normal(size=3) * 0.3
            b = c + rng.normal(size=3) * 0.3
            n = len(o.crossings(F, a, b))
            assert n == o.crossings_brute(F, a, b)
            hits += n
    assert hits > 200


def test_ghost_transparency_and_crossing_geometry():
    """The ghost is transparent in View_F and a segment through it reports 2 crossings on
    the cube at M_Fbar with the cube's outward normals."""
    w = S.config1(16, 16)
    o = B.Oracle(w.scene, w.edits)
    old_c, new_c = S.CUBE_CENTER, S.CUBE_CENTER + S.CUBE_MOVE
    # a ray along -x through the old cube position but above the new one is not blocked in N
    org = np.array([0.99, old_c[1], old_c[2] - 0.12])
    r_new = o.closest(0, org, [-1, 0, 0])
    r_old = o.closest(1, org, [-1, 0, 0])
    assert r_old[0] < r_new[0]
    cr = o.crossings(0, org, org + np.array([-0.95, 0, 0]))
    assert len(cr) == 2
    assert cr[0][1] == pytest.approx(old_c[0] + 0.15, abs=1e-6)
    assert cr[0][4:7] == pytest.approx([1, 0, 0], abs=1e-12)


def test_area_sampling_uniform_and_pdf():
    w = S.config1(16, 16)
    o = B.Oracle(w.scene, w.edits)
    assert o.set_area(0) == pytest.approx(6 * 0.09, rel=1e-6)   # rigid motion preserves area
    assert o.set_area(1) == pytest.approx(o.set_area(0), rel=1e-12)
    rng = np.random.default_rng(9)
    N = 12000
    tris = np.array([o.sample_set(0, 0, *rng.random(3))[6] for _ in range(N)])
    h = np.bincount(tris.astype(int) - int(tris.min()), minlength=12)
    chi = ((h - N / 12) ** 2 / (N / 12)).sum()
    assert chi < 31.3  # p = 0.001, 11 dof


def test_material_only_edit_has_empty_ghost_set():
    w = S.config2(16, 16)
    o = B.Oracle(w.scene, w.edits)
    assert o.effective_mask(0x7F) == 0x47  # T4-T6 auto-disabled
    with pytest.raises(ValueError):
        o.sample_set(1, 0, 0.1, 0.2, 0.3)
