"""Pins of the oracle's residual estimator against exact special cases, closed forms and an
independent estimator (the oracle's primal NEE/BSDF-MIS path tracer), SURVEY 8(c) C11."""
import dataclasses
import math
import multiprocessing as mp

import numpy as np
import pytest

from oracle import binding as B
from rr_inputs import scenes as S


def _pool():
    return mp.get_context("fork").Pool(min(8, mp.cpu_count()))


# ---------------------------------------------------------------- exact special cases
@pytest.mark.parametrize("flags", [S.PAPER_FLAGS, S.TWO_WAY, 0, S.PAPER_FLAGS | S.VNDF])
def test_identity_edit_is_exactly_zero(flags):
    """old_xform == new_xform bitwise and equal materials: every record cancels bitwise (S:L181,
    S:L507); the object stays dynamic so T1-T3 and T7 all run (no API short-circuit)."""
    w = S.cornell_identity(16, 16, spp=4, max_depth=5)
    o = B.Oracle(w.scene, w.edits)
    assert o.effective_mask(0x7F) == 0x47
    args = dataclasses.replace(w.args, flags=flags)
    img, recs, _ = o.render_residual(args, records=True)
    assert np.count_nonzero(img) == 0
    assert len(recs) > 500
    techs = {r.tech for r in recs}
    assert techs == {1, 2, 3, 7}
    for r in recs:
        assert r.status == 0
        for c in range(3):
            assert r.term_p[c] + r.term_q[c] == 0.0


def test_albedo_scale_direct_only():
    """D = 2, Lambert albedo a -> k a on the cube: every record through the cube has term_N = -k term_O (exact
    up to the rounding of k a), every other record cancels exactly; the image is (k-1) x the cube's old direct radiance with the same samples."""
    k = 0.5
    w = S.cornell_albedo_scale(k, 16, 16, spp=8)
    o = B.Oracle(w.scene, w.edits)
    img, recs, _ = o.render_residual(w.args, records=True)
    old_sum = np.zeros(3)
    n = 0
    for r in recs:
        assert r.status == 0  # a Lambert albedo edit never diverges
        tn, to = (np.array(r.term_p), np.array(r.term_q)) if r.side == 0 else (np.array(r.term_q), np.array(r.term_p))
        if np.all(tn == -to):   # path does not touch the cube: exact cancellation
            continue
        np.testing.assert_allclose(tn, -k * to, rtol=1e-7, atol=1e-300)
        old_sum += to
        n += 1
    assert n > 100
    # image = (k - 1) * old direct radiance  ==  sum(new) + sum(old) with new = -k old
    np.testing.assert_allclose(img.sum((0, 1)), (k - 1) * (-old_sum), rtol=1e-9)
    # pixels that never see the cube stay exactly 0
    assert 0 < np.count_nonzero(img.sum(2)) < img.shape[0] * img.shape[1]


def test_pure_replay_has_unit_jacobian():
    """North star: 'the mapping Jacobian is 1 for pure replay' (R == 1 exactly)."""
    w = S.config1(16, 16, spp=4)
    o = B.Oracle(w.scene, w.edits)
    args = dataclasses.replace(w.args, flags=S.TWO_WAY)
    _, recs, _ = o.render_residual(args, records=True)
    assert len(recs) > 1000
    assert all(r.R == 1.0 for r in recs)
    args = dataclasses.replace(w.args, flags=S.PAPER_FLAGS)
    _, recs, st = o.render_residual(args, records=True)
    assert sum(s["reconnected"] for s in st) > 0
    assert any(r.R != 1.0 for r in recs)
    assert all(r.R > 0 and math.isfinite(r.R) for r in recs if r.status == 0)


def test_sharding_partition_is_exact():
    """Films of disjoint sample ranges add up to the film of the union."""
    w = S.config1(16, 16, spp=4)
    o = B.Oracle(w.scene, w.edits)
    n = o.sample_range(w.args)
    for l in (2, 4, 7):
        full, _, _ = o.residual(w.args, l, 1, 0, n)
        a, _, _ = o.residual(w.args, l, 1, 0, n // 3)
        b, _, _ = o.residual(w.args, l, 1, n // 3, n)
        np.testing.assert_allclose(a + b, full, rtol=1e-12, atol=1e-15)


# ---------------------------------------------------------------- closed forms
def _furnace_primal(seed):
    w = S.furnace(0.5, le=1.0, width=4, height=4, max_depth=4, dynamic=False)
    o = B.Oracle(w.scene, w.edits)
    img, _ = o.primal(0, seed, 256, 4)
    return img


def test_furnace_primal_closed_form():
    """Closed Lambert enclosure, albedo a, radiance Le: pixel = Le sum_{j<D} a^j (= 1.875)."""
    with _pool() as p:
        imgs = np.stack(p.map(_furnace_primal, range(16)))
    m = imgs.mean()
    s = imgs.reshape(16, -1).mean(1).std() / math.sqrt(16)
    assert abs(m - 1.875) < 4 * s + 1e-3, (m, s)


def _furnace_residual(seed):
    w = S.furnace(0.5, new_albedo=0.8, le=1.0, width=4, height=4, max_depth=4, spp=16)
    o = B.Oracle(w.scene, w.edits)
    img, _, _ = o.render_residual(dataclasses.replace(w.args, seed=seed))
    return img


def test_furnace_residual_closed_form():
    """Material edit a -> a' of the enclosure: E[residual] = Le sum_{j=1}^{D-1} (a'^j - a^j) (= 1.077)."""
    with _pool() as p:
        imgs = np.stack(p.map(_furnace_residual, range(16)))
    per = imgs.reshape(16, -1).mean(1)
    m, s = per.mean(), per.std() / math.sqrt(16)
    assert abs(m - 1.077) < 4 * s + 2e-3, (m, s)


# ---------------------------------------------------------------- MIS + per-technique correctness
def _render(a):
    cfg, W, seed, mask, flags, D = a
    w = S.load_config(cfg, width=W, height=W, spp=8, max_depth=D) if cfg in (1, 2) else S.occluder_reveal(W, W, 8, D)
    o = B.Oracle(w.scene, w.edits)
    img, _, _ = o.render_residual(dataclasses.replace(w.args, seed=seed, technique_mask=mask, flags=flags))
    return img


def _agree(ref, other, pix_frac=0.975):
    """paired per-seed difference of image sums must be 0 within 4 sigma; >= 97.5% pixels within 3.5 sigma (24 seeds, heavy tails)"""
    d = other - ref
    tot = d.sum((1, 2))
    m, s = tot.mean(0), tot.std(0) / math.sqrt(len(tot)) + 1e-12
    assert np.all(np.abs(m) < 4 * s + 1e-9), (m, s)
    pm = d.mean(0)
    ps = d.std(0) / math.sqrt(len(d)) + 1e-12
    frac = (np.abs(pm) <= 3.5 * ps + 1e-12).mean()
    assert frac >= pix_frac, frac


@pytest.mark.parametrize("cfg,D", [(1, 4), ("rev", 4)])
def test_masks_l_plus_7_agree_with_7(cfg, D):
    """For each l, mask {l,7} and mask {7} estimate the same residual."""
    cfg_ = 99 if cfg == "rev" else cfg
    seeds = range(24)
    with _pool() as p:
        ref = np.stack(p.map(_render, [(cfg_, 12, s, 0x40, S.TWO_WAY, D) for s in seeds]))
        for l in range(1, 7):
            other = np.stack(p.map(_render, [(cfg_, 12, s, 0x40 | (1 << (l - 1)), S.TWO_WAY, D) for s in seeds]))
            _agree(ref, other)
        full = np.stack(p.map(_render, [(cfg_, 12, s, 0x7F, S.PAPER_FLAGS, D) for s in seeds]))
        _agree(ref, full)
        # T6 "uniformly toward the light": a variance-only change
        t6l = np.stack(p.map(_render, [(cfg_, 12, s, 0x60, S.TWO_WAY | S.T6_TOWARD_LIGHT, D) for s in seeds]))
        _agree(ref, t6l)
        # T_obj on the first mid-path hit of a moved object: a mapping change only
        tobj = np.stack(p.map(_render, [(cfg_, 12, s, 0x40, S.TWO_WAY | S.TOBJ_MIDPATH, D) for s in seeds]))
        _agree(ref, tobj)
        # reconnection inside the two-ended techniques' emitter-side sub-walk
        for l in (3, 6):
            rb = np.stack(p.map(_render, [(cfg_, 12, s, 0x40 | (1 << (l - 1)), S.PAPER_FLAGS | S.RECONNECT_BIDIR, D)
                                          for s in seeds]))
            _agree(ref, rb)


def test_material_edit_masks_agree():
    seeds = range(24)
    with _pool() as p:
        ref = np.stack(p.map(_render, [(2, 12, s, 0x40, S.TWO_WAY, 4) for s in seeds]))
        for mask, flags in ((0x47, S.TWO_WAY), (0x47, S.PAPER_FLAGS), (0x41, S.PAPER_FLAGS), (0x44, S.TWO_WAY),
                            (0x44, S.PAPER_FLAGS | S.RECONNECT_BIDIR),
                            (0x47, S.PAPER_FLAGS | S.VNDF), (0x44, S.TWO_WAY | S.VNDF), (0x40, S.VNDF)):
            other = np.stack(p.map(_render, [(2, 12, s, mask, flags, 4) for s in seeds]))
            _agree(ref, other, pix_frac=0.95)  # GGX alpha 0.1 light-tracing splats are heavy-tailed


# Convergence to the independent primal reference, the MSE slope, two-way necessity and swap antisymmetry:
# tests/test_oracle_pins.py (default run, no skips).
