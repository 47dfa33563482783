"""The oracle against every known-answer example and property SPEC.md states
for the hot path (the reference ships no tests: CMakeLists.txt:11,19 point at
an absent tests/ tree, so SPEC.md's [OP] examples are the golden vectors)."""
import math

import numpy as np
import pytest

from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import FieldConfig, Roi, Rpc, TrainConfig


def unit_box():
    return [0, 0, 0, 1, 1, 1]


# ---- geometry ------------------------------------------------
def test_intersect_kats(oracle):
    assert oracle.intersect([-1, 0.5, 0.5], [1, 0, 0], unit_box()) == (1.0, 2.0)
    assert oracle.intersect([0.5, 0.5, 2], [0, 0, -1], unit_box()) == (1.0, 2.0)
    d = np.array([1, 1, 0]) / math.sqrt(2)
    t0, t1 = oracle.intersect([-0.5, -0.5, 0.5], d, unit_box())
    assert abs(t0 - math.sqrt(0.5)) < 1e-12 and abs(t1 - 3 * math.sqrt(0.5)) < 1e-12
    # miss, behind, grazing
    assert oracle.intersect([2, 2, 2], [1, 0, 0], unit_box()) is None
    assert oracle.intersect([0.5, 0.5, -1], [0, 0, -1], unit_box()) is None
    assert oracle.intersect([1.0, 0.5, 2], [0, 0, -1], unit_box()) == (1.0, 2.0)  # on the face: inclusive


def test_segment_kats(oracle):
    boxes = [[0, 0, 0, 1, 1, 1], [1, 0, 0, 2, 1, 1], [0, 1, 0, 1, 2, 1], [1, 1, 0, 2, 2, 1]]
    s = oracle.segments([0.5, 0.5, 2], [0, 0, -1], boxes)
    assert len(s) == 1 and s[0][0] == 0
    d = np.array([1, 0, -1]) / math.sqrt(2)
    s = oracle.segments([0.5, 0.5, 1.0], d, boxes)
    assert len(s) == 2 and s[0][2] == s[1][1]  # F1 == N2 exactly
    # low-incidence ray clipping the corner region between three tiles
    d = np.array([1.0, 1.3, -0.2])
    d /= np.linalg.norm(d)
    s = oracle.segments([0.6, 0.55, 0.95], d, boxes)
    assert len(s) == 3
    for k in range(len(s) - 1):
        assert s[k][2] <= s[k + 1][1] + 1e-12


def test_segment_partition_property(oracle):
    rng = np.random.default_rng(0)
    boxes = [[i, j, 0, i + 1, j + 1, 0.25] for j in range(3) for i in range(3)]
    for _ in range(200):
        o = np.array([rng.uniform(0, 3), rng.uniform(0, 3), 0.25])
        th = rng.uniform(0, math.radians(30))
        ph = rng.uniform(0, 2 * math.pi)
        d = np.array([math.sin(th) * math.cos(ph), math.sin(th) * math.sin(ph), -math.cos(th)])
        segs = oracle.segments(o, d, boxes)
        assert len(segs) <= 3
        total = sum(tf - tn for _, tn, tf in segs)
        # brute-force march of the union of boxes
        tex = 0.25 / math.cos(th)
        ts = np.arange(0, tex, 1e-4)
        p = o[None, :] + ts[:, None] * d[None, :]
        inside = (p[:, 0] >= 0) & (p[:, 0] <= 3) & (p[:, 1] >= 0) & (p[:, 1] <= 3)
        meas = inside.sum() * 1e-4
        assert abs(total - meas) <= 2e-3 * max(tex, 1e-3) + 2e-4
        for k in range(len(segs) - 1):
            assert abs(segs[k][2] - segs[k + 1][1]) < 1e-6


# ---- camera --------------------------------------------------
def identity_camera(z_coeff=0.0):
    c = Rpc()
    c.line_num[1] = 1.0  # row = L
    c.samp_num[2] = 1.0  # col = P
    c.line_num[3] = z_coeff
    c.line_den[0] = c.samp_den[0] = 1.0
    c.image_rows = c.image_cols = 10
    return c


def test_identity_camera(oracle):
    c = identity_camera()
    np.testing.assert_array_equal(oracle.project(c, [0.3, -0.2, 0.0]), [0.3, -0.2])
    st, xy, r, it = oracle.localize(c, [0.3, -0.2], 0.0)
    assert st == 0 and np.allclose(xy, [0.3, -0.2], atol=1e-12)
    # SPEC.md:144 says a z-independent projection is a degenerate baseline, but
    # the reference code (camera.cpp:112-115) measures the 3D baseline, which
    # keeps its z component: it returns a vertical ray.  The code is the oracle;
    # the degenerate case it rejects is z_max <= z_min.
    o, d = oracle.ray_from_pixel(c, 0, 0, 0.0, 1.0)
    np.testing.assert_array_equal(d, [0, 0, -1])
    assert oracle.ray_from_pixel(c, 0, 0, 1.0, 1.0) is None
    assert oracle.project(c, [2.0, 0.0, 0.0]) is None  # outside validity 1.5


def test_localize_roundtrip(oracle):
    scene = synth.make_scene(2, 2, n_views=3, seed=3)
    rng = np.random.default_rng(1)
    for cam in scene.cams:
        for _ in range(300):
            p = [rng.uniform(0, 256), rng.uniform(0, 256), rng.uniform(0, 40)]
            px = oracle.project(cam, p)
            st, xy, r, it = oracle.localize(cam, px, p[2])
            assert st == 0 and r < 1e-4
            assert abs(xy[0] - p[0]) < 1e-4 * cam.long_scale and abs(xy[1] - p[1]) < 1e-4 * cam.lat_scale


def test_ray_from_pixel_directions(oracle):
    roi = Roi(0, 128, 0, 128, 0, 40)
    nadir = synth.make_camera(roi, 0.5, 0.0, 0.0, nonlinear=0.0)
    o, d = oracle.ray_from_pixel(nadir, 100, 120, 0.0, 40.0)
    assert np.allclose(d, [0, 0, -1], atol=1e-6)
    obl = synth.make_camera(roi, 0.5, 20.0, 60.0, nonlinear=0.0)
    o, d = oracle.ray_from_pixel(obl, 150, 130, 0.0, 40.0)
    assert abs(d[2] + math.cos(math.radians(20))) < 1e-3
    assert abs(np.linalg.norm(d) - 1) < 1e-9


def test_crop_kats(oracle):
    scene = synth.make_scene(4, 4, n_views=2, seed=5)
    cam = scene.cams[0]
    box = [0, 0, 0, 128, 128, 40]
    r0 = oracle.crop_for_tile(cam, box, 0)
    r8 = oracle.crop_for_tile(cam, box, 8)
    assert r8[0] <= r0[0] and r8[1] >= r0[1] and r8[2] <= r0[2] and r8[3] >= r0[3]
    # crop coverage: random points of the box project inside the margin-0 rect
    rng = np.random.default_rng(2)
    for _ in range(2000):
        p = [rng.uniform(0, 128), rng.uniform(0, 128), rng.uniform(0, 40)]
        rc = oracle.project(cam, p)
        assert r0[0] <= rc[0] < r0[1] and r0[2] <= rc[1] < r0[3]


# ---- tiler ----------------------------------------------------
def test_grid_edges_shared(oracle):
    roi = Roi(100.0, 4100.0, 200.0, 4200.0, 0, 40)
    e, n = oracle.grid_edges(roi, 4, 4)
    assert e[3] == 100.0 + 3000.0 and n[2] == 200.0 + 2000.0
    assert e[0] == roi.easting_min and e[-1] == roi.easting_max


def test_candidate_superset(oracle):
    scene = synth.make_scene(3, 3, n_views=2, seed=7)
    boxes = []
    e, n = oracle.grid_edges(scene.roi, 3, 3)
    for r in range(3):
        for c in range(3):
            boxes.append([e[c], n[r], 0, e[c + 1], n[r + 1], 40])
    rng = np.random.default_rng(3)
    cam = scene.cams[1]
    for _ in range(300):
        ray = oracle.ray_from_pixel(cam, int(rng.integers(40, 700)), int(rng.integers(40, 700)), 0.0, 40.0)
        if ray is None:
            continue
        o, d = ray
        cand = set(oracle.candidate_tiles(scene.roi, 3, 3, o, d))
        for k, b in enumerate(boxes):
            if oracle.intersect(o, d, b) is not None:
                assert (k // 3, k % 3) in cand


# ---- sampler ----------------------------------------------------
FR_UNIT = [0, 0, 0, 1, 1, 1]  # frame origin + inv size of a [0,1]^3-ish tile


def test_sampler_uniform_grid(oracle):
    o, d = [0.5, 0.5, 3.0], [0, 0, -1]
    s = oracle.sample_ray(o, d, [(0, 1.0, 2.0)], [FR_UNIT], spm=4.0, zmin=0.0)
    np.testing.assert_array_equal(s["t"], np.array([1.0, 1.25, 1.5, 1.75, 2.0], np.float32))
    np.testing.assert_array_equal(s["endpoint"], [1, 0, 0, 0, 1])
    # last delta: remaining distance to the z_min exit (3 - 2 = 1), capped at 10
    assert s["delta"][-1] == 1.0


def test_sampler_duplicate_boundary(oracle):
    o, d = [0.5, 0.5, 3.0], [0, 0, -1]
    s = oracle.sample_ray(o, d, [(0, 0.0, 1.0), (1, 1.0, 2.0)], [FR_UNIT, FR_UNIT], spm=2.0)
    t = list(s["t"])
    assert t.count(1.0) == 2
    i = t.index(1.0)
    assert s["delta"][i] == 0.0 and s["slot"][i] == 0 and s["slot"][i + 1] == 1


def test_sampler_jitter_stratified(oracle):
    o, d = [0.5, 0.5, 3.0], [0, 0, -1]
    s = oracle.sample_ray(o, d, [(0, 1.0, 2.0)], [FR_UNIT], spm=10.0, jitter=True, key=123)
    t = s["t"].astype(np.float64)
    assert t[0] == 1.0 and t[-1] == 2.0 and np.all(np.diff(t) > 0)
    for j in range(1, 10):
        assert (j - 0.5) * 0.1 - 1e-6 <= t[j] - 1.0 <= (j + 0.5) * 0.1 + 1e-6


def test_sampler_occupancy_culling(oracle):
    # nadir ray down x=y=0.5 of a unit tile; voxels z in [0.4, 0.6) cleared
    res = 32
    occ = np.ones(res ** 3, np.float32)
    for z in range(res):
        if 0.4 <= (z + 0.5) / res < 0.6:
            occ[z * res * res:(z + 1) * res * res] = 0.0
    o, d = [0.5, 0.5, 1.0], [0, 0, -1]
    s = oracle.sample_ray(o, d, [(0, 0.0, 1.0)], [FR_UNIT], spm=64.0, occupancy=[occ])
    z = s["local"][:, 2]
    interior = s["endpoint"] == 0
    band = (z >= 13 / 32) & (z < 19 / 32)
    assert not np.any(band & interior)
    assert s["endpoint"][0] == 1 and s["endpoint"][-1] == 1


# ---- render + loss --------------------------------------------
def test_render_kats(oracle):
    rgb, dep, op, _, _ = oracle.render_ray([0, 0, 0], np.full((3, 3), 0.3), [1, 2, 3], [1, 1, 1])
    np.testing.assert_allclose(rgb, [0.5, 0.5, 0.5]) and op == 0
    c = [0.2, 0.7, 0.9]
    rgb, dep, op, _, _ = oracle.render_ray([10.0], [c], [4.0], [1.0])
    assert np.all(np.abs(rgb - np.array(c)) <= math.exp(-10) + 1e-6) and abs(dep - 4.0) < 1e-5


def test_render_weight_normalization_and_duplicate(oracle):
    rng = np.random.default_rng(4)
    for _ in range(50):
        n = int(rng.integers(2, 80))
        sg = rng.uniform(0, 5, n)
        de = rng.uniform(0, 1, n)
        de[n // 2] = 0.0  # boundary duplicate
        t = np.cumsum(de)
        rgbs = rng.uniform(0, 1, (n, 3))
        # weights from a black background: opacity + T_N = 1
        rgb, dep, op, _, _ = oracle.render_ray(sg, np.zeros((n, 3)), t, de, bg=(1, 1, 1))
        assert abs(rgb[0] - (1 - op)) < 1e-6  # rgb = T_N
        _, _, _, ds, dr = oracle.render_ray(sg, rgbs, t, de, g=[1, 1, 1])
        assert ds[n // 2] == 0.0 and np.all(dr[n // 2] == 0.0)


def test_color_loss_kat(oracle):
    """SPEC.md:376-377 through the oracle's color_loss (the code tfo_composite
    uses): rendered = target -> 0 and 0; rendered = target + 0.1 on all
    channels, 1 ray -> loss 0.01, gradient 0.2/3 per channel."""
    target = np.array([[0.2, 0.3, 0.4]], np.float32)
    L, g = oracle.color_loss(target, target)
    assert L == 0.0 and not np.any(g)
    L, g = oracle.color_loss(target + np.float32(0.1), target)
    assert abs(L - 0.01) < 1e-8
    np.testing.assert_allclose(g, np.full((1, 3), 0.2 / 3), rtol=1e-6)
    # B rays: mean over rays and channels, gradient 2 (r - t) / (3 B)
    rng = np.random.default_rng(2)
    r, t = rng.random((7, 3)).astype(np.float32), rng.random((7, 3)).astype(np.float32)
    L, g = oracle.color_loss(r, t)
    assert abs(L - np.mean((r.astype(np.float64) - t) ** 2)) < 1e-7
    np.testing.assert_allclose(g, 2 * (r - t) / 21.0, rtol=1e-6, atol=1e-8)


def test_render_gradient_fd(oracle):
    rng = np.random.default_rng(5)
    n = 12
    sg = rng.uniform(0, 3, n)
    de = rng.uniform(0.05, 0.5, n)
    t = np.cumsum(de)
    c = rng.uniform(0.1, 0.9, (n, 3))
    g = np.array([0.3, -0.2, 0.5])
    _, _, _, ds, dr = oracle.render_ray(sg, c, t, de, g=g)
    for k in range(n):
        e = 1e-2
        sp, sm = sg.copy(), sg.copy()
        sp[k] += e
        sm[k] -= e
        fp = oracle.render_ray(sp, c, t, de)[0] @ g
        fm = oracle.render_ray(sm, c, t, de)[0] @ g
        assert abs((fp - fm) / (2 * e) - ds[k]) < 2e-3 * (1 + abs(ds[k]))


# ---- field ---------------------------------------------------
def test_query_color_zero_weights(oracle):
    cfg = FieldConfig.defaults()
    enc, dnet, _ = oracle.tile_create(cfg, 0, 0, 1)
    color = np.zeros_like(oracle.color_create(cfg, 1))
    s, rgb = oracle.query_field(cfg, enc, dnet, color, [0.3, 0.4, 0.5], [0, 0, -1])
    np.testing.assert_array_equal(rgb, [0.5, 0.5, 0.5])
    assert s >= 0


def test_fresh_field_density_scale(oracle):
    cfg = FieldConfig.defaults()
    enc, dnet, occ = oracle.tile_create(cfg, 1, 2, 7)
    assert np.all(occ == 1.0) and np.abs(enc).max() <= 1e-4
    color = oracle.color_create(cfg, 7)
    rng = np.random.default_rng(0)
    for _ in range(200):
        s, rgb = oracle.query_field(cfg, enc, dnet, color, rng.uniform(0, 1, 3), [0, 0, -1])
        assert 0.9 < s < 1.1  # exp(~0)
        assert np.all((rgb > 0) & (rgb < 1))


def test_adam_kats(oracle):
    p = np.random.default_rng(0).normal(size=64).astype(np.float32)
    p0 = p.copy()
    g = np.zeros_like(p)
    m, v = np.zeros_like(p), np.zeros_like(p)
    s = oracle.adam_step(p, g, m, v, 0)
    assert s == 1 and np.array_equal(p, p0)
    g[:] = 0.5
    for _ in range(10):
        s = oracle.adam_step(p, g, m, v, s)
    assert np.all(p < p0) and s == 11
    g[3] = np.nan
    with pytest.raises(RuntimeError, match="group g"):
        oracle.adam_step(p, g, m, v, s)


# ---- scheduler ------------------------------------------------
def test_snake_path(oracle):
    assert oracle.snake_path(2, 2) == [(0, 0)]
    assert oracle.snake_path(4, 4) == [(0, 0), (0, 1), (0, 2), (1, 2), (1, 1), (1, 0), (2, 0), (2, 1), (2, 2)]
    for H, W in [(3, 5), (6, 6), (8, 8)]:
        p = oracle.snake_path(H, W)
        assert len(p) == (H - 1) * (W - 1) and len(set(p)) == len(p)
        for a, b in zip(p, p[1:]):
            assert abs(a[0] - b[0]) + abs(a[1] - b[1]) == 1
    with pytest.raises(ValueError):
        oracle.snake_path(1, 4)


def _session(oracle, H, W, views=2, batch=256, seed=0):
    from oracle.pyoracle import Session

    scene = synth.make_scene(H, W, tile_side=128.0, n_views=views, seed=seed)
    return Session(oracle, scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=batch), workers=4)


def test_advance_swaps_and_multiplicity(oracle):
    s = _session(oracle, 4, 4)
    counts = {}
    prev = None
    for pos in oracle.snake_path(4, 4):
        s.set_window(*pos)
        tiles = s.window_tiles()
        assert len(set(tiles)) == 4
        if prev is not None:
            # staying tiles keep their slot; exactly 2 leave, 2 enter
            stay = [k for k in range(4) if tiles[k] == prev[k]]
            assert len(stay) == 2
        for t in tiles:
            counts[t] = counts.get(t, 0) + 1
        prev = tiles
    assert counts[(1, 1)] == 4 and counts[(0, 1)] == 2 and counts[(0, 0)] == 1
    # (0,0)->(0,1) unloads (0,0),(1,0), loads (0,2),(1,2)
    s2 = _session(oracle, 4, 4)
    s2.set_window(0, 0)
    a = set(s2.window_tiles())
    s2.set_window(0, 1)
    b = set(s2.window_tiles())
    assert a - b == {(0, 0), (1, 0)} and b - a == {(0, 2), (1, 2)}


def test_accept_full_window(oracle):
    """2x2 grid: the window covers the whole grid -> every in-ROI ray accepted."""
    s = _session(oracle, 2, 2, views=1)
    s.set_window(0, 0)
    acc = s.build_accept()
    assert acc.size > 0
    o = oracle
    cam = s.scene.cams[0]
    e, n = o.grid_edges(s.scene.roi, 2, 2)
    boxes = [[e[c], n[r], 0, e[c + 1], n[r + 1], 40] for r in range(2) for c in range(2)]
    acc_set = set(int(x) for x in acc)
    rng = np.random.default_rng(0)
    for _ in range(300):
        row, col = int(rng.integers(0, cam.image_rows)), int(rng.integers(0, cam.image_cols))
        ray = o.ray_from_pixel(cam, row, col, 0.0, 40.0)
        if ray is None:
            continue
        hits = sum(o.intersect(*ray, b) is not None for b in boxes)
        key = (row << 20) | col
        crop_rects = [o.crop_for_tile(cam, b, 4) for b in boxes]
        in_crop = any(r and r[0] <= row < r[1] and r[2] <= col < r[3] for r in crop_rects)
        if in_crop:
            assert (key in acc_set) == (hits >= 1)
