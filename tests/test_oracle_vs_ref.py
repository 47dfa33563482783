"""Pins the oracle restatement (oracle/tf_oracle.cpp) bit-for-bit against the
reference sources compiled verbatim (oracle/_ref/libtfref.so: geometry.cpp,
tiler.cpp, camera.cpp, parallel.cpp, nn.hpp, rng.hpp from
/root/reference/proj/src/core, Eigen-subset shim in oracle/shim)."""
import ctypes as C

import numpy as np
import pytest

from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import FieldConfig, Roi


@pytest.fixture(scope="module")
def scene():
    return synth.make_scene(3, 3, n_views=4, seed=11)


def test_rng_bits(oracle, reflib):
    L = oracle.L
    for x in [0, 1, 2**63 + 5, 123456789]:
        assert L.tfo_splitmix64(x) == reflib.L.ref_splitmix64(x)
        for y in [0, 7, 2**40]:
            assert L.tfo_hash_combine(x, y) == reflib.L.ref_hash_combine(x, y)
    u = reflib.rng_draws(99, 3, 1000, arg=12345)
    assert u.max() < 12345


def test_project_localize_ray_bits(oracle, reflib, scene):
    rng = np.random.default_rng(0)
    n_checked = 0
    for cam in scene.cams:
        for _ in range(400):
            p = [rng.uniform(-20, 404), rng.uniform(-20, 404), rng.uniform(0, 40)]
            a, b = oracle.project(cam, p), reflib.project(cam, p)
            assert (a is None) == (b is None)
            if a is not None:
                assert np.array_equal(a, b)
            row, col = int(rng.integers(0, cam.image_rows)), int(rng.integers(0, cam.image_cols))
            la = oracle.localize(cam, [row, col], 40.0)
            lb = reflib.localize(cam, [row, col], 40.0)
            assert (la[0] == 0) == (lb[0] == 0)
            if la[0] == 0:
                assert np.array_equal(la[1], lb[1]) and la[2] == lb[2] and la[3] == lb[3]
            ra = oracle.ray_from_pixel(cam, row, col, 0.0, 40.0)
            rb = reflib.ray_from_pixel(cam, row, col, 0.0, 40.0)
            assert (ra is None) == (rb is None)
            if ra is not None:
                assert np.array_equal(ra[0], rb[0]) and np.array_equal(ra[1], rb[1])
                n_checked += 1
    assert n_checked > 1000


def test_grid_segments_candidates_bits(oracle, reflib, scene):
    roi = scene.roi
    for (H, W) in [(1, 1), (3, 3), (6, 6), (5, 7)]:
        r = Roi(roi.easting_min, roi.easting_min + W * 128.0 + 0.3, roi.northing_min,
                roi.northing_min + H * 128.0, 0.0, 40.0)
        ea, na = oracle.grid_edges(r, H, W)
        eb, nb = reflib.grid_edges(r, H, W)
        assert np.array_equal(ea, eb) and np.array_equal(na, nb)
    e, n = oracle.grid_edges(roi, 3, 3)
    boxes = np.array([[e[c], n[r], 0, e[c + 1], n[r + 1], 40] for r in range(2) for c in range(2)])
    rng = np.random.default_rng(1)
    for cam in scene.cams:
        for _ in range(300):
            row, col = int(rng.integers(0, cam.image_rows)), int(rng.integers(0, cam.image_cols))
            ray = reflib.ray_from_pixel(cam, row, col, 0.0, 40.0)
            if ray is None:
                continue
            o, d = ray
            assert oracle.segments(o, d, boxes) == reflib.segments(o, d, boxes)
            for b in boxes:
                assert oracle.intersect(o, d, b) == reflib.intersect(o, d, b)
            assert oracle.candidate_tiles(roi, 3, 3, o, d) == reflib.candidate_tiles(roi, 3, 3, o, d)
    # nadir rays exactly on the shared face (tie order = box order)
    o = np.array([e[1], n[0] + 17.0, 40.0])
    d = np.array([0.0, 0.0, -1.0])
    assert oracle.segments(o, d, boxes) == reflib.segments(o, d, boxes)


def test_crop_bits(oracle, reflib, scene):
    e, n = oracle.grid_edges(scene.roi, 3, 3)
    for cam in scene.cams:
        for r in range(3):
            for c in range(3):
                box = [e[c], n[r], 0, e[c + 1], n[r + 1], 40]
                for m in (0, 4, 8):
                    assert oracle.crop_for_tile(cam, box, m) == reflib.crop_for_tile(cam, box, m)


def test_to_local_bits(reflib, scene):
    """The sampler's local = (p - min) * inv_size matches LocalFrame::to_local."""
    rng = np.random.default_rng(2)
    e_, n_ = reflib.grid_edges(scene.roi, 3, 3)
    for _ in range(200):
        r, c = int(rng.integers(0, 3)), int(rng.integers(0, 3))
        box, inv = reflib.tile_frame(scene.roi, 3, 3, r, c)
        p = rng.uniform(-10, 400, 3)
        a = reflib.to_local(scene.roi, 3, 3, r, c, p)
        b = (p - box[:3]) * (1.0 / (box[3:] - box[:3]))
        assert np.array_equal(a, b)
        assert np.array_equal(inv, 1.0 / (box[3:] - box[:3]))


def test_field_init_bits(oracle, reflib):
    cfg = FieldConfig.defaults()
    for l in range(cfg.levels):
        assert oracle.L.tfo_level_resolution(C.byref(cfg), l) == reflib.L.ref_level_resolution(C.byref(cfg), l)
    # tile streams: Rng(hash_combine(seed, PURPOSE, row, col)) into HashGridT/MlpT::init
    seed, row, col = 1, 2, 3
    hc = oracle.L.tfo_hash_combine
    enc, dnet, _ = oracle.tile_create(cfg, row, col, seed)
    k_enc = hc(hc(hc(seed, 0x54454E43), row), col)
    k_dnet = hc(hc(hc(seed, 0x54444E54), row), col)
    assert np.array_equal(enc, reflib.hash_init(cfg, k_enc))
    assert np.array_equal(dnet, reflib.mlp_init([16, 64, 16], k_dnet))
    color = oracle.color_create(cfg, seed)
    assert np.array_equal(color, reflib.mlp_init([39, 64, 64, 3], hc(seed, 0x434F4C52)))


def test_field_point_bits(oracle, reflib):
    """Hash lookup + density MLP + colour MLP (forward and backward) of the
    restatement equal MlpT/HashGridT (nn.hpp) bit-for-bit."""
    cfg = FieldConfig.defaults()
    enc, dnet, _ = oracle.tile_create(cfg, 0, 1, 5)
    rng = np.random.default_rng(3)
    enc = (enc + rng.normal(0, 0.3, enc.shape)).astype(np.float32)
    color = oracle.color_create(cfg, 5)
    pts = rng.uniform(-0.1, 1.1, (64, 3)).astype(np.float32)
    feat, _ = reflib.hash_lookup_bwd(cfg, enc, pts)
    for i in range(16):
        dout, _, _ = reflib.mlp_fwd_bwd([16, 64, 16], dnet, feat[i])
        sig_ref = reflib.L.ref_density_activation(float(dout[0]), 1e4, None)
        d3 = np.array([0.1, -0.3, -0.95], np.float32)
        venc = np.zeros(24, np.float32)
        reflib.L.ref_encode_direction(d3.ctypes.data, 4, venc.ctypes.data)
        cin = np.concatenate([dout[1:], venc]).astype(np.float32)
        cout, _, _ = reflib.mlp_fwd_bwd([39, 64, 64, 3], color, cin)
        rgb_ref = (1.0 / (1.0 + np.exp(-cout.astype(np.float32)))).astype(np.float32)
        s, rgb = oracle.query_field(cfg, enc, dnet, color, pts[i], d3)
        assert np.float32(s) == np.float32(sig_ref)
        np.testing.assert_allclose(rgb, rgb_ref, rtol=1e-6)  # numpy exp vs libm expf


def test_backward_primitives_bits(oracle, reflib):
    """The oracle's reverse mode equals the reference's MlpT::backward_p
    (nn.hpp:116-157) and HashGridT::backward (nn.hpp:231-245), compiled
    verbatim into oracle/_ref, bit for bit: outputs, parameter gradients
    (accumulated over several points) and input gradients."""
    cfg = FieldConfig.defaults()
    rng = np.random.default_rng(17)
    for widths, seed in (([16, 64, 16], 3), ([39, 64, 64, 3], 4)):
        params = reflib.mlp_init(widths, seed)
        params = (params + rng.normal(0, 0.05, params.shape)).astype(np.float32)  # non-zero biases
        g_ref = np.zeros_like(params)
        g_orc = np.zeros_like(params)
        for _ in range(24):
            x = rng.normal(0, 1, widths[0]).astype(np.float32)
            d_out = rng.normal(0, 1, widths[-1]).astype(np.float32)
            o1, g1, di1 = reflib.mlp_fwd_bwd(widths, params, x, d_out)
            o2, g2, di2 = oracle.mlp_fwd_bwd(widths, params, x, d_out)
            assert o1.tobytes() == o2.tobytes()
            assert di1.tobytes() == di2.tobytes()
            assert g1.tobytes() == g2.tobytes()
            g_ref += g1
            g_orc += g2
        assert g_ref.tobytes() == g_orc.tobytes()
    enc, _, _ = oracle.tile_create(cfg, 1, 2, 9)
    enc = (enc + rng.normal(0, 0.3, enc.shape)).astype(np.float32)
    pts = rng.uniform(-0.05, 1.05, (256, 3)).astype(np.float32)
    pts[:8] = [[0, 0, 0], [1, 1, 1], [0.5, 0.5, 0.5], [1, 0, 0.25], [0.999999, 1e-7, 0.5],
               [0.0625, 0.125, 0.1875], [1.0001, -0.0001, 0.3], [0.3, 0.7, 1.0]]
    d_out = rng.normal(0, 1, (256, 16)).astype(np.float32)
    f1, g1 = reflib.hash_lookup_bwd(cfg, enc, pts, d_out)
    f2, g2 = oracle.hash_lookup_bwd(cfg, enc, pts, d_out)
    assert f1.tobytes() == f2.tobytes()
    assert g1.tobytes() == g2.tobytes()
    assert np.count_nonzero(g1) > 1000
