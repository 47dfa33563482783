"""Evaluation metrics (evalio).

CPU: the oracle restatement (oracle/evalio.py) against every SPEC example and
against an independent scipy.ndimage formulation of SSIM.  GPU: the CUDA
metrics (csrc/k_eval.cu) against the oracle, the tile-edge band mask bit-exact,
and the full-frame render (render_view) against render_pixels."""
import numpy as np
import pytest

from oracle import evalio


def _img(seed, shape=(40, 52, 3)):
    return np.random.default_rng(seed).random(shape)


def test_psnr_spec_examples():
    a = _img(0)
    assert evalio.psnr(a, a) == 99.0  # identical -> cap
    b = np.clip(a, 0, 0.8)
    assert abs(evalio.psnr(b + 0.1, b) - 20.0) < 1e-9  # uniform offset 0.1 -> 20 dB
    c = _img(1)
    assert evalio.psnr(a, c) == evalio.psnr(c, a)  # symmetry
    with pytest.raises(ValueError):
        evalio.psnr(a, a[:-1])


def test_ssim_spec_examples():
    a = _img(2)
    assert abs(evalio.ssim(a, a) - 1.0) < 1e-12  # identical
    rng = np.random.default_rng(3)
    binary = (rng.random((32, 32, 1)) > 0.5).astype(np.float64).repeat(3, axis=2)
    assert evalio.ssim(binary, 1.0 - binary) < 0.0  # anticorrelated
    b = _img(4)
    assert abs(evalio.ssim(a, b) - evalio.ssim(b, a)) < 1e-12  # symmetry
    with pytest.raises(ValueError):
        evalio.ssim(a[:10], a[:10])  # smaller than the window


def test_ssim_matches_scipy_formulation():
    """Independent check of the restatement: scipy's gaussian_filter with
    truncate = 5/1.5 is the same 11-tap window; crop to the valid region."""
    from scipy.ndimage import gaussian_filter

    a, b = _img(5, (48, 37, 3)), _img(6, (48, 37, 3)) * 0.5 + 0.2
    x, y = a.mean(2), b.mean(2)
    f = lambda z: gaussian_filter(z, 1.5, truncate=5 / 1.5, mode="constant")[5:-5, 5:-5]
    mx, my = f(x), f(y)
    sx, sy, sxy = f(x * x) - mx * mx, f(y * y) - my * my, f(x * y) - mx * my
    C1, C2 = 1e-4, 9e-4
    ref = (((2 * mx * my + C1) * (2 * sxy + C2)) / ((mx * mx + my * my + C1) * (sx + sy + C2))).mean()
    assert abs(evalio.ssim(a, b) - ref) < 1e-12


def test_depth_mae_spec_examples():
    d = np.random.default_rng(7).random((20, 30)) * 40
    assert evalio.depth_mae(d, d) == 0.0
    assert abs(evalio.depth_mae(d + 1.0, d) - 1.0) < 1e-12
    m = np.zeros(d.shape, np.uint8)
    m[3:9, 4:20] = 1
    e = d.copy()
    e[m == 0] += 100.0  # outside the mask: ignored
    assert abs(evalio.depth_mae(e + 0.5 * m, d, m) - 0.5) < 1e-12
    with pytest.raises(ValueError):
        evalio.depth_mae(d, d, np.zeros(d.shape))


# ------------------------------------------------------------------ GPU
def _ctx(scene=None):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_01631_b200 import synth
    from paper_2507_01631_b200.abi import FieldConfig, TrainConfig
    from paper_2507_01631_b200.tilefield import Context

    scene = scene or synth.make_scene(2, 2, tile_side=128.0, n_views=1, gsd=1.0, seed=3, max_off_nadir=25.0)
    return scene, Context(scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=4096), max_rays=4096)


@pytest.mark.gpu
def test_gpu_metrics_match_oracle():
    _, ctx = _ctx()
    rng = np.random.default_rng(11)
    for shape in ((64, 80, 3), (257, 301, 3), (11, 11, 3)):
        a = rng.random(shape).astype(np.float32)
        b = np.clip(a + rng.normal(0, 0.05, shape), 0, 1).astype(np.float32)
        assert abs(ctx.psnr(a, b) - evalio.psnr(a, b)) < 1e-6
        assert ctx.psnr(a, a) == 99.0
        assert abs(ctx.ssim(a, b) - evalio.ssim(a, b)) < 2e-5, shape
        assert abs(ctx.ssim(a, a) - 1.0) < 1e-5
        d1 = (rng.random(shape[:2]) * 40).astype(np.float32)
        d2 = (d1 + rng.normal(0, 0.3, shape[:2])).astype(np.float32)
        m = (rng.random(shape[:2]) > 0.3).astype(np.uint8)
        assert abs(ctx.depth_mae(d1, d2, m) - evalio.depth_mae(d1, d2, m)) < 1e-6
        assert abs(ctx.depth_mae(d1, d2) - evalio.depth_mae(d1, d2)) < 1e-6
    from paper_2507_01631_b200.tilefield import TileFieldError

    with pytest.raises(TileFieldError, match="smaller than the 11x11 window"):
        ctx.ssim(np.zeros((10, 20, 3), np.float32), np.zeros((10, 20, 3), np.float32))
    with pytest.raises(TileFieldError, match="empty mask"):
        ctx.depth_mae(d1, d2, np.zeros(d1.shape, np.uint8))


@pytest.mark.gpu
def test_gpu_edge_band_mask_bit_exact():
    from oracle.pyoracle import Oracle

    scene, ctx = _ctx()
    o = Oracle()
    e, n = o.grid_edges(scene.roi, scene.grid_rows, scene.grid_cols)
    cam = scene.cams[0]
    for band in (0, 3, 8):
        got = ctx.edge_band_mask(cam, band)
        ref = evalio.edge_band_mask(o, cam, scene.roi, np.asarray(e), np.asarray(n), band)
        np.testing.assert_array_equal(got, ref)
        assert 0 < got.mean() < 0.9


@pytest.mark.gpu
def test_gpu_render_view_matches_render_pixels():
    from oracle.pyoracle import Oracle
    from paper_2507_01631_b200.abi import FieldConfig
    from paper_2507_01631_b200.tilefield import tile_init

    scene, ctx = _ctx()
    fc = FieldConfig.defaults()
    tiles = [(r, c) for r in range(2) for c in range(2)]
    states = [tile_init(fc, 5, r, c) for r, c in tiles]
    rng = np.random.default_rng(1)
    for s in states:
        s["enc"] += rng.normal(0, 0.3, s["enc"].shape).astype(np.float32)
    ctx.render_setup(tiles, states, Oracle().color_create(fc, 5))
    cam = scene.cams[0]
    rgb, dep, op = ctx.render_view(cam)
    assert rgb.shape == (cam.image_rows, cam.image_cols, 3)
    px = np.stack([rng.integers(0, cam.image_rows, 500), rng.integers(0, cam.image_cols, 500)], 1).astype(np.int32)
    r2, d2, o2 = ctx.render_pixels(cam, px)
    np.testing.assert_array_equal(rgb[px[:, 0], px[:, 1]], r2)
    np.testing.assert_array_equal(op[px[:, 0], px[:, 1]], o2)
    # an evaluation pass: PSNR of the render against itself and against the view
    assert ctx.psnr(rgb, rgb) == 99.0
    assert 0.0 < ctx.psnr(rgb, scene.images[0].astype(np.float32) / 255.0) < 99.0
