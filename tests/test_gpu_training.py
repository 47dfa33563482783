"""End-to-end training parity on B200: the CUDA path and the CPU oracle train
the same window from the same initialisation, seeds and batch stream
(including the periodic occupancy updates), then render the same evaluation
pixels.  Stated margins (north star: "final PSNR and depth error within a
stated margin"): |PSNR_gpu - PSNR_ref| <= 0.5 dB, and the mean |depth_gpu -
depth_ref| over opaque pixels <= 0.5 m (5% of the 10 m z-extent of this scene).
"""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2507_01631_b200 import synth
from paper_2507_01631_b200.abi import FieldConfig, Roi, TrainConfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _psnr(a, b):
    mse = float(np.mean((a - b) ** 2))
    return 99.0 if mse == 0 else 10 * np.log10(1.0 / mse)


def test_training_psnr_and_depth_match_oracle():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle.pyoracle import Oracle, Session
    from paper_2507_01631_b200.tilefield import Context

    # one 64 m tile, 10 m z-extent, 2 views of a textured flat ground
    scene = synth.make_scene(1, 1, tile_side=64.0, z_extent=10.0, n_views=2, gsd=0.5, seed=9,
                             max_off_nadir=20.0)
    fc = FieldConfig.defaults()
    B, iters = 1024, 160
    tc = TrainConfig.defaults(batch_rays=B, seed=11)
    tc.samples_per_meter = 3.2  # ~32 samples over the 10 m extent
    ctx = Context(scene, fc, tc, max_rays=2048)
    ses = Session(Oracle(), scene, fc, tc, workers=os.cpu_count() or 8)
    ctx.set_window(0, 0)
    ses.set_window(0, 0)
    acc = ses.build_accept()
    np.testing.assert_array_equal(ctx.accept_list(), acc)
    lg = lr = None
    for it in range(iters):
        lg = ctx.train_step(it, 0, B)
        lr = ses.train_step(it, 0, B)
    # evaluation: 2048 accepted pixels, midpoint samples
    sel = acc[:: max(1, acc.size // 2048)][:2048]
    px = np.stack([(sel >> 40).astype(np.int32), ((sel >> 20) & 0xFFFFF).astype(np.int32),
                   (sel & 0xFFFFF).astype(np.int32)], axis=1)
    ctx.sample_pixels(px)
    ses.sample_pixels(px)
    target = ses.batch()["rays"]["target"]
    ctx.field_forward()
    ses.forward()
    g, r = ctx.composite(), ses.composite()
    p_gpu, p_ref = _psnr(g["rgb"], target), _psnr(r["rgb"], target)
    print(f"after {iters} its: loss gpu {lg:.5f} ref {lr:.5f}; PSNR gpu {p_gpu:.2f} ref {p_ref:.2f} dB")
    assert p_gpu > 15.0 and p_ref > 15.0  # both actually learned the views
    assert abs(p_gpu - p_ref) <= 0.5
    op = (g["opacity"] > 0.5) & (r["opacity"] > 0.5)
    if op.sum() > 100:
        mae = float(np.mean(np.abs(g["depth"][op] - r["depth"][op])))
        print(f"depth |gpu - ref| over {op.sum()} opaque pixels: {mae:.3f} m")
        assert mae <= 0.5


def test_cpp_host_example():
    """examples/train_window.cpp drives the snake through the C++ wrapper."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    exe = os.path.join(ROOT, "paper_2507_01631_b200", "bin", "train_window")
    if not os.path.exists(exe):
        from paper_2507_01631_b200 import build

        build.build_examples()
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    lines = [l for l in out.stdout.splitlines() if l.startswith("window")]
    assert len(lines) == 4 and all("accepted rays" in l for l in lines)


def _train_eval_heightfield(scene, window, B, iters, tc_seed, n_eval):
    """Both sides train the same window from the same init / batch stream
    (occupancy updates included), then render the same evaluation pixels of
    view 0 (midpoint samples).  Returns the metrics of both and the GT."""
    from oracle.pyoracle import Oracle, Session
    from paper_2507_01631_b200.tilefield import Context

    fc = FieldConfig.defaults()
    tc = TrainConfig.defaults(batch_rays=B, seed=tc_seed)
    ctx = Context(scene, fc, tc, max_rays=max(B, n_eval))
    ses = Session(Oracle(), scene, fc, tc, workers=os.cpu_count() or 8)
    ctx.set_window(*window)
    ses.set_window(*window)
    acc = ses.build_accept()
    np.testing.assert_array_equal(ctx.accept_list(), acc)
    for it in range(iters):
        ctx.train_step(it, 0, B)
        ses.train_step(it, 0, B)
    v0 = acc[(acc >> 40) == 0]
    sel = v0[:: max(1, v0.size // n_eval)][:n_eval]
    px = np.stack([(sel >> 40).astype(np.int32), ((sel >> 20) & 0xFFFFF).astype(np.int32),
                   (sel & 0xFFFFF).astype(np.int32)], axis=1)
    ctx.sample_pixels(px)
    ses.sample_pixels(px)
    target = ses.batch()["rays"]["target"]
    ctx.field_forward()
    ses.forward()
    g, r = ctx.composite(), ses.composite()
    gt = scene.depths[0][px[:, 1], px[:, 2]]
    return g, r, target, gt


def _report(name, g, r, target, gt):
    p_gpu, p_ref = _psnr(g["rgb"], target), _psnr(r["rgb"], target)
    op = (g["opacity"] > 0.5) & (r["opacity"] > 0.5)
    mae_gpu = float(np.mean(np.abs(g["depth"][op] - gt[op])))
    mae_ref = float(np.mean(np.abs(r["depth"][op] - gt[op])))
    mae_gr = float(np.mean(np.abs(g["depth"][op] - r["depth"][op])))
    print(f"{name}: PSNR gpu {p_gpu:.2f} ref {p_ref:.2f} dB; depth MAE vs GT gpu {mae_gpu:.3f} ref {mae_ref:.3f} m, "
          f"|gpu - ref| {mae_gr:.3f} m over {op.sum()} opaque pixels")
    return p_gpu, p_ref, mae_gpu, mae_ref, mae_gr, op.sum()


# Stated margins of the heightfield runs (north star: "final PSNR and depth
# error within a stated margin"): PSNR within 0.5 dB of the oracle; depth MAE
# against the exact ground truth within 2 m of the oracle's (5% of the 40 m
# z-extent), and the two depth maps within 1.5 m of each other on average.
# (The short oracle-affordable runs fit colour, not yet geometry: both sides'
# depth MAE against the ground truth is still large; the long GPU-only run
# below shows the geometry converging.)
PSNR_MARGIN_DB = 0.5
DEPTH_MARGIN_M = 2.0
DEPTH_PAIR_M = 1.5


def test_heightfield_config1_training_parity():
    """Config 1 shape on the SPEC.md:533-556 heightfield (ground + boxes,
    exact depth): one 128 m tile, 4 views of ~280^2 px at 0.5 m, 4,096 rays."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    scene = synth.make_heightfield_scene(1, 1, tile_side=128.0, z_extent=40.0, n_views=4, gsd=0.5, seed=3)
    g, r, target, gt = _train_eval_heightfield(scene, (0, 0), 4096, 120, 11, 4096)
    p_gpu, p_ref, mae_gpu, mae_ref, mae_gr, n_op = _report("config 1 heightfield", g, r, target, gt)
    assert p_gpu > 14.0 and p_ref > 14.0
    assert abs(p_gpu - p_ref) <= PSNR_MARGIN_DB
    assert n_op > 500
    assert abs(mae_gpu - mae_ref) <= DEPTH_MARGIN_M and mae_gr <= DEPTH_PAIR_M


def test_heightfield_config2_window_training_parity():
    """Config 2 shape on the heightfield: 3x3 grid, 8 views at 0.5 m, the
    2x2 window (0,0) with rays crossing tile seams, 16,384 rays."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    scene = synth.make_heightfield_scene(3, 3, tile_side=128.0, z_extent=40.0, n_views=8, gsd=0.5, seed=2)
    g, r, target, gt = _train_eval_heightfield(scene, (0, 0), 16384, 40, 7, 4096)
    p_gpu, p_ref, mae_gpu, mae_ref, mae_gr, n_op = _report("config 2 heightfield window", g, r, target, gt)
    assert abs(p_gpu - p_ref) <= PSNR_MARGIN_DB
    assert n_op > 500
    assert abs(mae_gpu - mae_ref) <= DEPTH_MARGIN_M and mae_gr <= DEPTH_PAIR_M


def test_heightfield_geometry_converges():
    """GPU-only, long: on the config-1 heightfield with 8 views the trained
    field's depth approaches the exact ground truth (depth MAE over opaque
    evaluation pixels from ~36 m at initialisation to < 10 m after 4,000
    iterations; measured r02: 8.0 m, median 7.0 m), with PSNR > 38 dB."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_01631_b200.tilefield import Context

    scene = synth.make_heightfield_scene(1, 1, tile_side=128.0, z_extent=40.0, n_views=8, gsd=0.5, seed=3)
    B = 4096
    ctx = Context(scene, FieldConfig.defaults(), TrainConfig.defaults(batch_rays=B, seed=11), max_rays=8192)
    ctx.set_window(0, 0)
    acc = ctx.accept_list()
    v0 = acc[(acc >> 40) == 0]
    sel = v0[:: max(1, v0.size // 8192)][:8192]
    px = np.stack([(sel >> 40).astype(np.int32), ((sel >> 20) & 0xFFFFF).astype(np.int32),
                   (sel & 0xFFFFF).astype(np.int32)], axis=1)
    gt = scene.depths[0][px[:, 1], px[:, 2]]

    def evaluate():
        ctx.sample_pixels(px)
        ctx.field_forward()
        g = ctx.composite()
        op = g["opacity"] > 0.5
        return _psnr(g["rgb"], ctx.batch()["rays"]["target"]), float(np.mean(np.abs(g["depth"][op] - gt[op])))

    _, mae0 = evaluate()
    for it in range(4000):
        ctx.train_step(it, 0, B)
    psnr, mae = evaluate()
    print(f"heightfield 8 views: depth MAE vs GT {mae0:.2f} m -> {mae:.2f} m, PSNR {psnr:.2f} dB")
    assert mae < 10.0 and mae < mae0 / 3 and psnr > 38.0
